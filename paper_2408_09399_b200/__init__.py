"""paper_2408_09399_b200: B200-native TMFG-DBHT hot path (arxiv 2408.09399).

Drop-in replacements for the reference package's hot-path entry points
(``tmfgclust``): the work runs in hand-written sm_100a kernels
(``_lib/libtmfg_b200.so``, C ABI in ``include/tmfg_b200.h``) and there is no CPU
fallback -- a missing library or GPU raises ``NativeUnavailable``.

``install()`` rebinds the reference package's module attributes so its own
pipeline (``tmfgclust.pipeline.run_stages``, which looks stage functions up on
the modules at call time, pipeline.py:191-223) runs on the B200.
"""

from . import _native
from ._native import NativeError, NativeUnavailable
from .apsp import (
    ApspParams,
    DistanceOracle,
    ExactOracle,
    HubOracle,
    WeightedTmfg,
    apsp_exact,
    apsp_hub,
    default_hub_count,
    query,
    select_hubs,
    to_weighted,
)
from .dbht import (
    BubbleAssignment,
    BubbleTree,
    DirectedBubbleTree,
    assign_vertices,
    bubble_sinks,
    build_bubble_tree,
    build_hierarchy,
    converging_bubbles,
    orient_edges,
)
from .linkage import (
    Dendrogram,
    complete_linkage,
    cut,
    dendrogram_from_merges,
    load_dendrogram,
    nn_chain_merges,
    save_dendrogram,
    serialize_dendrogram,
)
from .metrics import ari, edge_sum_delta
from .pipeline import (
    PipelineConfig,
    RunReport,
    StageError,
    compare_variants,
    load_input,
    parse_variant_token,
    run_pipeline,
    run_series,
    run_stages,
)
from .simmatrix import (
    DataError,
    Dataset,
    SortedNeighborLists,
    load_matrix,
    load_ucr_dataset,
    pearson_similarity,
    read_matrix_binary,
    save_matrix,
    sort_neighbor_lists,
    validate_similarity,
    write_matrix_binary,
)
from .tmfg import (
    GAIN_EPS,
    BuildConfig,
    TmfgGraph,
    TmfgState,
    TraceError,
    build_tmfg,
    build_tmfg_corr,
    build_tmfg_exact,
    build_tmfg_heap,
    edge_sum,
    gain,
    load_tmfg,
    refresh_max_corr,
    replay_trace,
    save_tmfg,
    select_initial_clique,
)

__version__ = "0.1.0"

# reference module -> names this package replaces in it
_INSTALL_MAP = {
    "simmatrix": ["pearson_similarity", "sort_neighbor_lists"],
    "tmfg": ["select_initial_clique", "build_tmfg_exact", "build_tmfg_corr", "build_tmfg_heap"],
    "apsp": ["to_weighted", "apsp_exact", "apsp_hub", "select_hubs"],
    "dbht": ["build_bubble_tree", "orient_edges", "bubble_sinks", "assign_vertices", "build_hierarchy"],
    "linkage": ["nn_chain_merges"],
}


# reference module -> exception classes this package raises that the reference's callers catch
# (tmfg.py:67-68 TraceError, simmatrix.py:18-19 DataError); install() makes this package raise
# the reference's own classes so ``except tmfgclust.tmfg.TraceError`` keeps working.
_EXCEPTIONS = {
    "TraceError": ("tmfg", ["tmfg", "dbht"]),
    "DataError": ("simmatrix", ["simmatrix", "tmfg"]),
}


def install(package=None) -> dict:
    """Route the reference package's hot path through this package.

    Rebinds the stage functions on the reference modules (and its top-level
    re-exports), and points this package's raise sites at the reference's
    exception classes.  Returns the replaced originals so
    ``uninstall(originals)`` can restore them.
    """
    import importlib
    import sys

    pkg = package or importlib.import_module("tmfgclust")
    this = sys.modules[__name__]
    saved = {}
    for mod_name, names in _INSTALL_MAP.items():
        mod = importlib.import_module(f"{pkg.__name__}.{mod_name}")
        for name in names:
            saved[(mod.__name__, name)] = getattr(mod, name)
            setattr(mod, name, getattr(this, name))
            if hasattr(pkg, name):
                saved[(pkg.__name__, name)] = getattr(pkg, name)
                setattr(pkg, name, getattr(this, name))
    for exc, (ref_mod, ours) in _EXCEPTIONS.items():
        ref_cls = getattr(importlib.import_module(f"{pkg.__name__}.{ref_mod}"), exc)
        for m in ours:
            mod = importlib.import_module(f"{__name__}.{m}")
            saved[(mod.__name__, exc)] = getattr(mod, exc)
            setattr(mod, exc, ref_cls)
    return saved


def uninstall(saved: dict) -> None:
    import importlib

    for (mod_name, name), fn in saved.items():
        setattr(importlib.import_module(mod_name), name, fn)
