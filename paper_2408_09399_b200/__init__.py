"""paper_2408_09399_b200: B200-native TMFG-DBHT hot path (arxiv 2408.09399).

Drop-in replacements for the reference package's hot-path entry points
(``tmfgclust``): the work runs in hand-written sm_100a kernels
(``_lib/libtmfg_b200.so``, C ABI in ``include/tmfg_b200.h``) and there is no CPU
fallback.
"""

from . import _native
from .simmatrix import (
    DataError,
    Dataset,
    SortedNeighborLists,
    pearson_similarity,
    sort_neighbor_lists,
    validate_similarity,
)
from .tmfg import (
    GAIN_EPS,
    BuildConfig,
    TmfgGraph,
    TraceError,
    build_tmfg,
    build_tmfg_heap,
    edge_sum,
    gain,
    select_initial_clique,
)

__version__ = "0.1.0"
