"""The C-ABI library: builds, loads without a GPU, exports every declared symbol,
and the product path refuses to run without CUDA (no CPU fallback)."""

from __future__ import annotations

import ctypes
import re

import pytest

from conftest import REPO


def declared_symbols() -> list[str]:
    text = (REPO / "include" / "tmfg_b200.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(tg_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_hot_path():
    syms = declared_symbols()
    for s in ("tg_pearson_f64", "tg_row_sort_f64", "tg_tmfg_heap", "tg_sssp_rows", "tg_truncated",
              "tg_group_max_batch", "tg_nn_chain_batch", "tg_assign_vertices", "tg_bubble_tree"):
        assert s in syms


def test_library_exports_every_declared_symbol():
    from paper_2408_09399_b200 import _native
    lib = ctypes.CDLL(str(_native.LIB_PATH))
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing
    assert lib.tg_abi_version() == 1


def test_python_binding_covers_the_header():
    from paper_2408_09399_b200 import _native
    assert set(declared_symbols()) <= set(_native.EXPORTED)
    _native.load(require_cuda=False)
    assert not _native.MISSING


def test_binary_is_sm100a():
    """The shared library carries sm_100a SASS (cuobjdump lists the ELF arch)."""
    import shutil
    import subprocess
    from paper_2408_09399_b200 import _native
    tool = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    out = subprocess.run([tool, "--list-elf", str(_native.LIB_PATH)], capture_output=True, text=True)
    assert "sm_100a" in out.stdout


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    import numpy as np
    from paper_2408_09399_b200 import _native, sort_neighbor_lists
    _native._lib = None
    with pytest.raises(_native.NativeUnavailable):
        _native.load()
    with pytest.raises(Exception):
        sort_neighbor_lists(np.eye(5))
