"""CPU checks of the C-ABI boundary: the library loads and exports every
entry point declared in include/hsb200.h; struct layouts agree."""

from __future__ import annotations

import ctypes
import os
import re

import pytest

from conftest import REPO


def _declared():
    src = open(os.path.join(REPO, "include", "hsb200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:int|void|const char\*)\s+(hs_\w+)\s*\(", src, re.M)))


def test_header_declares_entry_points():
    names = _declared()
    for must in ("hs_index_create", "hs_search_batch", "hs_lut16_scan", "hs_select_topk",
                 "hs_sparse_scan", "hs_quantize_lut", "hs_shard_merge_dev"):
        assert must in names


def test_library_exports_every_declared_symbol():
    from paper_1903_08690_b200 import _native

    lib = _native.lib()  # loads libhsb200.so (no GPU needed to load)
    missing = [n for n in _declared() if not hasattr(lib, n)]
    assert not missing, missing
    assert b"sm_100a" in lib.hs_version()


def test_host_library_exports():
    from paper_1903_08690_b200 import builder

    lib = builder._hostlib()
    for n in ("hsb_cache_sort", "hsb_top_t_thresholds", "hsb_gen_hybrid"):
        assert hasattr(lib, n)


def test_struct_sizes_match_c_layout():
    from paper_1903_08690_b200 import _native as nat

    # 64-bit layout: pointers 8 B, int32 padded to 8 where followed by a pointer
    assert ctypes.sizeof(nat.SearchParams) == 32
    assert ctypes.sizeof(nat.QueryBatch) == 56
    assert ctypes.sizeof(nat.IndexDesc) % 8 == 0


def test_search_without_gpu_fails_loudly():
    import numpy as np

    import paper_1903_08690_b200 as hs

    try:
        import torch

        if torch.cuda.is_available():
            pytest.skip("a GPU is visible")
    except Exception:
        pass
    with pytest.raises(RuntimeError, match="GPU"):
        hs.select_topk(np.array([1.0, 2.0]), 1)
