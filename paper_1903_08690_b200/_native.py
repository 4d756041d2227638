"""ctypes binding of libhsb200.so (the C ABI in include/hsb200.h).

There is no CPU fallback: if the CUDA library is missing or no GPU is
visible, every search entry point raises.  Status codes map to the
reference's exception types (ValueError / MemoryError / RuntimeError).
"""

from __future__ import annotations

import ctypes
import os
import threading

import numpy as np

from ._build import LIB_CUDA

HS_OK, HS_EINVAL, HS_ENOMEM, HS_ECUDA, HS_ENCCL, HS_EUNSUPPORTED = range(6)

P = ctypes.c_void_p
i32 = ctypes.c_int32
i64 = ctypes.c_int64
f64 = ctypes.c_double


class IndexDesc(ctypes.Structure):
    _fields_ = [
        ("n", i64), ("d_sparse", i64), ("d_dense", i64), ("order", P),
        ("n_active", i64), ("post_dims", P), ("post_ptr", P), ("post_ids", P), ("post_w", P),
        ("res_indptr", P), ("res_indices", P), ("res_data", P),
        ("n_subspaces", i32), ("n_centers", i32), ("subdims", P), ("centers", P), ("packed", P),
        ("has_sq", i32), ("sq_lo", P), ("sq_step", P), ("sq_codes", P),
        ("has_whitening", i32), ("wh_mean", P), ("wh_inverse_t", P),
        ("has_dataset", i32), ("ds_dense", P), ("ds_indptr", P), ("ds_indices", P), ("ds_data", P),
        ("sparse_weight", f64), ("dense_weight", f64), ("id_offset", i64),
    ]


class QueryBatch(ctypes.Structure):
    _fields_ = [("nq", i64), ("sp_indptr", P), ("sp_dims", P), ("sp_vals", P), ("dense", P),
                ("nnz", i64), ("max_row_nnz", i32)]


class SearchParams(ctypes.Structure):
    _fields_ = [("h", i32), ("overfetch", f64), ("retain", f64), ("exact_final_rerank", i32)]


_LIB = None
_LOCK = threading.Lock()


def lib():
    """Load libhsb200.so (building it in-tree if absent and nvcc exists)."""
    global _LIB
    if _LIB is not None:
        return _LIB
    with _LOCK:
        if _LIB is not None:
            return _LIB
        if not os.path.exists(LIB_CUDA):
            from ._build import build_cuda

            build_cuda()
        L = ctypes.CDLL(LIB_CUDA)
        L.hs_last_error.restype = ctypes.c_char_p
        L.hs_version.restype = ctypes.c_char_p
        L.hs_index_create.argtypes = [ctypes.POINTER(IndexDesc), ctypes.c_int, ctypes.POINTER(P)]
        L.hs_index_destroy.argtypes = [P]
        L.hs_index_destroy.restype = None
        L.hs_index_memory_bytes.argtypes = [P, ctypes.POINTER(i64)]
        L.hs_result_sizes.argtypes = [P, ctypes.POINTER(SearchParams), P]
        L.hs_search_batch.argtypes = [P, ctypes.POINTER(QueryBatch), ctypes.POINTER(SearchParams),
                                      P, P, P]
        L.hs_search_batch_dev.argtypes = [P, ctypes.POINTER(QueryBatch),
                                          ctypes.POINTER(SearchParams), P, P, P]
        L.hs_adc_table.argtypes = [P, P, i32, i32, P, i64, i64, P]
        L.hs_quantize_lut.argtypes = [P, i64, i32, i32, P, P, P, P]
        L.hs_lut16_scan.argtypes = [P, i64, i32, P, P, P, i64, P, P]
        L.hs_sparse_scan.argtypes = [P, ctypes.POINTER(QueryBatch), P]
        L.hs_sparse_scan_into.argtypes = [P, ctypes.POINTER(QueryBatch), P]
        L.hs_sq_decode.argtypes = [P, i64, i32, P, P, P, i64, P]
        L.hs_sq_residual_dot.argtypes = [P, i64, i32, P, P, P, i64, P, P]
        L.hs_stage1_scores.argtypes = [P, ctypes.POINTER(QueryBatch), P]
        L.hs_select_topk.argtypes = [P, i64, i64, i64, P, P]
        L.hs_exact_topk.argtypes = [P, ctypes.POINTER(QueryBatch), i32, P, P]
        L.hs_shard_merge_dev.argtypes = [P, P, i64, i64, i64, i32, P, P, P]
        L.hs_set_timing.argtypes = [P, ctypes.c_int]
        L.hs_index_launches.argtypes = [P, ctypes.POINTER(i64)]
        L.hs_last_kernel_times.argtypes = [P, P, i32, ctypes.POINTER(i32), ctypes.c_char_p, i32]
        L.hs_dense_encode.argtypes = [P, i64, i64, P, i32, P, P, i32, P, P, P, P, ctypes.c_int, P]
        _LIB = L
    return _LIB


def check(rc: int):
    if rc == HS_OK:
        return
    msg = lib().hs_last_error().decode(errors="replace")
    if rc in (HS_EINVAL, HS_EUNSUPPORTED):
        raise ValueError(msg)
    if rc == HS_ENOMEM:
        raise MemoryError(msg)
    raise RuntimeError(f"hsb200 status {rc}: {msg}")


def ptr(a) -> ctypes.c_void_p:
    """Host pointer of a C-contiguous numpy array (None -> NULL)."""
    if a is None:
        return None
    return ctypes.c_void_p(a.ctypes.data)


def require_gpu():
    """Raise unless a CUDA device is visible (no CPU fallback exists)."""
    L = lib()
    # cudaGetDeviceCount through the runtime the library links
    cnt = ctypes.c_int(0)
    try:
        rt = ctypes.CDLL("libcudart.so.12")
        rc = rt.cudaGetDeviceCount(ctypes.byref(cnt))
    except OSError:
        rc, cnt.value = 1, 0
    if rc != 0 or cnt.value == 0:
        raise RuntimeError("hsb200: no CUDA device visible; the search path is GPU-only "
                           "(there is no CPU fallback)")
    return L


def contig(a, dtype):
    return np.ascontiguousarray(a, dtype=dtype)
