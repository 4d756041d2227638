"""GPU search: the reference's hot-path functions on top of libhsb200.so.

    search_topk / search_batch   pipeline.py:226-300  (hs_search_batch)
    select_topk                  pipeline.py:165-189  (hs_select_topk)
    adc_table                    dense.py:212-220     (hs_adc_table)
    quantize_lut                 dense.py:248-260     (hs_quantize_lut)
    lut16_scan[_reference]       dense.py:263-317     (hs_lut16_scan)
    sparse_scan                  sparse.py:268-284    (hs_sparse_scan)
    brute_force_topk             harness.py:25-35     (hs_exact_topk)

Every function validates like the reference (same exception types and
message fragments) and then runs on the GPU; nothing here computes scores
on the host.  A reference-built `HybridIndex` is accepted as is: its arrays
are uploaded once and the device handle is cached on the object.
"""

from __future__ import annotations

import ctypes
import math
import threading

import numpy as np
import scipy.sparse as sp

from . import _native as nat
from .types import (
    LUT16_CENTERS,
    Accumulator,
    HybridDataset,
    HybridVector,
    InvertedIndex,
    PQCodes,
    QuantizedLUT,
    SearchResult,
    SparseVector,
    StageStats,
)

_HANDLE_ATTR = "_hsb200_handles"
_CACHE_LOCK = threading.Lock()


# ----------------------------------------------------------------------------
# device index handles
# ----------------------------------------------------------------------------
class DeviceIndex:
    """Owns one hs_index_t (device copy of an index) on one GPU."""

    def __init__(self, index=None, *, device=0, sparse_index=None, dataset=None,
                 sparse_weight=None, dense_weight=None, id_offset=0, with_dataset=True):
        L = nat.require_gpu()
        keep = []  # arrays that must outlive hs_index_create

        def K(a, dtype):
            a = nat.contig(a, dtype)
            keep.append(a)
            return a

        d = nat.IndexDesc()
        if index is not None:
            sidx = index.sparse_index
            cfg = index.config
            n, d_sparse, d_dense = int(index.n), int(index.d_sparse), int(index.d_dense)
            order = index.order
            res = index.sparse_residual
            di = index.dense_index
            ds = index.dataset if with_dataset else None
            sw = cfg.sparse_weight if sparse_weight is None else sparse_weight
            dw = cfg.dense_weight if dense_weight is None else dense_weight
        elif sparse_index is not None:
            sidx = sparse_index
            n, d_sparse, d_dense = int(sidx.n), int(sidx.d_sparse), 0
            order, res, di, ds = sidx.order, None, None, None
            sw, dw = 1.0, 1.0
        else:
            ds = dataset
            n, d_sparse, d_dense = int(ds.n), int(ds.d_sparse), int(ds.d_dense)
            order, res, di, sidx = np.arange(n), None, None, None
            sw = 1.0 if sparse_weight is None else sparse_weight
            dw = 1.0 if dense_weight is None else dense_weight
        if d_sparse >= 2 ** 32:
            raise ValueError("d_sparse must be < 2^32")
        d.n, d.d_sparse, d.d_dense = n, d_sparse, d_dense
        d.order = nat.ptr(K(order, np.int64))
        if sidx is not None:
            dims, ptr_, ids, w = _posting_arrays(sidx)
            d.n_active = len(dims)
            d.post_dims = nat.ptr(K(dims, np.uint32))
            d.post_ptr = nat.ptr(K(ptr_, np.int64))
            d.post_ids = nat.ptr(K(ids, np.uint32))
            d.post_w = nat.ptr(K(w, np.float32))
        else:
            d.n_active = 0
            d.post_ptr = nat.ptr(K(np.zeros(1), np.int64))
        if res is not None and n > 0:
            r = sp.csr_matrix(res)
            d.res_indptr = nat.ptr(K(r.indptr, np.int64))
            d.res_indices = nat.ptr(K(r.indices, np.uint32))
            d.res_data = nat.ptr(K(r.data, np.float32))
        if di is not None and d_dense > 0:
            cb = di.codebooks
            d.n_subspaces = cb.n_subspaces
            d.n_centers = cb.n_centers
            d.subdims = nat.ptr(K(cb.subdims, np.int32))
            d.centers = nat.ptr(K(np.concatenate([np.asarray(c, np.float32).reshape(-1)
                                                  for c in cb.centers]), np.float32))
            if di.codes.packed is not None:
                d.packed = nat.ptr(K(di.codes.packed, np.uint8))
            if di.residual is not None:
                d.has_sq = 1
                d.sq_lo = nat.ptr(K(di.residual.lo, np.float32))
                d.sq_step = nat.ptr(K(di.residual.step, np.float32))
                d.sq_codes = nat.ptr(K(di.residual.codes, np.uint8))
            if di.whitening is not None:
                d.has_whitening = 1
                d.wh_mean = nat.ptr(K(di.whitening.mean, np.float64))
                d.wh_inverse_t = nat.ptr(K(di.whitening.inverse_t, np.float64))
        elif d_dense > 0 and index is not None:
            raise ValueError("index has a dense dimension but no dense index")
        if ds is not None:
            dsp = sp.csr_matrix(ds.sparse)
            dsp.sort_indices()
            d.has_dataset = 1
            if d_dense > 0:
                d.ds_dense = nat.ptr(K(ds.dense, np.float32))
            d.ds_indptr = nat.ptr(K(dsp.indptr, np.int64))
            d.ds_indices = nat.ptr(K(dsp.indices, np.uint32))
            d.ds_data = nat.ptr(K(dsp.data, np.float32))
        d.sparse_weight = float(sw)
        d.dense_weight = float(dw)
        d.id_offset = int(id_offset)
        h = ctypes.c_void_p()
        nat.check(L.hs_index_create(ctypes.byref(d), int(device), ctypes.byref(h)))
        self._h = h
        self.device = device
        self.n, self.d_sparse, self.d_dense = n, d_sparse, d_dense
        self.has_dataset = ds is not None
        self.sparse_weight, self.dense_weight = float(sw), float(dw)

    @classmethod
    def from_handle(cls, h, device, n, d_sparse, d_dense, sparse_weight, dense_weight,
                    has_dataset=True):
        """Wrap an hs_index_t made elsewhere (hs_builder_finish)."""
        self = cls.__new__(cls)
        self._h = h
        self.device = int(device)
        self.n, self.d_sparse, self.d_dense = int(n), int(d_sparse), int(d_dense)
        self.has_dataset = bool(has_dataset)
        self.sparse_weight, self.dense_weight = float(sparse_weight), float(dense_weight)
        return self

    @property
    def handle(self):
        return self._h

    def memory_bytes(self) -> int:
        b = ctypes.c_int64()
        nat.check(nat.lib().hs_index_memory_bytes(self._h, ctypes.byref(b)))
        return int(b.value)

    def kernel_times(self) -> dict:
        ms = (ctypes.c_double * 64)()
        cnt = ctypes.c_int32()
        names = ctypes.create_string_buffer(4096)
        nat.check(nat.lib().hs_last_kernel_times(self._h, ms, 64, ctypes.byref(cnt), names, 4096))
        keys = names.value.decode().split(";") if cnt.value else []
        return {k: float(ms[i]) for i, k in enumerate(keys)}

    def set_timing(self, on: bool):
        nat.check(nat.lib().hs_set_timing(self._h, int(bool(on))))

    def launches(self) -> int:
        v = ctypes.c_int64()
        nat.check(nat.lib().hs_index_launches(self._h, ctypes.byref(v)))
        return int(v.value)

    def search_dev(self, qb, params, out_ids_ptr: int, out_scores_ptr: int, stream: int = 0):
        """Device-resident batch: qb fields are device pointers (see hs_search_batch_dev)."""
        nat.check(nat.lib().hs_search_batch_dev(self._h, ctypes.byref(qb), ctypes.byref(params),
                                                ctypes.c_void_p(out_ids_ptr),
                                                ctypes.c_void_p(out_scores_ptr),
                                                ctypes.c_void_p(stream)))

    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            nat.lib().hs_index_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _posting_arrays(sidx):
    """(dims, ptr, ids, w) from our InvertedIndex or the reference's dict form."""
    if hasattr(sidx, "ids") and hasattr(sidx, "ptr") and hasattr(sidx, "dims"):
        return sidx.dims, sidx.ptr, sidx.ids, sidx.w
    tmp = InvertedIndex(sidx.n, sidx.d_sparse, sidx.order, sidx.lists)
    return tmp.dims, tmp.ptr, tmp.ids, tmp.w


def device_index(index, device: int = 0) -> DeviceIndex:
    """Cached device handle for a (reference-compatible) HybridIndex."""
    if hasattr(index, "device_handle"):  # built on the GPU (devbuild.DeviceBuiltIndex)
        return index.device_handle(device)
    cfg = index.config
    key = (int(device), float(cfg.sparse_weight), float(cfg.dense_weight),
           index.dataset is not None, id(index.dataset))
    with _CACHE_LOCK:
        cache = index.__dict__.setdefault(_HANDLE_ATTR, {})
        h = cache.get(key)
        if h is None:
            cache.clear()
            h = DeviceIndex(index, device=device)
            cache[key] = h
    return h


# ----------------------------------------------------------------------------
# query marshalling
# ----------------------------------------------------------------------------
class QueryArrays:
    """CSR sparse parts + dense rows of a query set, host side."""

    def __init__(self, indptr, dims, vals, dense):
        self.indptr = nat.contig(indptr, np.int64)
        self.dims = nat.contig(dims, np.uint32)
        self.vals = nat.contig(vals, np.float32)
        self.dense = nat.contig(dense, np.float32)
        self.nq = len(self.indptr) - 1

    def batch(self) -> nat.QueryBatch:
        b = nat.QueryBatch()
        b.nq = self.nq
        b.sp_indptr = nat.ptr(self.indptr)
        b.sp_dims = nat.ptr(self.dims)
        b.sp_vals = nat.ptr(self.vals)
        b.dense = nat.ptr(self.dense) if self.dense.size else None
        b.nnz = int(self.indptr[-1] - self.indptr[0]) if self.nq else 0
        lens = np.diff(self.indptr)
        b.max_row_nnz = int(lens.max()) if self.nq else 0
        return b


def query_arrays(queries, d_dense: int) -> QueryArrays:
    if isinstance(queries, QueryArrays):
        return queries
    if hasattr(queries, "sparse") and hasattr(queries, "dense") and hasattr(queries, "n"):
        s = sp.csr_matrix(queries.sparse)
        dense = np.asarray(queries.dense, dtype=np.float32).reshape(s.shape[0], -1)
        return QueryArrays(s.indptr, s.indices, s.data, dense)
    if isinstance(queries, HybridVector) or hasattr(queries, "sparse") and hasattr(queries, "dense"):
        queries = [queries]
    qs = list(queries)
    lens = [len(q.sparse.dims) for q in qs]
    indptr = np.concatenate(([0], np.cumsum(lens))).astype(np.int64)
    dims = (np.concatenate([np.asarray(q.sparse.dims) for q in qs]) if qs else np.zeros(0))
    vals = (np.concatenate([np.asarray(q.sparse.values, np.float32) for q in qs]) if qs
            else np.zeros(0))
    dense_rows = [np.asarray(q.dense, np.float32).reshape(-1) for q in qs]
    for r in dense_rows:
        if r.shape[0] != d_dense:
            raise ValueError("query dense dimension mismatch")
    dense = np.stack(dense_rows) if qs and d_dense else np.zeros((len(qs), d_dense), np.float32)
    return QueryArrays(indptr, dims, vals, dense)


def _validate_queries(q: QueryArrays, d_sparse: int, d_dense: int):
    if q.dense.shape != (q.nq, d_dense) and not (d_dense == 0 and q.dense.size == 0):
        raise ValueError("query dense dimension mismatch")
    if q.dims.size:
        if int(q.dims.max()) >= d_sparse:
            raise ValueError("query sparse dimension out of range")


# ----------------------------------------------------------------------------
# the hot path
# ----------------------------------------------------------------------------
def resolve_params(index, h=None, overfetch=None, retain=None, exact_final_rerank=None):
    """hs_search_params for an index + overrides (validated like the reference)."""
    return _resolve(index, h, overfetch, retain, exact_final_rerank)


def _resolve(index, h, overfetch, retain, exact_final_rerank):
    cfg = index.config
    h = cfg.h if h is None else int(h)
    if h < 1:
        raise ValueError("h must be >= 1")
    alpha = cfg.overfetch if overfetch is None else overfetch
    beta = cfg.retain if retain is None else retain
    exact = cfg.exact_final_rerank if exact_final_rerank is None else exact_final_rerank
    if not (alpha >= beta >= 1.0):
        raise ValueError("need overfetch >= retain >= 1")
    if exact and index.dataset is None:
        raise ValueError("exact_final_rerank requires the original dataset")
    if index.dense_index is not None and index.dense_index.codes.n_centers != LUT16_CENTERS:
        raise ValueError("lut16_scan requires 16-center codes")
    p = nat.SearchParams()
    p.h, p.overfetch, p.retain, p.exact_final_rerank = h, float(alpha), float(beta), int(bool(exact))
    return p


def search_batch(index, queries, h: int | None = None, threads: int = 1, device: int = 0,
                 **overrides) -> list:
    """Batched three-stage search on the GPU; results in query order.

    `threads` is accepted for API compatibility and ignored: the whole batch
    runs as one GPU pipeline (results are identical for any value).
    """
    del threads
    p = _resolve(index, h, overrides.get("overfetch"), overrides.get("retain"),
                 overrides.get("exact_final_rerank"))
    q = query_arrays(queries, int(index.d_dense))
    _validate_queries(q, int(index.d_sparse), int(index.d_dense))
    if q.nq == 0:
        return []
    dev = device_index(index, device)
    counts = np.zeros(3, dtype=np.int64)
    nat.check(nat.lib().hs_result_sizes(dev.handle, ctypes.byref(p), nat.ptr(counts)))
    k1, k2, kh = (int(x) for x in counts)
    ids = np.empty((q.nq, kh), dtype=np.int64)
    scores = np.empty((q.nq, kh), dtype=np.float64)
    secs = np.zeros(3, dtype=np.float64)
    b = q.batch()
    call = lambda: nat.lib().hs_search_batch(dev.handle, ctypes.byref(b), ctypes.byref(p),  # noqa: E731
                                             nat.ptr(ids), nat.ptr(scores), nat.ptr(secs))
    if q.nq < 64:
        nat.check(call())
        per_q = (secs / q.nq).tolist()
        return [SearchResult(i_row, s_row, StageStats([k1, k2, kh], per_q.copy()))
                for i_row, s_row in zip(list(ids), list(scores))]
    # Large batches: the C call (which releases the GIL) runs on a worker
    # thread while this thread builds the result objects around row views of
    # the output arrays; the rows are filled when the call returns.
    started = threading.Event()

    def run():
        started.set()  # the ctypes call below releases the GIL
        nat.check(call())  # (hs_last_error is thread-local: check on this thread)

    fut = _worker().submit(run)
    started.wait()  # blocks (GIL released) until the worker is about to call in
    stats = [StageStats([k1, k2, kh], [0.0, 0.0, 0.0]) for _ in range(q.nq)]
    res = [SearchResult(i_row, s_row, st) for i_row, s_row, st in zip(list(ids), list(scores), stats)]
    fut.result()
    per_q = (secs / q.nq).tolist()
    for st in stats:
        st.seconds[:] = per_q
    return res


_WORKER = None
_WORKER_LOCK = threading.Lock()


def _worker():
    global _WORKER
    if _WORKER is None:
        with _WORKER_LOCK:
            if _WORKER is None:
                import concurrent.futures as cf

                _WORKER = cf.ThreadPoolExecutor(max_workers=4, thread_name_prefix="hsb200")
    return _WORKER


def search_topk(index, query, h: int | None = None, *, overfetch=None, retain=None,
                exact_final_rerank=None, device: int = 0) -> SearchResult:
    """Three-stage approximate top-h for one query (GPU)."""
    if len(np.asarray(query.dense).reshape(-1)) != int(index.d_dense):
        raise ValueError("query dense dimension mismatch")
    return search_batch(index, [query], h, overfetch=overfetch, retain=retain,
                        exact_final_rerank=exact_final_rerank, device=device)[0]


def stage1_scores(index, queries, device: int = 0) -> np.ndarray:
    """Stage-1 approximate scores, layout order, weights applied (pipeline.py:192-203)."""
    q = query_arrays(queries, int(index.d_dense))
    _validate_queries(q, int(index.d_sparse), int(index.d_dense))
    dev = device_index(index, device)
    out = np.empty((q.nq, int(index.n)), dtype=np.float64)
    b = q.batch()
    nat.check(nat.lib().hs_stage1_scores(dev.handle, ctypes.byref(b), nat.ptr(out)))
    return out


# ----------------------------------------------------------------------------
# unit functions
# ----------------------------------------------------------------------------
def select_topk(scores, k: int, tie_ids=None) -> np.ndarray:
    """Exact top-k positions by (score desc, tie id asc) on the GPU."""
    s = nat.contig(scores, np.float64)
    single = s.ndim == 1
    s2 = s.reshape(1, -1) if single else s
    nq, n = s2.shape
    k = min(int(k), n)
    if k <= 0:
        return np.empty(0 if single else (nq, 0), dtype=np.int64)
    nat.require_gpu()
    t = None if tie_ids is None else nat.contig(tie_ids, np.int64)
    if t is not None and t.size and (t.min() < 0 or t.max() >= 2 ** 32 - 1):
        # order-preserving remap to dense ranks keeps the tie order
        t = np.argsort(np.argsort(t, kind="stable"), kind="stable").astype(np.int64)
    out = np.empty((nq, k), dtype=np.int64)
    nat.check(nat.lib().hs_select_topk(nat.ptr(s2), nq, n, k, nat.ptr(t), nat.ptr(out)))
    return out[0] if single else out


def _subspace_meta(codebooks):
    sub = nat.contig(codebooks.subdims, np.int32)
    cen = nat.contig(np.concatenate([np.asarray(c, np.float32).reshape(-1)
                                     for c in codebooks.centers]), np.float32)
    return sub, cen


def adc_table(query_dense, codebooks) -> np.ndarray:
    """T[k][c] = <query slice k, center c> (f64), computed on the GPU."""
    q = np.asarray(query_dense, dtype=np.float64)
    if q.shape != (codebooks.d_dense,):
        raise ValueError("query dense dimension mismatch")
    nat.require_gpu()
    sub, cen = _subspace_meta(codebooks)
    K, l = codebooks.n_subspaces, codebooks.n_centers
    T = np.empty((K, l), dtype=np.float64)
    q = nat.contig(q, np.float64)
    nat.check(nat.lib().hs_adc_table(nat.ptr(cen), nat.ptr(sub), K, l, nat.ptr(q), 1,
                                     q.shape[0], nat.ptr(T)))
    return T


def _sq_rows(r, rows):
    codes = np.ascontiguousarray(r.codes, dtype=np.uint8)
    if codes.ndim != 2:
        raise ValueError("codes must be (n, d)")
    n, d = codes.shape
    if isinstance(rows, slice):
        idx = np.arange(n, dtype=np.int64)[rows]
    else:
        idx = np.asarray(rows)
        if idx.dtype == bool:
            idx = np.flatnonzero(idx)
        idx = np.where(idx < 0, idx + n, idx).astype(np.int64).reshape(-1)
    return codes, n, d, nat.contig(r.lo, np.float32), nat.contig(r.step, np.float32), \
        nat.contig(idx, np.int64)


def sq_residual_decode(r, rows=slice(None)) -> np.ndarray:
    """ScalarQuantResidual.decode (dense.py:369-371) on the GPU: f64 rows."""
    codes, n, d, lo, step, idx = _sq_rows(r, rows)
    nat.require_gpu()
    out = np.empty((len(idx), d), dtype=np.float64)
    nat.check(nat.lib().hs_sq_decode(nat.ptr(codes), n, d, nat.ptr(lo), nat.ptr(step),
                                     nat.ptr(idx), len(idx), nat.ptr(out)))
    return out


def sq_residual_dot(r, rows, q) -> np.ndarray:
    """ScalarQuantResidual.dot (dense.py:373-375) on the GPU: decode(rows) @ q."""
    codes, n, d, lo, step, idx = _sq_rows(r, rows)
    qv = nat.contig(np.asarray(q, dtype=np.float64).reshape(-1), np.float64)
    if qv.shape[0] != d:
        raise ValueError(f"shapes ({len(idx)},{d}) and ({qv.shape[0]},) not aligned")
    nat.require_gpu()
    out = np.empty(len(idx), dtype=np.float64)
    nat.check(nat.lib().hs_sq_residual_dot(nat.ptr(codes), n, d, nat.ptr(lo), nat.ptr(step),
                                           nat.ptr(idx), len(idx), nat.ptr(qv), nat.ptr(out)))
    return out


def sq_decode(r) -> np.ndarray:
    """sq_decode (dense.py:393-394): every row decoded, on the GPU."""
    return sq_residual_decode(r)


def quantize_lut(table) -> QuantizedLUT:
    """Shared-scale 8-bit LUT (bias, scale, u8 table, bias_total) on the GPU."""
    T = nat.contig(table, np.float64)
    if T.ndim != 2:
        raise ValueError("table must be 2-D")
    if not np.all(np.isfinite(T)):
        raise ValueError("lookup table contains non-finite values")
    nat.require_gpu()
    K, l = T.shape
    tab = np.empty((K, l), dtype=np.uint8)
    bias = np.empty(K, dtype=np.float64)
    scale = np.empty(1, dtype=np.float64)
    bt = np.empty(1, dtype=np.float64)
    nat.check(nat.lib().hs_quantize_lut(nat.ptr(T), 1, K, l, nat.ptr(tab), nat.ptr(bias),
                                        nat.ptr(scale), nat.ptr(bt)))
    return QuantizedLUT(bias=bias, scale=float(scale[0]), table=tab, _bias_total=float(bt[0]))


def _lut16(packed, n, K, qlut):
    tab = nat.contig(qlut.table, np.uint8)
    if tab.shape != (K, LUT16_CENTERS):
        raise ValueError("LUT shape does not match the codes")
    nat.require_gpu()
    pk = nat.contig(packed, np.uint8)
    bt = np.array([qlut.bias_total], dtype=np.float64)
    sc = np.array([qlut.scale], dtype=np.float64)
    tot = np.empty(n, dtype=np.int32)
    out = np.empty(n, dtype=np.float64)
    if n:
        nat.check(nat.lib().hs_lut16_scan(nat.ptr(pk), n, K, nat.ptr(tab), nat.ptr(bt), nat.ptr(sc),
                                          1, nat.ptr(tot), nat.ptr(out)))
    return out, tot


def lut16_scan(codes: PQCodes, qlut: QuantizedLUT) -> np.ndarray:
    """bias_total + scale * sum_k table[k][code_k] for every point (GPU)."""
    if codes.n_centers != LUT16_CENTERS:
        raise ValueError("lut16_scan requires 16-center codes")
    return _lut16(codes.packed, int(codes.n), int(codes.n_subspaces), qlut)[0]


def lut16_totals(codes: PQCodes, qlut: QuantizedLUT) -> np.ndarray:
    """The integer totals of the scan (for parity checks)."""
    if codes.n_centers != LUT16_CENTERS:
        raise ValueError("lut16_scan requires 16-center codes")
    return _lut16(codes.packed, int(codes.n), int(codes.n_subspaces), qlut)[1]


def lut16_scan_reference(codes: np.ndarray, qlut: QuantizedLUT) -> np.ndarray:
    """Same semantics from an unpacked (n, K) code matrix."""
    from .builder import pack_codes

    c = np.asarray(codes, dtype=np.uint8)
    return _lut16(pack_codes(c), c.shape[0], c.shape[1], qlut)[0]


def _lines_touched(sidx, qdims, line_capacity):
    """Cache-line instrumentation of the reference Accumulator (sparse.py:261-265)."""
    dims, ptr, ids, _ = _posting_arrays(sidx)
    total = 0
    for j in np.asarray(qdims, dtype=np.int64):
        k = int(np.searchsorted(dims, j))
        if k < len(dims) and dims[k] == j:
            seg = ids[ptr[k]:ptr[k + 1]].astype(np.int64) // line_capacity
            if seg.size:
                total += 1 + int(np.count_nonzero(seg[1:] != seg[:-1]))
    return total


def sparse_scan(index, query: SparseVector, acc: Accumulator, device: int = 0) -> Accumulator:
    """acc.scores[layout slot] += sum_j q_j * w over the query's posting lists (GPU)."""
    q = query
    dims = np.asarray(q.dims, dtype=np.int64)
    if dims.size and int(dims.max()) >= int(index.d_sparse):
        raise ValueError("query dimension out of range for this index")
    with _CACHE_LOCK:
        cache = index.__dict__.setdefault(_HANDLE_ATTR, {})
        h = cache.get(("sparse", device))
        if h is None:
            h = DeviceIndex(sparse_index=index, device=device)
            cache[("sparse", device)] = h
    qa = QueryArrays(np.array([0, dims.size]), dims, q.values, np.zeros((1, 0), np.float32))
    b = qa.batch()
    if np.any(acc.scores):
        # non-zero accumulator: products added onto it one dim at a time, in
        # the query's (ascending) dim order, like sparse.py:277-282
        out = np.ascontiguousarray(acc.scores, dtype=np.float64).reshape(1, -1).copy()
        nat.check(nat.lib().hs_sparse_scan_into(h.handle, ctypes.byref(b), nat.ptr(out)))
    else:
        out = np.empty((1, int(index.n)), dtype=np.float64)
        nat.check(nat.lib().hs_sparse_scan(h.handle, ctypes.byref(b), nat.ptr(out)))
    acc.scores[:] = out[0]
    acc.lines_touched += _lines_touched(index, dims, acc.line_capacity)
    return acc


def brute_force_topk(dataset: HybridDataset, query, h: int, sparse_weight: float = 1.0,
                     dense_weight: float = 1.0, device: int = 0):
    """Exact top-h by hybrid inner product, ties to the lower id (GPU)."""
    ids, sc = brute_force_batch(dataset, [query], h, sparse_weight, dense_weight, device)
    return ids[0], sc[0]


def brute_force_batch(dataset: HybridDataset, queries, h: int, sparse_weight: float = 1.0,
                      dense_weight: float = 1.0, device: int = 0):
    key = ("exact", device, float(sparse_weight), float(dense_weight))
    with _CACHE_LOCK:
        cache = dataset.__dict__.setdefault(_HANDLE_ATTR, {})
        dev = cache.get(key)
        if dev is None:
            dev = DeviceIndex(dataset=dataset, device=device, sparse_weight=sparse_weight,
                              dense_weight=dense_weight)
            cache[key] = dev
    q = query_arrays(queries, int(dataset.d_dense))
    _validate_queries(q, int(dataset.d_sparse), int(dataset.d_dense))
    kh = min(int(h), int(dataset.n))
    ids = np.empty((q.nq, kh), dtype=np.int64)
    sc = np.empty((q.nq, kh), dtype=np.float64)
    b = q.batch()
    nat.check(nat.lib().hs_exact_topk(dev.handle, ctypes.byref(b), int(h), nat.ptr(ids),
                                      nat.ptr(sc)))
    return ids, sc


def exact_topk(index, queries, h: int, device: int = 0):
    """Exact top-h over the index's own raw dataset (brute_force_topk semantics,
    harness.py:25-35, with the index's weights); works for GPU-built indices,
    whose dataset lives only on the device."""
    dev = device_index(index, device)
    q = query_arrays(queries, int(index.d_dense))
    _validate_queries(q, int(index.d_sparse), int(index.d_dense))
    kh = min(int(h), int(index.n))
    ids = np.empty((q.nq, kh), dtype=np.int64)
    sc = np.empty((q.nq, kh), dtype=np.float64)
    b = q.batch()
    nat.check(nat.lib().hs_exact_topk(dev.handle, ctypes.byref(b), int(h), nat.ptr(ids),
                                      nat.ptr(sc)))
    return ids, sc


def recall_at_h(returned_ids, truth_ids, h: int) -> float:
    return len(np.intersect1d(np.asarray(returned_ids), np.asarray(truth_ids))) / h
