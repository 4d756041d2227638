"""CPU restatement of the reference index build, plus a numpy generator of the
BASELINE data laws.

TEST INFRASTRUCTURE ONLY (like hybrid_oracle.py): used by `bench.py
--impl reference` to build the reference arm's index with no product
library loaded, and by tests as a checker.  Nothing in the product package
imports it.

Follows /root/reference/pkg/src/hybridsearch:
    top_t_thresholds   sparse.py:66-80   (sort per column instead of a loop)
    prune_split        sparse.py:83-103
    cache_sort         sparse.py:106-163 (one lexsort over padded rank lists:
                       same order as the packed-key sort + _refine_equal_runs)
    build_inverted     sparse.py:219-235
    whiten_fit/apply   dense.py:333-357
    train_codebooks    dense.py:65-135   (k-means++ seeding, Lloyd, repair)
    pq_encode          dense.py:138-153
    pack_codes         dense.py:156-170
    sq_encode          dense.py:381-390
    build_index        pipeline.py:119-162
The products are pinned to the reference's own build fixtures in
tests/test_oracle_build.py (bit-identical integer products).
"""

from __future__ import annotations

import math
from types import SimpleNamespace

import numpy as np
import scipy.sparse as sp


# ---------------------------------------------------------------------------
# sparse part
# ---------------------------------------------------------------------------
def top_t_thresholds(matrix, t):
    """eta[j] = t-th largest |v| of column j, 0 when nnz_j <= t (sparse.py:66-80)."""
    d = matrix.shape[1]
    if t == 0:
        return np.full(d, np.inf)
    csc = sp.csc_matrix(matrix)
    csc.sort_indices()
    nnz = np.diff(csc.indptr)
    absv = np.abs(csc.data.astype(np.float64))
    col = np.repeat(np.arange(d), nnz)
    o = np.lexsort((absv, col))  # ascending |v| within each column
    sv = absv[o]
    eta = np.zeros(d, dtype=np.float64)
    big = np.flatnonzero(nnz > t)
    eta[big] = sv[csc.indptr[big] + nnz[big] - t]
    return eta


def resolve_thresholds(config, matrix):
    d = matrix.shape[1]
    if config.data_threshold is not None:
        eta = np.broadcast_to(np.asarray(config.data_threshold, dtype=np.float64), (d,)).copy()
    elif config.top_t is None:
        eta = np.zeros(d)
    else:
        eta = top_t_thresholds(matrix, config.top_t)
    eps = np.broadcast_to(np.asarray(config.residual_threshold, dtype=np.float64), (d,)).copy()
    if np.any(eps > eta):
        raise ValueError("residual_min must be <= data_min in every dimension")
    return eta, eps


def prune_split(matrix, config):
    """(data part, residual part) CSR (sparse.py:83-103)."""
    m = sp.csr_matrix(matrix)
    eta, eps = resolve_thresholds(config, m)
    absv = np.abs(m.data.astype(np.float64))
    in_data = absv >= eta[m.indices]
    in_res = ~in_data & (absv >= eps[m.indices])

    def sel(mask):
        out = sp.csr_matrix((np.where(mask, m.data, 0).astype(m.data.dtype), m.indices.copy(),
                             m.indptr.copy()), shape=m.shape)
        out.eliminate_zeros()
        return out

    return sel(in_data), sel(in_res)


def cache_sort(data_part):
    """Layout permutation order[slot] = original id (sparse.py:106-163).

    Points sorted by their activity over the dims ranked (nnz desc, dim asc),
    descending lexicographically, stably: each point's ascending rank list
    with an +inf terminator, compared ascending, ties by id.
    """
    m = sp.csr_matrix(data_part)
    n, d = m.shape
    nnz = np.bincount(m.indices, minlength=d)
    ranked = np.lexsort((np.arange(d), -nnz))
    ranked = ranked[nnz[ranked] > 0]
    if n == 0 or len(ranked) == 0:
        return np.arange(n, dtype=np.int64)
    rank = np.empty(d, dtype=np.int64)
    rank[ranked] = np.arange(len(ranked))
    lens = np.diff(m.indptr)
    L = int(lens.max()) + 1
    inf = len(ranked)
    pad = np.full((n, L), inf, dtype=np.int64)
    r = rank[m.indices]
    row = np.repeat(np.arange(n), lens)
    o = np.lexsort((r, row))  # ranks ascending within each row
    pos = np.arange(m.nnz) - np.repeat(m.indptr[:-1], lens)
    pad[row[o], pos] = r[o]
    keys = [np.arange(n)] + [pad[:, j] for j in range(L - 1, -1, -1)]
    return np.lexsort(keys).astype(np.int64)


def build_inverted(data_part, order):
    """Posting lists (dims asc, layout slots asc) as CSR arrays (sparse.py:219-235)."""
    m = sp.csr_matrix(data_part)
    n, d = m.shape
    pos = np.empty(n, dtype=np.int64)
    pos[order] = np.arange(n)
    lens = np.diff(m.indptr)
    slots = pos[np.repeat(np.arange(n), lens)]
    o = np.lexsort((slots, m.indices))
    cols = m.indices[o]
    dims, counts = np.unique(cols, return_counts=True)
    return SimpleNamespace(n=n, d_sparse=d, order=np.asarray(order, dtype=np.int64),
                           dims=dims.astype(np.int64),
                           ptr=np.concatenate(([0], np.cumsum(counts))).astype(np.int64),
                           ids=slots[o].astype(np.uint32), w=m.data[o].astype(np.float32))


# ---------------------------------------------------------------------------
# dense part
# ---------------------------------------------------------------------------
def whiten_fit(X, ridge_scale=1e-6):
    X = np.asarray(X, dtype=np.float64)
    mean = X.mean(axis=0)
    d = X.shape[1]
    cov = np.cov(X, rowvar=False, bias=True).reshape(d, d)
    if np.trace(cov) == 0.0:
        eye = np.eye(d)
        return SimpleNamespace(forward=eye, inverse_t=eye.copy(), mean=mean)
    ridge = ridge_scale * np.trace(cov) / d
    w, V = np.linalg.eigh(cov + ridge * np.eye(d))
    return SimpleNamespace(forward=(V * (w ** -0.5)) @ V.T, inverse_t=(V * (w ** 0.5)) @ V.T,
                           mean=mean)


def whiten_apply(t, v):
    return (np.asarray(v, dtype=np.float64) - t.mean) @ t.forward.T


def subspace_widths(d, K):
    base, rem = divmod(d, K)
    return np.array([base + 1] * rem + [base] * (K - rem), dtype=np.int64)


def _kmeanspp(x, k, rng):
    n = x.shape[0]
    c = np.empty((k, x.shape[1]))
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


def _dist(x, sq, c):
    return sq[:, None] - 2.0 * (x @ c.T) + np.sum(c ** 2, axis=1)[None, :]


def _lloyd(x, k, iters, rng):
    c = _kmeanspp(x, k, rng)
    sq = np.sum(x ** 2, axis=1)
    d2 = _dist(x, sq, c)
    for _ in range(iters):
        a = np.argmin(d2, axis=1)
        cnt = np.bincount(a, minlength=k)
        for e in np.flatnonzero(cnt == 0):
            big = int(np.argmax(cnt))
            mem = np.flatnonzero(a == big)
            far = mem[int(np.argmax(d2[mem, big]))]
            a[far] = e
            cnt[big] -= 1
            cnt[e] = 1
        for j in range(k):
            if cnt[j]:
                c[j] = x[a == j].mean(axis=0)
        d2 = _dist(x, sq, c)
    return c


def train_codebooks(X, K, n_centers=16, n_iters=25, seed=0, sample=None):
    X = np.asarray(X, dtype=np.float64)
    n, d = X.shape
    widths = subspace_widths(d, K)
    seqs = np.random.SeedSequence(seed).spawn(1 + K)
    if sample is not None and n_centers <= sample < n:
        X = X[np.sort(np.random.default_rng(seqs[0]).choice(n, size=sample, replace=False))]
    edges = np.concatenate(([0], np.cumsum(widths)))

    def one(k):  # each subspace owns its RNG stream: thread order cannot matter
        return _lloyd(np.ascontiguousarray(X[:, edges[k]:edges[k + 1]]), n_centers, n_iters,
                      np.random.default_rng(seqs[1 + k])).astype(np.float32)

    import os
    from concurrent.futures import ThreadPoolExecutor

    with ThreadPoolExecutor(max_workers=max(1, min(K, os.cpu_count() or 1))) as ex:
        centers = list(ex.map(one, range(K)))
    return SimpleNamespace(subdims=widths, centers=centers, n_subspaces=K, n_centers=n_centers,
                           d_dense=d)


def pq_encode(X, cb):
    X = np.asarray(X, dtype=np.float64)
    edges = np.concatenate(([0], np.cumsum(cb.subdims)))
    codes = np.empty((X.shape[0], cb.n_subspaces), dtype=np.uint8)
    for k in range(cb.n_subspaces):
        sub = X[:, edges[k]:edges[k + 1]]
        c = cb.centers[k].astype(np.float64)
        d2 = np.sum(sub ** 2, axis=1)[:, None] - 2.0 * (sub @ c.T) + np.sum(c ** 2, axis=1)[None, :]
        codes[:, k] = np.argmin(d2, axis=1)
    return codes


def pack_codes(codes):
    n, K = codes.shape
    packed = np.zeros(((K + 1) // 2, n), dtype=np.uint8)
    packed[:] = codes[:, 0::2].T
    if K > 1:
        packed[: K // 2] |= codes[:, 1::2].T << 4
    return packed


def reconstruct(cb, codes):
    edges = np.concatenate(([0], np.cumsum(cb.subdims)))
    out = np.empty((codes.shape[0], cb.d_dense), dtype=np.float32)
    for k in range(cb.n_subspaces):
        out[:, edges[k]:edges[k + 1]] = cb.centers[k][codes[:, k]]
    return out


def sq_encode(X):
    X = np.asarray(X, dtype=np.float64)
    lo = X.min(axis=0) if X.shape[0] else np.zeros(X.shape[1])
    hi = X.max(axis=0) if X.shape[0] else np.zeros(X.shape[1])
    step = (hi - lo) / 256.0
    safe = np.where(step > 0, step, 1.0)
    codes = np.clip(np.floor((X - lo) / safe), 0, 255).astype(np.uint8)
    return SimpleNamespace(lo=lo.astype(np.float32), step=step.astype(np.float32), codes=codes)


def build_index(dataset, config):
    """build_index (pipeline.py:119-162): a duck-typed index hybrid_oracle searches."""
    data_part, residual_part = prune_split(dataset.sparse, config)
    order = cache_sort(data_part)
    sidx = build_inverted(data_part, order)
    res = residual_part[order].tocsr()
    res.sort_indices()
    dense_index = None
    if dataset.dense.shape[1] > 0:
        vec = dataset.dense.astype(np.float64)
        wt = None
        if config.use_whitening:
            wt = whiten_fit(vec)
            vec = whiten_apply(wt, vec)
        K = config.pq_subspaces or max(1, math.ceil(vec.shape[1] / 2))
        cb = train_codebooks(vec, K, n_centers=config.pq_centers, n_iters=config.kmeans_iters,
                             seed=config.seed, sample=config.train_sample)
        codes = pq_encode(vec, cb)[order]
        residual = sq_encode(vec[order] - reconstruct(cb, codes))
        dense_index = SimpleNamespace(
            codebooks=cb, whitening=wt, residual=residual,
            codes=SimpleNamespace(n=dataset.sparse.shape[0], n_subspaces=K,
                                  n_centers=config.pq_centers, packed=pack_codes(codes)))
    return SimpleNamespace(config=config, n=dataset.sparse.shape[0],
                           d_sparse=dataset.sparse.shape[1], d_dense=dataset.dense.shape[1],
                           order=order, sparse_index=sidx, sparse_residual=res,
                           dense_index=dense_index, dataset=dataset)


# ---------------------------------------------------------------------------
# numpy generator of the BASELINE data laws
# ---------------------------------------------------------------------------
_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def _mix64(z):
    with np.errstate(over="ignore"):  # uint64 arithmetic wraps mod 2^64 on purpose
        z = (z + np.uint64(0x9E3779B97F4A7C15)) & _M64
        z = ((z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)) & _M64
        z = ((z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)) & _M64
        return z ^ (z >> np.uint64(31))


def feistel(x, d, seed):
    """The seeded bijection of [0, d) the generators share (4 Feistel rounds on
    2w bits + cycle walking; hostbuild.cpp / devbuild.cu restate the same map)."""
    bits = 2
    while (1 << bits) < d:
        bits += 2
    half = np.uint64(bits // 2)
    mask = np.uint64((1 << (bits // 2)) - 1)
    keys = [_mix64(np.uint64(seed) ^ np.uint64(0xA5A5A5A5 + r)) for r in range(4)]

    def once(v):
        L, R = v >> half, v & mask
        for r in range(4):
            F = _mix64(R ^ keys[r]) & mask
            L, R = R, L ^ F
        return (L << half) | R

    with np.errstate(over="ignore"):
        y = once(np.asarray(x, dtype=np.uint64))
        bad = y >= np.uint64(d)
        while bad.any():
            y[bad] = once(y[bad])
            bad = y >= np.uint64(d)
    return y.astype(np.int64)


def generate(n, d_sparse, d_dense, mean_nnz, zipf_s, value_law="absnormal",
             dense_fp16=False, seed=0, perm_seed=0x5EED19030869):
    """A dataset with the law (not byte-identical to the GPU generator: the
    reference arm times the search on its own index of the same law)."""
    rng = np.random.default_rng(seed)
    k = np.minimum(rng.poisson(mean_nnz, size=n), d_sparse) if d_sparse else np.zeros(n, int)
    table = min(d_sparse, 1 << 22)
    if d_sparse:
        p = np.arange(1, table + 1, dtype=np.float64) ** -zipf_s
        cdf = np.cumsum(p)
        tail = 0.0
        if d_sparse > table:
            a, b = table + 0.5, d_sparse + 0.5
            tail = (a ** (1 - zipf_s) - b ** (1 - zipf_s)) / (zipf_s - 1)
        total = cdf[-1] + tail
    indptr = np.concatenate(([0], np.cumsum(k))).astype(np.int64)
    ranks = np.empty(int(indptr[-1]), dtype=np.int64)
    for i in range(n):  # distinct ranks per row (rejection)
        need, got = int(k[i]), np.empty(0, dtype=np.int64)
        while len(got) < need:
            u = rng.random(2 * (need - len(got)) + 8) * total
            r = np.searchsorted(cdf, u)
            t = u >= cdf[-1]
            if t.any():
                x = (table + 0.5) ** (1 - zipf_s) - (u[t] - cdf[-1]) * (zipf_s - 1)
                r[t] = np.clip(np.floor(x ** (1 / (1 - zipf_s)) - 0.5), table, d_sparse - 1)
            got = np.concatenate((got, r))
            _, first = np.unique(got, return_index=True)
            got = got[np.sort(first)]
        ranks[indptr[i]:indptr[i + 1]] = got[:need]
    dims = feistel(ranks, max(d_sparse, 1), perm_seed) if len(ranks) else ranks
    z = rng.standard_normal(len(ranks))
    vals = np.exp(z) if value_law == "lognormal" else np.abs(z)
    dense = rng.standard_normal((n, d_dense))
    ss = np.add.reduceat(vals ** 2, indptr[:-1]) if len(vals) else np.zeros(n)
    ss = np.where(k > 0, ss, 0.0) + np.sum(dense ** 2, axis=1)
    inv = np.where(ss > 0, 1.0 / np.sqrt(ss), 1.0)
    vals = (vals * np.repeat(inv, k)).astype(np.float32)
    dense = (dense * inv[:, None]).astype(np.float32)
    if dense_fp16:
        dense = dense.astype(np.float16).astype(np.float32)
    m = sp.csr_matrix((vals, dims, indptr), shape=(n, d_sparse))
    m.sort_indices()
    return SimpleNamespace(sparse=m, dense=dense, n=n, d_sparse=d_sparse, d_dense=d_dense)
