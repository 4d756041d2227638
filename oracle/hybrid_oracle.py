"""CPU oracle for the hybrid sparse+dense search hot path.

TEST INFRASTRUCTURE ONLY.  Nothing in the product package
(`paper_1903_08690_b200`) may import this module; only `tests/`,
`__graft_entry__.smoke()` and the `cpu_baseline` / `--impl reference` legs of
`bench.py` use it, and only as the checker / the timed CPU baseline.

This is a numpy restatement of the reference algorithm
(`/root/reference/pkg/src/hybridsearch`, the `hybridsearch` 0.1.0 package),
written against its semantics, not copied.  Each function names the reference
lines it follows.  It is pinned against golden vectors produced by the
reference itself (`tests/golden/make_golden.py`, checked by
`tests/test_oracle_golden.py`).

The index argument is duck-typed: anything exposing the reference
`HybridIndex` attribute names works (`config`, `n`, `d_sparse`, `d_dense`,
`order`, `sparse_index` with either `.lists` (reference dict form) or the
array form `.dims/.ptr/.ids/.w`, `sparse_residual` (CSR), `dense_index`,
`dataset`).
"""

from __future__ import annotations

import math

import numpy as np

_CHUNK = 256  # dense.py:22 — subspaces per 16-bit accumulation chunk


# --------------------------------------------------------------------------
# top-k selection                                     pipeline.py:165-189
# --------------------------------------------------------------------------
def select_topk(scores, k, tie_ids=None):
    """Positions of the k best entries by (score desc, tie id asc).

    Restates `select_topk` (pipeline.py:165-189) as a full lexicographic sort,
    which the reference documents as its definition (pipeline.py:168-170).
    """
    scores = np.asarray(scores, dtype=np.float64)
    n = scores.shape[0]
    k = min(int(k), n)
    if k <= 0:
        return np.empty(0, dtype=np.int64)
    ties = np.arange(n, dtype=np.int64) if tie_ids is None else np.asarray(tie_ids)
    # numpy treats -0.0 == 0.0; lexsort on -scores keeps that equivalence.
    perm = np.lexsort((ties, -scores))
    return perm[:k].astype(np.int64)


# --------------------------------------------------------------------------
# dense side: ADC table, LUT quantisation, LUT16 scan  dense.py:212-317
# --------------------------------------------------------------------------
def subspace_edges(subdims):
    """Contiguous subspace boundaries (dense.py:45-47)."""
    return np.concatenate(([0], np.cumsum(np.asarray(subdims, dtype=np.int64))))


def adc_table(qw, centers, subdims):
    """T[k][c] = <center c of subspace k, query slice k>  (dense.py:212-220).

    Uses numpy's matrix-vector product exactly like the reference so the
    oracle inherits the same BLAS arithmetic.
    """
    qw = np.asarray(qw, dtype=np.float64)
    edges = subspace_edges(subdims)
    K = len(centers)
    l = centers[0].shape[0]
    out = np.empty((K, l), dtype=np.float64)
    for k in range(K):
        out[k] = centers[k].astype(np.float64) @ qw[edges[k]:edges[k + 1]]
    return out


def quantize_lut(table):
    """(bias[K] f64, scale f64, u8 table[K,l])          (dense.py:248-260).

    bias = per-row min; scale = max(T - bias) / 255; entries rounded half to
    even then clipped; a zero scale yields the all-zero table.
    """
    T = np.asarray(table, dtype=np.float64)
    if not np.isfinite(T).all():
        raise ValueError("lookup table contains non-finite values")
    bias = T.min(axis=1)
    shifted = T - bias[:, None]
    spread = float(shifted.max()) if T.size else 0.0
    scale = spread / 255.0
    if scale == 0.0:
        q = np.zeros(T.shape, dtype=np.uint8)
    else:
        q = np.clip(np.rint(shifted / scale), 0, 255).astype(np.uint8)
    return bias, scale, q


def bias_total(bias):
    """`QuantizedLUT.bias_total` = numpy's own sum of the bias row (dense.py:243-245)."""
    return float(np.sum(np.asarray(bias, dtype=np.float64)))


def pairwise_sum(a):
    """Explicit restatement of numpy's pairwise summation for 1-D f64 arrays.

    Used to pin the recipe the CUDA kernel implements:
    blocks of < 8 are summed sequentially, up to 128 with 8 interleaved lanes
    combined as ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)) plus a sequential tail, and
    longer arrays split at a multiple of 8 near the middle.
    """
    a = [float(x) for x in a]

    def rec(lo, n):
        if n < 8:
            s = 0.0 if n == 0 else a[lo]
            for i in range(1, n):
                s += a[lo + i]
            return s
        if n <= 128:
            r = a[lo:lo + 8]
            i = 8
            while i < n - (n % 8):
                for j in range(8):
                    r[j] += a[lo + i + j]
                i += 8
            s = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]))
            while i < n:
                s += a[lo + i]
                i += 1
            return s
        n2 = (n // 2) - ((n // 2) % 8)
        return rec(lo, n2) + rec(lo + n2, n - n2)

    # the reduction starts from the additive identity (+0.0), so an all -0.0
    # input sums to +0.0 like np.sum
    return 0.0 + rec(0, len(a))


def lut16_totals_scalar(codes, qtable):
    """Scalar integer totals with 16-bit wrap per 256-subspace chunk.

    Restates `lut16_scan_reference` (dense.py:263-281) without the final affine
    step; codes is (n, K) uint8 with values < 16.  Pure Python: small n only.
    """
    codes = np.asarray(codes)
    n, K = codes.shape
    out = np.zeros(n, dtype=np.int64)
    for i in range(n):
        total = 0
        acc = 0
        for k in range(K):
            acc = (acc + int(qtable[k, codes[i, k]])) & 0xFFFF
            if (k + 1) % _CHUNK == 0:
                total += acc
                acc = 0
        out[i] = total + acc
    return out


def lut16_totals(packed, K, qtable):
    """Vectorised integer totals from pair-major packed codes.

    Restates `lut16_scan` (dense.py:297-317) with `_pair_table`
    (dense.py:288-294): byte b of pair p contributes table[2p][b & 15] and,
    if subspace 2p+1 exists, table[2p+1][b >> 4].  Accumulation is per
    256-subspace chunk in uint16 (wrapping), then widened.
    """
    packed = np.asarray(packed, dtype=np.uint8)
    npairs, n = packed.shape
    lo_nib = np.arange(256) & 0x0F
    hi_nib = np.arange(256) >> 4
    total = np.zeros(n, dtype=np.int64)
    for c0 in range(0, npairs, _CHUNK // 2):
        acc = np.zeros(n, dtype=np.uint16)
        for p in range(c0, min(c0 + _CHUNK // 2, npairs)):
            pt = qtable[2 * p].astype(np.uint16)[lo_nib]
            if 2 * p + 1 < K:
                pt = pt + qtable[2 * p + 1].astype(np.uint16)[hi_nib]
            acc += pt[packed[p]]
        total += acc
    return total


def lut16_scores(totals, bias_tot, scale):
    """bias_total + scale * f64(total)  — unfused (dense.py:280, dense.py:317)."""
    return bias_tot + scale * np.asarray(totals, dtype=np.float64)


def pack_codes(codes):
    """(n, K) 4-bit codes -> (ceil(K/2), n) pair-major bytes, low nibble = even
    subspace (dense.py:156-170)."""
    codes = np.asarray(codes, dtype=np.uint8)
    n, K = codes.shape
    out = np.zeros(((K + 1) // 2, n), dtype=np.uint8)
    out[:] = codes[:, 0::2].T
    if K > 1:
        out[: K // 2] |= (codes[:, 1::2].T << 4).astype(np.uint8)
    return out


# --------------------------------------------------------------------------
# sparse side                                         sparse.py:268-284
# --------------------------------------------------------------------------
def _posting_list(sidx, dim):
    """(ids u32, w f32) for one dim, from either index representation."""
    lists = getattr(sidx, "lists", None)
    if isinstance(lists, dict):
        return lists.get(int(dim))
    dims = np.asarray(sidx.dims)
    j = int(np.searchsorted(dims, dim))
    if j >= len(dims) or dims[j] != dim:
        return None
    lo, hi = int(sidx.ptr[j]), int(sidx.ptr[j + 1])
    return sidx.ids[lo:hi], sidx.w[lo:hi]


def sparse_scan(sidx, n, d_sparse, qdims, qvals, acc=None):
    """f64 accumulator in layout order (sparse.py:268-284).

    For each query dim in the order given (ascending), acc[ids] += f64(q) *
    f64(w).  Raises on an out-of-range dim like the reference (sparse.py:274-275).
    `acc` (optional) is the initial accumulator (Accumulator.scores), updated
    in place and returned.
    """
    qdims = np.asarray(qdims, dtype=np.int64)
    qvals = np.asarray(qvals, dtype=np.float32)
    if len(qdims) and int(qdims.max()) >= d_sparse:
        raise ValueError("query dimension out of range for this index")
    if acc is None:
        acc = np.zeros(n, dtype=np.float64)
    for j, v in zip(qdims, qvals):
        entry = _posting_list(sidx, j)
        if entry is None:
            continue
        ids, w = entry
        acc[np.asarray(ids, dtype=np.int64)] += float(v) * np.asarray(w).astype(np.float64)
    return acc


# --------------------------------------------------------------------------
# pipeline                                            pipeline.py:192-322
# --------------------------------------------------------------------------
def dense_query(index, qd):
    """(qw, offset): whitened query and mean-shift constant (pipeline.py:216-223,
    dense.py:351-357)."""
    wt = index.dense_index.whitening
    if wt is None:
        return qd, 0.0
    qw = qd @ wt.inverse_t.T
    return qw, float(qd @ wt.mean)


def query_lut(index, qdense):
    """Per-query LUT products: qw, offset, u8 table, bias, scale, bias_total."""
    cfg = index.config
    di = index.dense_index
    qd = np.asarray(qdense, dtype=np.float64) * cfg.dense_weight
    qw, offset = dense_query(index, qd)
    cb = di.codebooks
    T = adc_table(qw, cb.centers, cb.subdims)
    bias, scale, q = quantize_lut(T)
    return dict(qd=qd, qw=qw, offset=offset, T=T, bias=bias, scale=scale,
                table=q, bias_total=bias_total(bias))


def effective_sparse_values(index, qvals):
    """Stage-1 query values after sparse_weight, in f32 (pipeline.py:196-198)."""
    w = index.config.sparse_weight
    qvals = np.asarray(qvals, dtype=np.float32)
    if w != 1.0 and len(qvals):
        return (qvals * w).astype(np.float32)
    return qvals


def stage1_scores(index, qdims, qvals, qdense, want_parts=False):
    """Approximate scores for every layout slot (pipeline.py:192-213)."""
    sidx = index.sparse_index
    acc = sparse_scan(sidx, index.n, index.d_sparse, qdims,
                      effective_sparse_values(index, qvals))
    parts = dict(sparse=acc)
    scores = acc
    if index.dense_index is not None:
        lut = query_lut(index, qdense)
        codes = index.dense_index.codes
        if codes.n_centers != 16:
            raise ValueError("lut16_scan requires 16-center codes")
        totals = lut16_totals(codes.packed, codes.n_subspaces, lut["table"])
        dense = lut16_scores(totals, lut["bias_total"], lut["scale"]) + lut["offset"]
        scores = acc + dense
        parts.update(lut=lut, totals=totals, dense=dense)
    return (scores, parts) if want_parts else scores


def sq_residual_dot(residual, rows, qw):
    """Stage-2 SQ residual inner products (dense.py:369-375)."""
    c = residual.codes[rows].astype(np.float64)
    dec = residual.lo.astype(np.float64) + residual.step.astype(np.float64) * (c + 0.5)
    return dec @ np.asarray(qw, dtype=np.float64)


def dot_recipe(x, y):
    """One f64 dot product in the OpenBLAS `dgemv_t` order the kernels follow
    (SURVEY Appendix A.1): four FMA lanes over blocks of 4 combined as
    (L0+L2)+(L1+L3); a one-element tail is FMA'd onto that, a longer tail is
    summed as fma(x0, y0, x1*y1) (+ fma for a third) and then added.  Exact
    rational arithmetic stands in for the hardware FMA, so the result does not
    depend on this host's BLAS, thread count or batch shape (numpy's own
    `A @ v` rounds rows differently in the remainder kernels of a thread's
    row block).  Small inputs only (pure Python)."""
    from fractions import Fraction

    x = [float(v) for v in x]
    y = [float(v) for v in y]

    def fma(a, b, c):
        return float(Fraction(a) * Fraction(b) + Fraction(c))

    w = len(x)
    lanes = [0.0, 0.0, 0.0, 0.0]
    m = w - (w % 4)
    for i in range(0, m, 4):
        for j in range(4):
            lanes[j] = fma(x[i + j], y[i + j], lanes[j])
    base = (lanes[0] + lanes[2]) + (lanes[1] + lanes[3])
    rem = w - m
    if rem == 0:
        return base
    if rem == 1:
        return fma(x[m], y[m], base) if m else x[m] * y[m]
    p = fma(x[m], y[m], x[m + 1] * y[m + 1])
    for k in range(m + 2, w):
        p = fma(x[k], y[k], p)
    return base + p if m else p


def sparse_residual_dot(index, layout_rows, qdims, qvals):
    """Stage-3 residual term (pipeline.py:303-310)."""
    res = index.sparse_residual
    if len(qdims) == 0 or res.nnz == 0:
        return np.zeros(len(layout_rows), dtype=np.float64)
    qvec = np.zeros(index.d_sparse, dtype=np.float64)
    qvec[np.asarray(qdims, dtype=np.int64)] = np.asarray(qvals, dtype=np.float32).astype(np.float64)
    return res[layout_rows] @ qvec


def exact_scores(dataset, qdims, qvals, qdense, ids, sparse_weight=1.0, dense_weight=1.0):
    """Exact weighted hybrid scores for original ids (pipeline.py:313-322)."""
    qd = np.asarray(qdense, dtype=np.float32).astype(np.float64) * dense_weight
    out = dataset.dense[ids].astype(np.float64) @ qd
    if len(qdims):
        qvec = np.zeros(dataset.d_sparse, dtype=np.float64)
        qvec[np.asarray(qdims, dtype=np.int64)] = (
            np.asarray(qvals, dtype=np.float32).astype(np.float64) * sparse_weight)
        out = out + dataset.sparse[ids] @ qvec
    return out


def search_topk(index, qdims, qvals, qdense, h=None, overfetch=None, retain=None,
                exact_final_rerank=None, trace=None):
    """Three-stage search for one query (pipeline.py:226-279).

    Returns (ids int64 original, scores f64, candidates [k1, k2, kh]).  When
    `trace` is a dict it receives the intermediate stage outputs.
    """
    cfg = index.config
    h = cfg.h if h is None else h
    qdims = np.asarray(qdims, dtype=np.int64)
    qvals = np.asarray(qvals, dtype=np.float32)
    qdense = np.asarray(qdense, dtype=np.float32)
    if h < 1:
        raise ValueError("h must be >= 1")
    if len(qdense) != index.d_dense:
        raise ValueError("query dense dimension mismatch")
    if len(qdims) and int(qdims.max()) >= index.d_sparse:
        raise ValueError("query sparse dimension out of range")
    alpha = cfg.overfetch if overfetch is None else overfetch
    beta = cfg.retain if retain is None else retain
    exact = cfg.exact_final_rerank if exact_final_rerank is None else exact_final_rerank
    if not (alpha >= beta >= 1.0):
        raise ValueError("need overfetch >= retain >= 1")
    orig = np.asarray(index.order, dtype=np.int64)

    s1, parts = stage1_scores(index, qdims, qvals, qdense, want_parts=True)
    k1 = min(index.n, math.ceil(alpha * h))
    cand1 = select_topk(s1, k1, tie_ids=orig)

    s2 = s1[cand1]
    di = index.dense_index
    if di is not None and di.residual is not None:
        qw, _ = dense_query(index, qdense.astype(np.float64) * cfg.dense_weight)
        s2 = s2 + sq_residual_dot(di.residual, cand1, qw)
    k2 = min(len(cand1), math.ceil(beta * h))
    keep = select_topk(s2, k2, tie_ids=orig[cand1])
    cand2 = cand1[keep]
    s2 = s2[keep]

    if exact:
        if getattr(index, "dataset", None) is None:
            raise ValueError("exact_final_rerank requires the original dataset")
        final = exact_scores(index.dataset, qdims, qvals, qdense, orig[cand2],
                             cfg.sparse_weight, cfg.dense_weight)
    else:
        final = s2 + sparse_residual_dot(index, cand2, qdims, qvals) * cfg.sparse_weight
    kh = min(h, len(cand2))
    top = select_topk(final, kh, tie_ids=orig[cand2])
    if trace is not None:
        trace.update(stage1=s1, parts=parts, cand1=cand1, cand2=cand2,
                     scores2=s2, final=final)
    return orig[cand2[top]], final[top], [len(cand1), len(cand2), kh]


def query_parts(queries, i):
    """(dims, values, dense) of query row i of a CSR+dense query set."""
    sp = queries.sparse
    lo, hi = sp.indptr[i], sp.indptr[i + 1]
    return (sp.indices[lo:hi].astype(np.int64), sp.data[lo:hi].astype(np.float32),
            queries.dense[i])


def search_batch(index, queries, h=None, threads=1, **overrides):
    """Order-preserving map of search_topk over a query set (pipeline.py:282-300)."""
    nq = queries.sparse.shape[0]
    run = lambda i: search_topk(index, *query_parts(queries, i), h, **overrides)
    if threads > 1 and nq > 1:
        from concurrent.futures import ThreadPoolExecutor

        with ThreadPoolExecutor(max_workers=threads) as pool:
            return list(pool.map(run, range(nq)))
    return [run(i) for i in range(nq)]


def brute_force_topk(dataset, qdims, qvals, qdense, h, sparse_weight=1.0, dense_weight=1.0):
    """Exact top-h ground truth, ties to the lower id (harness.py:25-35)."""
    s = exact_scores(dataset, qdims, qvals, qdense, np.arange(dataset.sparse.shape[0]),
                     sparse_weight, dense_weight)
    top = select_topk(s, min(h, len(s)))
    return top, s[top]


def recall_at_h(returned, truth, h):
    """|returned ∩ truth| / h (harness.py:38-40)."""
    return len(np.intersect1d(np.asarray(returned), np.asarray(truth))) / h


def merge_shards(ids_list, scores_list, h):
    """Top-h over the union of per-shard results by (score desc, id asc).

    No reference counterpart (the reference is single-index); this is the
    definition the multi-GPU merge must meet.
    """
    ids = np.concatenate([np.asarray(x, dtype=np.int64) for x in ids_list])
    sc = np.concatenate([np.asarray(x, dtype=np.float64) for x in scores_list])
    top = select_topk(sc, h, tie_ids=ids)
    return ids[top], sc[top]
