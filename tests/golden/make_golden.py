"""Generate golden fixtures by running the REFERENCE implementation.

Run in the dev container (where `/root/reference` exists):

    python tests/golden/make_golden.py

It imports `hybridsearch` from `/root/reference/pkg/src`, builds small indices
with the reference's own `build_index`, runs the reference's own search /
LUT / scan functions and stores inputs + outputs as compressed `.npz` files in
this directory.  The fixtures travel with the repo; nothing at test time reads
`/root/reference`.
"""

from __future__ import annotations

import json
import math
import os
import sys

import numpy as np
import scipy.sparse as sp

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))


def _ref():
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import hybridsearch as hs  # noqa: F401
    from hybridsearch import dense, pipeline, sparse, harness  # noqa: F401
    return hs


def save(name, **arrays):
    path = os.path.join(HERE, name + ".npz")
    np.savez_compressed(path, **arrays)
    print(f"wrote {path} ({os.path.getsize(path) / 1024:.1f} KiB)")


def csr_arrays(prefix, m):
    m = m.tocsr()
    return {f"{prefix}_indptr": m.indptr.astype(np.int64),
            f"{prefix}_indices": m.indices.astype(np.int64),
            f"{prefix}_data": m.data.astype(np.float32),
            f"{prefix}_shape": np.asarray(m.shape, dtype=np.int64)}


def index_arrays(idx):
    """Flatten a reference HybridIndex into named arrays."""
    out = {"order": idx.order.astype(np.int64),
           "n": np.int64(idx.n), "d_sparse": np.int64(idx.d_sparse),
           "d_dense": np.int64(idx.d_dense)}
    dims = np.array(sorted(idx.sparse_index.lists), dtype=np.int64)
    ptr = [0]
    ids, ws = [], []
    for j in dims:
        a, w = idx.sparse_index.lists[int(j)]
        ids.append(a)
        ws.append(w)
        ptr.append(ptr[-1] + len(a))
    out["post_dims"] = dims
    out["post_ptr"] = np.asarray(ptr, dtype=np.int64)
    out["post_ids"] = (np.concatenate(ids) if ids else np.zeros(0)).astype(np.uint32)
    out["post_w"] = (np.concatenate(ws) if ws else np.zeros(0)).astype(np.float32)
    out.update(csr_arrays("res", idx.sparse_residual))
    di = idx.dense_index
    out["has_dense"] = np.int64(di is not None)
    if di is not None:
        cb = di.codebooks
        out["subdims"] = cb.subdims.astype(np.int64)
        out["centers_flat"] = np.concatenate([c.reshape(-1) for c in cb.centers]).astype(np.float32)
        out["n_centers"] = np.int64(cb.n_centers)
        out["packed"] = di.codes.packed
        out["has_sq"] = np.int64(di.residual is not None)
        if di.residual is not None:
            out["sq_lo"] = di.residual.lo
            out["sq_step"] = di.residual.step
            out["sq_codes"] = di.residual.codes
        out["has_whitening"] = np.int64(di.whitening is not None)
        if di.whitening is not None:
            out["wh_mean"] = di.whitening.mean
            out["wh_forward"] = di.whitening.forward
            out["wh_inverse_t"] = di.whitening.inverse_t
    return out


def config_json(cfg):
    from dataclasses import asdict
    d = asdict(cfg)
    return json.dumps({k: (v.tolist() if isinstance(v, np.ndarray) else v) for k, v in d.items()})


def gen_lut16():
    """Criterion-4 style LUT16 instances (test_acceptance.py:140-163 pattern)."""
    hs = _ref()
    dn = hs.dense
    rng = np.random.default_rng(2024)
    cases = {}
    Ks = [1, 2, 5, 8, 32, 33, 64, 128, 255, 256, 257, 300]
    for i, K in enumerate(Ks):
        n = 257 if K < 256 else 61
        codes = rng.integers(0, 16, size=(n, K), dtype=np.uint8)
        table = rng.normal(size=(K, 16)) * float(rng.uniform(0.1, 5.0))
        if i == 3:   # exact grid + ties
            table = np.round(table * 4) / 4
        q = dn.quantize_lut(table)
        pq = dn.PQCodes.from_codes(codes, 16)
        vec = dn.lut16_scan(pq, q)
        ref = dn.lut16_scan_reference(codes, q)
        assert np.array_equal(vec, ref)
        cases[f"k{i}_codes"] = codes
        cases[f"k{i}_table"] = table
        cases[f"k{i}_bias"] = q.bias
        cases[f"k{i}_scale"] = np.float64(q.scale)
        cases[f"k{i}_qtable"] = q.table
        cases[f"k{i}_bias_total"] = np.float64(q.bias_total)
        cases[f"k{i}_packed"] = pq.packed
        cases[f"k{i}_scores"] = vec
    # zero-scale constant table (test_dense.py:204-208 pattern)
    q = dn.quantize_lut(np.full((5, 16), -1.25))
    pq = dn.PQCodes.from_codes(np.zeros((7, 5), dtype=np.uint8), 16)
    cases["zero_scores"] = dn.lut16_scan(pq, q)
    cases["Ks"] = np.asarray(Ks)
    save("lut16", **cases)


def gen_adc():
    """ADC tables for several subspace widths, fed by whitened-like queries."""
    hs = _ref()
    dn = hs.dense
    rng = np.random.default_rng(77)
    out = {}
    specs = [(16, 8), (128, 64), (9, 4), (7, 7), (12, 3), (256, 128), (10, 3)]
    for i, (d, K) in enumerate(specs):
        X = rng.normal(size=(400, d))
        cb = dn.train_codebooks(X, K, n_iters=3, seed=i)
        qs = rng.normal(size=(6, d)) * rng.uniform(0.05, 3.0)
        tabs = np.stack([dn.adc_table(q, cb) for q in qs])
        qluts = [dn.quantize_lut(t) for t in tabs]
        out[f"a{i}_subdims"] = cb.subdims.astype(np.int64)
        out[f"a{i}_centers"] = np.concatenate([c.reshape(-1) for c in cb.centers]).astype(np.float32)
        out[f"a{i}_q"] = qs
        out[f"a{i}_T"] = tabs
        out[f"a{i}_qtable"] = np.stack([q.table for q in qluts])
        out[f"a{i}_bias_total"] = np.array([q.bias_total for q in qluts])
        out[f"a{i}_scale"] = np.array([q.scale for q in qluts])
    out["n_specs"] = np.int64(len(specs))
    save("adc", **out)


def _dataset(hs, kind, seed):
    if kind == "synth":
        ds, qs = hs.generate_synthetic(hs.SynthConfig(
            n=3000, d_sparse=400, d_dense=16, n_queries=12, seed=seed))
        return ds, qs
    if kind == "odd":
        ds, qs = hs.generate_synthetic(hs.SynthConfig(
            n=1500, d_sparse=300, d_dense=9, n_queries=8, seed=seed))
        return ds, qs
    if kind == "dense_only":
        rng = np.random.default_rng(seed)
        X = rng.standard_normal((4000, 32)).astype(np.float32)
        X /= np.linalg.norm(X, axis=1, keepdims=True)
        Q = rng.standard_normal((10, 32)).astype(np.float32)
        ds = hs.HybridDataset(sp.csr_matrix((4000, 0), dtype=np.float32), X)
        qs = hs.HybridDataset(sp.csr_matrix((10, 0), dtype=np.float32), Q)
        return ds, qs
    if kind == "sparse_only":
        ds, qs = hs.generate_synthetic(hs.SynthConfig(
            n=2500, d_sparse=600, d_dense=0, n_queries=10, seed=seed,
            zipf_alpha=1.2, nnz_scale=0.8))
        return ds, qs
    raise KeyError(kind)


PIPELINE_CASES = {
    # name: (dataset kind, seed, config kwargs, list of search settings)
    "pipe_default": ("synth", 3, dict(kmeans_iters=6, train_sample=3000), [
        dict(h=20), dict(h=10, overfetch=20.0, retain=20.0, exact_final_rerank=True),
        dict(h=7, overfetch=5.0, retain=2.0)]),
    "pipe_nowhite": ("synth", 4, dict(kmeans_iters=6, train_sample=3000, use_whitening=False,
                                      sparse_weight=0.5, dense_weight=2.0), [
        dict(h=10), dict(h=10, overfetch=8.0, retain=8.0, exact_final_rerank=True)]),
    "pipe_unpruned": ("synth", 5, dict(kmeans_iters=6, train_sample=3000, top_t=None,
                                       use_whitening=False), [
        dict(h=10, overfetch=20.0, retain=20.0, exact_final_rerank=True)]),
    "pipe_odd": ("odd", 6, dict(kmeans_iters=6, train_sample=1500, pq_subspaces=4), [
        dict(h=10), dict(h=5, overfetch=30.0, retain=10.0, exact_final_rerank=True)]),
    "pipe_dense_only": ("dense_only", 7, dict(kmeans_iters=6, train_sample=4000,
                                              pq_subspaces=16, use_whitening=False), [
        dict(h=25, overfetch=4.0, retain=4.0)]),
    "pipe_sparse_only": ("sparse_only", 8, dict(top_t=None), [
        dict(h=10, overfetch=1.0, retain=1.0)]),
}


def gen_pipeline(name):
    hs = _ref()
    pl = hs.pipeline
    kind, seed, cfg_kw, settings = PIPELINE_CASES[name]
    ds, qs = _dataset(hs, kind, seed)
    cfg = hs.HybridIndexConfig(seed=seed, **cfg_kw)
    idx = hs.build_index(ds, cfg)
    out = index_arrays(idx)
    out["config"] = np.array(config_json(cfg))
    out.update(csr_arrays("ds", ds.sparse))
    out["ds_dense"] = ds.dense
    out.update(csr_arrays("q", qs.sparse))
    out["q_dense"] = qs.dense
    out["settings"] = np.array(json.dumps(settings))
    nq = qs.n
    # stage-1 traces for every query (pipeline.py:192-213)
    s1 = np.stack([pl._stage1_scores(idx, qs.point(i)) for i in range(nq)])
    out["stage1"] = s1
    if idx.dense_index is not None:
        tabs, bt, sc, off = [], [], [], []
        for i in range(nq):
            qd = qs.dense[i].astype(np.float64) * cfg.dense_weight
            qw, o = pl._dense_query(idx, qd)
            q = hs.quantize_lut(hs.adc_table(qw, idx.dense_index.codebooks))
            tabs.append(q.table)
            bt.append(q.bias_total)
            sc.append(q.scale)
            off.append(o)
        out["qtable"] = np.stack(tabs)
        out["bias_total"] = np.asarray(bt)
        out["scale"] = np.asarray(sc)
        out["offset"] = np.asarray(off)
    for si, st in enumerate(settings):
        h = st.get("h")
        kw = {k: v for k, v in st.items() if k != "h"}
        res = hs.search_batch(idx, qs, h, **kw)
        out[f"s{si}_ids"] = np.stack([r.ids for r in res])
        out[f"s{si}_scores"] = np.stack([r.scores for r in res])
        out[f"s{si}_cands"] = np.asarray([r.stages.candidates for r in res])
        # stage-1 candidate ids (pipeline.py:250-252)
        k1 = min(idx.n, math.ceil((kw.get("overfetch") or cfg.overfetch) * h))
        out[f"s{si}_cand1"] = np.stack([
            pl.select_topk(s1[i], k1, tie_ids=idx.order) for i in range(nq)])
    # brute force ground truth (harness.py:25-35)
    truth = [hs.brute_force_topk(ds, qs.point(i), 10, cfg.sparse_weight, cfg.dense_weight)
             for i in range(nq)]
    out["truth10_ids"] = np.stack([t[0] for t in truth])
    out["truth10_scores"] = np.stack([t[1] for t in truth])
    save(name, **out)


def gen_sparse_scan():
    hs = _ref()
    rng = np.random.default_rng(31)
    n, d = 700, 90
    rows = []
    for i in range(n):
        k = rng.poisson(6)
        dims = np.sort(rng.choice(d, size=min(k, d), replace=False))
        rows.append((dims, rng.normal(size=len(dims)).astype(np.float32)))
    indptr = np.cumsum([0] + [len(r[0]) for r in rows])
    mat = sp.csr_matrix((np.concatenate([r[1] for r in rows]),
                         np.concatenate([r[0] for r in rows]), indptr), shape=(n, d))
    order = hs.cache_sort(mat)
    idx = hs.build_inverted(mat, order)
    out = {"order": order}
    dims = np.array(sorted(idx.lists), dtype=np.int64)
    ptr = [0]
    ids, ws = [], []
    for j in dims:
        a, w = idx.lists[int(j)]
        ids.append(a)
        ws.append(w)
        ptr.append(ptr[-1] + len(a))
    out.update(post_dims=dims, post_ptr=np.asarray(ptr), post_ids=np.concatenate(ids),
               post_w=np.concatenate(ws), n=np.int64(n), d_sparse=np.int64(d))
    accs, qd, qv, qp = [], [], [], [0]
    for t in range(20):
        k = int(rng.integers(0, 12))
        dq = np.sort(rng.choice(d, size=k, replace=False))
        vq = rng.normal(size=k).astype(np.float32)
        acc = hs.Accumulator.zeros(n)
        hs.sparse_scan(idx, hs.SparseVector(dq, vq), acc)
        accs.append(acc.scores)
        qd.append(dq)
        qv.append(vq)
        qp.append(qp[-1] + k)
    out.update(q_ptr=np.asarray(qp), q_dims=np.concatenate(qd).astype(np.int64),
               q_vals=np.concatenate(qv).astype(np.float32), acc=np.stack(accs))
    out.update(csr_arrays("mat", mat))
    save("sparse_scan", **out)


def gen_build():
    """Reference build products on a small synthetic dataset, for the host
    builder's parity (order, postings, codes, SQ)."""
    hs = _ref()
    ds, qs = hs.generate_synthetic(hs.SynthConfig(n=1200, d_sparse=250, d_dense=12,
                                                  n_queries=2, seed=11))
    out = {}
    out.update(csr_arrays("ds", ds.sparse))
    out["ds_dense"] = ds.dense
    for tag, kw in (("t128", dict()), ("t5", dict(top_t=5)), ("none", dict(top_t=None)),
                    ("thr", dict(data_threshold=0.3, residual_threshold=0.1))):
        cfg = hs.HybridIndexConfig(seed=11, kmeans_iters=4, train_sample=1200, **kw)
        idx = hs.build_index(ds, cfg)
        for k, v in index_arrays(idx).items():
            out[f"{tag}_{k}"] = v
        out[f"{tag}_config"] = np.array(config_json(cfg))
    save("build", **out)


if __name__ == "__main__":
    which = sys.argv[1:] or ["lut16", "adc", "sparse_scan", "build"] + list(PIPELINE_CASES)
    for w in which:
        if w in PIPELINE_CASES:
            gen_pipeline(w)
        else:
            globals()["gen_" + w]()
