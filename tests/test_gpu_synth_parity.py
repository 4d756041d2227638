"""GPU parity on the BASELINE data laws (seeded generator), scaled down so the
CPU oracle finishes in seconds: cfg1/cfg2-shaped hybrid data with K=64/128,
dense-only (cfg3-shaped) and sparse-only unpruned (cfg4-shaped)."""

from __future__ import annotations

import numpy as np
import pytest

import paper_1903_08690_b200 as hs
from paper_1903_08690_b200 import synth
from oracle import hybrid_oracle as O

pytestmark = pytest.mark.gpu


def _scaled(name, n, nq, **over):
    ds, qs, cfg = synth.make_config(name, n=n, n_queries=nq)
    kw = dict(cfg.index)
    kw.update(over)
    kw.setdefault("kmeans_iters", 4)
    kw["train_sample"] = min(n, 20_000)
    idx = hs.build_index(ds, hs.HybridIndexConfig(**kw))
    return ds, qs, cfg, idx


def _check_search(idx, qs, h, a, b, exact, n_oracle=None):
    res = hs.search_batch(idx, qs, h, overfetch=a, retain=b, exact_final_rerank=exact)
    n_oracle = qs.n if n_oracle is None else n_oracle
    for i in range(n_oracle):
        ids, sc, _ = O.search_topk(idx, *O.query_parts(qs, i), h, overfetch=a, retain=b,
                                   exact_final_rerank=exact)
        assert res[i].ids.tolist() == ids.tolist(), i
        np.testing.assert_allclose(res[i].scores, sc, rtol=1e-9)
    return res


@pytest.mark.parametrize("name,n,top_t", [("cfg2", 30_000, 128), ("cfg1", 40_000, 128),
                                          ("cfg1", 20_000, None)])
def test_hybrid_law_search_matches_oracle(name, n, top_t):
    ds, qs, cfg, idx = _scaled(name, n, 12, top_t=top_t)
    s = cfg.search
    _check_search(idx, qs, s["h"], s["overfetch"], s["retain"], s["exact_final_rerank"])
    _check_search(idx, qs, 10, 5.0, 2.0, False)


def test_stage1_scores_and_totals_k128():
    ds, qs, cfg, idx = _scaled("cfg2", 20_000, 6)
    s1 = hs.stage1_scores(idx, qs)
    for i in range(qs.n):
        ref = O.stage1_scores(idx, *O.query_parts(qs, i))
        # whitening offset is a BLAS ddot the GPU does not reproduce bit-for-bit
        np.testing.assert_allclose(s1[i], ref, rtol=1e-12, atol=1e-15)


def test_dense_only_law_top100():
    ds, qs, cfg, idx = _scaled("cfg3", 60_000, 8)
    res = _check_search(idx, qs, 100, 1.0, 1.0, False)
    assert all(len(r.ids) == 100 for r in res)


def test_sparse_only_unpruned_law_top10():
    law = synth.CONFIGS["cfg4"]
    ds = synth.generate(law.data, 0, n=50_000)
    qs = synth.generate(law.data, 1, n=10, mean_nnz=law.query_mean_nnz)
    idx = hs.build_index(ds, hs.HybridIndexConfig(top_t=None))
    _check_search(idx, qs, 10, 1.0, 1.0, False)
    acc_gpu = hs.stage1_scores(idx, qs)
    for i in range(qs.n):
        assert np.array_equal(acc_gpu[i], O.stage1_scores(idx, *O.query_parts(qs, i)))


def test_device_entry_point_matches_host_entry_point():
    import torch

    ds, qs, cfg, idx = _scaled("cfg2", 30_000, 16)
    s = cfg.search
    host = hs.search_batch(idx, qs, s["h"], overfetch=s["overfetch"], retain=s["retain"],
                           exact_final_rerank=True)
    dev = hs.device_index(idx)
    p = hs.search.resolve_params(idx, s["h"], s["overfetch"], s["retain"], True)
    from paper_1903_08690_b200 import _native as nat

    sp_ = qs.sparse
    t = [torch.as_tensor(np.asarray(sp_.indptr, np.int64)).cuda(),
         torch.as_tensor(np.asarray(sp_.indices, np.int32)).cuda(),
         torch.as_tensor(np.asarray(sp_.data, np.float32)).cuda(),
         torch.as_tensor(np.ascontiguousarray(qs.dense, np.float32)).cuda()]
    b = nat.QueryBatch()
    b.nq, b.sp_indptr, b.sp_dims, b.sp_vals, b.dense = qs.n, *[x.data_ptr() for x in t]
    b.nnz, b.max_row_nnz = int(sp_.nnz), int(np.diff(sp_.indptr).max())
    kh = s["h"]
    ids = torch.empty((qs.n, kh), dtype=torch.int64, device="cuda")
    sc = torch.empty((qs.n, kh), dtype=torch.float64, device="cuda")
    torch.cuda.synchronize()
    dev.search_dev(b, p, ids.data_ptr(), sc.data_ptr(), torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    for i in range(qs.n):
        assert ids[i].tolist() == host[i].ids.tolist()
        assert sc[i].tolist() == host[i].scores.tolist()


def test_multi_chunk_tiles_many_queries():
    """Tiles spanning many 4096-point chunks (the bench regime): 300 queries over
    100K points => 2 tiles x 13 chunks per CTA."""
    ds, qs, cfg, idx = _scaled("cfg2", 100_000, 300)
    s = cfg.search
    _check_search(idx, qs, s["h"], s["overfetch"], s["retain"], True, n_oracle=6)


def test_bucketed_and_streamed_sparse_paths_agree(monkeypatch):
    """The sparse pre-pass (postings bucketed per chunk) and the in-kernel
    cursor stream must give identical stage-1 scores and results."""
    ds, qs, cfg, idx = _scaled("cfg2", 60_000, 40)
    s = cfg.search
    a = hs.search_batch(idx, qs, s["h"], overfetch=s["overfetch"], retain=s["retain"],
                        exact_final_rerank=True)
    s1a = hs.stage1_scores(idx, qs)
    monkeypatch.setenv("HSB200_NO_BUCKETS", "1")
    b = hs.search_batch(idx, qs, s["h"], overfetch=s["overfetch"], retain=s["retain"],
                        exact_final_rerank=True)
    s1b = hs.stage1_scores(idx, qs)
    assert np.array_equal(s1a, s1b)
    for x, y in zip(a, b):
        assert x.ids.tolist() == y.ids.tolist()
        assert x.scores.tolist() == y.scores.tolist()


@pytest.mark.parametrize("name,n,nq", [("cfg2", 40_000, 200), ("cfg3", 70_000, 150),
                                       ("cfg1", 30_000, 130)])
def test_tensor_core_lut16_path_matches_oracle_and_prmt(name, n, nq, monkeypatch):
    """Batches >= 16 queries take the tcgen05 kind::i8 LUT16 pass; results must be
    identical to the PRMT CUDA-core path and to the oracle."""
    ds, qs, cfg, idx = _scaled(name, n, nq)
    s = cfg.search
    kw = dict(overfetch=s["overfetch"], retain=s["retain"],
              exact_final_rerank=s["exact_final_rerank"])
    tc = hs.search_batch(idx, qs, s["h"], **kw)
    monkeypatch.setenv("HSB200_NO_TC", "1")
    ref = hs.search_batch(idx, qs, s["h"], **kw)
    for a, b in zip(tc, ref):
        assert a.ids.tolist() == b.ids.tolist()
        assert a.scores.tolist() == b.scores.tolist()
    for i in range(0, qs.n, max(1, qs.n // 6)):
        ids, sc, _ = O.search_topk(idx, *O.query_parts(qs, i), s["h"], **kw)
        assert tc[i].ids.tolist() == ids.tolist()
        np.testing.assert_allclose(tc[i].scores, sc, rtol=1e-9)


@pytest.mark.parametrize("name,n,nq,sample,cap", [
    ("cfg2", 60_000, 200, 4096, None),   # hybrid: filtered dense + touched points
    ("cfg3", 80_000, 150, 4096, None),   # dense only
    ("cfg2", 60_000, 130, 2048, 1),      # tiny list segments: overflowed queries rerun unfiltered
])
def test_threshold_filtered_stage1_matches_unfiltered_and_oracle(name, n, nq, sample, cap,
                                                                 monkeypatch):
    """The filtered tensor-core stage 1 (sample threshold -> filter epilogue ->
    candidate scoring) must select exactly what the unfiltered scan selects."""
    ds, qs, cfg, idx = _scaled(name, n, nq)
    s = cfg.search
    kw = dict(overfetch=s["overfetch"], retain=s["retain"],
              exact_final_rerank=s["exact_final_rerank"])
    monkeypatch.setenv("HSB200_FUSE_SAMPLE", str(sample))
    if cap:
        monkeypatch.setenv("HSB200_FUSE_CAP", str(cap))
    dev = hs.device_index(idx)
    dev.set_timing(True)
    fused = hs.search_batch(idx, qs, s["h"], **kw)
    assert "fuse" in dev.kernel_times()  # the filtered path ran
    monkeypatch.setenv("HSB200_NO_FUSE", "1")
    ref = hs.search_batch(idx, qs, s["h"], **kw)
    for a, b in zip(fused, ref):
        assert a.ids.tolist() == b.ids.tolist()
        assert a.scores.tolist() == b.scores.tolist()
    for i in range(0, qs.n, max(1, qs.n // 5)):
        ids, sc, _ = O.search_topk(idx, *O.query_parts(qs, i), s["h"], **kw)
        assert fused[i].ids.tolist() == ids.tolist()
        np.testing.assert_allclose(fused[i].scores, sc, rtol=1e-9)


@pytest.mark.parametrize("name,n,nq,top_t,negate", [
    ("cfg2", 60_000, 160, 128, True),    # negative query values: sparse lower bound lb < 0
    ("cfg1", 40_000, 150, None, False),  # unpruned lists: points repeat inside chunk buckets
    ("cfg1", 40_000, 150, None, True),
])
def test_filtered_stage1_negative_values_and_repeats(name, n, nq, top_t, negate, monkeypatch):
    """The totals-only sample threshold must stay a lower bound when products
    are negative (lb < 0), and the per-point bucket aggregation must sum
    repeated points in the reference's dim order; both checked against the
    unfiltered scan, the exact-sample threshold and the oracle."""
    ds, qs, cfg, idx = _scaled(name, n, nq, top_t=top_t)
    if negate:
        sp = qs.sparse.copy()
        sp.data[::3] *= -1.0
        qs = hs.HybridDataset(sp, qs.dense)
    s = cfg.search
    kw = dict(overfetch=s["overfetch"], retain=s["retain"],
              exact_final_rerank=s["exact_final_rerank"])
    monkeypatch.setenv("HSB200_FUSE_SAMPLE", "4096")
    dev = hs.device_index(idx)
    dev.set_timing(True)
    fused = hs.search_batch(idx, qs, s["h"], **kw)
    assert "fuse" in dev.kernel_times()
    monkeypatch.setenv("HSB200_EXACT_SAMPLE", "1")
    exact = hs.search_batch(idx, qs, s["h"], **kw)
    monkeypatch.delenv("HSB200_EXACT_SAMPLE")
    monkeypatch.setenv("HSB200_NO_FUSE", "1")
    ref = hs.search_batch(idx, qs, s["h"], **kw)
    for a, b, c in zip(fused, exact, ref):
        assert a.ids.tolist() == c.ids.tolist()
        assert b.ids.tolist() == c.ids.tolist()
        assert a.scores.tolist() == c.scores.tolist()
    for i in range(0, qs.n, max(1, qs.n // 5)):
        ids, sc, _ = O.search_topk(idx, *O.query_parts(qs, i), s["h"], **kw)
        assert fused[i].ids.tolist() == ids.tolist()
        np.testing.assert_allclose(fused[i].scores, sc, rtol=1e-9)


@pytest.mark.parametrize("name,n,nq,sample,cap,over", [
    ("cfg2", 60_000, 1, 4096, None, {}),      # single hybrid query (K=128)
    ("cfg2", 60_000, 7, 4096, None, {}),
    ("cfg3", 80_000, 5, 4096, None, {}),      # dense only (K=64)
    ("cfg1", 50_000, 12, 4096, None, {"pq_subspaces": 25}),  # K not a multiple of the 8-row slice
    ("cfg2", 60_000, 9, 2048, 1, {}),         # tiny list segments: overflow -> unfiltered rerun
])
def test_streamed_lut16_path_matches_unfiltered_and_oracle(name, n, nq, sample, cap, over,
                                                           monkeypatch):
    """Batches below the tensor-core minimum take the HBM-bound streamed LUT16
    scan (k_lut16_stream: sample totals -> threshold -> filter) in the filtered
    stage 1; it must select exactly what the unfiltered PRMT scan selects."""
    ds, qs, cfg, idx = _scaled(name, n, nq, **over)
    s = cfg.search
    kw = dict(overfetch=s["overfetch"], retain=s["retain"],
              exact_final_rerank=s["exact_final_rerank"])
    monkeypatch.setenv("HSB200_FUSE_SAMPLE", str(sample))
    if cap:
        monkeypatch.setenv("HSB200_FUSE_CAP", str(cap))
    dev = hs.device_index(idx)
    dev.set_timing(True)
    fused = hs.search_batch(idx, qs, s["h"], **kw)
    assert "lut16_stream" in dev.kernel_times()  # the streamed filtered path ran
    monkeypatch.setenv("HSB200_NO_FUSE", "1")
    ref = hs.search_batch(idx, qs, s["h"], **kw)
    for a, b in zip(fused, ref):
        assert a.ids.tolist() == b.ids.tolist()
        assert a.scores.tolist() == b.scores.tolist()
    for i in range(qs.n):
        ids, sc, _ = O.search_topk(idx, *O.query_parts(qs, i), s["h"], **kw)
        assert fused[i].ids.tolist() == ids.tolist()
        np.testing.assert_allclose(fused[i].scores, sc, rtol=1e-9)


@pytest.mark.parametrize("static", ["0", "1"])
def test_streamed_lut16_block_scheduling(static, monkeypatch):
    """k_lut16_stream hands out code blocks by ticket (HSB200_STREAM_STATIC=1:
    a fixed stride); the assignment must not change results, launch after
    launch (the ticket counter re-arms itself at the end of every launch)."""
    ds, qs, cfg, idx = _scaled("cfg2", 70_000, 6)
    s = cfg.search
    kw = dict(overfetch=s["overfetch"], retain=s["retain"],
              exact_final_rerank=s["exact_final_rerank"])
    monkeypatch.setenv("HSB200_FUSE_SAMPLE", "4096")
    dev = hs.device_index(idx)
    dev.set_timing(True)
    monkeypatch.setenv("HSB200_NO_FUSE", "1")
    base = hs.search_batch(idx, qs, s["h"], **kw)
    monkeypatch.delenv("HSB200_NO_FUSE")
    monkeypatch.setenv("HSB200_STREAM_STATIC", static)
    for _ in range(3):
        got = hs.search_batch(idx, qs, s["h"], **kw)
        assert "lut16_stream" in dev.kernel_times()
        for a, b in zip(got, base):
            assert a.ids.tolist() == b.ids.tolist()
            assert a.scores.tolist() == b.scores.tolist()


@pytest.mark.parametrize("name,n,nq,sub,direct", [
    ("cfg2", 70_000, 70, 64, None), ("cfg3", 80_000, 5, 32, None),
    ("cfg2", 70_000, 3, 100000, None),
    ("cfg2", 70_000, 70, 64, 16), ("cfg3", 80_000, 5, 32, 4)])  # open bin hit: two-pass fallback
def test_sample_threshold_two_level_selection(name, n, nq, sub, direct, monkeypatch):
    """k_sample_tlim finds the k1-th largest sample total with a first selection
    over a strided sub-sample (a lower bound L) and one full pass with a direct
    histogram of (total - L), falling back to two 8-bit passes when the k1-th
    largest lands in the open-ended last bin (HSB200_TLIM_DIRECT shrinks the
    histogram so that happens).  HSB200_TLIM_SUBGROUPS shrinks the
    sub-sample so the small test samples take that path (the last case: a
    sub-sample larger than the sample, i.e. the direct path); results must
    equal the unfiltered stage 1 for tensor-core and streamed batches."""
    ds, qs, cfg, idx = _scaled(name, n, nq)
    s = cfg.search
    kw = dict(overfetch=s["overfetch"], retain=s["retain"],
              exact_final_rerank=s["exact_final_rerank"])
    monkeypatch.setenv("HSB200_FUSE_SAMPLE", "8192")
    monkeypatch.setenv("HSB200_TLIM_SUBGROUPS", str(sub))
    if direct:
        monkeypatch.setenv("HSB200_TLIM_DIRECT", str(direct))
    dev = hs.device_index(idx)
    dev.set_timing(True)
    fused = hs.search_batch(idx, qs, s["h"], **kw)
    assert "fuse" in dev.kernel_times()
    monkeypatch.setenv("HSB200_NO_FUSE", "1")
    ref = hs.search_batch(idx, qs, s["h"], **kw)
    for a, b in zip(fused, ref):
        assert a.ids.tolist() == b.ids.tolist()
        assert a.scores.tolist() == b.scores.tolist()


@pytest.mark.parametrize("K,nq", [(100, 193), (97, 70), (200, 100), (128, 385), (128, 17), (128, 40),
                                  (64, 16), (64, 33), (108, 200), (72, 150), (32, 300)])
def test_tensor_core_group_shapes(K, nq, monkeypatch):
    """Tensor-core scan shapes around the CTA-pair / single-CTA switch: K = 100
    and 97 (pairs, 192-query groups, K not a multiple of the 8-subspace chunk,
    odd K), K = 200 (single CTA, narrow groups), batches that leave a 1-query
    or partial last group (193, 385), and the smallest tensor-core batches
    (16-40 queries: 32- and 64-query groups), K = 108 and 72 (chunk counts per
    block whose fixed producer assignment would outrun the TMEM ring: chunks go
    by global index there) and K = 32 with 300 queries (the group width is
    capped so the ring keeps four slots) — filtered stage 1 against the
    unfiltered scan and the oracle."""
    ds, qs, cfg, idx = _scaled("cfg2", 70_000, nq, pq_subspaces=K)
    s = cfg.search
    kw = dict(overfetch=s["overfetch"], retain=s["retain"],
              exact_final_rerank=s["exact_final_rerank"])
    monkeypatch.setenv("HSB200_FUSE_SAMPLE", "4096")
    dev = hs.device_index(idx)
    dev.set_timing(True)
    fused = hs.search_batch(idx, qs, s["h"], **kw)
    assert "lut16_tc" in dev.kernel_times() and "fuse" in dev.kernel_times()
    monkeypatch.setenv("HSB200_NO_FUSE", "1")
    monkeypatch.setenv("HSB200_NO_TC", "1")
    ref = hs.search_batch(idx, qs, s["h"], **kw)
    for a, b in zip(fused, ref):
        assert a.ids.tolist() == b.ids.tolist()
        assert a.scores.tolist() == b.scores.tolist()
    for i in range(0, qs.n, max(1, qs.n // 4)):
        ids, sc, _ = O.search_topk(idx, *O.query_parts(qs, i), s["h"], **kw)
        assert fused[i].ids.tolist() == ids.tolist()
        np.testing.assert_allclose(fused[i].scores, sc, rtol=1e-9)


def test_tensor_core_global_chunk_assignment_forced(monkeypatch):
    """HSB200_TC_ROT=1 forces the producers' global-index chunk assignment
    (normally chosen only for shapes that need it) on the K = 128 pair kernel."""
    ds, qs, cfg, idx = _scaled("cfg2", 70_000, 200)
    s = cfg.search
    kw = dict(overfetch=s["overfetch"], retain=s["retain"],
              exact_final_rerank=s["exact_final_rerank"])
    monkeypatch.setenv("HSB200_FUSE_SAMPLE", "4096")
    base = hs.search_batch(idx, qs, s["h"], **kw)
    monkeypatch.setenv("HSB200_TC_ROT", "1")
    rot = hs.search_batch(idx, qs, s["h"], **kw)
    for a, b in zip(rot, base):
        assert a.ids.tolist() == b.ids.tolist()
        assert a.scores.tolist() == b.scores.tolist()
