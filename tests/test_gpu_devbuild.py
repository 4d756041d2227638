"""GPU index build from a GPU-resident dataset (devbuild.py, hs_builder_*;
SURVEY §8(f) row f1) and the on-device generator.

Integer products (top_t thresholds, data-part split, cache_sort layout order,
postings, residual) must equal the reference build's bit for bit (golden
fixtures written by the reference, tests/golden/make_golden.py).  Dense
products equal the reference's exactly without whitening; with whitening the
mean / covariance come from a GPU f64 reduction in another summation order,
so the whitening matrices agree to ~1e-12 and codes to all but rare near-ties.
A GPU-generated config-5-law replica is built on the GPU and searched on the
GPU; the CPU oracle on the downloaded index gives the same ids.
"""

from __future__ import annotations

import numpy as np
import pytest

import paper_1903_08690_b200 as hs
from paper_1903_08690_b200 import synth
from conftest import csr_from, golden, golden_config, golden_index
from oracle import hybrid_oracle as O

pytestmark = pytest.mark.gpu


def _sparse_equal(idx, z, prefix=""):
    g = lambda k: z[prefix + k]  # noqa: E731
    assert np.array_equal(idx.order, g("order"))
    s = idx.sparse_index
    assert np.array_equal(s.dims, g("post_dims"))
    assert np.array_equal(s.ptr, g("post_ptr"))
    assert np.array_equal(s.ids, g("post_ids"))
    assert np.array_equal(s.w, g("post_w"))
    r = csr_from(z, prefix + "res")
    assert np.array_equal(idx.sparse_residual.indptr, r.indptr)
    assert np.array_equal(idx.sparse_residual.indices, r.indices)
    assert np.array_equal(idx.sparse_residual.data, r.data)


def _dense_close(idx, z, prefix="", exact=False):
    g = lambda k: z[prefix + k]  # noqa: E731
    if not int(g("has_dense")):
        assert idx.dense_index is None
        return
    di = idx.dense_index
    assert np.array_equal(di.codebooks.subdims, g("subdims"))
    flat = np.concatenate([c.reshape(-1) for c in di.codebooks.centers])
    if exact:
        assert np.array_equal(flat, g("centers_flat"))
        assert np.array_equal(di.codes.packed, g("packed"))
        assert np.array_equal(di.residual.lo, g("sq_lo"))
        assert np.array_equal(di.residual.step, g("sq_step"))
        assert np.array_equal(di.residual.codes, g("sq_codes"))
    else:
        np.testing.assert_allclose(di.whitening.inverse_t, g("wh_inverse_t"), rtol=1e-9, atol=1e-12)
        np.testing.assert_allclose(di.whitening.mean, g("wh_mean"), rtol=1e-12, atol=1e-15)
        np.testing.assert_allclose(flat, g("centers_flat"), rtol=1e-5, atol=1e-6)
        agree = np.mean(di.codes.packed == g("packed"))
        assert agree >= 0.999, agree


@pytest.mark.parametrize("tag", ["t128", "t5", "none", "thr"])
def test_device_build_matches_reference_build(tag):
    z = golden("build")
    ds = hs.HybridDataset(csr_from(z, "ds"), z["ds_dense"])
    cfg = golden_config(z, tag + "_config")
    dd = hs.DeviceDataset.upload(ds, 0)
    b = dd.build(cfg)
    idx = b.host_index(ds)
    _sparse_equal(idx, z, tag + "_")
    _dense_close(idx, z, tag + "_")
    # the top_t thresholds: the t-th largest |v| of every dim with more than t entries
    if cfg.data_threshold is None and cfg.top_t:
        sp_ = b.sparse_products()
        csc = ds.sparse.tocsc()
        for j, thr in zip(sp_["head_dims"], sp_["head_thr"]):
            col = np.abs(csc.data[csc.indptr[j]:csc.indptr[j + 1]].astype(np.float64))
            assert len(col) > cfg.top_t
            assert thr == np.partition(col, len(col) - cfg.top_t)[len(col) - cfg.top_t]


@pytest.mark.parametrize("name", ["pipe_default", "pipe_nowhite", "pipe_unpruned",
                                  "pipe_dense_only", "pipe_sparse_only"])
def test_device_build_pipeline_fixtures(name):
    z = golden(name)
    ref = golden_index(z)
    dd = hs.DeviceDataset.upload(ref.dataset, 0)
    idx = dd.build(ref.config).host_index(ref.dataset)
    _sparse_equal(idx, z)
    _dense_close(idx, z, exact=not ref.config.use_whitening)


def test_device_build_unwhitened_equals_host_build():
    """Without whitening every product is bit-identical to the host builder's
    (which the CPU suite pins to the reference)."""
    ds, qs, cfg = synth.make_config("cfg1", n=30_000, n_queries=8)
    icfg = cfg.index_config(use_whitening=False, kmeans_iters=4, train_sample=8000)
    host = hs.build_index(ds, icfg)
    dev = hs.DeviceDataset.upload(ds, 0).build(icfg).host_index(ds)
    assert np.array_equal(dev.order, host.order)
    for a in ("dims", "ptr", "ids", "w"):
        assert np.array_equal(getattr(dev.sparse_index, a), getattr(host.sparse_index, a))
    assert (dev.sparse_residual != host.sparse_residual).nnz == 0
    for c1, c2 in zip(dev.dense_index.codebooks.centers, host.dense_index.codebooks.centers):
        assert np.array_equal(c1, c2)
    assert np.array_equal(dev.dense_index.codes.packed, host.dense_index.codes.packed)
    assert np.array_equal(dev.dense_index.residual.codes, host.dense_index.residual.codes)
    assert np.array_equal(dev.dense_index.residual.lo, host.dense_index.residual.lo)


def test_upload_rejects_non_canonical_rows():
    """hs_builder_upload checks the CSR itself (columns strictly ascending)."""
    import ctypes

    from paper_1903_08690_b200 import _native as nat
    from paper_1903_08690_b200 import devbuild

    h = ctypes.c_void_p()
    keep = (np.array([0, 3], np.int64), np.array([5, 2, 7], np.uint32), np.ones(3, np.float32))
    args = [nat.ptr(keep[0]), nat.ptr(keep[1]), nat.ptr(keep[2]), None, 0, 0, ctypes.byref(h)]
    with pytest.raises(ValueError, match="ascending"):
        nat.check(devbuild._lib().hs_builder_upload(1, 10, 0, *args))
    with pytest.raises(ValueError, match="out of range"):
        nat.check(devbuild._lib().hs_builder_upload(1, 6, 0, *args))


def test_generator_shards_and_law():
    law = synth.replica_law(synth.CONFIGS["cfg5"].data, 40_000)
    full = hs.DeviceDataset.generate(law, seed=0, n=4000).download()
    part = hs.DeviceDataset.generate(law, seed=0, n=1500, row0=2500).download()
    assert (full.sparse[2500:] != part.sparse).nnz == 0
    assert np.array_equal(full.dense[2500:], part.dense)
    s = full.sparse
    lens = np.diff(s.indptr)
    assert abs(lens.mean() - law.mean_nnz) < 1.0
    for i in range(0, 4000, 97):  # distinct ascending dims, in range
        row = s.indices[s.indptr[i]:s.indptr[i + 1]]
        assert np.all(np.diff(row) > 0) and row.max(initial=0) < law.d_sparse
    # rows L2-normalised over the concatenation (f32 sparse, fp16 dense)
    nrm = np.sqrt(np.asarray(s.multiply(s).sum(axis=1)).ravel()
                  + np.sum(full.dense.astype(np.float64) ** 2, axis=1))
    assert np.all(np.abs(nrm - 1.0) < 2e-3)
    # fp16-exact dense values
    assert np.array_equal(full.dense.astype(np.float16).astype(np.float32), full.dense)


def test_generated_replica_build_and_search_match_oracle():
    """cfg5 law at a size the oracle handles: GPU generate -> GPU build ->
    GPU search; the oracle searches the downloaded index with the same queries."""
    cfg = synth.CONFIGS["cfg5"]
    law = synth.replica_law(cfg.data, 60_000)
    dd = hs.DeviceDataset.generate(law, seed=0)
    qlaw = synth.HybridLaw(law.n, law.d_sparse, law.d_dense, law.mean_nnz, law.zipf_s,
                           law.value_law, dense_fp16=False)
    qs = hs.DeviceDataset.generate(qlaw, seed=1, n=64).download()
    icfg = cfg.index_config(kmeans_iters=5, train_sample=20_000)
    b = dd.build(icfg)
    host = b.host_index()
    # the host builder on the downloaded dataset: same sparse products
    ref = hs.build_index(host.dataset, icfg)
    assert np.array_equal(host.order, ref.order)
    assert np.array_equal(host.sparse_index.ids, ref.sparse_index.ids)
    assert np.array_equal(host.sparse_index.w, ref.sparse_index.w)
    assert (host.sparse_residual != ref.sparse_residual).nnz == 0
    gidx = b.finish()
    s = dict(cfg.search, overfetch=5.0, retain=5.0)
    h = s["h"]
    kw = dict(overfetch=s["overfetch"], retain=s["retain"], exact_final_rerank=True)
    res = hs.search_batch(gidx, qs, h, **kw)
    host.config.h = h
    for i in range(qs.n):
        ids, sc, _ = O.search_topk(host, *O.query_parts(qs, i), h, **kw)
        assert res[i].ids.tolist() == ids.tolist(), i
        np.testing.assert_allclose(res[i].scores, sc, rtol=1e-12)
    # non-exact stage 3: the residual read from the raw rows
    q16 = hs.HybridDataset(qs.sparse[:16], qs.dense[:16])
    res2 = hs.search_batch(gidx, q16, h, overfetch=5.0, retain=2.0, exact_final_rerank=False)
    for i in range(len(res2)):
        ids, sc, _ = O.search_topk(host, *O.query_parts(qs, i), h, overfetch=5.0, retain=2.0,
                                   exact_final_rerank=False)
        assert res2[i].ids.tolist() == ids.tolist(), i
        np.testing.assert_allclose(res2[i].scores, sc, rtol=1e-12)
    # exact truth from the device-held dataset
    t_ids, t_sc = hs.exact_topk(gidx, qs, 10)
    for i in range(0, qs.n, 8):
        e_ids, e_sc = O.brute_force_topk(host.dataset, *O.query_parts(qs, i), 10)
        assert t_ids[i].tolist() == e_ids.tolist()
