"""The host index builder reproduces the reference build_index products
(layout order, postings, residual CSR, codebooks, packed codes, SQ store,
whitening) on the reference-generated fixtures (CPU only)."""

from __future__ import annotations

import json

import numpy as np
import pytest

import paper_1903_08690_b200 as hs
from conftest import PIPELINE_CASES, csr_from, golden, golden_config, golden_index


def _compare(idx, z, prefix=""):
    g = lambda k: z[prefix + k]
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
    if int(g("has_dense")):
        di = idx.dense_index
        assert np.array_equal(di.codebooks.subdims, g("subdims"))
        flat = np.concatenate([c.reshape(-1) for c in di.codebooks.centers])
        assert np.array_equal(flat, g("centers_flat"))
        assert np.array_equal(di.codes.packed, g("packed"))
        if int(g("has_sq")):
            assert np.array_equal(di.residual.lo, g("sq_lo"))
            assert np.array_equal(di.residual.step, g("sq_step"))
            assert np.array_equal(di.residual.codes, g("sq_codes"))
        if int(g("has_whitening")):
            assert np.array_equal(di.whitening.inverse_t, g("wh_inverse_t"))
            assert np.array_equal(di.whitening.mean, g("wh_mean"))


@pytest.mark.parametrize("tag", ["t128", "t5", "none", "thr"])
def test_build_variants_match_reference(tag):
    z = golden("build")
    ds = hs.HybridDataset(csr_from(z, "ds"), z["ds_dense"])
    cfg = golden_config(z, tag + "_config")
    idx = hs.build_index(ds, cfg)
    _compare(idx, z, tag + "_")


@pytest.mark.parametrize("name", PIPELINE_CASES)
def test_pipeline_fixture_indices_match_reference(name):
    z = golden(name)
    ref = golden_index(z)
    idx = hs.build_index(ref.dataset, ref.config)
    _compare(idx, z)


def test_cache_sort_lexicographic_definition():
    """cache_sort == stable descending-lexicographic sort of activity patterns
    over dims ranked by (nnz desc, dim asc), beyond 64 dims (sparse.py:106-136)."""
    import scipy.sparse as sp

    rng = np.random.default_rng(3)
    n, d = 300, 120
    m = sp.random(n, d, density=0.05, random_state=4, format="csr", dtype=np.float32)
    m.data[:] = 1.0
    order = hs.cache_sort(m)
    nnz = np.asarray((m != 0).sum(axis=0)).ravel()
    ranked = np.lexsort((np.arange(d), -nnz))
    ranked = ranked[nnz[ranked] > 0]
    pat = (m[:, ranked] != 0).toarray().astype(np.int8)
    keys = [np.arange(n)] + [-pat[:, j] for j in range(pat.shape[1] - 1, -1, -1)]
    oracle = np.lexsort(keys)
    assert order.tolist() == oracle.tolist()


def test_order_fn_hook_and_bijection_check():
    z = golden("build")
    ds = hs.HybridDataset(csr_from(z, "ds"), z["ds_dense"])
    cfg = hs.HybridIndexConfig(seed=1, kmeans_iters=2, train_sample=ds.n)
    rev = hs.build_index(ds, cfg, order_fn=lambda mat: np.arange(mat.shape[0])[::-1])
    assert rev.order.tolist() == list(range(ds.n))[::-1]
    with pytest.raises(ValueError):
        hs.build_index(ds, cfg, order_fn=lambda mat: np.zeros(mat.shape[0], dtype=int))
