"""The oracle's numpy restatement of build_index (oracle/build_oracle.py, the
reference arm's index builder) reproduces the reference build fixtures."""

from __future__ import annotations

import numpy as np
import pytest

from conftest import PIPELINE_CASES, csr_from, golden, golden_config, golden_index
from oracle import build_oracle as B
from oracle import hybrid_oracle as O


def _compare(idx, z, prefix=""):
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
    if int(g("has_dense")):
        di = idx.dense_index
        flat = np.concatenate([c.reshape(-1) for c in di.codebooks.centers])
        assert np.array_equal(flat, g("centers_flat"))
        assert np.array_equal(di.codes.packed, g("packed"))
        assert np.array_equal(di.residual.codes, g("sq_codes"))
        assert np.array_equal(di.residual.lo, g("sq_lo"))


@pytest.mark.parametrize("tag", ["t128", "t5", "none", "thr"])
def test_oracle_build_matches_reference(tag):
    z = golden("build")
    from types import SimpleNamespace

    ds = SimpleNamespace(sparse=csr_from(z, "ds"), dense=z["ds_dense"])
    _compare(B.build_index(ds, golden_config(z, tag + "_config")), z, tag + "_")


@pytest.mark.parametrize("name", [c for c in PIPELINE_CASES if c != "pipe_odd"])
def test_oracle_build_pipeline_fixtures(name):
    z = golden(name)
    ref = golden_index(z)
    idx = B.build_index(ref.dataset, ref.config)
    _compare(idx, z)
    # and the oracle search over it returns the reference's final ids
    import json

    st = json.loads(str(z["settings"]))[0]
    kw = {k: v for k, v in st.items() if k != "h"}
    from conftest import golden_queries

    qs = golden_queries(z)
    for i in range(min(qs.n, 5)):
        ids, _, _ = O.search_topk(idx, *O.query_parts(qs, i), st["h"], **kw)
        assert ids.tolist() == z["s0_ids"][i].tolist()


def test_numpy_generator_law():
    ds = B.generate(3000, 200_000, 16, 20.0, 1.1, dense_fp16=True, seed=3)
    lens = np.diff(ds.sparse.indptr)
    assert abs(lens.mean() - 20.0) < 1.0
    for i in range(0, 3000, 101):
        row = ds.sparse.indices[ds.sparse.indptr[i]:ds.sparse.indptr[i + 1]]
        assert np.all(np.diff(row) > 0)
    nrm = np.sqrt(np.asarray(ds.sparse.multiply(ds.sparse).sum(axis=1)).ravel()
                  + np.sum(ds.dense.astype(np.float64) ** 2, axis=1))
    assert np.all(np.abs(nrm - 1) < 2e-3)
    # the Feistel map is a bijection
    perm = B.feistel(np.arange(1000), 1000, 7)
    assert np.array_equal(np.sort(perm), np.arange(1000))
