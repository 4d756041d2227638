"""GPU dense build (`hs_dense_encode`): PQ codes, packing
and the SQ residual in layout order, bit-identical to the reference build
products (golden fixtures) and to the host builder at larger sizes."""

from __future__ import annotations

import numpy as np
import pytest

import paper_1903_08690_b200 as hs
from paper_1903_08690_b200 import builder as B
from conftest import PIPELINE_CASES, csr_from, golden, golden_config, golden_index
from test_builder_golden import _compare

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("tag", ["t128", "t5", "none", "thr"])
def test_gpu_build_variants_match_reference(tag):
    z = golden("build")
    ds = hs.HybridDataset(csr_from(z, "ds"), z["ds_dense"])
    cfg = golden_config(z, tag + "_config")
    _compare(hs.build_index(ds, cfg, device=0), z, tag + "_")


@pytest.mark.parametrize("name", PIPELINE_CASES)
def test_gpu_build_pipeline_fixtures_match_reference(name):
    z = golden(name)
    ref = golden_index(z)
    _compare(hs.build_index(ref.dataset, ref.config, device=0), z)


def _codebooks(rng, d, K_wide):
    subdims = np.array([2] * K_wide + [1] * (d - 2 * K_wide), dtype=np.int64)
    centers = [rng.standard_normal((16, int(w))).astype(np.float32) for w in subdims]
    return hs.Codebooks(subdims=subdims, centers=centers)


@pytest.mark.parametrize("n,d,K_wide", [(200_003, 256, 128), (50_000, 9, 4), (1, 3, 1), (0, 4, 2)])
def test_gpu_encode_equals_host_encode(n, d, K_wide):
    rng = np.random.default_rng(n + d)
    cb = _codebooks(rng, d, K_wide)
    vec = rng.standard_normal((n, d))
    if n > 10:
        vec[3] = vec[7]  # duplicate rows
        flat = np.concatenate([c[5] for c in cb.centers])  # a row sitting on centers: zero residuals
        vec[11] = flat.astype(np.float64)
        vec[:, 0] = np.round(vec[:, 0], 1)  # many exact ties between candidates
    order = rng.permutation(n).astype(np.int64)
    t = {}
    pq, sq = B.dense_encode_gpu(vec, order, cb, 0, timing=t)
    codes = B.pq_encode(vec, cb)[order] if n else np.zeros((0, cb.n_subspaces), np.uint8)
    assert np.array_equal(pq.packed, B.pack_codes(codes))
    if n:
        ref = B.sq_residual(vec, order, codes, cb)
        assert np.array_equal(sq.lo.view(np.uint32) & 0x7FFFFFFF, ref.lo.view(np.uint32) & 0x7FFFFFFF)
        assert np.array_equal(sq.step, ref.step)
        assert np.array_equal(sq.codes, ref.codes)
    assert t["dense_encode_s"] >= 0.0


def test_gpu_encode_rejects_unsupported():
    rng = np.random.default_rng(0)
    cb = hs.Codebooks(subdims=np.array([3, 1]), centers=[rng.standard_normal((16, 3)).astype(np.float32),
                                                          rng.standard_normal((16, 1)).astype(np.float32)])
    with pytest.raises(ValueError, match="wider than 2"):
        B.dense_encode_gpu(rng.standard_normal((10, 4)), np.arange(10), cb, 0)
