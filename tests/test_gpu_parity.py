"""GPU parity: the CUDA path (through the C ABI) against the reference goldens
and the CPU oracle on identical inputs.

Bars (BASELINE.json north_star): LUT quantisation, integer PQ totals and
top-k ids (ties by id) bit-exact; float sparse / rerank scores within 1e-4
relative (asserted much tighter where the arithmetic is reproducible).
"""

from __future__ import annotations

import json

import numpy as np
import pytest

import paper_1903_08690_b200 as hs
from conftest import PIPELINE_CASES, golden, golden_index, golden_queries
from oracle import hybrid_oracle as O

pytestmark = pytest.mark.gpu

RTOL = 1e-4  # north_star float tolerance (relative)


def test_quantize_lut_bit_exact():
    z = golden("lut16")
    for i, K in enumerate(z["Ks"]):
        q = hs.quantize_lut(z[f"k{i}_table"])
        assert np.array_equal(q.table, z[f"k{i}_qtable"]), K
        assert np.array_equal(q.bias, z[f"k{i}_bias"])
        assert q.scale == float(z[f"k{i}_scale"])
        assert q.bias_total == float(z[f"k{i}_bias_total"])
    q = hs.quantize_lut(np.full((4, 16), 2.5))
    assert q.scale == 0.0 and not q.table.any() and q.bias_total == 10.0
    bad = np.zeros((2, 16))
    bad[1, 3] = np.inf
    with pytest.raises(ValueError):
        hs.quantize_lut(bad)


def test_lut16_scan_bit_exact():
    z = golden("lut16")
    for i, K in enumerate(z["Ks"]):
        qlut = hs.QuantizedLUT(bias=z[f"k{i}_bias"], scale=float(z[f"k{i}_scale"]),
                               table=z[f"k{i}_qtable"])
        codes = hs.PQCodes(n=z[f"k{i}_codes"].shape[0], n_subspaces=int(K), n_centers=16,
                           packed=z[f"k{i}_packed"])
        out = hs.lut16_scan(codes, qlut)
        assert np.array_equal(out, z[f"k{i}_scores"]), K
        tot = hs.lut16_totals(codes, qlut)
        assert np.array_equal(tot, O.lut16_totals(z[f"k{i}_packed"], int(K), z[f"k{i}_qtable"]))
        assert np.array_equal(hs.lut16_scan_reference(z[f"k{i}_codes"], qlut), out)
    qlut = hs.quantize_lut(np.full((5, 16), -1.25))
    pq = hs.PQCodes.from_codes(np.zeros((7, 5), dtype=np.uint8), 16)
    np.testing.assert_array_equal(hs.lut16_scan(pq, qlut), np.full(7, -6.25))
    wide = hs.PQCodes.from_codes(np.zeros((3, 2), dtype=np.uint8), 256)
    with pytest.raises(ValueError):
        hs.lut16_scan(wide, qlut)


def test_lut16_criterion4_random_instances():
    """Acceptance criterion 4 pattern (test_acceptance.py:140-163): bit identity with
    the scalar semantics and error <= K*s/2 + 1e-4 vs the float ADC."""
    rng = np.random.default_rng(4)
    for _ in range(40):
        K = int(rng.integers(1, 41))
        n = 1000
        codes = rng.integers(0, 16, size=(n, K), dtype=np.uint8)
        table = rng.normal(size=(K, 16)) * float(rng.uniform(0.1, 5.0))
        b, s, q = O.quantize_lut(table)
        qlut = hs.quantize_lut(table)
        assert np.array_equal(qlut.table, q) and qlut.scale == s
        out = hs.lut16_scan(hs.PQCodes.from_codes(codes, 16), qlut)
        ref = O.lut16_scores(O.lut16_totals(O.pack_codes(codes), K, q), O.bias_total(b), s)
        assert np.array_equal(out, ref)
        exact = np.zeros(n)
        for k in range(K):
            exact += table[k][codes[:, k]]
        assert np.max(np.abs(out - exact)) <= K * s / 2 + 1e-4


def test_adc_table_recipe_matches_reference_blas():
    z = golden("adc")
    mism = 0
    total = 0
    for i in range(int(z["n_specs"])):
        sub = z[f"a{i}_subdims"]
        flat = z[f"a{i}_centers"]
        centers, off = [], 0
        for w in sub:
            centers.append(flat[off:off + 16 * int(w)].reshape(16, int(w)))
            off += 16 * int(w)
        cb = hs.Codebooks(subdims=sub, centers=centers)
        for j, q in enumerate(z[f"a{i}_q"]):
            T = hs.adc_table(q, cb)
            mism += int(np.sum(T != z[f"a{i}_T"][j]))
            total += T.size
            np.testing.assert_allclose(T, z[f"a{i}_T"][j], rtol=1e-13, atol=1e-15)
    # the dgemv recipe reproduces the dev container's OpenBLAS exactly
    assert mism == 0, f"{mism}/{total} ADC entries differ"


def test_select_topk_known_answers_and_ties():
    assert hs.select_topk(np.array([1.0, 3.0, 2.0]), 5).tolist() == [1, 2, 0]
    assert hs.select_topk(np.ones(6), 3).tolist() == [0, 1, 2]
    assert hs.select_topk(np.array([1.0, 1.0, 1.0, 0.0]), 2,
                          tie_ids=np.array([30, 20, 10, 0])).tolist() == [2, 1]
    rng = np.random.default_rng(1)
    for _ in range(30):
        n = int(rng.integers(1, 3000))
        s = rng.integers(-4, 5, size=n).astype(np.float64)
        k = int(rng.integers(1, n + 5))
        t = rng.permutation(n)
        assert hs.select_topk(s, k, tie_ids=t).tolist() == O.select_topk(s, k, t).tolist()
    # large k (global path) and large n (streamed path)
    s = rng.integers(0, 50, size=20000).astype(np.float64)
    assert hs.select_topk(s, 5000).tolist() == O.select_topk(s, 5000).tolist()
    assert hs.select_topk(s, 300).tolist() == O.select_topk(s, 300).tolist()
    # keys that share their leading bytes (the radix select starts at the first
    # differing byte), all-equal keys (tie ids only), signs and infinities mixed
    for n, k in [(5000, 100), (70000, 1000), (3000, 2999)]:
        t = rng.permutation(n)
        near = 1.0 + rng.random(n) * 1e-9
        near[rng.integers(0, n, size=n // 10)] = near[0]          # exact ties at many levels
        assert hs.select_topk(near, k, tie_ids=t).tolist() == O.select_topk(near, k, t).tolist()
        same = np.full(n, -0.375)
        assert hs.select_topk(same, k, tie_ids=t).tolist() == O.select_topk(same, k, t).tolist()
        mixed = rng.standard_normal(n) * 1e-3
        mixed[::7] = -np.inf
        mixed[3::11] = 0.0
        assert hs.select_topk(mixed, k, tie_ids=t).tolist() == O.select_topk(mixed, k, t).tolist()


def test_sparse_scan_bit_exact():
    z = golden("sparse_scan")
    idx = hs.InvertedIndex(int(z["n"]), int(z["d_sparse"]), z["order"], dims=z["post_dims"],
                           ptr=z["post_ptr"], ids=z["post_ids"], w=z["post_w"])
    qp = z["q_ptr"]
    for t in range(len(qp) - 1):
        q = hs.SparseVector(z["q_dims"][qp[t]:qp[t + 1]], z["q_vals"][qp[t]:qp[t + 1]])
        acc = hs.Accumulator.zeros(int(z["n"]))
        hs.sparse_scan(idx, q, acc)
        assert np.array_equal(acc.scores, z["acc"][t]), t
    with pytest.raises(ValueError):
        hs.sparse_scan(idx, hs.SparseVector([int(z["d_sparse"])], [1.0]),
                       hs.Accumulator.zeros(int(z["n"])))


def test_sparse_scan_single_list_known_answer():
    import scipy.sparse as sp

    m = sp.csr_matrix(np.array([[0, 0, 0, 2.0, 0], [0, 0, 0, -1.0, 0]], dtype=np.float32))
    idx = hs.build_inverted(m, np.arange(2))
    acc = hs.Accumulator.zeros(2)
    hs.sparse_scan(idx, hs.SparseVector([3], [0.5]), acc)
    assert acc.scores.tolist() == [1.0, -0.5] and acc.lines_touched == 1


@pytest.mark.parametrize("name", PIPELINE_CASES)
def test_stage1_scores_vs_reference(name):
    z = golden(name)
    idx = golden_index(z)
    qs = golden_queries(z)
    s1 = hs.stage1_scores(idx, qs)
    ref = z["stage1"]
    if idx.dense_index is None or idx.dense_index.whitening is None:
        # no BLAS-ordered term: bit-exact
        assert np.array_equal(s1, ref)
    else:
        # whitening (dgemv, reproduced) + offset (ddot, not reproduced): ulp-level
        np.testing.assert_allclose(s1, ref, rtol=1e-12, atol=1e-14)


@pytest.mark.parametrize("name", PIPELINE_CASES)
def test_search_vs_reference(name):
    z = golden(name)
    idx = golden_index(z)
    qs = golden_queries(z)
    settings = json.loads(str(z["settings"]))
    for si, st in enumerate(settings):
        kw = {k: v for k, v in st.items() if k != "h"}
        res = hs.search_batch(idx, qs, st["h"], **kw)
        ids = np.stack([r.ids for r in res])
        sc = np.stack([r.scores for r in res])
        assert ids.tolist() == z[f"s{si}_ids"].tolist(), (name, si)
        np.testing.assert_allclose(sc, z[f"s{si}_scores"], rtol=1e-12, atol=1e-14)
        assert [r.stages.candidates for r in res] == z[f"s{si}_cands"].tolist()
        # one-at-a-time equals batched (search_topk / search_batch contract)
        one = hs.search_topk(idx, qs.point(0), st["h"], **kw)
        assert one.ids.tolist() == ids[0].tolist()
        np.testing.assert_array_equal(one.scores, sc[0])


def test_search_vs_live_oracle_unpruned():
    z = golden("pipe_unpruned")
    idx = golden_index(z)
    qs = golden_queries(z)
    for h, a, b, ex in [(10, 20.0, 20.0, True), (5, 3.0, 2.0, False), (40, 1.0, 1.0, False)]:
        res = hs.search_batch(idx, qs, h, overfetch=a, retain=b, exact_final_rerank=ex)
        for i in range(qs.n):
            ids, sc, _ = O.search_topk(idx, *O.query_parts(qs, i), h, overfetch=a, retain=b,
                                       exact_final_rerank=ex)
            assert res[i].ids.tolist() == ids.tolist()
            np.testing.assert_allclose(res[i].scores, sc, rtol=RTOL)


def test_exhaustive_search_equals_brute_force():
    """test_pipeline.py:128-137 pattern: overfetch = retain = n/h with exact rerank."""
    z = golden("pipe_default")
    idx = golden_index(z)
    qs = golden_queries(z)
    h = 20
    res = hs.search_batch(idx, qs, h, overfetch=idx.n / h, retain=idx.n / h,
                          exact_final_rerank=True)
    t_ids, t_sc = hs.brute_force_batch(idx.dataset, qs, h)
    for i in range(qs.n):
        assert res[i].ids.tolist() == t_ids[i].tolist()
        np.testing.assert_allclose(res[i].scores, t_sc[i], rtol=1e-9)
        ids, sc = O.brute_force_topk(idx.dataset, *O.query_parts(qs, i), h)
        assert t_ids[i].tolist() == ids.tolist()
        np.testing.assert_allclose(t_sc[i], sc, rtol=1e-12)


def test_brute_force_matches_reference_truth(pipeline_case):
    name, z = pipeline_case
    idx = golden_index(z)
    qs = golden_queries(z)
    ids, sc = hs.brute_force_batch(idx.dataset, qs, 10, idx.config.sparse_weight,
                                   idx.config.dense_weight)
    assert ids.tolist() == z["truth10_ids"].tolist()
    np.testing.assert_allclose(sc, z["truth10_scores"], rtol=1e-12, atol=1e-14)


def test_validation_errors():
    z = golden("pipe_default")
    idx = golden_index(z)
    qs = golden_queries(z)
    q = qs.point(0)
    with pytest.raises(ValueError):
        hs.search_topk(idx, q, 0)
    with pytest.raises(ValueError):
        hs.search_topk(idx, hs.HybridVector(q.sparse, np.zeros(idx.d_dense + 1)), 3)
    with pytest.raises(ValueError, match="range"):
        hs.search_topk(idx, hs.HybridVector(hs.SparseVector([idx.d_sparse], [1.0]), q.dense), 3)
    with pytest.raises(ValueError):
        hs.search_topk(idx, q, 3, overfetch=1.0, retain=2.0)
    nods = golden_index(z, with_dataset=False)
    with pytest.raises(ValueError, match="dataset"):
        hs.search_topk(nods, q, 3, exact_final_rerank=True)


def test_h_equals_n_and_empty_query():
    z = golden("pipe_odd")
    idx = golden_index(z)
    qs = golden_queries(z)
    n = idx.n
    res = hs.search_batch(idx, qs, 50, overfetch=n / 50, retain=n / 50)
    for r in res:
        assert len(set(r.ids.tolist())) == 50
        assert np.all(np.diff(r.scores) <= 1e-12)
    empty = hs.HybridVector(hs.SparseVector([], []), qs.dense[0])
    r = hs.search_topk(idx, empty, 10, exact_final_rerank=True)
    ids, sc, _ = O.search_topk(idx, [], [], qs.dense[0], 10, exact_final_rerank=True)
    assert r.ids.tolist() == ids.tolist()
