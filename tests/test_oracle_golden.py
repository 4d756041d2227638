"""Pin the CPU oracle (oracle/hybrid_oracle.py) to the reference's own outputs.

The fixtures were produced by running the reference package
(tests/golden/make_golden.py); these tests run without it and without a GPU.
"""

from __future__ import annotations

import json
import math

import numpy as np
import pytest

from conftest import PIPELINE_CASES, golden, golden_index, golden_queries
from oracle import hybrid_oracle as O


def test_lut16_quantize_and_scan_match_reference():
    z = golden("lut16")
    for i, K in enumerate(z["Ks"]):
        table = z[f"k{i}_table"]
        bias, scale, q = O.quantize_lut(table)
        assert np.array_equal(q, z[f"k{i}_qtable"]), K
        assert np.array_equal(bias, z[f"k{i}_bias"])
        assert scale == float(z[f"k{i}_scale"])
        bt = O.bias_total(bias)
        assert bt == float(z[f"k{i}_bias_total"])
        assert O.pairwise_sum(bias) == bt
        tot = O.lut16_totals(z[f"k{i}_packed"], int(K), q)
        assert np.array_equal(O.lut16_scores(tot, bt, scale), z[f"k{i}_scores"]), K
        codes = z[f"k{i}_codes"]
        small = slice(0, 40)
        assert np.array_equal(O.lut16_totals_scalar(codes[small], q), tot[small])
        assert np.array_equal(O.pack_codes(codes), z[f"k{i}_packed"])
    np.testing.assert_array_equal(z["zero_scores"], np.full(7, -6.25))


def test_quantize_lut_known_answers():
    # constant table -> zero scale, bias_total 10 (test_dense.py:159-164 semantics)
    bias, scale, q = O.quantize_lut(np.full((4, 16), 2.5))
    assert scale == 0.0 and not q.any() and O.bias_total(bias) == 10.0
    with pytest.raises(ValueError):
        bad = np.zeros((2, 16))
        bad[1, 3] = np.inf
        O.quantize_lut(bad)
    # round half to even
    t = np.array([[0.0, 0.5, 1.5, 2.5, 254.5, 255.0] + [0.0] * 10])
    _, s, q = O.quantize_lut(t)
    assert s == 1.0
    assert q[0, :6].tolist() == [0, 0, 2, 2, 254, 255]


def test_adc_tables_match_reference():
    z = golden("adc")
    for i in range(int(z["n_specs"])):
        sub = z[f"a{i}_subdims"]
        flat = z[f"a{i}_centers"]
        centers, off = [], 0
        for w in sub:
            centers.append(flat[off:off + 16 * int(w)].reshape(16, int(w)))
            off += 16 * int(w)
        for j, q in enumerate(z[f"a{i}_q"]):
            T = O.adc_table(q, centers, sub)
            assert np.array_equal(T, z[f"a{i}_T"][j])
            _, s, qt = O.quantize_lut(T)
            assert np.array_equal(qt, z[f"a{i}_qtable"][j])


def test_select_topk_known_answers():
    assert O.select_topk(np.array([1.0, 3.0, 2.0]), 5).tolist() == [1, 2, 0]
    assert O.select_topk(np.ones(6), 3).tolist() == [0, 1, 2]
    assert O.select_topk(np.array([1.0, 1.0, 1.0, 0.0]), 2,
                         tie_ids=np.array([30, 20, 10, 0])).tolist() == [2, 1]
    assert O.select_topk(np.array([-0.0, 0.0, -1.0]), 2).tolist() == [0, 1]
    rng = np.random.default_rng(0)
    for _ in range(50):
        s = rng.integers(-4, 5, size=rng.integers(1, 40)).astype(np.float64)
        k = int(rng.integers(1, 45))
        ref = np.lexsort((np.arange(len(s)), -s))[:min(k, len(s))]
        assert O.select_topk(s, k).tolist() == ref.tolist()


def test_sparse_scan_matches_reference():
    z = golden("sparse_scan")

    class Idx:  # array-form inverted index
        dims, ptr, ids, w = z["post_dims"], z["post_ptr"], z["post_ids"], z["post_w"]

    qp = z["q_ptr"]
    for t in range(len(qp) - 1):
        dq = z["q_dims"][qp[t]:qp[t + 1]]
        vq = z["q_vals"][qp[t]:qp[t + 1]]
        acc = O.sparse_scan(Idx, int(z["n"]), int(z["d_sparse"]), dq, vq)
        assert np.array_equal(acc, z["acc"][t])
    with pytest.raises(ValueError):
        O.sparse_scan(Idx, int(z["n"]), int(z["d_sparse"]), [int(z["d_sparse"])], [1.0])


@pytest.mark.parametrize("name", PIPELINE_CASES)
def test_pipeline_matches_reference(name):
    z = golden(name)
    idx = golden_index(z)
    qs = golden_queries(z)
    settings = json.loads(str(z["settings"]))
    for i in range(qs.n):
        dims, vals, dense = O.query_parts(qs, i)
        s1 = O.stage1_scores(idx, dims, vals, dense)
        assert np.array_equal(s1, z["stage1"][i]), (name, i)
        for si, st in enumerate(settings):
            kw = {k: v for k, v in st.items() if k != "h"}
            ids, scores, cands = O.search_topk(idx, dims, vals, dense, st["h"], **kw)
            assert ids.tolist() == z[f"s{si}_ids"][i].tolist(), (name, si, i)
            assert np.array_equal(scores, z[f"s{si}_scores"][i])
            assert cands == z[f"s{si}_cands"][i].tolist()
        t_ids, t_sc = O.brute_force_topk(idx.dataset, dims, vals, dense, 10,
                                         idx.config.sparse_weight, idx.config.dense_weight)
        assert t_ids.tolist() == z["truth10_ids"][i].tolist()
        assert np.array_equal(t_sc, z["truth10_scores"][i])


def test_merge_shards_definition():
    ids = [np.array([5, 1]), np.array([9, 3])]
    sc = [np.array([2.0, 1.0]), np.array([2.0, 1.5])]
    mid, msc = O.merge_shards(ids, sc, 3)
    assert mid.tolist() == [5, 9, 3] and msc.tolist() == [2.0, 2.0, 1.5]
