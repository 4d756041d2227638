"""Multi-rank path: id-range shards + all-gather + merge.

CPU: world_size-2 gloo process group; each rank's per-shard search is the CPU
oracle (test infrastructure) so the sharding, the collective plumbing and the
merge ordering are checked without a GPU.  GPU: two shards on one device,
per-shard CUDA search, the device merge kernel (K7) vs the oracle.
"""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest

import paper_1903_08690_b200 as hs
from paper_1903_08690_b200 import sharded
from oracle import hybrid_oracle as O


def _data():
    from paper_1903_08690_b200 import synth

    ds, qs, cfg = synth.make_config("cfg1", n=4000, n_queries=6)
    return ds, qs


CFG = dict(kmeans_iters=3, train_sample=2000, pq_subspaces=64, top_t=None, use_whitening=False)


def test_shard_bounds_cover_and_disjoint():
    for n in (0, 1, 7, 100, 1001):
        for world in (1, 2, 3, 8):
            spans = [sharded.shard_bounds(n, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            for (a, b), (c, d) in zip(spans, spans[1:]):
                assert b == c and a <= b
    with pytest.raises(ValueError):
        sharded.shard_bounds(10, 2, 2)


def test_merge_host_ordering():
    ids = np.array([[[5, 1, -1]], [[9, 3, 2]]])
    sc = np.array([[[2.0, 1.0, -np.inf]], [[2.0, 1.5, 1.0]]])
    mi, ms = sharded.merge_host(ids, sc, 4)
    assert mi[0].tolist() == [5, 9, 3, 1] and ms[0].tolist() == [2.0, 2.0, 1.5, 1.0]


def _oracle_local(shard, queries, h, overrides):
    res = [O.search_topk(shard.index, *O.query_parts(queries, i), h, **overrides)
           for i in range(queries.n)]
    kh = max(len(r[0]) for r in res)
    ids = np.full((queries.n, kh), -1, dtype=np.int64)
    sc = np.full((queries.n, kh), -np.inf)
    for i, r in enumerate(res):
        ids[i, :len(r[0])] = r[0] + shard.lo
        sc[i, :len(r[1])] = r[1]
    return ids, sc


def _small_data():
    """40 points over two ranks with h=30: each 20-point shard returns
    kh = 20 < h columns (k1 is capped by the shard's n)."""
    from paper_1903_08690_b200 import synth

    ds, qs, cfg = synth.make_config("cfg1", n=40, n_queries=4)
    return ds, qs


def _worker(rank, world, port, out_q, small=False):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        ds, qs = _small_data() if small else _data()
        h = 30 if small else 10
        shard = sharded.build_shard(ds, hs.HybridIndexConfig(**CFG), rank, world)
        s = sharded.ShardedSearcher(shard, local_search=_oracle_local, merge=sharded.merge_host)
        res = s.search_batch(qs, h, overfetch=5.0, retain=3.0, exact_final_rerank=True)
        out_q.put((rank, [r.ids.tolist() for r in res], [r.scores.tolist() for r in res]))
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_two_rank_gloo_matches_oracle_per_shard_merge():
    import multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = []
    try:
        got = [q.get(timeout=240) for _ in procs]
    finally:
        for p in procs:
            p.join(timeout=60)
            if p.is_alive():
                p.kill()
    assert all(p.exitcode == 0 for p in procs)
    got.sort()
    assert got[0][1] == got[1][1]  # every rank holds the merged result
    # expected: oracle on each shard, merged by (score desc, id asc)
    ds, qs = _data()
    ids_l, sc_l = [], []
    for r in range(2):
        shard = sharded.build_shard(ds, hs.HybridIndexConfig(**CFG), r, 2)
        i, s = _oracle_local(shard, qs, 10, dict(overfetch=5.0, retain=3.0,
                                                 exact_final_rerank=True))
        ids_l.append(i)
        sc_l.append(s)
    mi, ms = sharded.merge_host(np.stack(ids_l), np.stack(sc_l), 10)
    assert got[0][1] == [row.tolist() for row in mi]
    # with exact rerank the shard scores are exact hybrid dot products
    for qi in range(qs.n):
        t_ids, _ = O.brute_force_topk(ds, *O.query_parts(qs, qi), 10)
        assert len(np.intersect1d(t_ids, mi[qi])) >= 8


@pytest.mark.gpu
def test_two_shards_on_one_gpu_device_merge():
    import torch

    ds, qs = _data()
    shards = [sharded.build_shard(ds, hs.HybridIndexConfig(**CFG), r, 2) for r in range(2)]
    outs = []
    for sh in shards:
        s = sharded.ShardedSearcher.__new__(sharded.ShardedSearcher)
        s.shard, s.device, s._dev = sh, 0, None
        outs.append(s._gpu_local_search(sh, qs, 10, dict(overfetch=5.0, retain=3.0,
                                                         exact_final_rerank=True)))
    g_ids = torch.stack([o[0] for o in outs])
    g_sc = torch.stack([o[1] for o in outs])
    mi, ms = sharded.ShardedSearcher._gpu_merge(None, g_ids, g_sc, 10)
    ids_l = [_oracle_local(sh, qs, 10, dict(overfetch=5.0, retain=3.0, exact_final_rerank=True))
             for sh in shards]
    ei, es = sharded.merge_host(np.stack([x[0] for x in ids_l]), np.stack([x[1] for x in ids_l]), 10)
    assert mi.cpu().numpy().tolist() == ei.tolist()
    np.testing.assert_allclose(ms.cpu().numpy(), es, rtol=1e-12)


def test_two_rank_gloo_shards_smaller_than_h():
    """Ranks whose shard holds fewer than h points pad their local results to
    h columns before the all-gather (equal shapes on every rank)."""
    import multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q, True)) for r in range(2)]
    for p in procs:
        p.start()
    got = []
    try:
        got = [q.get(timeout=240) for _ in procs]
    finally:
        for p in procs:
            p.join(timeout=60)
            if p.is_alive():
                p.kill()
    assert all(p.exitcode == 0 for p in procs)
    got.sort()
    assert got[0][1] == got[1][1]
    ds, qs = _small_data()
    ids_l, sc_l = [], []
    for r in range(2):
        shard = sharded.build_shard(ds, hs.HybridIndexConfig(**CFG), r, 2)
        i, s = _oracle_local(shard, qs, 30, dict(overfetch=5.0, retain=3.0,
                                                 exact_final_rerank=True))
        assert i.shape[1] == 20
        pad = np.full((qs.n, 10), -1, dtype=np.int64)
        ids_l.append(np.concatenate([i, pad], axis=1))
        sc_l.append(np.concatenate([s, np.full((qs.n, 10), -np.inf)], axis=1))
    mi, ms = sharded.merge_host(np.stack(ids_l), np.stack(sc_l), 30)
    assert got[0][1] == [row[row >= 0].tolist() for row in mi]
    assert all(len(row) == 30 for row in got[0][1])  # 2 x 20 candidates cover h
