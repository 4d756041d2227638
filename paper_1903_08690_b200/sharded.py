"""Multi-GPU hybrid search: contiguous id-range shards, one per rank.

SURVEY §8(e).  The reference is single-index (SPEC.md:17 puts distributed
serving out of its scope); the paper shards data over servers
(PAPER.md:696-698).  Here each rank holds an independent, reference-
equivalent index over ids [lo, hi) (its own pruning thresholds, layout
order, codebooks, whitening), searches the replicated queries with the
three-stage pipeline, and returns its top-kh with GLOBAL ids (id_offset =
lo, monotone so id tie-breaking is preserved).  The per-shard results are
all-gathered (torch.distributed: NCCL over NVLink on GPUs, gloo on CPU) and
merged to the top-h by (score desc, id asc) on the device (K7,
hs_shard_merge_dev).  The merged result is the union-of-shards result, not
a single-index search with k1 global candidates (SURVEY §8(e) note).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from .builder import build_index
from .types import HybridDataset, HybridIndexConfig, SearchResult, StageStats


def shard_bounds(n: int, rank: int, world: int) -> tuple[int, int]:
    """[lo, hi) of shard `rank` in a contiguous split of n ids over `world`."""
    if not (0 <= rank < world):
        raise ValueError("rank out of range")
    return n * rank // world, n * (rank + 1) // world


def shard_dataset(dataset: HybridDataset, rank: int, world: int) -> HybridDataset:
    lo, hi = shard_bounds(dataset.n, rank, world)
    return HybridDataset(dataset.sparse[lo:hi], dataset.dense[lo:hi])


@dataclass
class Shard:
    index: object  # HybridIndex over the shard's rows (local ids 0..hi-lo)
    lo: int
    hi: int
    rank: int
    world: int


def build_shard(dataset: HybridDataset, config: HybridIndexConfig | None, rank: int, world: int,
                keep_dataset: bool = True) -> Shard:
    lo, hi = shard_bounds(dataset.n, rank, world)
    idx = build_index(shard_dataset(dataset, rank, world), config, keep_dataset=keep_dataset)
    return Shard(index=idx, lo=lo, hi=hi, rank=rank, world=world)


def merge_host(ids: np.ndarray, scores: np.ndarray, h: int):
    """Reference ordering of the merge on host arrays [G][nq][kh] (used by tests
    as the checker's counterpart; the product merges on the device)."""
    G, nq, kh = ids.shape
    out_i = np.full((nq, h), -1, dtype=np.int64)
    out_s = np.full((nq, h), -np.inf)
    for q in range(nq):
        i = ids[:, q, :].reshape(-1)
        s = scores[:, q, :].reshape(-1)
        keep = i >= 0
        i, s = i[keep], s[keep]
        o = np.lexsort((i, -s))[:h]
        out_i[q, :len(o)] = i[o]
        out_s[q, :len(o)] = s[o]
    return out_i, out_s


class ShardedSearcher:
    """Search one shard per rank and merge across the process group.

    local_search(shard, queries, h, overrides) -> (ids[nq][kh] global, scores)
    and merge(ids[G][nq][kh], scores, h) -> (ids, scores) default to the GPU
    implementations; they are injectable so the collective plumbing can be
    exercised on CPU ranks (gloo) in tests.
    """

    def __init__(self, shard: Shard, group=None, device=None, local_search=None, merge=None):
        import torch.distributed as dist

        self.shard = shard
        self.group = group
        self.dist = dist
        self.device = device
        self.local_search = local_search or self._gpu_local_search
        self.merge = merge
        self._dev = None

    # -- GPU default path (device tensors end to end) --
    def _dev_index(self):
        if self._dev is None:
            from .search import DeviceIndex

            self._dev = DeviceIndex(self.shard.index, device=self.device or 0,
                                    id_offset=self.shard.lo)
        return self._dev

    def _gpu_local_search(self, shard, queries, h, overrides):
        import torch

        from . import _native as nat
        from .search import query_arrays, resolve_params

        idx = shard.index
        dev = self._dev_index()
        p = resolve_params(idx, h, overrides.get("overfetch"), overrides.get("retain"),
                           overrides.get("exact_final_rerank"))
        counts = np.zeros(3, dtype=np.int64)
        nat.check(nat.lib().hs_result_sizes(dev.handle, p, nat.ptr(counts)))
        kh = int(counts[2])
        self._last_counts = [int(counts[0]), int(counts[1]), kh]
        q = query_arrays(queries, int(idx.d_dense))
        d = torch.device("cuda", self.device or 0)
        t = [torch.as_tensor(q.indptr).to(d), torch.as_tensor(q.dims.view(np.int32)).to(d),
             torch.as_tensor(q.vals).to(d), torch.as_tensor(q.dense).to(d)]
        b = nat.QueryBatch()
        b.nq = q.nq
        b.sp_indptr, b.sp_dims, b.sp_vals = t[0].data_ptr(), t[1].data_ptr(), t[2].data_ptr()
        b.dense = t[3].data_ptr() if q.dense.size else None
        b.nnz = int(q.indptr[-1])
        b.max_row_nnz = int(np.diff(q.indptr).max()) if q.nq else 0
        ids = torch.empty((q.nq, kh), dtype=torch.int64, device=d)
        sc = torch.empty((q.nq, kh), dtype=torch.float64, device=d)
        st = torch.cuda.current_stream(d)
        dev.search_dev(b, p, ids.data_ptr(), sc.data_ptr(), st.cuda_stream)
        return ids, sc

    def _gpu_merge(self, g_ids, g_sc, h):
        import torch

        from . import _native as nat

        G, nq, kh = g_ids.shape
        out_i = torch.empty((nq, h), dtype=torch.int64, device=g_ids.device)
        out_s = torch.empty((nq, h), dtype=torch.float64, device=g_ids.device)
        st = torch.cuda.current_stream(g_ids.device)
        nat.check(nat.lib().hs_shard_merge_dev(g_ids.data_ptr(), g_sc.data_ptr(), G, nq, kh, h,
                                               out_i.data_ptr(), out_s.data_ptr(),
                                               st.cuda_stream))
        return out_i, out_s

    def search_batch(self, queries, h: int | None = None, **overrides) -> list:
        import torch

        idx = self.shard.index
        h = idx.config.h if h is None else int(h)
        ids, sc = self.local_search(self.shard, queries, h, overrides)
        ids = torch.as_tensor(ids)
        sc = torch.as_tensor(sc)
        world = self.dist.get_world_size(self.group)
        nq, kh = ids.shape
        if kh < h:
            # a shard smaller than h (k2 is capped by the shard's n) returns
            # fewer columns: pad to h (-1 / -inf, dropped by the merge) so
            # every rank contributes the same shape to the all-gather
            pad_i = torch.full((nq, h - kh), -1, dtype=ids.dtype, device=ids.device)
            pad_s = torch.full((nq, h - kh), -np.inf, dtype=sc.dtype, device=sc.device)
            ids = torch.cat([ids, pad_i], dim=1)
            sc = torch.cat([sc, pad_s], dim=1)
            kh = h
        g_ids = torch.empty((world, nq, kh), dtype=ids.dtype, device=ids.device)
        g_sc = torch.empty((world, nq, kh), dtype=sc.dtype, device=sc.device)
        if ids.is_cuda:  # NCCL: one collective into the stacked buffer
            self.dist.all_gather_into_tensor(g_ids.view(-1), ids.contiguous().view(-1),
                                             group=self.group)
            self.dist.all_gather_into_tensor(g_sc.view(-1), sc.contiguous().view(-1),
                                             group=self.group)
        else:  # gloo (CPU ranks)
            self.dist.all_gather(list(g_ids.unbind(0)), ids.contiguous(), group=self.group)
            self.dist.all_gather(list(g_sc.unbind(0)), sc.contiguous(), group=self.group)
        if self.merge is not None:
            mi, ms = self.merge(g_ids.cpu().numpy(), g_sc.cpu().numpy(), h)
        else:
            mi, ms = self._gpu_merge(g_ids, g_sc, h)
            mi, ms = mi.cpu().numpy(), ms.cpu().numpy()
        out = []
        local = getattr(self, "_last_counts", None)
        for i in range(nq):
            keep = mi[i] >= 0
            cands = ([local[0], local[1], int(keep.sum())] if local is not None
                     else [int(keep.sum())] * 3)
            out.append(SearchResult(ids=mi[i][keep], scores=ms[i][keep],
                                    stages=StageStats(candidates=cands, seconds=[0.0, 0.0, 0.0])))
        return out
