#!/usr/bin/env python
"""Benchmark: hybrid search queries/sec at recall@10 on BASELINE configs[1] (cfg2).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload cfg2] [--queries Q] [--top-t 128|none]

A step = one `search_batch` over the Q-query batch (the whole three-stage
pipeline: LUT build, fused stage-1 scan + top-k1, SQ rerank, exact rerank).
`value`  : Q*K / device time with queries already resident in HBM (max over
           ranks; L2 flushed before every step, flush not timed).
`e2e`    : same metric through the public API `search_batch(index, queries)`
           with host buffers: H2D of the queries and D2H of the results inside
           the timed region (wall clock around the call, which syncs).
`roofline`: the fused stage-1 kernel (LUT16 scan + posting stream + per-tile
           top-k): algorithmic bytes / its CUDA-event time vs MEASURED_PEAKS.
`cpu_baseline`: the CPU oracle port (oracle/hybrid_oracle.py, a restatement of
           the reference search path) on a bounded query sample, all host threads.
`--impl reference`: that CPU path alone, printed as the reference arm.

Multi-GPU (torchrun, N>1): the cfg2 dataset is split into N contiguous id-range
shards, one per rank (each an independent index); every rank
searches the same queries on its shard, per-shard top-h are all-gathered over
NCCL and merged on device (K7).  Total work is fixed => scaling "strong".
"""

from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

METRIC = "hybrid search queries/sec at recall@10 (1–8 GPU); scan HBM GB/s vs peak"


def _peaks():
    try:
        with open(os.path.join(REPO, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def _tensor_peak():
    """Dense u8 tensor peak: 2x the measured bf16 rate (tcgen05 kind::i8 issues in
    the same cycles per MMA as kind::f16 with twice the K; tools/mma_bench.cu)."""
    try:
        with open(os.path.join(REPO, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return 2.0 * float(p["bf16_tflops"]), "2x measured bf16 (MEASURED_PEAKS.json)"
    except Exception:
        return 4500.0, "nominal dense int8 (fallback)"


def _traffic(workload):
    """ncu-measured DRAM bytes per launch of the dominant kernel, if captured
    (profiles/<round>/traffic_<workload>.json, written by tools/ncu_traffic.py)."""
    import glob

    for path in sorted(glob.glob(os.path.join(REPO, "profiles", "*", f"traffic_{workload}.json")),
                       reverse=True):
        try:
            with open(path) as f:
                t = json.load(f)
            t["source"] = os.path.relpath(path, REPO)
            return t
        except Exception:
            continue
    return {}


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index=0):
        self.dev = device_index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.dev), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=self._read, daemon=True)
            self._t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx.append(float(f[2]))
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": float(max(mx)),
                "reasons": sorted(reasons), "samples": len(sm)}


def build_workload(args, rank, world, device=None):
    """Seeded cfg data (this rank's id-range shard) + queries + index."""
    from paper_1903_08690_b200 import build_index, sharded, synth

    cfg = synth.CONFIGS[args.workload]
    n_total = args.n or cfg.data.n
    t0 = time.time()
    ds_full = synth.generate(cfg.data, seed=0, n=n_total)
    lo, _ = sharded.shard_bounds(n_total, rank, world)
    ds = sharded.shard_dataset(ds_full, rank, world) if world > 1 else ds_full
    qs = synth.generate(cfg.data, seed=1, n=args.queries, mean_nnz=cfg.query_mean_nnz)
    t_gen = time.time() - t0
    kw = {}
    if args.top_t is not None:
        kw["top_t"] = None if args.top_t == "none" else int(args.top_t)
    icfg = cfg.index_config(**kw)
    t0 = time.time()
    exact = cfg.search["exact_final_rerank"]
    idx = build_index(ds, icfg, keep_dataset=exact, device=device)
    if cfg.search["overfetch"] == 1.0 and idx.dense_index is not None:
        # "no rerank" configs: the stage-1 composition (cfg 3)
        idx.dense_index.residual = None
    t_build = time.time() - t0
    return cfg, ds_full, ds, qs, idx, icfg, lo, t_gen, t_build


def query_device_buffers(qs, d_dense, torch, dev):
    from paper_1903_08690_b200 import _native as nat

    s = qs.sparse
    indptr = torch.as_tensor(np.asarray(s.indptr, dtype=np.int64)).to(dev)
    dims = torch.as_tensor(np.asarray(s.indices, dtype=np.int32)).to(dev)
    vals = torch.as_tensor(np.asarray(s.data, dtype=np.float32)).to(dev)
    dense = torch.as_tensor(np.ascontiguousarray(qs.dense, dtype=np.float32)).to(dev)
    b = nat.QueryBatch()
    b.nq = qs.n
    b.sp_indptr = indptr.data_ptr()
    b.sp_dims = dims.data_ptr()
    b.sp_vals = vals.data_ptr()
    b.dense = dense.data_ptr() if d_dense else None
    b.nnz = int(s.nnz)
    lens = np.diff(s.indptr)
    b.max_row_nnz = int(lens.max()) if len(lens) else 0
    hold = (indptr, dims, vals, dense)
    h2d = sum(int(t.numel() * t.element_size()) for t in hold)
    return b, hold, h2d


def cpu_oracle_qps(idx, qs, sample, threads):
    """The CPU port of the reference search path on `sample` queries."""
    from oracle import hybrid_oracle as O
    from paper_1903_08690_b200 import HybridDataset

    sub = HybridDataset(qs.sparse[:sample], qs.dense[:sample])
    s = idx.config
    O.search_batch(idx, HybridDataset(qs.sparse[:1], qs.dense[:1]), s.h, threads=1)  # warm
    t0 = time.perf_counter()
    O.search_batch(idx, sub, None, threads=threads)
    dt = time.perf_counter() - t0
    return sample / dt, dt


def run_reference_arm(args, rank, world):
    """--impl reference: the CPU port of the reference path, rank 0 only."""
    if rank != 0:
        return
    cfg, ds_full, ds, qs, idx, icfg, lo, t_gen, t_build = build_workload(args, 0, 1)
    s = cfg.search
    idx.config.h = s["h"]
    idx.config.overfetch = s["overfetch"]
    idx.config.retain = s["retain"]
    idx.config.exact_final_rerank = s["exact_final_rerank"]
    threads = os.cpu_count() or 1
    sample = min(args.cpu_sample, qs.n)
    from oracle import hybrid_oracle as O
    from paper_1903_08690_b200 import HybridDataset

    sub = HybridDataset(qs.sparse[:sample], qs.dense[:sample])
    for _ in range(args.warmup):
        O.search_batch(idx, HybridDataset(qs.sparse[:1], qs.dense[:1]), None, threads=1)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        O.search_batch(idx, sub, None, threads=threads)
        times.append(time.perf_counter() - t0)
    qps = sample * len(times) / sum(times)
    line = {
        "impl": "reference", "metric": METRIC, "value": qps, "unit": "queries/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * sum(times) / len(times), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "u8+f64", "data": "synthetic",
        "config": {"workload": f"{args.workload} ({cfg.note}), sample of {sample} queries/step",
                   "n": int(ds.n), "queries_per_step": sample},
        "cpu_baseline": {"value": qps, "unit": "queries/s", "cores": threads, "kind": "port",
                         "sample": f"{sample} queries of {args.workload} per step, "
                                   f"oracle search_batch(threads={threads})"},
        "e2e": {"value": qps, "unit": "queries/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="cfg2")
    ap.add_argument("--queries", type=int, default=None)
    ap.add_argument("--n", type=int, default=None)
    ap.add_argument("--top-t", default=None)
    ap.add_argument("--cpu-sample", type=int, default=None)
    ap.add_argument("--cpu-seconds", type=float, default=10.0,
                    help="target CPU work of the cpu_baseline sample")
    ap.add_argument("--truth-queries", type=int, default=None)
    ap.add_argument("--qb1", type=int, default=16,
                    help="single-query launches timed for the Qb=1 scan roofline")
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    from paper_1903_08690_b200 import synth

    if args.queries is None:
        args.queries = synth.CONFIGS[args.workload].n_queries
    big = args.workload in ("cfg3", "cfg4")
    if args.cpu_sample is None:
        args.cpu_sample = 8 if big else 24
    if args.truth_queries is None:
        args.truth_queries = 200 if big else args.queries
    if args.impl == "reference":
        run_reference_arm(args, rank, world)
        return

    import torch

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=dev)

    import paper_1903_08690_b200 as hs
    from paper_1903_08690_b200 import _native as nat

    cfg, ds_full, ds, qs, idx, icfg, id_lo, t_gen, t_build = build_workload(args, rank, world,
                                                                            device=local)
    s = cfg.search
    h = s["h"]
    dev_index = (hs.device_index(idx, local) if world == 1
                 else hs.DeviceIndex(idx, device=local, id_offset=id_lo))
    params = hs.search.resolve_params(idx, h, s["overfetch"], s["retain"], s["exact_final_rerank"])
    counts = np.zeros(3, dtype=np.int64)
    nat.check(nat.lib().hs_result_sizes(dev_index.handle, params, nat.ptr(counts)))
    k1, k2, kh = (int(x) for x in counts)
    nq = qs.n

    qb, hold, h2d_bytes = query_device_buffers(qs, idx.d_dense, torch, dev)
    out_ids = torch.empty((nq, kh), dtype=torch.int64, device=dev)
    out_sc = torch.empty((nq, kh), dtype=torch.float64, device=dev)
    if world > 1:
        g_ids = torch.empty((world, nq, kh), dtype=torch.int64, device=dev)
        g_sc = torch.empty((world, nq, kh), dtype=torch.float64, device=dev)
        m_ids = torch.empty((nq, h), dtype=torch.int64, device=dev)
        m_sc = torch.empty((nq, h), dtype=torch.float64, device=dev)
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)
    torch.cuda.synchronize()
    stream = torch.cuda.Stream(dev)
    torch.cuda.set_stream(stream)

    def step():
        dev_index.search_dev(qb, params, out_ids.data_ptr(), out_sc.data_ptr(),
                             stream.cuda_stream)
        if world > 1:
            dist.all_gather_into_tensor(g_ids.view(-1), out_ids.view(-1))
            dist.all_gather_into_tensor(g_sc.view(-1), out_sc.view(-1))
            nat.check(nat.lib().hs_shard_merge_dev(
                g_ids.data_ptr(), g_sc.data_ptr(), world, nq, kh, h, m_ids.data_ptr(),
                m_sc.data_ptr(), stream.cuda_stream))

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    # ---- timed region: device-resident queries, L2 flushed before each step ----
    l0 = dev_index.launches()
    times = []
    with ClockSampler(local) as clk:
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        for _ in range(args.steps):
            flush.zero_()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            step()
            e1.record(stream)
            e1.synchronize()
            times.append(e0.elapsed_time(e1))
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
    launches = dev_index.launches() - l0
    if world > 1:
        launches += args.steps  # shard merge kernel
    t_total = float(sum(times))
    if dist:
        tt = torch.tensor([t_total], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_total = float(tt.item())
    value = nq * args.steps / (t_total / 1e3)

    # ---- e2e through the public API with host buffers (N=1) ----
    e2e = None
    if world == 1:
        for _ in range(2):
            hs.search_batch(idx, qs, h, overfetch=s["overfetch"], retain=s["retain"],
                            exact_final_rerank=s["exact_final_rerank"])
        et = []
        for _ in range(args.steps):
            flush.zero_()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            hs.search_batch(idx, qs, h, overfetch=s["overfetch"], retain=s["retain"],
                            exact_final_rerank=s["exact_final_rerank"])
            et.append(time.perf_counter() - t0)
        d2h = nq * kh * (8 + 8)
        e2e = {"value": nq * len(et) / sum(et), "unit": "queries/s",
               "h2d_bytes_per_step": int(h2d_bytes), "d2h_bytes_per_step": int(d2h),
               "ms_per_step": 1e3 * sum(et) / len(et)}

    # ---- per-kernel breakdown (separate profiled steps; timing adds syncs) ----
    dev_index.set_timing(True)
    ktimes = {}
    for _ in range(2):
        flush.zero_()
        torch.cuda.synchronize()
        step()
        torch.cuda.synchronize()
        for k, v in dev_index.kernel_times().items():
            ktimes[k] = ktimes.get(k, 0.0) + v / 2
    qb1 = None
    if world == 1 and args.qb1 > 0:
        # Qb=1: one query per launch, stage-1 kernel time per pass over the codes
        from paper_1903_08690_b200 import HybridDataset

        t1 = []
        for i in range(min(args.qb1, nq)):
            one = HybridDataset(qs.sparse[i:i + 1], qs.dense[i:i + 1])
            b1, hold1, _ = query_device_buffers(one, idx.d_dense, torch, dev)
            o_i = torch.empty((1, kh), dtype=torch.int64, device=dev)
            o_s = torch.empty((1, kh), dtype=torch.float64, device=dev)
            flush.zero_()
            torch.cuda.synchronize()
            dev_index.search_dev(b1, params, o_i.data_ptr(), o_s.data_ptr(), stream.cuda_stream)
            torch.cuda.synchronize()
            kt = dev_index.kernel_times()
            if i > 0:  # first launch warms the per-launch path
                t1.append(kt.get("stage1", 0.0))
        qb1 = float(np.mean(t1)) if t1 else None
    dev_index.set_timing(False)

    # ---- results (rank-local then merged) and recall@10 vs exact brute force ----
    torch.cuda.synchronize()
    if world > 1:
        res_ids = m_ids.cpu().numpy()
    else:
        res_ids = out_ids.cpu().numpy()
    recall = None
    if rank == 0:
        truth_q = min(nq, args.truth_queries)
        from paper_1903_08690_b200 import HybridDataset

        qsub = HybridDataset(qs.sparse[:truth_q], qs.dense[:truth_q])
        t_ids, _ = hs.brute_force_batch(ds_full, qsub, 10, icfg.sparse_weight, icfg.dense_weight,
                                        device=local)
        rec = [len(np.intersect1d(res_ids[i, :10], t_ids[i])) / 10 for i in range(truth_q)]
        recall = float(np.mean(rec))

    # ---- roofline of the dominant kernel ----
    # tensor-core path (cfg2/cfg3): k_lut16_tc, bound by the tensor cores:
    #   algorithmic work = the one-hot LUT16 product, 2*N*Q*16K u8 ops per step
    # posting-stream path (cfg4 / small batches): k_stage1, bound by HBM:
    #   algorithmic bytes = 8 B per streamed posting (+ N*ceil(K/2) code bytes
    #   per query when the CUDA-core LUT16 scan runs), SURVEY 8(d)
    di = idx.dense_index
    npairs = (di.codes.n_subspaces + 1) // 2 if di is not None else 0
    K = di.codes.n_subspaces if di is not None else 0
    sidx = idx.sparse_index
    # postings streamed per query: sum of list lengths over the query dims
    lens = np.diff(sidx.ptr)
    pos = np.searchsorted(sidx.dims, qs.sparse.indices)
    pos = np.minimum(pos, max(len(sidx.dims) - 1, 0))
    hit = (len(sidx.dims) > 0) & (sidx.dims[pos] == qs.sparse.indices) if len(sidx.dims) else \
        np.zeros(qs.sparse.nnz, bool)
    postings = int(lens[pos][hit].sum()) if len(sidx.dims) else 0
    tc_ms = ktimes.get("lut16_tc")
    s1_ms = ktimes.get("stage1")
    roof = None
    traffic = _traffic(args.workload)
    if tc_ms and K:
        ops = 2.0 * idx.n * nq * 16 * K
        tpeak, tkind = _tensor_peak()
        achieved = ops / (tc_ms / 1e3) / 1e12
        roof = {"bound": "tensor", "achieved": achieved, "peak": tpeak, "unit": "TFLOP/s",
                "frac": achieved / tpeak, "traffic": traffic.get("dram_bytes_per_launch"),
                "kernel": "k_lut16_tc (tcgen05 kind::i8, threshold-filter epilogue)",
                "peak_kind": tkind, "ops_per_step": ops, "kernel_ms_per_step": tc_ms,
                "traffic_source": traffic.get("source"),
                "note": "u8 ops of the one-hot x LUT product (2*N*Q*16*K per step); the "
                        "kernel writes only threshold-passing candidates, so its HBM "
                        "traffic is the code stream, not the N*Q score matrix"}
    elif s1_ms:
        alg_bytes = 8 * postings + (nq * idx.n * npairs if K else 0)
        peak, peak_kind = _peaks()
        achieved = alg_bytes / (s1_ms / 1e3) / 1e9
        roof = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "traffic": traffic.get("dram_bytes_per_launch"),
                "kernel": "k_stage1 (posting stream + selection)", "peak_kind": peak_kind,
                "alg_bytes_per_step": alg_bytes, "kernel_ms_per_step": s1_ms,
                "traffic_source": traffic.get("source"),
                "note": "alg bytes = 8 B per streamed posting (u32 id + f32 weight)"
                        + (" + N*ceil(K/2) code bytes per query" if K else "")}
    if roof is not None and qb1:
        peak, peak_kind = _peaks()
        per_query_bytes = (idx.n * npairs + K * 16) + 8 * postings / max(nq, 1)
        a1 = per_query_bytes / (qb1 / 1e3) / 1e9
        roof["qb1"] = {"stage1_ms": qb1, "alg_bytes": per_query_bytes, "achieved_gbs": a1,
                       "peak_gbs": peak, "frac": a1 / peak,
                       "note": "latency path: one query per launch (CUDA-core LUT16 + "
                               "posting stream, HBM-bound), L2 flushed before each launch"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        threads = os.cpu_count() or 1
        sample = min(args.cpu_sample, nq)
        idx.config.h = h
        idx.config.overfetch = s["overfetch"]
        idx.config.retain = s["retain"]
        idx.config.exact_final_rerank = s["exact_final_rerank"]
        qps_cpu, dt = cpu_oracle_qps(idx, qs, sample, threads)
        if dt < 0.5 * args.cpu_seconds and sample < nq:
            # the first sample sizes the real one: ~--cpu-seconds of CPU work
            sample = min(nq, max(sample + 1, int(sample * args.cpu_seconds / max(dt, 1e-3))))
            qps_cpu, dt = cpu_oracle_qps(idx, qs, sample, threads)
        cpu = {"value": qps_cpu, "unit": "queries/s", "cores": threads, "kind": "port",
               "sample": f"first {sample} of {nq} {args.workload} queries, oracle "
                         f"search_batch(threads={threads}), {dt:.1f} s"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "queries/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_total / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "u8+f64",
            "data": "synthetic (seeded BASELINE-law generator, SURVEY App. B)",
            "config": {
                "workload": f"{args.workload}: {cfg.note}",
                "n": int(idx.n * world if world > 1 else idx.n), "d_sparse": int(idx.d_sparse),
                "d_dense": int(idx.d_dense), "pq_subspaces": K, "queries_per_step": nq,
                "h": h, "k1": k1, "k2": k2, "top_t": icfg.top_t,
                "exact_final_rerank": s["exact_final_rerank"],
                "recall_at_10": recall, "l2": "flushed (256 MiB write) before every step, untimed",
                "parallelism": f"id-range shards x{world}" if world > 1 else "single GPU",
                "postings_per_query": postings / max(nq, 1),
                "gen_s": round(t_gen, 1), "build_s": round(t_build, 1),
            },
            "e2e": e2e, "roofline": roof, "cpu_baseline": cpu, "clocks": clk.summary(),
            "gpu_launches": int(launches),
            "kernel_ms_per_step": {k: round(v, 4) for k, v in ktimes.items()},
        }
        print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
