#!/usr/bin/env python
"""Benchmark: hybrid search queries/sec at recall@10 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload cfg5|cfg2|cfg3|cfg4|cfg1] [--queries Q] [--n N]

Default workload: BASELINE `configs[4]` (cfg5) — N=10^8 points, 10^9 sparse
dims (Zipf 1.1, mean 50 nnz), 256 dense dims stored fp16, PQ 128x16, 10^4
queries, top-100 after exact rerank of 1000 candidates per shard.  It fits one
B200 (~150 GB resident), so N=1 runs it whole; with N ranks each GPU holds the
id range [r*N/G, (r+1)*N/G) (scaling "strong": total work fixed).  Data are
seeded synthetic with the BASELINE laws, generated ON THE GPU
that searches them (rows keyed by global id) and indexed there
(devbuild.py; the host cannot hold cfg5).  cfg1-cfg4 keep the host generator
and host build (`--workload`).

A step = one search of the whole Q-query batch through the three-stage
pipeline (LUT build, tensor-core stage 1 + top-k1, SQ rerank, exact rerank)
and, for N>1, the NCCL all-gather of per-shard top-h and the device merge.
`value` : Q*K / device time (CUDA events on the search stream, max over
          ranks), queries resident in HBM; L2 flushed (256 MiB write) before
          every step, untimed.
`e2e`   : same metric through the public API with host buffers: H2D of the
          queries and D2H of the results inside the timed region.
`roofline`: the dominant kernel (k_lut16_tc, tcgen05 kind::i8) vs the u8
          tensor peak, plus the Qb=1 HBM view (single-query launches).
`parity`: GPU results vs the CPU oracle (oracle/hybrid_oracle.py) on the
          same inputs: for cfg5 a GPU-generated, GPU-built cfg5-law replica
          searched by both (>= 200 queries) plus full-scale sampled checks of
          the exact-rerank scores; for cfg1-4 the cpu_baseline sample.
`cpu_baseline`: the oracle port on the box's host cores, on a bounded sample.
`--impl reference`: the reference arm — the oracle port alone, on an index
          built by oracle/build_oracle.py (numpy; no product library loaded).
"""

from __future__ import annotations

import argparse
import json
import math
import os
import socket
import subprocess
import sys
import threading
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

METRIC = "hybrid search queries/sec at recall@10 (1–8 GPU); scan HBM GB/s vs peak"
REPLICA_N = 200_000      # cfg5-law replica for parity and the CPU baseline
PARITY_QUERIES = 256


def _peaks():
    try:
        with open(os.path.join(REPO, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def _tensor_peak():
    """Dense u8 tensor peak.  The kind::i8 MMA rate measured on this pool's B200
    (tools/mma_bench2 -> profiles/*/u8_peak.json) when recorded; else 2x the
    measured bf16 rate of MEASURED_PEAKS.json (kind::i8 issues in the same
    cycles per MMA as kind::f16 with twice the K) — cuBLAS bf16 runs
    power-capped well below the clock this scan holds, so that figure
    understates the u8 ceiling; else the nominal number."""
    import glob

    for path in sorted(glob.glob(os.path.join(REPO, "profiles", "*", "u8_peak.json")),
                       reverse=True):
        try:
            with open(path) as f:
                p = json.load(f)
            return float(p["u8_tops"]), ("measured tcgen05 kind::i8 MMA rate (tools/mma_bench2, "
                                         + os.path.relpath(path, REPO) + ")")
        except Exception:
            continue
    try:
        with open(os.path.join(REPO, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return 2.0 * float(p["bf16_tflops"]), "2x measured bf16 (MEASURED_PEAKS.json)"
    except Exception:
        return 4500.0, "nominal dense int8 (fallback)"


def _bf16x2_peak():
    try:
        with open(os.path.join(REPO, "MEASURED_PEAKS.json")) as f:
            return 2.0 * float(json.load(f)["bf16_tflops"])
    except Exception:
        return None


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


def _cpu_info():
    model = "unknown"
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    model = ln.split(":", 1)[1].strip()
                    break
    except Exception:
        pass
    blas = "unknown"
    try:
        cfg = np.show_config(mode="dicts")
        b = cfg.get("Build Dependencies", {}).get("blas", {})
        blas = f"{b.get('name', '?')} {b.get('version', '')}".strip()
    except Exception:
        pass
    return {"cpu_model": model, "numpy": np.__version__, "blas": blas}


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
        sm, mx, pw, reasons = [], [], [], set()
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
            try:
                pw.append(float(f[3]))
            except ValueError:
                pass
            for nm, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": float(max(mx)),
                "sm_mhz_min": float(min(sm)), "power_w_median": float(np.median(pw)) if pw else None,
                "power_w_max": float(max(pw)) if pw else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _relaunch(args):
    """`--gpus N` outside torchrun: start N ranks with torch.distributed.run."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
           f"--master-port={_free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    sys.exit(subprocess.call(cmd, env=env))


# ---------------------------------------------------------------------------
# workloads
# ---------------------------------------------------------------------------
class Work:
    """Everything one rank needs: index, device handle, queries, settings."""


def _gpu_query_law(cfg):
    from paper_1903_08690_b200 import synth

    L = cfg.data
    return synth.HybridLaw(L.n, L.d_sparse, L.d_dense, cfg.query_mean_nnz, L.zipf_s, L.value_law,
                           dense_fp16=False)


def setup_gpu_built(args, rank, world, device):
    """cfg5: this rank's id range generated and indexed on its GPU."""
    import paper_1903_08690_b200 as hs
    from paper_1903_08690_b200 import sharded, synth

    cfg = synth.CONFIGS[args.workload]
    n_total = args.n or cfg.data.n
    law = cfg.data if n_total == cfg.data.n else synth.replica_law(cfg.data, n_total)
    lo, hi = sharded.shard_bounds(n_total, rank, world)
    w = Work()
    w.cfg, w.law, w.n_total, w.lo, w.hi = cfg, law, n_total, lo, hi
    t0 = time.time()
    qlaw = synth.HybridLaw(law.n, law.d_sparse, law.d_dense, cfg.query_mean_nnz, law.zipf_s,
                           law.value_law, dense_fp16=False)
    w.qs = hs.DeviceDataset.generate(qlaw, seed=1, n=args.queries, device=device).download()
    dd = hs.DeviceDataset.generate(law, seed=0, n=hi - lo, row0=lo, device=device)
    w.t_gen = time.time() - t0
    w.nnz = dd.nnz
    t0 = time.time()
    w.icfg = cfg.index_config()
    b = dd.build(w.icfg)
    w.index = b.finish(id_offset=lo)
    w.t_build = time.time() - t0
    w.build_timing = dict(w.index.build_timing)
    w.dev = w.index.handle
    w.gpu_built = True
    w.postings = None
    return w


def setup_host_built(args, rank, world, device):
    """cfg1-cfg4: host generator + host build (dense encode on the GPU)."""
    import paper_1903_08690_b200 as hs
    from paper_1903_08690_b200 import build_index, sharded, synth

    cfg = synth.CONFIGS[args.workload]
    n_total = args.n or cfg.data.n
    w = Work()
    w.cfg, w.law, w.n_total = cfg, cfg.data, n_total
    t0 = time.time()
    ds_full = synth.generate(cfg.data, seed=0, n=n_total)
    w.lo, w.hi = sharded.shard_bounds(n_total, rank, world)
    ds = sharded.shard_dataset(ds_full, rank, world) if world > 1 else ds_full
    w.qs = synth.generate(cfg.data, seed=1, n=args.queries, mean_nnz=cfg.query_mean_nnz)
    w.t_gen = time.time() - t0
    kw = {}
    if args.top_t is not None:
        kw["top_t"] = None if args.top_t == "none" else int(args.top_t)
    w.icfg = cfg.index_config(**kw)
    t0 = time.time()
    exact = cfg.search["exact_final_rerank"]
    idx = build_index(ds, w.icfg, keep_dataset=True, device=device)
    if cfg.search["overfetch"] == 1.0 and idx.dense_index is not None:
        # "no rerank" configs: the stage-1 composition (cfg 3)
        idx.dense_index.residual = None
    w.t_build = time.time() - t0
    w.build_timing = {}
    w.index, w.ds = idx, ds
    w.nnz = int(ds.sparse.nnz)
    w.dev = (hs.device_index(idx, device) if world == 1
             else hs.DeviceIndex(idx, device=device, id_offset=w.lo))
    del exact
    w.gpu_built = False
    sidx = idx.sparse_index
    lens = np.diff(sidx.ptr)
    if len(sidx.dims):
        pos = np.minimum(np.searchsorted(sidx.dims, w.qs.sparse.indices), len(sidx.dims) - 1)
        hit = sidx.dims[pos] == w.qs.sparse.indices
        w.postings = int(lens[pos][hit].sum())
    else:
        w.postings = 0
    return w


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


def exact_truth(dev, qs, h):
    """Exact top-h (GPU, f64) over this rank's shard, global ids."""
    import ctypes

    from paper_1903_08690_b200 import _native as nat
    from paper_1903_08690_b200.search import query_arrays

    q = query_arrays(qs, int(dev.d_dense))
    kh = min(h, int(dev.n))
    ids = np.empty((q.nq, kh), dtype=np.int64)
    sc = np.empty((q.nq, kh), dtype=np.float64)
    b = q.batch()
    nat.check(nat.lib().hs_exact_topk(dev.handle, ctypes.byref(b), int(h), nat.ptr(ids),
                                      nat.ptr(sc)))
    return ids, sc


def _sub(qs, a, b):
    from paper_1903_08690_b200 import HybridDataset

    return HybridDataset(qs.sparse[a:b], qs.dense[a:b])


def _time_oracle(index, qs, sample, threads, s):
    """Oracle search over `sample` queries on `threads` host threads; also the
    single-thread split between stage 1 (scales with N) and stages 2-3."""
    from oracle import hybrid_oracle as O

    kw = dict(overfetch=s["overfetch"], retain=s["retain"],
              exact_final_rerank=s["exact_final_rerank"])
    O.search_topk(index, *O.query_parts(qs, 0), s["h"], **kw)  # warm
    t0 = time.perf_counter()
    res = O.search_batch(index, _sub(qs, 0, sample), s["h"], threads=threads, **kw)
    dt = time.perf_counter() - t0
    # share of the per-query time that scales with N: stage-1 scoring +
    # selection minus the query's LUT build (single thread, median of 3)
    t1s, tall = [], []
    for i in range(min(3, sample)):
        parts = O.query_parts(qs, i)
        a, b = [], []
        for _ in range(3):
            u0 = time.perf_counter()
            sc = O.stage1_scores(index, *parts)
            O.select_topk(sc, min(index.n, math.ceil(s["overfetch"] * s["h"])),
                          tie_ids=np.asarray(index.order, dtype=np.int64))
            u1 = time.perf_counter()
            if index.dense_index is not None:
                O.query_lut(index, parts[2])
            u2 = time.perf_counter()
            O.search_topk(index, *parts, s["h"], **kw)
            u3 = time.perf_counter()
            a.append((u1 - u0) - (u2 - u1))
            b.append(u3 - u2)
        t1s.append(float(np.median(a)))
        tall.append(float(np.median(b)))
    f1 = min(1.0, max(0.0, float(np.sum(t1s)) / max(float(np.sum(tall)), 1e-12)))
    return res, dt, f1


def replica_parity(args, device, s, want_cpu):
    """cfg5-law replica generated and built on the GPU, searched on the GPU and
    by the oracle on the downloaded index (same bytes, same queries)."""
    import paper_1903_08690_b200 as hs
    from paper_1903_08690_b200 import synth
    from oracle import build_oracle as BO

    cfg = synth.CONFIGS[args.workload]
    law = synth.replica_law(cfg.data, args.replica_n)
    qlaw = _gpu_query_law(cfg)
    qlaw.d_sparse = law.d_sparse
    t0 = time.time()
    dd = hs.DeviceDataset.generate(law, seed=0, device=device)
    qs = hs.DeviceDataset.generate(qlaw, seed=1, n=args.parity_queries, device=device).download()
    icfg = cfg.index_config()
    b = dd.build(icfg)
    host = b.host_index()
    # build parity: the oracle's numpy build of the downloaded dataset
    ob = BO.build_index(host.dataset, icfg)
    bp = {"order_equal": bool(np.array_equal(ob.order, host.order)),
          "postings_equal": bool(np.array_equal(ob.sparse_index.ids, host.sparse_index.ids)
                                 and np.array_equal(ob.sparse_index.w, host.sparse_index.w)
                                 and np.array_equal(ob.sparse_index.ptr, host.sparse_index.ptr)),
          "residual_equal": bool((ob.sparse_residual != host.sparse_residual).nnz == 0),
          "pq_codes_agree": float(np.mean(ob.dense_index.codes.packed
                                          == host.dense_index.codes.packed)),
          "sq_codes_agree": float(np.mean(ob.dense_index.residual.codes
                                          == host.dense_index.residual.codes))}
    del ob
    gidx = b.finish()
    res = hs.search_batch(gidx, qs, s["h"], overfetch=s["overfetch"], retain=s["retain"],
                          exact_final_rerank=s["exact_final_rerank"])
    host.config.h = s["h"]
    threads = os.cpu_count() or 1
    ores, dt, f1 = _time_oracle(host, qs, qs.n, threads, s)
    mism, worst = 0, 0.0
    for r, (oi, osc, _) in zip(res, ores):
        if r.ids.tolist() != oi.tolist():
            mism += 1
        if len(osc):
            worst = max(worst, float(np.max(np.abs(r.scores - osc) / np.maximum(np.abs(osc),
                                                                               1e-300))))
    # stage-1 scores of every point (whitening on): the one place where the GPU
    # does not reproduce a BLAS call bit for bit (the ddot of the whitening
    # offset, pipeline.py:223) — report how far that goes
    s1 = None
    try:
        from oracle import hybrid_oracle as O2

        nq1 = min(8, qs.n)
        g1 = hs.stage1_scores(gidx, _sub(qs, 0, nq1))
        worst1, neq = 0.0, 0
        for i in range(nq1):
            o1 = O2.stage1_scores(host, *O2.query_parts(qs, i))
            neq += int(np.count_nonzero(g1[i] != o1))
            worst1 = max(worst1, float(np.max(np.abs(g1[i] - o1) / np.maximum(np.abs(o1), 1e-300))))
        s1 = {"queries": nq1, "points": int(law.n), "scores_not_bit_equal": neq,
              "max_rel_err": worst1}
        del g1
    except Exception as e:  # noqa: BLE001
        s1 = {"error": repr(e)}
    out = {"replica": f"cfg5 law at N={law.n}, d_sparse={law.d_sparse} (GPU-generated, "
                      f"GPU-built, downloaded for the oracle)",
           "queries": int(qs.n), "id_mismatch": int(mism), "max_rel_err": worst,
           "build": bp, "stage1_scores": s1, "seconds": round(time.time() - t0, 1)}
    # operating points on the replica: the reference defaults
    # (top_t = 128) and the unpruned scan index (top_t = None), recall@10 of
    # the GPU results against GPU exact truth
    kw = dict(overfetch=s["overfetch"], retain=s["retain"],
              exact_final_rerank=s["exact_final_rerank"])
    t_ids, _ = exact_truth(gidx.handle, qs, 10)

    def _recall(rr):
        return float(np.mean([len(np.intersect1d(r.ids[:10], t_ids[i])) / 10
                              for i, r in enumerate(rr)]))

    ops = {f"top_t={icfg.top_t}": {"recall_at_10": _recall(res)}}
    try:
        # (finish() moved the first builder's arrays into its index: generate again)
        dd2 = hs.DeviceDataset.generate(law, seed=0, device=device)
        b2 = dd2.build(cfg.index_config(top_t=None))
        g2 = b2.finish()
        res2 = hs.search_batch(g2, qs, s["h"], **kw)
        t0u = time.perf_counter()
        hs.search_batch(g2, qs, s["h"], **kw)
        ops["top_t=None"] = {"recall_at_10": _recall(res2),
                             "gpu_qps_replica": qs.n / (time.perf_counter() - t0u)}
        t0u = time.perf_counter()
        hs.search_batch(gidx, qs, s["h"], **kw)
        ops[f"top_t={icfg.top_t}"]["gpu_qps_replica"] = qs.n / (time.perf_counter() - t0u)
        g2.handle.close()
        del b2, g2, dd2
    except Exception as e:  # noqa: BLE001
        ops["top_t=None"] = {"error": repr(e)}
    out["operating_points"] = ops
    cpu = None
    if want_cpu:
        # single-thread figure (BASELINE.md §3 asks for threads=1 beside all cores)
        n1 = min(qs.n, 24)
        t0u = time.perf_counter()
        from oracle import hybrid_oracle as O1

        O1.search_batch(host, _sub(qs, 0, n1), s["h"], threads=1, **kw)
        dt1 = time.perf_counter() - t0u
        per_q = dt / qs.n
        scale = cfg.data.n / law.n
        est = per_q * (f1 * scale + (1.0 - f1))
        cpu = {"value": 1.0 / est, "unit": "queries/s", "cores": threads, "kind": "port",
               "sample": f"{qs.n} queries of the cfg5-law replica (N={law.n}), oracle "
                         f"search_batch(threads={threads}) {dt:.1f} s; per-query time "
                         f"extrapolated to N={cfg.data.n}: the share that scales with N "
                         f"(stage-1 scan + select, {f1:.3f}, measured single-thread) x"
                         f"{scale:.0f}, the rest (LUT build, stages 2-3) constant",
               "replica_qps_measured": qs.n / dt,
               "replica_qps_threads1": n1 / dt1,
               "value_threads1": 1.0 / ((dt1 / n1) * (f1 * scale + (1.0 - f1)))}
        cpu.update(_cpu_info())
    gidx.handle.close()
    return out, cpu


def blas_recipe_check():
    """The f64 dot recipe the kernels reproduce (common.cuh dot_recipe: the
    OpenBLAS dgemv_t order) checked against THIS host's numpy/BLAS: the ADC
    table (dense.py:212-220, widths 1-3) and the SQ residual dot
    (dense.py:373-375, d = 256), GPU vs numpy on the same random inputs."""
    import paper_1903_08690_b200 as hs
    from oracle import hybrid_oracle as O

    rng = np.random.default_rng(123)
    out = {}
    bad = tot = 0
    for widths in ([2] * 128, [1] * 64, [3] * 40 + [2] * 4):
        sub = np.asarray(widths, dtype=np.int64)
        d = int(sub.sum())
        cents = [rng.standard_normal((16, w)).astype(np.float32) for w in widths]
        cb = hs.Codebooks(subdims=sub, centers=cents)
        for _ in range(4):
            q = rng.standard_normal(d)
            g = hs.adc_table(q, cb)
            o = O.adc_table(q, cents, sub)
            bad += int(np.count_nonzero(g != o))
            tot += g.size
    out["adc_table"] = {"entries": tot, "mismatch": bad}
    r = hs.ScalarQuantResidual(lo=rng.standard_normal(256).astype(np.float32),
                               step=(rng.random(256) * 0.01).astype(np.float32),
                               codes=rng.integers(0, 256, size=(4096, 256), dtype=np.uint8))
    bad = tot = 0
    for _ in range(4):
        q = rng.standard_normal(256)
        rows = rng.integers(0, 4096, size=1000)
        g = r.dot(rows, q)
        o = O.sq_residual_dot(r, rows, q)
        bad += int(np.count_nonzero(g != o))
        tot += g.size
    out["sq_residual_dot"] = {"rows": tot, "mismatch": bad}
    out["ok"] = out["adc_table"]["mismatch"] == 0 and bad == 0
    return out


def fullscale_checks(w, res_ids, res_sc, nq_check, s):
    """Exact-rerank scores of the returned ids recomputed on the host from the
    rows gathered out of the device index (rank-local ids)."""
    from oracle import hybrid_oracle as O

    worst, checked = 0.0, 0
    for i in range(min(nq_check, res_ids.shape[0])):
        ids = res_ids[i]
        ids = ids[ids >= 0]
        loc = ids - w.lo
        mine = (loc >= 0) & (loc < w.hi - w.lo)
        if not mine.any():
            continue
        rows = w.index.gather_rows(loc[mine])
        qd, qv, qdense = O.query_parts(w.qs, i)
        ex = O.exact_scores(rows, qd, qv, qdense, np.arange(rows.n),
                            w.icfg.sparse_weight, w.icfg.dense_weight)
        got = res_sc[i][: len(ids)][mine]
        worst = max(worst, float(np.max(np.abs(got - ex) / np.maximum(np.abs(ex), 1e-300))))
        checked += int(mine.sum())
    out = {"queries": int(min(nq_check, res_ids.shape[0])), "rows_checked": checked,
           "max_rel_err_exact_scores": worst}
    # two independent scans at full scale: the same queries one at a time take the
    # streamed PRMT scan (k_lut16_stream) instead of the tensor-core pass of the
    # batch; ids and scores must be identical
    try:
        import paper_1903_08690_b200 as hs

        kw = dict(overfetch=s["overfetch"], retain=s["retain"],
                  exact_final_rerank=s["exact_final_rerank"])
        nq1 = min(8, res_ids.shape[0])
        bad_i = bad_s = 0
        for i in range(nq1):
            r = hs.search_batch(w.index, _sub(w.qs, i, i + 1), s["h"], **kw)[0]
            ids = res_ids[i][res_ids[i] >= 0]
            bad_i += int(r.ids.tolist() != ids.tolist())
            bad_s += int(r.scores.tolist() != res_sc[i][: len(ids)].tolist())
        out["tc_vs_streamed_scan"] = {"queries": nq1, "id_mismatch": bad_i, "score_mismatch": bad_s}
    except Exception as e:  # noqa: BLE001
        out["tc_vs_streamed_scan"] = {"error": repr(e)}
    return out


# ---------------------------------------------------------------------------
# reference arm
# ---------------------------------------------------------------------------
def run_reference_arm(args, rank, world):
    """--impl reference: the oracle port on the host cores (rank 0 only), on an
    index built by oracle/build_oracle.py (no product library loaded)."""
    if rank != 0:
        return
    from oracle import build_oracle as BO
    from oracle import hybrid_oracle as O
    from types import SimpleNamespace

    spec = _workload_spec(args.workload)
    s = spec["search"]
    gpu_built = args.workload == "cfg5"
    n_full = args.n or spec["n"]
    n_rep = min(n_full, args.replica_n) if gpu_built else n_full
    scale_d = n_rep / spec["n"]
    d_sparse = max(1000, int(round(spec["d_sparse"] * scale_d))) if spec["d_sparse"] else 0
    t0 = time.time()
    ds = BO.generate(n_rep, d_sparse, spec["d_dense"], spec["mean_nnz"], spec["zipf_s"],
                     spec["value_law"], spec["dense_fp16"], seed=0)
    qs = BO.generate(max(64, args.ref_queries), d_sparse, spec["d_dense"], spec["q_mean_nnz"],
                     spec["zipf_s"], spec["value_law"], False, seed=1)
    icfg = SimpleNamespace(**spec["index"])
    index = BO.build_index(ds, icfg)
    index.config.h = s["h"]
    t_setup = time.time() - t0
    threads = os.cpu_count() or 1
    kw = dict(overfetch=s["overfetch"], retain=s["retain"],
              exact_final_rerank=s["exact_final_rerank"])
    # per-step sample: ~args.ref_step_seconds of work
    u0 = time.perf_counter()
    O.search_batch(index, _sub(qs, 0, 4), s["h"], threads=threads, **kw)
    per = (time.perf_counter() - u0) / 4
    sample = int(min(qs.n, max(8, args.ref_step_seconds / max(per, 1e-4) * min(threads, 8))))
    for _ in range(args.warmup):
        O.search_batch(index, _sub(qs, 0, min(4, sample)), s["h"], threads=threads, **kw)
    times = []
    for k in range(args.steps):
        a = (k * sample) % max(1, qs.n - sample + 1)
        t1 = time.perf_counter()
        O.search_batch(index, _sub(qs, a, a + sample), s["h"], threads=threads, **kw)
        times.append(time.perf_counter() - t1)
    qps_rep = sample * len(times) / sum(times)
    f1 = 1.0
    note = ""
    qps = qps_rep
    if gpu_built and n_rep < n_full:
        _, _, f1 = _time_oracle(index, qs, 4, 1, s)
        scale = n_full / n_rep
        qps = 1.0 / ((1.0 / qps_rep) * (f1 * scale + 1.0 - f1))
        note = (f"; QPS extrapolated to N={n_full} from the N={n_rep} replica: the share "
                f"that scales with N (stage-1 scan + select, {f1:.3f}) x{scale:.0f}, the rest "
                f"(LUT build, stages 2-3) constant")
    Q = args.queries or spec["queries"]
    line = {
        "impl": "reference", "metric": METRIC, "value": qps, "unit": "queries/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * Q / qps, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "u8+f64", "data": "synthetic (seeded BASELINE-law "
        "generator, numpy: oracle/build_oracle.py)",
        "config": _config_dict(args.workload, spec, n_full, Q),
        "cpu_baseline": {"value": qps, "unit": "queries/s", "cores": threads, "kind": "port",
                         "sample": f"{sample} queries per step of the {args.workload} law at "
                                   f"N={n_rep}, oracle search_batch(threads={threads}), index "
                                   f"from oracle/build_oracle.py{note}",
                         "measured_qps_at_sample_n": qps_rep, "setup_s": round(t_setup, 1),
                         **_cpu_info()},
        "e2e": {"value": qps, "unit": "queries/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def _workload_spec(name):
    """Plain-data description of a BASELINE workload (no product import)."""
    specs = {
        "cfg1": dict(n=100_000, d_sparse=1_000_000, d_dense=128, mean_nnz=50.0, zipf_s=1.1,
                     value_law="absnormal", dense_fp16=False, q_mean_nnz=50.0, queries=1000,
                     index=dict(pq_subspaces=64, kmeans_iters=10),
                     search=dict(h=10, overfetch=20.0, retain=20.0, exact_final_rerank=True)),
        "cfg2": dict(n=1_000_000, d_sparse=10_000_000, d_dense=256, mean_nnz=100.0, zipf_s=1.1,
                     value_law="lognormal", dense_fp16=False, q_mean_nnz=100.0, queries=1000,
                     index=dict(pq_subspaces=128),
                     search=dict(h=10, overfetch=50.0, retain=50.0, exact_final_rerank=True)),
        "cfg3": dict(n=10_000_000, d_sparse=0, d_dense=128, mean_nnz=0.0, zipf_s=1.1,
                     value_law="absnormal", dense_fp16=False, q_mean_nnz=0.0, queries=10_000,
                     index=dict(pq_subspaces=64),
                     search=dict(h=100, overfetch=1.0, retain=1.0, exact_final_rerank=False)),
        "cfg4": dict(n=10_000_000, d_sparse=100_000_000, d_dense=0, mean_nnz=80.0, zipf_s=1.05,
                     value_law="absnormal", dense_fp16=False, q_mean_nnz=30.0, queries=10_000,
                     index=dict(top_t=None),
                     search=dict(h=10, overfetch=1.0, retain=1.0, exact_final_rerank=False)),
        "cfg5": dict(n=100_000_000, d_sparse=1_000_000_000, d_dense=256, mean_nnz=50.0,
                     zipf_s=1.1, value_law="absnormal", dense_fp16=True, q_mean_nnz=50.0,
                     queries=10_000, index=dict(pq_subspaces=128),
                     search=dict(h=100, overfetch=10.0, retain=10.0, exact_final_rerank=True)),
    }
    sp_ = dict(specs[name])
    base = dict(overfetch=10.0, retain=3.0, h=20, top_t=128, data_threshold=None,
                residual_threshold=0.0, pq_subspaces=None, pq_centers=16, use_whitening=True,
                exact_final_rerank=False, sparse_weight=1.0, dense_weight=1.0, kmeans_iters=25,
                train_sample=50_000, line_capacity=16, seed=0)
    base.update(sp_["index"])
    sp_["index"] = base
    return sp_


def _config_dict(name, spec, n, Q):
    s = spec["search"]
    k1 = min(n, math.ceil(s["overfetch"] * s["h"]))
    return {"workload": name, "n": int(n), "d_sparse": int(spec["d_sparse"]),
            "d_dense": int(spec["d_dense"]), "pq_subspaces": spec["index"]["pq_subspaces"],
            "queries_per_step": int(Q), "h": s["h"], "k1": int(k1),
            "k2": int(min(k1, math.ceil(s["retain"] * s["h"]))),
            "top_t": spec["index"]["top_t"], "exact_final_rerank": s["exact_final_rerank"]}


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="cfg5")
    ap.add_argument("--queries", type=int, default=None)
    ap.add_argument("--n", type=int, default=None)
    ap.add_argument("--top-t", default=None)
    ap.add_argument("--cpu-sample", type=int, default=None)
    ap.add_argument("--cpu-seconds", type=float, default=10.0,
                    help="target CPU work of the cpu_baseline sample (cfg1-4)")
    ap.add_argument("--truth-queries", type=int, default=None)
    ap.add_argument("--qb1", type=int, default=16,
                    help="single-query launches timed for the Qb=1 scan roofline")
    ap.add_argument("--replica-n", type=int, default=REPLICA_N)
    ap.add_argument("--parity-queries", type=int, default=PARITY_QUERIES)
    ap.add_argument("--ref-queries", type=int, default=512)
    ap.add_argument("--ref-step-seconds", type=float, default=3.0)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-parity", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        _relaunch(args)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference_arm(args, rank, world)
        return

    from paper_1903_08690_b200 import synth

    if args.queries is None:
        args.queries = synth.CONFIGS[args.workload].n_queries
    gpu_built = args.workload == "cfg5"
    big = args.workload in ("cfg3", "cfg4", "cfg5")
    if args.cpu_sample is None:
        args.cpu_sample = 8 if big else 24
    if args.truth_queries is None:
        args.truth_queries = 100 if big else args.queries

    import torch

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=dev)

    import paper_1903_08690_b200 as hs
    from paper_1903_08690_b200 import _native as nat
    from paper_1903_08690_b200 import sharded

    cfg = synth.CONFIGS[args.workload]
    s = cfg.search
    h = s["h"]

    # parity replica first (small; freed before the full-size index is built)
    parity, cpu = None, None
    if gpu_built and rank == 0 and not args.no_parity:
        parity, cpu = replica_parity(args, local, s, want_cpu=(world == 1 and not args.no_cpu))
        torch.cuda.synchronize()

    w = (setup_gpu_built if gpu_built else setup_host_built)(args, rank, world, local)
    idx, dev_index, qs = w.index, w.dev, w.qs
    params = hs.search.resolve_params(idx, h, s["overfetch"], s["retain"], s["exact_final_rerank"])
    counts = np.zeros(3, dtype=np.int64)
    nat.check(nat.lib().hs_result_sizes(dev_index.handle, params, nat.ptr(counts)))
    k1, k2, kh = (int(x) for x in counts)
    nq = qs.n
    if world > 1:  # ranks agree on the per-shard result width (pad to h)
        t = torch.tensor([kh], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        kh_all = int(t.item())
    else:
        kh_all = kh

    qb, hold, h2d_bytes = query_device_buffers(qs, idx.d_dense, torch, dev)
    out_ids = torch.full((nq, kh_all), -1, dtype=torch.int64, device=dev)
    out_sc = torch.full((nq, kh_all), -math.inf, dtype=torch.float64, device=dev)
    if world > 1:
        g_ids = torch.empty((world, nq, kh_all), dtype=torch.int64, device=dev)
        g_sc = torch.empty((world, nq, kh_all), dtype=torch.float64, device=dev)
        m_ids = torch.empty((nq, h), dtype=torch.int64, device=dev)
        m_sc = torch.empty((nq, h), dtype=torch.float64, device=dev)
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)
    torch.cuda.synchronize()
    stream = torch.cuda.Stream(dev)
    torch.cuda.set_stream(stream)
    # per-shard outputs are written into the first kh columns (row stride kh)
    o_ids = out_ids if kh == kh_all else torch.empty((nq, kh), dtype=torch.int64, device=dev)
    o_sc = out_sc if kh == kh_all else torch.empty((nq, kh), dtype=torch.float64, device=dev)

    def step(qbuf=qb):
        dev_index.search_dev(qbuf, params, o_ids.data_ptr(), o_sc.data_ptr(), stream.cuda_stream)
        if kh != kh_all:
            out_ids[:, :kh].copy_(o_ids)
            out_sc[:, :kh].copy_(o_sc)
        if world > 1:
            dist.all_gather_into_tensor(g_ids.view(-1), out_ids.view(-1))
            dist.all_gather_into_tensor(g_sc.view(-1), out_sc.view(-1))
            nat.check(nat.lib().hs_shard_merge_dev(
                g_ids.data_ptr(), g_sc.data_ptr(), world, nq, kh_all, h, m_ids.data_ptr(),
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

    # results of the last timed step (merged for N > 1)
    torch.cuda.synchronize()
    res_ids = (m_ids if world > 1 else out_ids).cpu().numpy()
    res_sc = (m_sc if world > 1 else out_sc).cpu().numpy()
    loc_ids, loc_sc = out_ids.cpu().numpy(), out_sc.cpu().numpy()

    # ---- e2e through the public API with host buffers ----
    e2e_steps = max(1, min(args.steps, 10))
    if world == 1:
        kw = dict(overfetch=s["overfetch"], retain=s["retain"],
                  exact_final_rerank=s["exact_final_rerank"])
        for _ in range(2):
            hs.search_batch(idx, qs, h, **kw)
        et = []
        for _ in range(e2e_steps):
            flush.zero_()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            hs.search_batch(idx, qs, h, **kw)
            et.append(time.perf_counter() - t0)
        d2h = nq * kh * (8 + 8)
    else:
        # host queries -> each GPU, shard search, all-gather, merge, merged
        # result back to the host (every step, inside the timed region)
        pin = [t.cpu().pin_memory() for t in hold]
        et = []
        for it in range(e2e_steps + 2):
            flush.zero_()
            torch.cuda.synchronize()
            dist.barrier()
            t0 = time.perf_counter()
            with torch.cuda.stream(stream):
                for dst, src in zip(hold, pin):
                    dst.copy_(src, non_blocking=True)
                step()
                mi, ms = m_ids.to("cpu", non_blocking=False), m_sc.to("cpu", non_blocking=False)
            stream.synchronize()
            tt = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device=dev)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            if it >= 2:
                et.append(float(tt.item()))
        d2h = nq * h * (8 + 8)
        del mi, ms
    e2e = {"value": nq * len(et) / sum(et), "unit": "queries/s",
           "h2d_bytes_per_step": int(h2d_bytes), "d2h_bytes_per_step": int(d2h),
           "ms_per_step": 1e3 * sum(et) / len(et),
           "path": ("search_batch(index, queries) host buffers" if world == 1 else
                    "host queries -> GPUs, shard search, NCCL all-gather, merge, D2H")}

    # ---- per-kernel breakdown (separate profiled steps; timing adds syncs) ----
    dev_index.set_timing(True)
    ktimes = {}
    for _ in range(2):
        flush.zero_()
        torch.cuda.synchronize()
        dev_index.search_dev(qb, params, o_ids.data_ptr(), o_sc.data_ptr(), stream.cuda_stream)
        torch.cuda.synchronize()
        for k, v in dev_index.kernel_times().items():
            ktimes[k] = ktimes.get(k, 0.0) + v / 2
    qb1 = None
    qb1_kernel = None
    qb1_kt = {}
    t1_all = []
    if world == 1 and args.qb1 > 0:
        t1 = []
        for i in range(min(args.qb1, nq)):
            b1, hold1, _ = query_device_buffers(_sub(qs, i, i + 1), idx.d_dense, torch, dev)
            oi = torch.empty((1, kh), dtype=torch.int64, device=dev)
            os_ = torch.empty((1, kh), dtype=torch.float64, device=dev)
            flush.zero_()
            torch.cuda.synchronize()
            dev_index.search_dev(b1, params, oi.data_ptr(), os_.data_ptr(), stream.cuda_stream)
            torch.cuda.synchronize()
            kt = dev_index.kernel_times()
            if i > 0:  # first launch warms the per-launch path
                # the scan kernel alone: the streamed LUT16 filter pass of the
                # filtered stage 1, or the fused k_stage1 where that does not apply
                t1.append(kt.get("lut16_stream", kt.get("stage1", 0.0)))
                t1_all.append(sum(kt.values()))
                qb1_kt = dict(kt)
                qb1_kernel = "k_lut16_stream" if "lut16_stream" in kt else "k_stage1"
        qb1 = float(np.mean(t1)) if t1 else None
    dev_index.set_timing(False)

    # ---- recall@10 vs exact brute force (GPU f64 truth, merged over shards) ----
    truth_q = min(nq, args.truth_queries)
    qsub = _sub(qs, 0, truth_q)
    t_ids, t_sc = exact_truth(dev_index, qsub, 10)
    if world > 1:
        ti = torch.as_tensor(t_ids).to(dev)
        ts = torch.as_tensor(t_sc).to(dev)
        gi = [torch.empty_like(ti) for _ in range(world)]
        gs = [torch.empty_like(ts) for _ in range(world)]
        dist.all_gather(gi, ti)
        dist.all_gather(gs, ts)
        t_ids, _ = sharded.merge_host(torch.stack(gi).cpu().numpy(),
                                      torch.stack(gs).cpu().numpy(), 10)
    rec = [len(np.intersect1d(res_ids[i, :10], t_ids[i])) / 10 for i in range(truth_q)]
    recall = float(np.mean(rec))
    # true top-10 found anywhere in the returned top-h (cfg3's "10@100")
    recall_10_at_h = float(np.mean([len(np.intersect1d(res_ids[i], t_ids[i])) / 10
                                    for i in range(truth_q)]))

    # ---- full-scale sampled checks (exact scores of the returned rows) ----
    full_check = None
    if w.gpu_built and not args.no_parity:
        full_check = fullscale_checks(w, loc_ids, loc_sc, 16, s)

    # ---- parity (host-built workloads): the cpu_baseline sample vs the oracle ----
    if not w.gpu_built and rank == 0 and world == 1 and not args.no_cpu:
        threads = os.cpu_count() or 1
        sample = min(args.cpu_sample, nq)
        idx.config.h = h
        ores, dt, _ = _time_oracle(idx, qs, sample, threads, s)
        if dt < 0.5 * args.cpu_seconds and sample < nq:
            sample = min(nq, max(sample + 1, int(sample * args.cpu_seconds / max(dt, 1e-3))))
            ores, dt, _ = _time_oracle(idx, qs, sample, threads, s)
        mism, worst = 0, 0.0
        for i, (oi, osc, _) in enumerate(ores):
            got = res_ids[i][res_ids[i] >= 0]
            if got.tolist() != oi.tolist():
                mism += 1
            if len(osc):
                worst = max(worst, float(np.max(np.abs(res_sc[i][:len(osc)] - osc)
                                                / np.maximum(np.abs(osc), 1e-300))))
        parity = {"queries": int(sample), "id_mismatch": int(mism), "max_rel_err": worst,
                  "against": "oracle/hybrid_oracle.py on the same index and queries"}
        # single-thread figure beside the all-cores one
        from oracle import hybrid_oracle as O1

        n1 = max(1, min(sample, 4 if big else 12))
        t0u = time.perf_counter()
        O1.search_batch(idx, _sub(qs, 0, n1), h, threads=1, overfetch=s["overfetch"],
                        retain=s["retain"], exact_final_rerank=s["exact_final_rerank"])
        dt1 = time.perf_counter() - t0u
        cpu = {"value": sample / dt, "unit": "queries/s", "cores": threads, "kind": "port",
               "sample": f"first {sample} of {nq} {args.workload} queries, oracle "
                         f"search_batch(threads={threads}), {dt:.1f} s",
               "value_threads1": n1 / dt1, "threads1_sample": f"first {n1} queries, {dt1:.1f} s",
               **_cpu_info()}
    if parity is not None and full_check is not None:
        parity["full_scale"] = full_check
    if parity is not None and rank == 0:
        parity["blas_recipe"] = blas_recipe_check()

    # ---- roofline of the dominant kernel ----
    di = idx.dense_index
    K = di.codebooks.n_subspaces if di is not None else 0
    npairs = (K + 1) // 2
    n_local = int(w.hi - w.lo)
    tc_ms = ktimes.get("lut16_tc")
    s1_ms = ktimes.get("stage1")
    roof = None
    traffic = _traffic(args.workload)
    postings = w.postings
    if tc_ms and K:
        ops = 2.0 * n_local * nq * 16 * K
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
        # other denominators: the analytic kind::i8 issue rate at the SM clock this
        # run held (16384 u8 ops per SM per clock: one M=128, N=256, K=32 MMA per
        # 128 cycles — the floor tools/mma_bench2.cu measures), and 2x the
        # MEASURED_PEAKS bf16 rate (cuBLAS, power-capped at a lower clock: the
        # scan now exceeds it)
        mhz = (clk.summary() or {}).get("sm_mhz")
        if mhz:
            ipk = 148 * 16384 * float(mhz) * 1e6 / 1e12
            roof["issue_peak"] = ipk
            roof["frac_of_issue_peak"] = achieved / ipk
        # SURVEY 8(d)'s byte view of the same pass: one read of the code matrix per group
        # of Qb queries (the pass is compute-bound by design, so this sits far below HBM)
        # (query group of k_lut16_tc: CTA pairs hold 2 x 96 tables for K > 96, one CTA 160 below)
        qb_grp = 192 if K > 96 else 160
        hbm_pk, _ = _peaks()
        passes = -(-nq // qb_grp)
        cs_bytes = float(passes) * n_local * npairs
        roof["code_stream"] = {"Qb": qb_grp, "passes_per_step": passes, "bytes_per_step": cs_bytes,
                               "achieved_gbs": cs_bytes / (tc_ms / 1e3) / 1e9,
                               "frac_of_hbm": cs_bytes / (tc_ms / 1e3) / 1e9 / hbm_pk}
        # the algorithmic work behind those ops: one table lookup-add per (point, query,
        # subspace); the one-hot product spends 32 u8 ops on each
        roof["lookup_adds_per_s"] = float(n_local) * nq * K / (tc_ms / 1e3)
        b2 = _bf16x2_peak()
        if b2:
            roof["peak_2x_measured_bf16"] = b2
            roof["frac_of_2x_measured_bf16"] = achieved / b2
    elif s1_ms:
        alg_bytes = 8 * (postings or 0) + (nq * n_local * npairs if K else 0)
        peak, peak_kind = _peaks()
        achieved = alg_bytes / (s1_ms / 1e3) / 1e9
        roof = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "traffic": traffic.get("dram_bytes_per_launch"),
                "frac_of_nominal_8tbs": achieved / 8000.0,
                "kernel": "k_stage1 (posting stream + selection)", "peak_kind": peak_kind,
                "alg_bytes_per_step": alg_bytes, "kernel_ms_per_step": s1_ms,
                "traffic_source": traffic.get("source"),
                "note": "alg bytes = 8 B per streamed posting (u32 id + f32 weight)"
                        + (" + N*ceil(K/2) code bytes per query" if K else "")}
    if roof is not None and qb1:
        peak, peak_kind = _peaks()
        per_query_bytes = (n_local * npairs + K * 16) + 8 * (postings or 0) / max(nq, 1)
        streamed = qb1_kernel == "k_lut16_stream"
        if streamed:  # the scan kernel reads the codes only (postings go through the buckets)
            per_query_bytes = n_local * npairs + K * 16
        a1 = per_query_bytes / (qb1 / 1e3) / 1e9
        roof["qb1"] = {"scan_ms": qb1, "kernel": qb1_kernel, "alg_bytes": per_query_bytes,
                       "achieved_gbs": a1, "peak_gbs": peak, "frac": a1 / peak,
                       "frac_of_nominal_8tbs": a1 / 8000.0,
                       "query_ms_all_kernels": float(np.mean(t1_all)) if t1_all else None,
                       "query_kernels_ms": {k: round(v, 4) for k, v in qb1_kt.items()},
                       "note": ("single-query path: one query per launch, L2 flushed before "
                                "each launch; scan_ms = the code-stream kernel alone "
                                "(k_lut16_stream filter pass: TMA-staged nibble codes, PRMT "
                                "LUT16, threshold filter), alg bytes = N*ceil(K/2) code bytes "
                                "+ the query's tables; query_ms_all_kernels = every kernel of "
                                "the query (LUT build, sample, scan, candidate scoring, "
                                "select, reranks)") if streamed else
                               ("latency path: one query per launch (CUDA-core LUT16 + "
                                "posting stream, HBM-bound), L2 flushed before each launch"
                                + ("" if postings is not None else "; code bytes only"))}

    if rank == 0:
        spec = _workload_spec(args.workload)
        conf = _config_dict(args.workload, spec, w.n_total, nq)
        conf.update({
            "note": cfg.note, "recall_at_10": recall, "recall_10_at_h": recall_10_at_h,
            "truth_queries": truth_q,
            "l2": "flushed (256 MiB write) before every step, untimed",
            "parallelism": f"id-range shards x{world}" if world > 1 else "single GPU",
            "data_gen": "on-GPU generator (devbuild.cu)" if w.gpu_built else "host generator",
            "index_build": "GPU (hs_builder_*)" if w.gpu_built else "host (+GPU dense encode)",
            "nnz": int(w.nnz), "postings_per_query": (postings / max(nq, 1)
                                                      if postings is not None else None),
            "gen_s": round(w.t_gen, 1), "build_s": round(w.t_build, 1),
            "build_phases_s": {k: round(v, 2) for k, v in w.build_timing.items()},
            "index_bytes_rank0": int(dev_index.memory_bytes()),
            "index_postings_rank0": int(getattr(idx, "nnz_post", 0) or
                                        (len(idx.sparse_index.ids)
                                         if getattr(idx, "sparse_index", None) is not None
                                         and hasattr(idx.sparse_index, "ids") else 0)),
        })
        line = {
            "metric": METRIC, "value": value, "unit": "queries/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_total / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "u8+f64",
            "data": "synthetic (seeded BASELINE-law generator, SURVEY App. B)",
            "config": conf,
            "e2e": e2e, "roofline": roof, "cpu_baseline": cpu, "parity": parity,
            "clocks": clk.summary(), "gpu_launches": int(launches),
            "kernel_ms_per_step": {k: round(v, 4) for k, v in ktimes.items()},
        }
        print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
