"""Probe of k_lut16_stream (single-query LUT16 scan): one GPU-built index, then
single-query searches under each block-scheduling setting, reporting the scan
kernel's time (CUDA events of the per-kernel breakdown) and its share of the
HBM peak.  Results (ids, scores) must agree across settings.

    python tools/stream_probe.py [n] [K] [settings...]     e.g.  10000000 64 d s
'd' = ticket (dynamic) block scheduling, the default; 's' = static stride.
"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1903_08690_b200 as hs  # noqa: E402
from paper_1903_08690_b200 import _native as nat, synth  # noqa: E402
from bench import query_device_buffers, _sub  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 10_000_000
K = int(sys.argv[2]) if len(sys.argv) > 2 else 64
settings = sys.argv[3:] or ["d", "s"]
d = 2 * K
law = synth.HybridLaw(n, max(1000, n * 10), d, 50.0, 1.1, "absnormal", dense_fp16=True)
qlaw = synth.HybridLaw(n, law.d_sparse, d, 50.0, 1.1, "absnormal", dense_fp16=False)
dev = torch.device("cuda", 0)
torch.cuda.set_device(0)
dd = hs.DeviceDataset.generate(law, seed=0)
qs = hs.DeviceDataset.generate(qlaw, seed=1, n=24).download()
icfg = hs.HybridIndexConfig(pq_subspaces=K, pq_centers=16, seed=0, kmeans_iters=2)
idx = dd.build(icfg).finish()
dix = idx.handle
h = 100
params = hs.search.resolve_params(idx, h, 10.0, 10.0, True)
counts = np.zeros(3, dtype=np.int64)
nat.check(nat.lib().hs_result_sizes(dix.handle, params, nat.ptr(counts)))
kh = int(counts[2])
flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)
stream = torch.cuda.Stream(dev)
torch.cuda.set_stream(stream)
peak = json.load(open(os.path.join(os.path.dirname(__file__), "..", "MEASURED_PEAKS.json")))["hbm_gbs"]
code_bytes = n * ((K + 1) // 2)
# share of table rows with an entry >= 128 (the rows that need the mask-and-blend lookup)
try:
    from paper_1903_08690_b200 import whiten_apply
    di = idx.dense_index
    fr = []
    for i in range(qs.n):
        qd = np.asarray(qs.dense[i], dtype=np.float64)
        if di.whitening is not None:
            qd = whiten_apply(di.whitening, qd, "query")
        ql = hs.quantize_lut(hs.adc_table(qd, di.codebooks))
        fr.append(float((np.asarray(ql.table) >= 128).any(axis=1).mean()))
    print("big-row share per query: mean %.3f min %.3f max %.3f" % (np.mean(fr), min(fr), max(fr)), flush=True)
except Exception as e:  # noqa: BLE001
    print("big-row share: n/a (%r)" % (e,), flush=True)
ref = None
out = {}
for s in settings:
    os.environ["HSB200_STREAM_STATIC"] = "1" if s.endswith("s") else "0"
    dix.set_timing(True)
    ts, res = [], []
    for i in range(qs.n):
        b1, hold, _ = query_device_buffers(_sub(qs, i, i + 1), idx.d_dense, torch, dev)
        oi = torch.empty((1, kh), dtype=torch.int64, device=dev)
        osc = torch.empty((1, kh), dtype=torch.float64, device=dev)
        flush.zero_()
        torch.cuda.synchronize()
        dix.search_dev(b1, params, oi.data_ptr(), osc.data_ptr(), stream.cuda_stream)
        torch.cuda.synchronize()
        kt = dix.kernel_times()
        if i >= 2:
            ts.append(kt["lut16_stream"])
        res.append((oi.cpu().numpy().copy(), osc.cpu().numpy().copy()))
    dix.set_timing(False)
    if ref is None:
        ref = res
    same = all(np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1]) for a, b in zip(ref, res))
    ms = float(np.median(ts))
    out[s] = {"scan_ms_median": ms, "scan_ms_min": float(np.min(ts)),
              "gbs": code_bytes / ms / 1e6, "frac": code_bytes / ms / 1e6 / peak,
              "same_results": bool(same)}
    print(s, out[s], flush=True)
print(json.dumps({"n": n, "K": K, "peak_gbs": peak, "settings": out}))
