"""Time the GPU dense build (hs_dense_encode) against the host builder at a
cfg2/cfg5-like shape (d=256, K=128 two-dim subspaces, 16 centers)."""
import json
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_1903_08690_b200 as hs  # noqa: E402
from paper_1903_08690_b200 import builder as B  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 2_000_000
d, K = 256, 128
rng = np.random.default_rng(0)
vec = rng.standard_normal((n, d))
order = rng.permutation(n).astype(np.int64)
cb = hs.Codebooks(subdims=np.full(K, 2, np.int64),
                  centers=[rng.standard_normal((16, 2)).astype(np.float32) for _ in range(K)])
B.dense_encode_gpu(vec[:1000], order[order < 1000] if False else np.arange(1000), cb, 0)  # warm
t = {}
t0 = time.time()
pq, sq = B.dense_encode_gpu(vec, order, cb, 0, timing=t)
wall_gpu = time.time() - t0
t0 = time.time()
codes = B.pq_encode(vec, cb)[order]
ref_sq = B.sq_residual(vec, order, codes, cb)
wall_host = time.time() - t0
same = bool(np.array_equal(pq.packed, B.pack_codes(codes)) and np.array_equal(sq.codes, ref_sq.codes)
            and np.array_equal(sq.step, ref_sq.step))
alg = n * d * 8 * 2 + n * (K // 2) + n * d  # vectors read twice + codes + sq out
print(json.dumps({"n": n, "d": d, "K": K, "kernel_s": t["dense_encode_s"],
                  "kernel_gbs": alg / t["dense_encode_s"] / 1e9, "call_wall_s": wall_gpu,
                  "host_wall_s": wall_host, "identical": same}))
