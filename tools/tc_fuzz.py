"""Shape fuzz of the tensor-core stage 1: random subspace counts and batch sizes
(the chunk count per block, the group width and the ring depth all follow from
them), filtered tensor-core results against the unfiltered CUDA-core scan.

    python tools/tc_fuzz.py [trials] [seed] [small]      # small: batches of 1-15 queries (streamed scan)
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["HSB200_FUSE_SAMPLE"] = "4096"
import numpy as np  # noqa: E402

import paper_1903_08690_b200 as hs  # noqa: E402
from paper_1903_08690_b200 import synth  # noqa: E402

trials = int(sys.argv[1]) if len(sys.argv) > 1 else 16
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 0)
small = len(sys.argv) > 3 and sys.argv[3] == 'small'
bad = 0
for t in range(trials):
    K = int(rng.integers(4, 129))
    nq = int(rng.choice([1, 2, 5, 9, 15] if small else [16, 31, 64, 97, 192, 193, 250, 385, 600]))
    name = "cfg2" if K > 64 else "cfg1"
    ds, qs, cfg = synth.make_config(name, n=70_000, n_queries=nq)
    kw = dict(cfg.index)
    kw.update(pq_subspaces=K, kmeans_iters=2, train_sample=6000)
    idx = hs.build_index(ds, hs.HybridIndexConfig(**kw))
    s = cfg.search
    skw = dict(overfetch=s["overfetch"], retain=s["retain"], exact_final_rerank=True)
    dev = hs.device_index(idx)
    dev.set_timing(True)
    for _ in range(2):  # twice: the second run reuses every ring / counter state
        a = hs.search_batch(idx, qs, s["h"], **skw)
    used_tc = "lut16_tc" in dev.kernel_times() or "lut16_stream" in dev.kernel_times()
    os.environ["HSB200_NO_TC"] = "1"
    os.environ["HSB200_NO_FUSE"] = "1"
    b = hs.search_batch(idx, qs, s["h"], **skw)
    del os.environ["HSB200_NO_TC"], os.environ["HSB200_NO_FUSE"]
    same = all(x.ids.tolist() == y.ids.tolist() and x.scores.tolist() == y.scores.tolist()
               for x, y in zip(a, b))
    bad += 0 if same else 1
    print(f"trial {t}: K={K} nq={nq} tc={used_tc} same={same}", flush=True)
print("tc fuzz:", trials, "trials,", bad, "mismatching")
sys.exit(1 if bad else 0)
