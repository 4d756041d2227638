"""Small searches that reach every mbarrier / TMA / tcgen05 kernel of the hot
path, for compute-sanitizer (racecheck, synccheck, memcheck): a 96-query batch
(k_lut16_tc totals + filter, k_fuse_cands, k_select_radix, k_stage2/3), a
3-query batch (k_lut16_stream totals + filter), the unfiltered k_stage1, and a
sparse-only unpruned index (posting stream).  Sizes are tiny: the sanitizer
slows kernels down by two orders of magnitude.

    compute-sanitizer --tool racecheck python tools/sanitize_probe.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("HSB200_FUSE_SAMPLE", "4096")

import paper_1903_08690_b200 as hs  # noqa: E402
from paper_1903_08690_b200 import synth  # noqa: E402


def scaled(name, n, nq, **over):
    ds, qs, cfg = synth.make_config(name, n=n, n_queries=nq)
    kw = dict(cfg.index)
    kw.update(over)
    kw["kmeans_iters"] = 2
    kw["train_sample"] = min(n, 8000)
    return qs, cfg, hs.build_index(ds, hs.HybridIndexConfig(**kw))


def run(idx, qs, cfg, label):
    s = cfg.search
    r = hs.search_batch(idx, qs, s["h"], overfetch=s["overfetch"], retain=s["retain"],
                        exact_final_rerank=s["exact_final_rerank"])
    print(label, "ok:", len(r), "queries,", len(r[0].ids), "ids each", flush=True)


qs, cfg, idx = scaled("cfg2", 40_000, 96)
run(idx, qs, cfg, "hybrid K=128, 96 queries (tensor-core filtered stage 1)")
run(idx, hs.HybridDataset(qs.sparse[:3], qs.dense[:3]), cfg,
    "hybrid K=128, 3 queries (streamed LUT16 filtered stage 1)")
os.environ["HSB200_NO_FUSE"] = "1"
run(idx, hs.HybridDataset(qs.sparse[:2], qs.dense[:2]), cfg,
    "hybrid K=128, 2 queries (unfiltered k_stage1)")
del os.environ["HSB200_NO_FUSE"]
qs, cfg, idx = scaled("cfg4", 40_000, 4)
run(idx, qs, cfg, "sparse-only unpruned, 4 queries (posting stream)")
print("sanitize probe done", flush=True)
