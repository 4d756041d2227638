import os, sys, numpy as np
sys.path.insert(0, '.')
os.environ.setdefault("HSB200_LIB_TAG", "prof")
import paper_1903_08690_b200 as hs
from paper_1903_08690_b200 import synth
cfg = synth.CONFIGS["cfg5"]
law = synth.replica_law(cfg.data, int(sys.argv[1]) if len(sys.argv) > 1 else 10_000_000)
qlaw = synth.HybridLaw(law.n, law.d_sparse, law.d_dense, 50.0, law.zipf_s, law.value_law, dense_fp16=False)
dd = hs.DeviceDataset.generate(law, seed=0)
qs = hs.DeviceDataset.generate(qlaw, seed=1, n=192).download()
g = dd.build(cfg.index_config(kmeans_iters=2)).finish()
print("search", flush=True)
r = hs.search_batch(g, qs, 100, overfetch=10.0, retain=10.0, exact_final_rerank=True)
print("done", flush=True)
