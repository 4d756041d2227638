"""Where does the host-API (e2e) time go?  Times the pieces of search_batch.

python tools/e2e_probe.py [--workload cfg2]
"""

import argparse
import ctypes
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="cfg2")
    ap.add_argument("--queries", type=int, default=None)
    ap.add_argument("--n", type=int, default=None)
    ap.add_argument("--top-t", default=None)
    ap.add_argument("--reps", type=int, default=5)
    args = ap.parse_args()
    import bench
    import paper_1903_08690_b200 as hs
    from paper_1903_08690_b200 import _native as nat, search as S, synth

    if args.queries is None:
        args.queries = synth.CONFIGS[args.workload].n_queries
    cfg, ds_full, ds, qs, idx, icfg, lo, tg, tb = bench.build_workload(args, 0, 1)
    s = cfg.search
    h = s["h"]
    kw = dict(overfetch=s["overfetch"], retain=s["retain"], exact_final_rerank=s["exact_final_rerank"])
    for _ in range(2):
        hs.search_batch(idx, qs, h, **kw)
    rows = []
    for _ in range(args.reps):
        t0 = time.perf_counter()
        p = S._resolve(idx, h, kw["overfetch"], kw["retain"], kw["exact_final_rerank"])
        q = S.query_arrays(qs, int(idx.d_dense))
        S._validate_queries(q, int(idx.d_sparse), int(idx.d_dense))
        dev = S.device_index(idx, 0)
        counts = np.zeros(3, dtype=np.int64)
        nat.check(nat.lib().hs_result_sizes(dev.handle, ctypes.byref(p), nat.ptr(counts)))
        k1, k2, kh = (int(x) for x in counts)
        ids = np.empty((q.nq, kh), dtype=np.int64)
        sc = np.empty((q.nq, kh), dtype=np.float64)
        secs = np.zeros(3)
        b = q.batch()
        t1 = time.perf_counter()
        nat.check(nat.lib().hs_search_batch(dev.handle, ctypes.byref(b), ctypes.byref(p),
                                            nat.ptr(ids), nat.ptr(sc), nat.ptr(secs)))
        t2 = time.perf_counter()
        per_q = (secs / q.nq).tolist()
        res = [hs.SearchResult(ids=ids[i], scores=sc[i],
                               stages=hs.StageStats(candidates=[k1, k2, kh], seconds=list(per_q)))
               for i in range(q.nq)]
        t3 = time.perf_counter()
        t4 = time.perf_counter()
        hs.search_batch(idx, qs, h, **kw)
        t5 = time.perf_counter()
        rows.append((1e3 * (t1 - t0), 1e3 * (t2 - t1), 1e3 * (t3 - t2), 1e3 * (t5 - t4),
                     1e3 * secs.sum()))
        del res
    for r in rows:
        print("prep %.2f ms  c_call %.2f ms  pack %.2f ms  | full %.2f ms  | stage_sum %.2f ms" % r)
    dev = S.device_index(idx, 0)
    dev.set_timing(True)
    hs.search_batch(idx, qs, h, **kw)
    print("kernels", {k: round(v, 3) for k, v in dev.kernel_times().items()})
    dev.set_timing(False)


if __name__ == "__main__":
    main()
