"""Run selected queries of a workload with per-kernel CUDA-event profiling (gsi profile mode).

  python tools/profile_query.py --config C5b --scale 20 --qidx 8 [--reps 2] [--no-fp]
Used standalone for timings and under `ncu -k regex:k_join ...` for counter captures.
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import workloads as W  # noqa: E402
from paper_1906_03420_b200 import gsi  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C5b")
ap.add_argument("--scale", type=int, default=None)
ap.add_argument("--nlv", type=int, default=None)
ap.add_argument("--qidx", type=int, nargs="+", default=[8])
ap.add_argument("--k", type=int, default=12)
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--no-fp", action="store_true")
ap.add_argument("--table", action="store_true")
ap.add_argument("--enum", action="store_true", help="count_ahead off: enumerate every match of the last level")
a = ap.parse_args()
over = {}
if a.scale:
    over["scale"] = a.scale
if a.nlv:
    over["nlv"] = a.nlv
g = W.make_config(a.config, device="cuda", **over)
adj = W._Adj(g, device="cuda")
qs = {i: W.random_walk_query(g, a.k, 1000 + i, adj) for i in a.qidx}
del adj
graph = gsi.build(g)
for i, q in qs.items():
    for rep in range(a.reps):
        prof = rep == a.reps - 1
        torch.cuda.synchronize()
        t = time.time()
        r = gsi.query(graph, q, profile=prof, fingerprint=not a.no_fp, want_table=a.table, count_ahead=not a.enum)
        torch.cuda.synchronize()
        ms = 1000 * (time.time() - t)
    s = r.stats()
    kern = {gsi.KCLASS[c]: {"ms": round(s["ms_kernel"][c], 3), "launches": s["launches"][c],
                            "alg_GB": round(s["alg_bytes"][c] / 1e9, 3),
                            "alg_GBps": round(s["alg_bytes"][c] / 1e9 / (s["ms_kernel"][c] / 1e3), 1)
                            if s["ms_kernel"][c] else 0} for c in range(6)}
    print(json.dumps({"q": i, "count": r.count, "wall_ms": round(ms, 2), "rows": s["rows"][:q.n],
                      "gba": s["gba"][1:q.n], "chunks": s["n_chunks"], "kernels": kern,
                      "ms_filter": s["ms_filter"], "ms_join": s["ms_join"], "ms_alloc": s["ms_host_alloc"],
                      "ms_sync": s["ms_host_sync"]}), flush=True)
