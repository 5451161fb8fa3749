"""Small-query latency breakdown (C2 / C4): per query the host wall time around a synchronous
gsi_query_run and the library's phase times (filter, plan, join; host sync / allocation), and
a GSI_TRACE device timeline of one query.

  python tools/small_latency.py [--configs C2 C4] [--queries 16]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import workloads as W  # noqa: E402
from paper_1906_03420_b200 import gsi  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--configs", nargs="+", default=["C2", "C4"])
ap.add_argument("--queries", type=int, default=16)
ap.add_argument("--reps", type=int, default=7)
a = ap.parse_args()
for cfg in a.configs:
    g = W.make_config(cfg, device="cuda")
    adj = W._Adj(g, device="cuda")
    qs = [W.random_walk_query(g, 12, 1000 + i, adj) for i in range(a.queries)]
    graph = gsi.build(g)
    torch.cuda.synchronize()
    ps = [gsi.prepare(graph, q) for q in qs]
    rows = []
    for p in ps:
        gsi.gsi_query_run(graph, p, fingerprint=False)
        ts = []
        for _ in range(a.reps):
            t = time.perf_counter()
            r = gsi.gsi_query_run(graph, p, fingerprint=False)
            ts.append(1e3 * (time.perf_counter() - t))
        s = r.stats()
        rows.append({"wall_ms": float(np.median(ts)), "ms_total": s["ms_total"], "ms_filter": s["ms_filter"],
                     "ms_plan": s["ms_plan"], "ms_join": s["ms_join"], "ms_host_sync": s["ms_host_sync"],
                     "ms_host_alloc": s["ms_host_alloc"], "launches": s["total_launches"],
                     "small": s["variants"].get("small", 0), "count": r.count})
    keys = ["wall_ms", "ms_total", "ms_filter", "ms_plan", "ms_join", "ms_host_sync", "ms_host_alloc", "launches"]
    print(json.dumps({"config": cfg, "median": {k: float(np.median([x[k] for x in rows])) for k in keys},
                      "per_query": rows}), flush=True)
    # one profiled query: per-launch device timeline
    r = gsi.gsi_query_run(graph, ps[0], fingerprint=False, profile=True)
    s = r.stats()
    print(json.dumps({"config": cfg, "profiled_q0": {"ms_kernel": s["ms_kernel"], "launches": s["launches"],
                                                    "ms_total": s["ms_total"]}}), flush=True)
    os.environ["GSI_TRACE"] = "1"
    gsi.gsi_query_run(graph, ps[0], fingerprint=False, profile=True)
    os.environ.pop("GSI_TRACE")
    del ps, graph
    gsi.gsi_trim_workspace()
    torch.cuda.empty_cache()
