"""Per-query workload calibration on the GPU: count, time, per-level |M_t| and |GBA|.

  python tools/calibrate.py --config C5b --scale 22 --nlv 10 --queries 20 --timeout 10
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
ap.add_argument("--nle", type=int, default=None)
ap.add_argument("--queries", type=int, default=20)
ap.add_argument("--k", type=int, default=12)
ap.add_argument("--timeout", type=float, default=10.0)
ap.add_argument("--fp", action="store_true", help="fingerprint on: enumerate every match")
a = ap.parse_args()
over = {}
if a.scale:
    over["scale"] = a.scale
if a.nlv:
    over["nlv"] = a.nlv
if a.nle:
    over["nle"] = a.nle
t = time.time()
g = W.make_config(a.config, device="cuda", **over)
adj = W._Adj(g, device="cuda")
qs = [W.random_walk_query(g, a.k, 1000 + i, adj) for i in range(a.queries)]
del adj
print(f"gen {time.time() - t:.1f}s n={g.n} m={g.m}", flush=True)
t = time.time()
graph = gsi.build(g)
print(f"build {time.time() - t:.2f}s {graph.info()}", flush=True)
tot_c, tot_ms = 0, 0.0
for i, q in enumerate(qs):
    t = time.time()
    r = gsi.query(graph, q, timeout_s=a.timeout, partial_on_timeout=True, fingerprint=a.fp)
    torch.cuda.synchronize()
    ms = 1000 * (time.time() - t)
    s = r.stats()
    tot_c += r.count
    tot_ms += ms
    print(json.dumps({"q": i, "E": q.m, "count": r.count, "ms": round(ms, 2), "capped": s["capped"],
                      "rows": s["rows"][:q.n], "gba": s["gba"][1:q.n], "chunks": s["n_chunks"], "ms_filter": round(s["ms_filter"], 3), "ms_plan": round(s["ms_plan"], 3),
                      "ms_join": round(s["ms_join"], 3), "launches": s["total_launches"],
                      "cand": s["cand"][:q.n]}), flush=True)
print(f"TOTAL matches={tot_c} ms={tot_ms:.1f} matches/s={tot_c / (tot_ms / 1e3):.3e}")
