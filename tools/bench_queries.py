"""Per-query modes of the bench workload: count-only (count-ahead), count-ahead off and
fingerprinted (every final match read and hashed), with the counts, device times and the
kernel variants each mode launched.

  python tools/bench_queries.py [--config C5m] [--queries 16] [--modes count enum fp] [--timeout 30]
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

MODES = {"count": dict(fingerprint=False), "enum": dict(fingerprint=False, count_ahead=False),
         "fp": dict(fingerprint=True), "table": dict(fingerprint=False, want_table=True)}

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C5m")
ap.add_argument("--queries", type=int, default=16)
ap.add_argument("--qidx", type=int, nargs="*", default=None)
ap.add_argument("--k", type=int, default=12)
ap.add_argument("--modes", nargs="+", default=["count", "enum", "fp"])
ap.add_argument("--timeout", type=float, default=30.0)
ap.add_argument("--profile", action="store_true")
a = ap.parse_args()
g = W.make_config(a.config, device="cuda")
adj = W._Adj(g, device="cuda")
idx = a.qidx if a.qidx else list(range(a.queries))
qs = {i: W.random_walk_query(g, a.k, 1000 + i, adj) for i in idx}
del adj
torch.cuda.empty_cache()
graph = gsi.build(g)
for i, q in qs.items():
    out = {"q": i}
    for m in a.modes:
        torch.cuda.synchronize()
        t = time.time()
        try:
            r = gsi.query(graph, q, timeout_s=a.timeout, partial_on_timeout=True, profile=a.profile, **MODES[m])
        except gsi.GsiError as e:
            out[m] = {"error": str(e)}
            continue
        torch.cuda.synchronize()
        s = r.stats()
        d = {"count": r.count, "ms": round(1000 * (time.time() - t), 2), "capped": s["capped"],
             "variants": s["variants"]}
        if m == "fp":
            d["fp"] = [str(x) for x in r.fingerprint()]
        if a.profile:
            d["kernel_ms"] = {gsi.KCLASS[c]: round(s["ms_kernel"][c], 3) for c in range(6) if s["ms_kernel"][c]}
        out[m] = d
    print(json.dumps(out), flush=True)
