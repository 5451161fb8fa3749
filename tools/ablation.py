"""NEXT-3 / NEXT-2: the paper's join-phase ablations on B200 (Tables VI-VIII,
L1467-1641; load balance and duplicate removal, §VI).

Runs the bench-style random-walk queries of a workload through the paper-style engine
(`gsi_query_opts.ablation`, one warp per row of M) with the techniques added one by one —
GSI- (CR lookup, two-step output, naive set operation, no write cache), +DS (PCSR), +PC
(Prealloc-Combine), +SO (GPU-friendly set operation), +WC (write cache), +LB (4-layer balance,
heavy rows by 8-CTA clusters), +DR (block duplicate removal, Alg. 5) — and then the B200
default path (fused per-level kernels) and its one-launch small-query path.  Every variant
must give the same count and fingerprint (asserted).  Device time per query = the library's
own ms_total with the host waiting on the result.

  python tools/ablation.py --config C3 --nlv 10 --queries 16 [--md out.md]
Under `ncu --metrics <ld/st sector counters>` the same script gives the load/store trends.
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

E, CR, TWO, NOWC, NAIVE = gsi.ABL_ENGINE, gsi.ABL_CR, gsi.ABL_TWO_STEP, gsi.ABL_NO_WCACHE, gsi.ABL_NAIVE_SO
NOLB, NODR = gsi.ABL_NO_LB, gsi.ABL_NO_DR
LADDER = [("GSI- (CR, two-step, naive SO, no WC, no LB, no DR)", dict(ablation=E | CR | TWO | NAIVE | NOWC | NOLB | NODR)),
          ("+DS (PCSR)", dict(ablation=E | TWO | NAIVE | NOWC | NOLB | NODR)),
          ("+PC (Prealloc-Combine)", dict(ablation=E | NAIVE | NOWC | NOLB | NODR)),
          ("+SO (GPU-friendly set op)", dict(ablation=E | NOWC | NOLB | NODR)),
          ("+WC (write cache)", dict(ablation=E | NOLB | NODR)),
          ("+LB (4-layer balance: block / 8-CTA cluster rows)", dict(ablation=E | NODR)),
          ("+DR (block duplicate removal) = paper GSI", dict(ablation=E)),
          ("B200 fused per-level path", dict(small=False)),
          ("B200 default (small-query path when it fits)", dict())]

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C3")
ap.add_argument("--nlv", type=int, default=None)
ap.add_argument("--queries", type=int, default=16)
ap.add_argument("--k", type=int, default=8)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--max-count", type=float, default=2e8, help="skip queries with more matches")
ap.add_argument("--md", default=None)
ap.add_argument("--only", type=int, default=None, help="run only ladder step i (for ncu)")
a = ap.parse_args()
over = {"nlv": a.nlv} if a.nlv else {}
g = W.make_config(a.config, device="cuda", **over)
graph = gsi.build(g)
adj = W._Adj(g, device="cuda")
qs = [W.random_walk_query(g, a.k, 1000 + i, adj) for i in range(a.queries)]
del adj
ps = [gsi.prepare(graph, q) for q in qs]
ref = [gsi.gsi_query_run(graph, p, fingerprint=True) for p in ps]
keep = [i for i, r in enumerate(ref) if 0 < r.count <= a.max_count]
rows = []
for li, (name, kw) in enumerate(LADDER):
    if a.only is not None and li != a.only:
        continue
    ms = []
    for i in keep:
        best = None
        for _ in range(a.reps):
            torch.cuda.synchronize()
            t = time.perf_counter()
            r = gsi.gsi_query_run(graph, ps[i], fingerprint=True, **kw)
            torch.cuda.synchronize()
            el = 1000 * (time.perf_counter() - t)
            best = el if best is None else min(best, el)
        assert r.count == ref[i].count and r.fingerprint() == ref[i].fingerprint(), (name, i)
        ms.append(best)
    rows.append((name, float(np.sum(ms)), float(np.mean(ms))))
    print(json.dumps({"variant": name, "total_ms": rows[-1][1], "mean_ms": rows[-1][2], "queries": len(keep)}),
          flush=True)
if a.md and a.only is None:
    lines = [f"# NEXT-3 join-phase ablations on B200 — {a.config}{' |L_V|=' + str(a.nlv) if a.nlv else ''}, "
             f"{len(keep)} {a.k}-vertex walk queries (seeds 1000+), {sum(ref[i].count for i in keep)} matches", "",
             "Wall time per query around a synchronous gsi_query_run (fingerprint on: every match hashed), best of "
             f"{a.reps}; every variant's count and fingerprint equal the default path's (asserted).", "",
             "| variant | total ms | mean ms/query | speedup vs previous |", "|---|---|---|---|"]
    prev = None
    for name, tot, mean in rows:
        sp = f"{prev / tot:.2f}x" if prev else "-"
        lines.append(f"| {name} | {tot:.2f} | {mean:.3f} | {sp} |")
        prev = tot
    open(a.md, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))
