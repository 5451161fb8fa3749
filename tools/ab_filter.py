"""A/B of library builds on the filter alone: per config, the median CUDA-event time of the
filter launch over 16 walk queries (profiled runs, count mode), one process per library.

  python tools/ab_filter.py [--configs C4 C5m] --libs LIB1.so LIB2.so ...
"""
import argparse
import json
import os
import subprocess
import sys

ap = argparse.ArgumentParser()
ap.add_argument("--configs", nargs="+", default=["C4", "C5m"])
ap.add_argument("--child", action="store_true")
ap.add_argument("--libs", nargs="*", default=[])
a = ap.parse_args()
if not a.child:
    for lib in a.libs:
        env = dict(os.environ, GSI_LIB=os.path.abspath(lib))
        out = subprocess.run([sys.executable, __file__, "--child", "--configs", *a.configs], env=env,
                             capture_output=True, text=True)
        for line in out.stdout.splitlines():
            print(lib, line, flush=True)
        if out.returncode:
            print(lib, out.stderr[-800:])
    sys.exit(0)

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import workloads as W  # noqa: E402
from paper_1906_03420_b200 import gsi  # noqa: E402

for cfg in a.configs:
    g = W.make_config(cfg, device="cuda")
    adj = W._Adj(g, device="cuda")
    qs = [W.random_walk_query(g, 12, 1000 + i, adj) for i in range(16)]
    del adj
    torch.cuda.empty_cache()
    graph = gsi.build(g)
    ps = [gsi.prepare(graph, q) for q in qs]
    ms, loads = [], []
    for p in ps:
        gsi.gsi_query_run(graph, p, fingerprint=False, timeout_s=2.0, partial_on_timeout=True)
        s = gsi.gsi_query_run(graph, p, fingerprint=False, profile=True, timeout_s=2.0, partial_on_timeout=True).stats()
        ms.append(s["ms_kernel"][0])
        loads.append(s["alg_bytes"][0])
    print(json.dumps({"config": cfg, "filter_ms_median": round(float(np.median(ms)), 4),
                      "filter_ms_mean": round(float(np.mean(ms)), 4),
                      "alg_GBps_median": round(float(np.median(np.array(loads) / 1e9 / (np.array(ms) / 1e3))), 1)}),
          flush=True)
    del ps, graph
    gsi.gsi_trim_workspace()
    torch.cuda.empty_cache()
