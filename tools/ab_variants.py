"""A/B of library builds on the bench's 16 C5m queries in fingerprint mode (the headline pass):
per kernel variant the summed CUDA-event ms (profiled pass, queries one at a time) and the
summed wall ms of an unprofiled pass.  One process per library (GSI_LIB is read at import).

  python tools/ab_variants.py LIB1.so LIB2.so ...
"""
import json
import os
import subprocess
import sys

if len(sys.argv) > 1 and sys.argv[1] != "--child":
    for lib in sys.argv[1:]:
        env = dict(os.environ, GSI_LIB=os.path.abspath(lib))
        out = subprocess.run([sys.executable, __file__, "--child"], env=env, capture_output=True, text=True)
        line = [l for l in out.stdout.splitlines() if l.startswith("{")]
        print(lib, line[-1] if line else out.stderr[-600:], flush=True)
    sys.exit(0)

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import time  # noqa: E402

import torch  # noqa: E402

import workloads as W  # noqa: E402
from paper_1906_03420_b200 import gsi  # noqa: E402

g = W.make_config("C5m", device="cuda")
adj = W._Adj(g, device="cuda")
qs = [W.random_walk_query(g, 12, 1000 + i, adj) for i in range(16)]
del adj
torch.cuda.empty_cache()
graph = gsi.build(g)
ps = [gsi.prepare(graph, q) for q in qs]
for p in ps:   # warm-up (workspace growth, term tables)
    gsi.gsi_query_run(graph, p, fingerprint=True)
torch.cuda.synchronize()
t = time.time()
cnt = 0
for p in ps:
    cnt += gsi.gsi_query_run(graph, p, fingerprint=True).count
torch.cuda.synchronize()
wall = 1000 * (time.time() - t)
var = {}
for p in ps:
    s = gsi.gsi_query_run(graph, p, fingerprint=True, profile=True).stats()
    for i, name in enumerate(gsi.KVARIANT):
        if s["ms_variant"][i]:
            var[name] = var.get(name, 0.0) + s["ms_variant"][i]
print(json.dumps({"wall_ms": round(wall, 1), "count": cnt, "variant_ms": {k: round(v, 1) for k, v in sorted(var.items())}}))
