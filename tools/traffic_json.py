"""Write profiles/ncu_traffic.json from a committed `--set full` capture summary: DRAM bytes
(read + write) per launch of the join-class kernels, which bench.py reports as roofline.traffic.

  python tools/traffic_json.py profiles/r1/r1j_join_metrics.md C5m "C5m query 11 join launches"
"""
import json
import os
import sys

path, config, what = sys.argv[1], sys.argv[2], sys.argv[3]
rows = [l.strip().strip("|").split("|") for l in open(path) if l.startswith("|")]
hdr = [h.strip() for h in rows[0]]
ri, wi = hdr.index("dram__bytes_read.sum"), hdr.index("dram__bytes_write.sum")
scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
units = [x.strip() for x in rows[2]]
assert units[0] == "(unit)", "summary lacks the unit row (re-run tools/ncu_summary.py full)"
tot, n = 0.0, 0
for r in rows[3:]:
    r = [x.strip() for x in r]
    tot += float(r[ri]) * scale[units[ri]] + float(r[wi]) * scale[units[wi]]
    n += 1
out_p = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "ncu_traffic.json")
d = json.load(open(out_p)) if os.path.exists(out_p) else {}
d.setdefault(config, {})["join"] = {"dram_bytes_per_launch": tot / max(n, 1), "launches": n,
                                     "source": f"{os.path.relpath(path)}: {what}"}
json.dump(d, open(out_p, "w"), indent=1)
print(d)
