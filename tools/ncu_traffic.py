"""Summarise an ncu launch list with DRAM counters per kernel variant, and record it in
profiles/ncu_traffic.json (bench.py reports it as roofline.traffic / roofline.ncu_dram_frac).

The capture (one bench step's queries, every launch, L2 not flushed so the warm-cache
behaviour of the real run is kept):
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
      --clock-control none --cache-control none -k regex:'^k_' --csv --log-file L.csv \
      python tools/bench_queries.py --modes count
  python tools/ncu_traffic.py L.csv C5m "<what>" [--md out.md] [--record]
"""
import argparse
import collections
import csv
import json
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

# kernel name prefix -> gsi KVARIANT name (bench.py's roofline.kernel)
VARIANTS = [("k_join<2>", "join_next"), ("k_join<0>", "join_count"), ("k_join<1>", "join_table"),
            ("k_join<3>", "join_cahead"), ("k_count_fast", "count_fast"), ("k_next_lean", "next_lean"),
            ("k_cahead_warp", "cahead_warp"), ("k_cahead_lean<0, 0>", "cahead_lean"),
            ("k_cahead_lean<1, 0>", "cahead_lean"), ("k_cahead_lean<0, 1>", "final_lean"),
            ("k_cahead_lean<1, 1>", "final_lean"), ("k_final_fp", "final_fp"),
            ("k_filter_partition", "filter_partition"), ("k_refilter", "refilter"),
            ("k_probe_ahead", "probe_ahead"), ("k_small", "small"), ("k_filter(", "filter"),
            ("k_fused_cahead", "fused_cahead"), ("k_final_table", "final_table"), ("k_surv_scan", "surv_scan"),
            ("k_fp_terms", "fp_terms"), ("k_abl_heavy", "abl_heavy"), ("k_abl_join", "ablation"),
            ("k_filter_ml", "filter_ml")]


def variant_of(name: str) -> str:
    n = name.replace("(anonymous namespace)::", "").replace("<unnamed>::", "").replace("unnamed>::", "")
    if n.startswith("void "):
        n = n[5:].replace("unnamed>::", "")
    for pre, v in VARIANTS:
        if n.startswith(pre):
            return v
    return n.split("(")[0]


def load(path):
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[start]
    ix = {h: i for i, h in enumerate(hdr)}
    per = collections.OrderedDict()
    for r in rows[start + 1:]:
        if len(r) < len(hdr):
            continue
        key = (r[ix["ID"]], r[ix["Kernel Name"]])
        d = per.setdefault(key, {})
        v = float(r[ix["Metric Value"]].replace(",", ""))
        unit = r[ix["Metric Unit"]]
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "ns": 1e-9,
                 "usecond": 1e-6, "us": 1e-6, "msecond": 1e-3, "ms": 1e-3, "second": 1.0, "s": 1.0}.get(unit, 1.0)
        d[r[ix["Metric Name"]]] = v * scale
    return per


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("config")
    ap.add_argument("what")
    ap.add_argument("--md", default=None)
    ap.add_argument("--record", action="store_true", help="write profiles/ncu_traffic.json")
    a = ap.parse_args()
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] \
        if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6548.5
    per = load(a.csv)
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
    for (_, name), d in per.items():
        v = variant_of(name)
        x = agg[v]
        x[0] += 1
        x[1] += d.get("gpu__time_duration.sum", 0.0)
        x[2] += d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)
    tot = sum(x[1] for x in agg.values())
    lines = [f"# ncu DRAM traffic per kernel variant — {a.config}: {a.what}", "",
             f"source: `{os.path.relpath(a.csv, ROOT)}`; peak {peak} GB/s (MEASURED_PEAKS.json hbm_gbs)", "",
             "| variant | launches | ms | share | DRAM GB | DRAM GB/s | frac of peak |", "|---|---|---|---|---|---|---|"]
    out = {}
    for v, (n, t, b) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        gbs = b / t / 1e9 if t else 0.0
        lines.append(f"| {v} | {n} | {t * 1e3:.3f} | {t / tot:.3f} | {b / 1e9:.3f} | {gbs:.1f} | {gbs / peak:.3f} |")
        out[v] = {"dram_bytes_per_launch": b / n, "ms_per_launch": t * 1e3 / n, "launches": n,
                  "dram_frac": gbs / peak, "share": t / tot,
                  "source": f"{os.path.relpath(a.csv, ROOT)}: {a.what}"}
    txt = "\n".join(lines) + "\n"
    print(txt)
    if a.md:
        open(a.md, "w").write(txt)
    if a.record:
        p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
        d = json.load(open(p)) if os.path.exists(p) else {}
        for v, e in out.items():   # merge: keep what other captures recorded for other variants
            d.setdefault(a.config, {}).setdefault(v, {}).update(e)
        json.dump(d, open(p, "w"), indent=1)


if __name__ == "__main__":
    main()
