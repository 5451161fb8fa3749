"""Summarise an `ncu --set full` capture (.ncu-rep) of one kernel launch into markdown (the key
speed-of-light, pipe, memory and stall counters) and optionally record its pipe activity in
profiles/ncu_traffic.json under the kernel variant (bench.py reports it beside the roofline).

  python tools/ncu_full_summary.py REP.ncu-rep CONFIG VARIANT "<what>" --md OUT.md [--record]
"""
import argparse
import csv
import io
import json
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "l1tex__t_sector_hit_rate.pct", "lts__t_sector_hit_rate.pct", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__occupancy_limit_registers",
        "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
        "smsp__thread_inst_executed_per_inst_executed.ratio", "sm__cycles_elapsed.avg.per_second"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("config")
    ap.add_argument("variant")
    ap.add_argument("what")
    ap.add_argument("--md", required=True)
    ap.add_argument("--record", action="store_true")
    a = ap.parse_args()
    raw = subprocess.run(["ncu", "-i", a.rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    lines = [f"# ncu --set full — {a.config} {a.variant}: {a.what}", "", f"source: `{os.path.relpath(a.rep, ROOT)}`", "",
             "| launch | metric | value | unit |", "|---|---|---|---|"]
    first = None
    for li, r in enumerate(rows[2:]):
        d = {}
        for k in KEYS:
            if k in hdr:
                v = r[hdr.index(k)]
                d[k] = v
                lines.append(f"| {li} {r[hdr.index('Kernel Name')][:40]} | {k} | {v} | {units[hdr.index(k)]} |")
        first = first or d
    txt = "\n".join(lines) + "\n"
    open(a.md, "w").write(txt)
    print(txt)
    if a.record and first:
        p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
        js = json.load(open(p)) if os.path.exists(p) else {}
        e = js.setdefault(a.config, {}).setdefault(a.variant, {})
        f = lambda k: float(first[k].replace(",", "")) if k in first else None
        e["alu_pipe_active"] = f("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active") / 100.0
        e["fma_pipe_active"] = f("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active") / 100.0
        e["issue_active"] = f("smsp__issue_active.avg.pct_of_peak_sustained_active") / 100.0
        e["full_capture"] = f"{os.path.relpath(a.md, ROOT)}: {a.what}"
        json.dump(js, open(p, "w"), indent=1)


if __name__ == "__main__":
    main()
