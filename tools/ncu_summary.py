"""Summarise ncu outputs into profiles/ (committed evidence).

  python tools/ncu_summary.py launches gpurun_out/launches.csv     # per-kernel share of device time
  python tools/ncu_summary.py full gpurun_out/prof.ncu-rep          # key metrics of a --set full capture
"""
import collections
import csv
import io
import subprocess
import sys


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr_i = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[hdr_i]
    ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    tot = collections.defaultdict(float)
    cnt = collections.Counter()
    for r in rows[hdr_i + 1:]:
        if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
            continue
        name = r[ki].split("(")[0]
        name = name.replace("void ", "").split("<")[0].split("::")[-1]
        try:
            v = float(r[vi].replace(",", ""))
        except ValueError:
            continue
        tot[name] += v
        cnt[name] += 1
    # graph-build kernels (graph.cu) run once, outside the timed region: listed apart, and the
    # shares are over the query kernels only (what a bench step launches)
    build = {"k_chains", "k_claim1", "k_debug_lookup", "k_empty_list", "k_entries", "k_fill_groups", "k_group_deg",
             "k_home", "k_key_flags", "k_kid_inclusive", "k_label_starts", "k_label_tables", "k_need_empty",
             "k_place", "k_scatter_ci", "k_signatures", "k_unique", "k_validate_edges", "k_validate_vl"}
    q_t = sum(v for k, v in tot.items() if k not in build)
    print("Query kernels (the bench step; share of their total):\n")
    print(f"| kernel | launches | total ns | share |\n|---|---|---|---|")
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        if k not in build:
            print(f"| {k} | {cnt[k]} | {v:.0f} | {v / q_t:.1%} |")
    b_t = sum(v for k, v in tot.items() if k in build)
    print(f"\nGraph build (once, untimed): {sum(cnt[k] for k in build)} launches, {b_t:.0f} ns")


KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "smsp__thread_inst_executed_per_inst_executed.ratio", "l1tex__t_sector_hit_rate.pct",
        "lts__t_bytes.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "launch__grid_size", "launch__occupancy_limit_registers", "sm__maximum_warps_per_active_cycle_pct"]


def full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[0]
    idx = {k: hdr.index(k) for k in KEYS if k in hdr}
    ki = hdr.index("Kernel Name")
    print("| kernel | " + " | ".join(idx) + " |")
    print("|---" * (len(idx) + 1) + "|")
    print("| (unit) | " + " | ".join(rows[1][i] for i in idx.values()) + " |")
    for r in rows[2:]:
        name = r[ki].split("(")[0].replace("void ", "").split("<")[0].split("::")[-1]
        print(f"| {name} | " + " | ".join(r[i] for i in idx.values()) + " |")


if __name__ == "__main__" and sys.argv[1] in ("launches", "full"):
    {"launches": launches, "full": full}[sys.argv[1]](sys.argv[2])


def stalls(path, launch=0, top=15):
    """Stall-reason breakdown and the hottest SASS lines of one captured launch."""
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass",
                          "--launch-skip", str(launch), "--launch-count", "1"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    kname = rows[0][1] if rows and len(rows[0]) > 1 else "?"
    h = rows[1]
    S = h.index("Warp Stall Sampling (All Samples)")
    src = h.index("Source")

    def f(x):
        try:
            return float(x)
        except ValueError:
            return None
    data = [r for r in rows[2:] if len(r) > S and f(r[S]) is not None]
    stall_cols = [i for i, c in enumerate(h) if c.startswith("stall_") and "Not Issued" not in c]
    tot = sum(f(r[S]) for r in data) or 1.0
    agg = collections.Counter()
    for r in data:
        for i in stall_cols:
            v = f(r[i])
            if v:
                agg[h[i]] += v
    print(f"kernel: {kname.split('(')[0]}  (launch {launch}; {int(tot)} warp samples)\n")
    print("| stall reason | share |\n|---|---|")
    for k_, v in agg.most_common(10):
        print(f"| {k_[6:]} | {v / tot:.1%} |")
    print("\n| samples | SASS |\n|---|---|")
    seen = set()
    for r in sorted(data, key=lambda r: -f(r[S])):
        if r[0] in seen:
            continue
        seen.add(r[0])
        print(f"| {int(f(r[S]))} | `{r[src].strip()[:70]}` |")
        if len(seen) >= top:
            break


def details(path, launch=0):
    out = subprocess.run(["ncu", "-i", path, "--page", "details", "--csv", "--launch-skip", str(launch),
                          "--launch-count", "1"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[0]
    si, mi, vi, ui = h.index("Section Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
    keep = ("GPU Speed Of Light Throughput", "Memory Workload Analysis", "Compute Workload Analysis",
            "Occupancy", "Scheduler Statistics", "Warp State Statistics", "Launch Statistics")
    print("| section | metric | value |\n|---|---|---|")
    for r in rows[1:]:
        if r[si] in keep and r[mi]:
            print(f"| {r[si]} | {r[mi]} | {r[vi]} {r[ui]} |")


if __name__ == "__main__" and len(sys.argv) > 1 and sys.argv[1] in ("stalls", "details"):
    fn = {"stalls": stalls, "details": details}[sys.argv[1]]
    fn(sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 0)
