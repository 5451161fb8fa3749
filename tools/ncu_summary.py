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
    all_t = sum(tot.values())
    print(f"| kernel | launches | total ns | share |\n|---|---|---|---|")
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        print(f"| {k} | {cnt[k]} | {v:.0f} | {v / all_t:.1%} |")


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
    for r in rows[2:]:
        name = r[ki].split("(")[0].replace("void ", "").split("<")[0].split("::")[-1]
        print(f"| {name} | " + " | ".join(r[i] for i in idx.values()) + " |")


if __name__ == "__main__":
    {"launches": launches, "full": full}[sys.argv[1]](sys.argv[2])
