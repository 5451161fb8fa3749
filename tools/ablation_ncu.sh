#!/bin/bash
# Load/store trends of the NEXT-2/NEXT-3 ladder (tools/ablation.py --only i) under ncu:
# global load / store sectors, DRAM bytes and device time summed over the step's kernels.
# usage: bash tools/ablation_ncu.sh <tag> <config> <nlv> <k>
tag=${1:-r2e}; cfg=${2:-C3}; nlv=${3:-10}; k=${4:-8}
out=gpurun_out; mkdir -p $out
for i in 0 1 2 3 4 5 6 7; do
  timeout 600 ncu --metrics gpu__time_duration.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_st.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none -k regex:'^k_' --csv --log-file $out/${tag}_abl_$i.csv \
    python tools/ablation.py --config $cfg --nlv $nlv --k $k --queries 16 --reps 1 --only $i > $out/${tag}_abl_$i.log 2>&1
done
python - "$tag" <<'PY'
import csv, sys, collections
tag = sys.argv[1]
names = ["GSI-", "+DS", "+PC", "+SO", "+WC", "+LB", "+DR (paper GSI)", "B200 fused"]
print("| step | kernels | ms | ld sectors (M) | st sectors (M) | DRAM GB |")
print("|---|---|---|---|---|---|")
for i, nm in enumerate(names):
    try:
        rows = list(csv.reader(open(f"gpurun_out/{tag}_abl_{i}.csv")))
    except FileNotFoundError:
        continue
    st = next(j for j, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[st]; ix = {h: j for j, h in enumerate(hdr)}
    tot = collections.Counter(); ids = set()
    for r in rows[st + 1:]:
        if len(r) < len(hdr): continue
        ids.add(r[ix["ID"]])
        v = float(r[ix["Metric Value"]].replace(",", "")); u = r[ix["Metric Unit"]]
        sc = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "sector": 1}.get(u, 1)
        tot[r[ix["Metric Name"]]] += v * sc
    print(f"| {nm} | {len(ids)} | {tot['gpu__time_duration.sum']:.2f} | {tot['l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum']/1e6:.2f} | "
          f"{tot['l1tex__t_sectors_pipe_lsu_mem_global_op_st.sum']/1e6:.2f} | "
          f"{(tot['dram__bytes_read.sum'] + tot['dram__bytes_write.sum'])/1e9:.3f} |")
PY
