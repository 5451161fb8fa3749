#!/bin/bash
# round-2 GPU session Z: final-state evidence — J_NEXT capture (heaviest launch), fp launch list (recorded), bench
out=gpurun_out; mkdir -p $out
timeout 1500 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"k_join<\(int\)2>" -s 159 -c 1 -o $out/z_join_next python tools/bench_queries.py --modes fp > $out/z_jn.log 2>&1; tail -1 $out/z_jn.log
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --cache-control none \
  -k regex:'^k_' --csv --log-file $out/z_fp_launches.csv python tools/bench_queries.py --modes fp > $out/z_fp_launches.log 2>&1; tail -1 $out/z_fp_launches.log
python tools/ncu_traffic.py $out/z_fp_launches.csv C5m "bench step, fp mode (headline), ncu serialised launch list (r2z)" --md $out/z_fp_traffic.md | head -14
