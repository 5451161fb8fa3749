#!/bin/bash
# round-2 GPU session W: final-state ncu evidence — k_filter_tw (C4), k_join<J_NEXT> (bench q0), fp launch list
out=gpurun_out; mkdir -p $out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_filter_tw" -s 1 -c 1 -o $out/w_filter_c4 python tools/small_latency.py --configs C4 --queries 1 --reps 1 > $out/w_filter.log 2>&1; tail -1 $out/w_filter.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_join<2>" -s 4 -c 3 -o $out/w_join_next python tools/bench_queries.py --qidx 0 --modes fp > $out/w_jn.log 2>&1; tail -1 $out/w_jn.log
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --cache-control none \
  -k regex:'^k_' --csv --log-file $out/w_fp_launches.csv python tools/bench_queries.py --modes fp > $out/w_fp_launches.log 2>&1; tail -2 $out/w_fp_launches.log
python tools/ncu_traffic.py $out/w_fp_launches.csv C5m "bench step, fp mode (headline), ncu serialised launch list (r2w)" --md $out/w_fp_traffic.md | head -12
