#!/bin/bash
# round-2 GPU session AK: C4 launch list over 10 queries, final bench line
out=gpurun_out; mkdir -p $out
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --cache-control none \
  -k regex:'^k_' --csv --log-file $out/ak_c4_launches.csv python tools/small_latency.py --configs C4 --queries 10 --reps 1 > $out/ak_c4.log 2>&1; tail -1 $out/ak_c4.log
python tools/ncu_traffic.py $out/ak_c4_launches.csv C4 "10 C4 walk queries (small path), ncu serialised launch list (r2ak)" --md $out/ak_c4_traffic.md | head -12
timeout 1500 python bench.py > $out/ak_bench.json 2> $out/ak_bench.err; tail -c 300 $out/ak_bench.json; tail -3 $out/ak_bench.err
