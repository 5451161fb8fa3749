#!/bin/bash
# round-2 GPU session D: bench (fixed profiler), parity + ext, table-mode ncu, scale-test timings
out=gpurun_out; mkdir -p $out
timeout 1500 python bench.py > $out/d_bench.json 2> $out/d_bench.err; tail -c 400 $out/d_bench.json; tail -2 $out/d_bench.err
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_ext.py -q --timeout 600 --durations=12 > $out/d_pytest_parity.log 2>&1; tail -16 $out/d_pytest_parity.log
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --cache-control none \
  -k regex:'^k_' --csv --log-file $out/d_table_launches.csv python tools/bench_queries.py --qidx 2 3 10 14 --modes table > $out/d_table_launches.log 2>&1
python tools/ncu_traffic.py $out/d_table_launches.csv C5m "table mode, queries 2 3 10 14" --md $out/d_table_traffic.md | head -12
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_final_table -c 1 -o $out/d_ftab python tools/bench_queries.py --qidx 10 --modes table > $out/d_ftab.log 2>&1; tail -2 $out/d_ftab.log
timeout 1800 python -m pytest tests/test_gpu_scale.py -v --timeout 1200 --durations=0 > $out/d_pytest_scale.log 2>&1; tail -14 $out/d_pytest_scale.log
