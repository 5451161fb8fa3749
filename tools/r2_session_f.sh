#!/bin/bash
# round-2 GPU session F: parity, bench, small-query latency, ncu captures of the three hot kernels
out=gpurun_out; mkdir -p $out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_ext.py -q --timeout 600 -x > $out/f_pytest_parity.log 2>&1; tail -2 $out/f_pytest_parity.log
timeout 600 python tools/small_latency.py > $out/f_small.log 2> $out/f_small.err; grep median $out/f_small.log | cut -c1-400
timeout 1500 python bench.py > $out/f_bench.json 2> $out/f_bench.err; tail -c 300 $out/f_bench.json; tail -1 $out/f_bench.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_final_fp -s 30 -c 1 -o $out/f_ffp python tools/bench_queries.py --qidx 0 --modes fp > $out/f_ffp.log 2>&1; tail -1 $out/f_ffp.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_final_table -c 1 -o $out/f_ftab python tools/bench_queries.py --qidx 10 --modes table > $out/f_ftab.log 2>&1; tail -1 $out/f_ftab.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_next_lean -s 20 -c 1 -o $out/f_nl python tools/bench_queries.py --qidx 0 --modes fp > $out/f_nl.log 2>&1; tail -1 $out/f_nl.log
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --cache-control none \
  -k regex:'^k_' --csv --log-file $out/f_fp_launches.csv python tools/bench_queries.py --modes fp > $out/f_fp_launches.log 2>&1
python tools/ncu_traffic.py $out/f_fp_launches.csv C5m "bench step, fp mode" --md $out/f_fp_traffic.md | head -10
