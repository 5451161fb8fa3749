#!/bin/bash
# round-2 GPU session C: new-code parity, table/fp per-query profile, bench, ncu launch list + full capture
out=gpurun_out; mkdir -p $out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_ext.py -q --timeout 600 --durations=12 -x > $out/c_pytest_parity.log 2>&1; tail -16 $out/c_pytest_parity.log
timeout 600 python tools/bench_queries.py --qidx 2 3 7 10 13 --modes table fp --profile > $out/c_table_prof.log 2>&1; tail -6 $out/c_table_prof.log
timeout 1200 python bench.py > $out/c_bench.json 2> $out/c_bench.err; tail -c 600 $out/c_bench.json; tail -2 $out/c_bench.err
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --cache-control none \
  -k regex:'^k_' --csv --log-file $out/c_fp_launches.csv python tools/bench_queries.py --modes fp > $out/c_fp_launches.log 2>&1
python tools/ncu_traffic.py $out/c_fp_launches.csv C5m "bench step (16 queries), fp mode, warm L2" --md $out/c_fp_traffic.md | head -20
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_final_fp -s 30 -c 1 -o $out/c_ffp python tools/bench_queries.py --qidx 0 --modes fp > $out/c_ffp.log 2>&1; tail -2 $out/c_ffp.log
