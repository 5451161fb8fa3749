#!/bin/bash
# round-2 GPU session E: parity (changed kernels), bench, ncu (fp list, final_fp, next_lean, final_table)
out=gpurun_out; mkdir -p $out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_ext.py -q --timeout 600 -x > $out/e_pytest_parity.log 2>&1; tail -3 $out/e_pytest_parity.log
timeout 1500 python bench.py > $out/e_bench.json 2> $out/e_bench.err; tail -c 300 $out/e_bench.json; tail -1 $out/e_bench.err
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --cache-control none \
  -k regex:'^k_' --csv --log-file $out/e_fp_launches.csv python tools/bench_queries.py --modes fp > $out/e_fp_launches.log 2>&1
python tools/ncu_traffic.py $out/e_fp_launches.csv C5m "bench step, fp mode" --md $out/e_fp_traffic.md | head -12
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_final_fp -s 30 -c 1 -o $out/e_ffp python tools/bench_queries.py --qidx 0 --modes fp > $out/e_ffp.log 2>&1; tail -1 $out/e_ffp.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_next_lean -s 20 -c 1 -o $out/e_nl python tools/bench_queries.py --qidx 0 --modes fp > $out/e_nl.log 2>&1; tail -1 $out/e_nl.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_final_table -c 1 -o $out/e_ftab python tools/bench_queries.py --qidx 10 --modes table > $out/e_ftab.log 2>&1; tail -1 $out/e_ftab.log
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --cache-control none \
  -k regex:'^k_' --csv --log-file $out/e_table_launches.csv python tools/bench_queries.py --qidx 2 3 10 14 --modes table > $out/e_table_launches.log 2>&1
python tools/ncu_traffic.py $out/e_table_launches.csv C5m "table mode, queries 2 3 10 14" --md $out/e_table_traffic.md | head -8
