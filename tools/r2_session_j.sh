#!/bin/bash
# round-2 GPU session J: compacting filter (FW 1/8), warp-planned small path with on-chip rows
out=gpurun_out; mkdir -p $out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_ext.py -q --timeout 600 -x > $out/j_pytest.log 2>&1; tail -3 $out/j_pytest.log
GSI_TRACE=1 timeout 600 python tools/small_latency.py --queries 16 > $out/j_small.log 2> $out/j_small.err; grep -E "median|profiled" $out/j_small.log | cut -c1-300; grep -E "trace" $out/j_small.err | tail -4
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_filter|k_small_query" -s 2 -c 2 -o $out/j_c2_ncu python tools/small_latency.py --configs C2 --queries 1 --reps 1 > $out/j_ncu_c2.log 2>&1; tail -1 $out/j_ncu_c2.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_filter|k_small_query" -s 2 -c 2 -o $out/j_c4_ncu python tools/small_latency.py --configs C4 --queries 1 --reps 1 > $out/j_ncu_c4.log 2>&1; tail -1 $out/j_ncu_c4.log
timeout 1500 python bench.py --steps 3 --warmup 3 > $out/j_bench.json 2> $out/j_bench.err; tail -c 300 $out/j_bench.json; tail -2 $out/j_bench.err
