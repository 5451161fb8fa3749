#!/bin/bash
# round-2 GPU session K: thread-per-word filter, small path phase times
out=gpurun_out; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_parity.py -q --timeout 600 -x -k "filter or signature or small or clique or tiny or medium" > $out/k_pytest.log 2>&1; tail -3 $out/k_pytest.log
GSI_TRACE=1 timeout 600 python tools/small_latency.py --queries 16 > $out/k_small.log 2> $out/k_small.err; grep -E "median|profiled" $out/k_small.log | cut -c1-300; grep -E "\[small\]" $out/k_small.err | tail -6; grep trace $out/k_small.err | tail -4
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_filter|k_small_query" -s 2 -c 2 -o $out/k_c4_ncu python tools/small_latency.py --configs C4 --queries 1 --reps 1 > $out/k_ncu_c4.log 2>&1; tail -1 $out/k_ncu_c4.log
timeout 900 python -m pytest tests/test_gpu_scale.py -q --timeout 800 -x -k "full_config" > $out/k_scale.log 2>&1; tail -2 $out/k_scale.log
timeout 1500 python bench.py --steps 3 --warmup 3 > $out/k_bench.json 2> $out/k_bench.err; tail -c 300 $out/k_bench.json; tail -2 $out/k_bench.err
