#!/bin/bash
# round-2 GPU session L: exact label bits + NC-templated rounds in k_filter_tw, planner from shared memory
out=gpurun_out; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_parity.py -q --timeout 600 -x -k "filter or signature or small or clique or tiny or medium" > $out/l_pytest.log 2>&1; tail -1 $out/l_pytest.log
timeout 600 python tools/small_latency.py --queries 16 --configs C4 C2 > $out/l_small.log 2> $out/l_small.err; grep -E "median|profiled" $out/l_small.log | cut -c1-200
GSI_TRACE=1 timeout 600 python tools/small_latency.py --queries 2 --configs C2 C4 > $out/l_small_tr.log 2> $out/l_small_tr.err; grep -E "\[small\]" $out/l_small_tr.err | tail -3
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_filter|k_small_query" -s 2 -c 2 -o $out/l_c4_ncu python tools/small_latency.py --configs C4 --queries 1 --reps 1 > $out/l_ncu_c4.log 2>&1; tail -1 $out/l_ncu_c4.log
timeout 900 python -m pytest tests/test_gpu_scale.py -q --timeout 800 -x -k "full_config" > $out/l_scale.log 2>&1; tail -1 $out/l_scale.log
