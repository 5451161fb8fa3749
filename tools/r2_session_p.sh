#!/bin/bash
# round-2 GPU session P: native-DMUL warp planner; J_NEXT launch-parameter A/B on the fp bench queries
out=gpurun_out; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_parity.py -q --timeout 600 -x -k "small or clique or tiny or medium or fig" > $out/p_pytest.log 2>&1; tail -1 $out/p_pytest.log
timeout 600 python tools/small_latency.py --queries 16 --configs C4 C2 > $out/p_small.log 2> $out/p_small.err; grep -E "median|profiled" $out/p_small.log | cut -c1-200
GSI_TRACE=1 timeout 600 python tools/small_latency.py --queries 2 --configs C2 C4 > $out/p_small_tr.log 2> $out/p_small_tr.err; grep -E "\[small\]" $out/p_small_tr.err | tail -3
timeout 1200 python tools/ab_variants.py build_ab/base/libgsi_b200.so build_ab/minb2/libgsi_b200.so build_ab/minb4/libgsi_b200.so build_ab/items4/libgsi_b200.so build_ab/items16/libgsi_b200.so build_ab/rows2/libgsi_b200.so > $out/p_ab.log 2>&1; cat $out/p_ab.log
