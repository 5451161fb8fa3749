#!/bin/bash
# round-2 GPU session O: integer planner, warp-mode levels — parity + latency
out=gpurun_out; mkdir -p $out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_ext.py -q --timeout 600 -x > $out/o_pytest.log 2>&1; tail -2 $out/o_pytest.log
timeout 600 python tools/small_latency.py --queries 16 --configs C4 C2 > $out/o_small.log 2> $out/o_small.err; grep -E "median|profiled" $out/o_small.log | cut -c1-200
GSI_TRACE=1 timeout 600 python tools/small_latency.py --queries 2 --configs C2 C4 > $out/o_small_tr.log 2> $out/o_small_tr.err; grep -E "\[small\]" $out/o_small_tr.err | tail -3
