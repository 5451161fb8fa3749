#!/bin/bash
# round-2 GPU session R: host plan + in-kernel M_1, warp-mode levels, single read-back
out=gpurun_out; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_parity.py -q --timeout 600 -x -k "small or clique or tiny or medium or fig or filter or order" > $out/r_pytest.log 2>&1; tail -1 $out/r_pytest.log
timeout 600 python tools/small_latency.py --queries 16 --configs C4 C2 > $out/r_small.log 2> $out/r_small.err; grep -E "median|profiled" $out/r_small.log | cut -c1-200
GSI_TRACE=1 timeout 600 python tools/small_latency.py --queries 2 --configs C2 C4 > $out/r_small_tr.log 2> $out/r_small_tr.err; grep -E "\[small\]|\[host\]|\[trace\]" $out/r_small_tr.err | tail -12
