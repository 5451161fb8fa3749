#!/bin/bash
# round-2 GPU session S: zero-copy filter publication
out=gpurun_out; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_parity.py -q --timeout 600 -x -k "small or clique or tiny or medium or fig or filter or order" > $out/s_pytest.log 2>&1; tail -1 $out/s_pytest.log
timeout 600 python tools/small_latency.py --queries 16 --configs C4 C2 > $out/s_small.log 2> $out/s_small.err; grep -E "median|profiled" $out/s_small.log | cut -c1-200
GSI_TRACE=1 timeout 600 python tools/small_latency.py --queries 2 --configs C2 C4 > $out/s_small_tr.log 2> $out/s_small_tr.err; grep -E "\[small\]|\[host\]|\[trace\]" $out/s_small_tr.err | tail -12
