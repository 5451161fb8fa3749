#!/bin/bash
# round-2 GPU session N: warp-mode small levels, planner timing detail, tw_all filter
out=gpurun_out; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_parity.py -q --timeout 600 -x -k "filter or signature or small or clique or tiny or medium" > $out/n_pytest.log 2>&1; tail -1 $out/n_pytest.log
timeout 600 python tools/small_latency.py --queries 16 --configs C4 C2 > $out/n_small.log 2> $out/n_small.err; grep -E "median|profiled" $out/n_small.log | cut -c1-200
GSI_TRACE=1 timeout 600 python tools/small_latency.py --queries 2 --configs C2 C4 > $out/n_small_tr.log 2> $out/n_small_tr.err; grep -E "\[small\]" $out/n_small_tr.err | tail -3
