#!/bin/bash
# round-2 GPU session AL: C(u) bitmap on chip in k_small_query (small graphs)
out=gpurun_out; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_ext.py -q --timeout 600 -x -k "small or clique or tiny or medium or fig or path or star or square or ml or line" > $out/al_pytest.log 2>&1; tail -1 $out/al_pytest.log
timeout 900 python -m pytest tests/test_gpu_scale.py -q --timeout 800 -x -k "full_config" > $out/al_scale.log 2>&1; tail -1 $out/al_scale.log
timeout 600 python tools/small_latency.py --queries 16 --configs C2 C3 C4 > $out/al_small.log 2> $out/al_small.err; grep -E "median" $out/al_small.log | cut -c1-120
GSI_TRACE=1 timeout 600 python tools/small_latency.py --queries 2 --configs C2 > $out/al_small_tr.log 2> $out/al_small_tr.err; grep -E "\[small\]" $out/al_small_tr.err | tail -2
