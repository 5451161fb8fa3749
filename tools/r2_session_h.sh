#!/bin/bash
# round-2 GPU session H: the whole GPU suite on HEAD, small-query trace, default bench line
out=gpurun_out; mkdir -p $out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $out/h_smi.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q --timeout 1500 --durations=15 > $out/h_pytest_gpu.log 2>&1; tail -20 $out/h_pytest_gpu.log | cut -c1-200
GSI_TRACE=1 timeout 600 python tools/small_latency.py --queries 8 > $out/h_small.log 2> $out/h_small.err; grep median $out/h_small.log | cut -c1-300; grep "trace" $out/h_small.err | tail -8
timeout 1500 python bench.py > $out/h_bench.json 2> $out/h_bench.err; tail -c 400 $out/h_bench.json; tail -3 $out/h_bench.err
