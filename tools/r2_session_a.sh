#!/bin/bash
# round-2 first GPU session: parity tests, scale tests, bench line
out=gpurun_out; mkdir -p $out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $out/a_gpu.txt 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py -q --timeout 600 -x > $out/a_pytest_parity.log 2>&1; tail -5 $out/a_pytest_parity.log
timeout 1800 python -m pytest tests/test_gpu_scale.py -q --timeout 1500 > $out/a_pytest_scale.log 2>&1; tail -5 $out/a_pytest_scale.log
timeout 1200 python bench.py > $out/a_bench.json 2> $out/a_bench.err; tail -c 3000 $out/a_bench.json; tail -5 $out/a_bench.err
