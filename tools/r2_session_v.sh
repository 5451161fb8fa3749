#!/bin/bash
# round-2 GPU session V: whole GPU suite + default bench line on the current tree
out=gpurun_out; mkdir -p $out
timeout 2700 python -m pytest tests -m gpu -q --timeout 1500 -x --durations=10 > $out/v_pytest_gpu.log 2>&1; tail -14 $out/v_pytest_gpu.log | cut -c1-160
timeout 1500 python bench.py > $out/v_bench.json 2> $out/v_bench.err; tail -c 400 $out/v_bench.json; tail -3 $out/v_bench.err
