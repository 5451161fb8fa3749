#!/bin/bash
# round-2 GPU session B: parity + NEXT-4 tests, bench line, scale tests (durations)
out=gpurun_out; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_ext.py -q --timeout 600 --durations=15 > $out/b_pytest_parity.log 2>&1; tail -5 $out/b_pytest_parity.log
timeout 1200 python bench.py --no-small > $out/b_bench.json 2> $out/b_bench.err; tail -c 1500 $out/b_bench.json; tail -3 $out/b_bench.err
timeout 1500 python -m pytest tests/test_gpu_scale.py -q --timeout 900 --durations=0 > $out/b_pytest_scale.log 2>&1; tail -12 $out/b_pytest_scale.log
