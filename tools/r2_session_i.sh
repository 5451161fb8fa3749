#!/bin/bash
# round-2 GPU session I: device-planned small path — parity, latency trace, ncu of filter + small kernel
out=gpurun_out; mkdir -p $out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_ext.py -q --timeout 600 -x > $out/i_pytest.log 2>&1; tail -3 $out/i_pytest.log
GSI_TRACE=1 timeout 600 python tools/small_latency.py --queries 16 > $out/i_small.log 2> $out/i_small.err; grep median $out/i_small.log | cut -c1-300; grep -E "trace|host" $out/i_small.err | tail -24
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_filter|k_small_query" -s 4 -c 4 -o $out/i_small_ncu python tools/small_latency.py --queries 2 --reps 1 > $out/i_ncu.log 2>&1; tail -2 $out/i_ncu.log
timeout 2000 python -m pytest tests/test_gpu_scale.py -q --timeout 1500 -k "bench_kernels or many_roots" --durations=5 > $out/i_scale.log 2>&1; tail -8 $out/i_scale.log
