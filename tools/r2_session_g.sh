#!/bin/bash
# round-2 GPU session G: small-query host trace, filter parity, ablation ladder (+ncu), scale tests
out=gpurun_out; mkdir -p $out
GSI_TRACE=1 timeout 600 python tools/small_latency.py --queries 8 > $out/g_small.log 2> $out/g_small.err; grep median $out/g_small.log | cut -c1-300; grep "\[host\]" $out/g_small.err | tail -8
timeout 900 python -m pytest tests/test_gpu_parity.py -q --timeout 600 -k "filter or signature or fig1 or tiny or medium or large_counts" > $out/g_pytest_filter.log 2>&1; tail -2 $out/g_pytest_filter.log
timeout 900 python -m pytest tests/test_gpu_ext.py -q --timeout 600 -k "ml_signatures" > $out/g_pytest_mlf.log 2>&1; tail -1 $out/g_pytest_mlf.log
timeout 900 python tools/ablation.py --config C3 --nlv 10 --k 8 --queries 16 --md $out/g_ablation_C3.md > $out/g_ablation_C3.log 2>&1; tail -12 $out/g_ablation_C3.md
bash tools/ablation_ncu.sh g C3 10 8 > $out/g_ablation_ncu.md 2>&1; cat $out/g_ablation_ncu.md
timeout 2400 python -m pytest tests/test_gpu_scale.py -v --timeout 1500 --durations=0 > $out/g_pytest_scale.log 2>&1; grep -E "PASSED|FAILED|passed|failed|s call" $out/g_pytest_scale.log | tail -14
