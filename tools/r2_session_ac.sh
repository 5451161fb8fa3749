#!/bin/bash
# round-2 GPU session AC: bulk-copy (UBLKCP) plane-0 prefetch in k_filter_tw — parity + A/B
out=gpurun_out; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_parity.py -q --timeout 600 -x -k "filter" > $out/ac_pytest.log 2>&1; tail -1 $out/ac_pytest.log
timeout 900 python -m pytest tests/test_gpu_scale.py -q --timeout 800 -x -k "full_config" > $out/ac_scale.log 2>&1; tail -1 $out/ac_scale.log
timeout 1200 python tools/ab_filter.py --configs C4 C5m C5a --libs paper_1906_03420_b200/lib/libgsi_b200.so build_ab/head/libgsi_b200.so > $out/ac_ab.log 2>&1; cat $out/ac_ab.log
timeout 600 python tools/small_latency.py --queries 16 --configs C4 C2 > $out/ac_small.log 2> $out/ac_small.err; grep -E "median" $out/ac_small.log | cut -c1-120
