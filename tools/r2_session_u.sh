#!/bin/bash
# round-2 GPU session U: cheaper label test in k_filter_tw
out=gpurun_out; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_parity.py -q --timeout 600 -x -k "filter" > $out/u_pytest.log 2>&1; tail -1 $out/u_pytest.log
timeout 1200 python tools/ab_filter.py --configs C4 C5m C5a --libs paper_1906_03420_b200/lib/libgsi_b200.so build_ab/twp1/libgsi_b200.so > $out/u_ab.log 2>&1; cat $out/u_ab.log
timeout 600 python tools/small_latency.py --queries 16 --configs C4 C2 > $out/u_small.log 2> $out/u_small.err; grep -E "median|profiled" $out/u_small.log | cut -c1-160
