#!/bin/bash
# round-2 GPU session T: filter A/B (plane loads per round for short queues), filter parity
out=gpurun_out; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_parity.py -q --timeout 600 -x -k "filter" > $out/t_pytest.log 2>&1; tail -1 $out/t_pytest.log
timeout 1200 python tools/ab_filter.py --configs C4 C5m C5a --libs build_ab/twp1/libgsi_b200.so build_ab/twp2/libgsi_b200.so build_ab/twp3/libgsi_b200.so > $out/t_ab.log 2>&1; cat $out/t_ab.log
