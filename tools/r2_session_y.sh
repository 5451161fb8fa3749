#!/bin/bash
# round-2 GPU session Y: J_NEXT write loop (shared column map, multiply-high row index) — parity + A/B
out=gpurun_out; mkdir -p $out
timeout 1200 python -m pytest tests/test_gpu_parity.py -q --timeout 600 -x -k "random or medium or clique or table or shared or count_ahead or path" > $out/y_pytest.log 2>&1; tail -1 $out/y_pytest.log
timeout 1200 python tools/ab_variants.py paper_1906_03420_b200/lib/libgsi_b200.so build_ab/jn3/libgsi_b200.so > $out/y_ab.log 2>&1; cat $out/y_ab.log
