#!/bin/bash
# round-2 GPU session AN: k_next_lean all-kept fast copy — parity + A/B
out=gpurun_out; mkdir -p $out
timeout 1200 python -m pytest tests/test_gpu_parity.py -q --timeout 600 -x -k "shared or count_ahead or random or medium or table" > $out/an_pytest.log 2>&1; tail -1 $out/an_pytest.log
timeout 900 python -m pytest tests/test_gpu_scale.py -q --timeout 800 -x -k "modes_agree" > $out/an_scale.log 2>&1; tail -1 $out/an_scale.log
timeout 1200 python tools/ab_variants.py paper_1906_03420_b200/lib/libgsi_b200.so build_ab/head/libgsi_b200.so paper_1906_03420_b200/lib/libgsi_b200.so > $out/an_ab.log 2>&1; cat $out/an_ab.log
