#!/bin/bash
# round-2 GPU session AE: k_final_fp with the term table as a template parameter and per-row counts — parity + A/B
out=gpurun_out; mkdir -p $out
timeout 1200 python -m pytest tests/test_gpu_parity.py -q --timeout 600 -x -k "fingerprint or fp or shared or count_ahead or table or random or medium" > $out/ae_pytest.log 2>&1; tail -1 $out/ae_pytest.log
timeout 900 python -m pytest tests/test_gpu_scale.py -q --timeout 800 -x -k "modes_agree" > $out/ae_scale.log 2>&1; tail -1 $out/ae_scale.log
timeout 1200 python tools/ab_variants.py paper_1906_03420_b200/lib/libgsi_b200.so build_ab/head/libgsi_b200.so paper_1906_03420_b200/lib/libgsi_b200.so > $out/ae_ab.log 2>&1; cat $out/ae_ab.log
