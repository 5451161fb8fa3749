#!/bin/bash
# round-2 GPU session AJ: k_final_fp occupancy A/B
out=gpurun_out; mkdir -p $out
timeout 1500 python tools/ab_variants.py paper_1906_03420_b200/lib/libgsi_b200.so build_ab/fpminb5/libgsi_b200.so build_ab/fpminb6/libgsi_b200.so > $out/aj_ab.log 2>&1; cat $out/aj_ab.log
