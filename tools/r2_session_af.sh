#!/bin/bash
# round-2 GPU session AF: k_final_fp lane-own threshold A/B
out=gpurun_out; mkdir -p $out
timeout 1500 python tools/ab_variants.py paper_1906_03420_b200/lib/libgsi_b200.so build_ab/even8/libgsi_b200.so build_ab/even4/libgsi_b200.so build_ab/even24/libgsi_b200.so > $out/af_ab.log 2>&1; cat $out/af_ab.log
