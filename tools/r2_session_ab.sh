#!/bin/bash
# round-2 GPU session AB: k_next_lean probe-ahead hoist A/B
out=gpurun_out; mkdir -p $out
timeout 1200 python tools/ab_variants.py paper_1906_03420_b200/lib/libgsi_b200.so build_ab/nl_hoist/libgsi_b200.so paper_1906_03420_b200/lib/libgsi_b200.so build_ab/nl_hoist/libgsi_b200.so > $out/ab_ab.log 2>&1; cat $out/ab_ab.log
