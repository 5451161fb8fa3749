#!/bin/bash
# round-2 GPU session AG: k_final_fp capture on the final tree (same launch as r2f)
out=gpurun_out; mkdir -p $out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_final_fp -s 30 -c 1 -o $out/ag_final_fp python tools/bench_queries.py --qidx 0 --modes fp > $out/ag_ffp.log 2>&1; tail -1 $out/ag_ffp.log
