#!/bin/bash
# round-2 GPU session X: ncu --set full of the heaviest k_join<J_NEXT> launch of the fp bench step
out=gpurun_out; mkdir -p $out
timeout 1500 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"k_join<\(int\)2>" -s 159 -c 1 -o $out/x_join_next python tools/bench_queries.py --modes fp > $out/x_jn.log 2>&1; tail -2 $out/x_jn.log
