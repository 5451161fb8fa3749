#!/bin/bash
# round-2 GPU session AA: final bench line
out=gpurun_out; mkdir -p $out
timeout 1500 python bench.py > $out/aa_bench.json 2> $out/aa_bench.err; tail -c 300 $out/aa_bench.json; tail -3 $out/aa_bench.err
