#!/bin/bash
# round-2 GPU session AH: final bench line
out=gpurun_out; mkdir -p $out
timeout 1500 python bench.py > $out/ah_bench.json 2> $out/ah_bench.err; tail -c 300 $out/ah_bench.json; tail -3 $out/ah_bench.err
