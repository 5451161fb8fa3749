#!/bin/bash
# round-2 GPU session Q: planner step timing
out=gpurun_out; mkdir -p $out
GSI_TRACE=1 timeout 600 python tools/small_latency.py --queries 2 --configs C2 > $out/q_small_tr.log 2> $out/q_small_tr.err; grep -E "\[small\]" $out/q_small_tr.err | tail -3
