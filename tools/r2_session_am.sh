#!/bin/bash
# round-2 GPU session AM: 100-query calibration (SURVEY §8(d) statistic: mean over 100 queries, p50/p95)
out=gpurun_out; mkdir -p $out
for c in C2 C3 C4 C5a C5m; do
  timeout 900 python tools/calibrate.py --config $c --queries 100 --timeout 10 > $out/am_calib_${c}.log 2>&1; tail -1 $out/am_calib_${c}.log
done
timeout 1200 python tools/calibrate.py --config C5m --queries 100 --timeout 10 --fp > $out/am_calib_C5m_fp.log 2>&1; tail -1 $out/am_calib_C5m_fp.log
