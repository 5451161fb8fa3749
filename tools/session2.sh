#!/bin/bash
# round-2 GPU session: scale parity tests, bench line, ncu DRAM-per-variant capture
tag=${1:-r2a}
out=gpurun_out; mkdir -p $out
timeout 2400 python -m pytest tests/test_gpu_scale.py -x -q --timeout 2400 > $out/pytest_scale_$tag.log 2>&1; tail -3 $out/pytest_scale_$tag.log
timeout 1500 python bench.py > $out/bench_$tag.json 2> $out/bench_$tag.err; tail -c 4000 $out/bench_$tag.json; tail -3 $out/bench_$tag.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --cache-control none \
  -k regex:'^k_' --csv --log-file $out/traffic_$tag.csv python tools/bench_queries.py --modes count > $out/traffic_$tag.log 2>&1
python tools/ncu_traffic.py $out/traffic_$tag.csv C5m "bench step (16 queries), count mode, warm L2" | head -14
