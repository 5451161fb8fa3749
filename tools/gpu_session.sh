#!/bin/bash
# One gpurun session: GPU tests, the bench line, ncu launch list and a full capture of the
# dominant kernel.  Usage (under gpurun): bash tools/gpu_session.sh <tag> [bench args...]
tag=${1:-r1}; shift
out=gpurun_out
mkdir -p $out
python -m pytest tests -m gpu -x -q --timeout 900 > $out/pytest_gpu_$tag.log 2>&1; tail -2 $out/pytest_gpu_$tag.log
timeout 900 python __graft_entry__.py smoke > $out/smoke_$tag.log 2>&1; tail -1 $out/smoke_$tag.log
timeout 1200 python bench.py "$@" > $out/bench_$tag.json 2> $out/bench_$tag.err; tail -c 3000 $out/bench_$tag.json; tail -3 $out/bench_$tag.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'^k_' \
    --csv --log-file $out/launches_$tag.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-enumerated --query-timeout 0 "$@" > $out/bench_ncu_$tag.log 2>&1
tail -2 $out/bench_ncu_$tag.log | cut -c1-300
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_join|k_cahead|k_next' -s 8 -c 6 -o $out/join_full_$tag \
    python tools/profile_query.py --config C5m --qidx 11 --reps 1 --no-fp > $out/ncu_full_$tag.log 2>&1
tail -2 $out/ncu_full_$tag.log | cut -c1-300
timeout 900 python tools/calibrate.py --config C5m --queries 100 --timeout 2 > $out/calib_$tag.log 2>&1; tail -1 $out/calib_$tag.log
