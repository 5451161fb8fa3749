#!/bin/bash
# Copy one gpu_session.sh run's evidence into profiles/<round>/: bench line, launch list,
# full-capture metrics / details / stalls of the captured k_join launches.
# usage: bash tools/summarize_session.sh <tag> [round]
tag=$1; rnd=${2:-r1}
src=gpurun_out; dst=profiles/$rnd
mkdir -p $dst
cp $src/bench_$tag.json $dst/${tag}_bench.json
python tools/ncu_summary.py launches $src/launches_$tag.csv > $dst/${tag}_launches.md
gzip -c $src/launches_$tag.csv > $dst/${tag}_launches.csv.gz
if [ -f $src/join_full_$tag.ncu-rep ]; then
  python tools/ncu_summary.py full $src/join_full_$tag.ncu-rep > $dst/${tag}_join_metrics.md
  n=$(($(wc -l < $dst/${tag}_join_metrics.md) - 3))
  for i in $(seq 0 $((n - 1))); do
    python tools/ncu_summary.py details $src/join_full_$tag.ncu-rep $i > $dst/${tag}_join_details_launch$i.md
    python tools/ncu_summary.py stalls $src/join_full_$tag.ncu-rep $i > $dst/${tag}_join_stalls_launch$i.md
  done
fi
[ -f $src/calib_$tag.log ] && cp $src/calib_$tag.log $dst/${tag}_calib_100q.log
ls $dst | grep "^$tag"
