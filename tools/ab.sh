#!/bin/bash
# A/B: per-query wall / join / filter ms for library variants (GSI_LIB) on one workload.
# usage: bash tools/ab.sh "<profile_query args>" lib1.so lib2.so ...
args=$1; shift
for lib in "$@"; do
  echo "== $lib"
  GSI_LIB=$lib timeout 600 python tools/profile_query.py $args --no-fp 2>&1 | python -c "
import sys, json
tot = [0, 0]
for l in sys.stdin:
    if l.startswith('{'):
        d = json.loads(l); tot[0] += d['wall_ms']; tot[1] += d['kernels']['join']['ms']
        print(d['q'], d['count'], d['wall_ms'], 'join', round(d['kernels']['join']['ms'], 3), 'filt', round(d['kernels']['filter']['ms'], 3),
              'other', round(d['kernels']['other']['ms'], 3), 'n_other', d['kernels']['other']['launches'], 'hjoin', round(d['ms_join'], 2), 'alloc', round(d['ms_alloc'], 2), 'sync', round(d['ms_sync'], 2))
print('TOTAL wall %.1f join %.1f' % tuple(tot))
"
done
