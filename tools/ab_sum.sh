#!/bin/bash
# A/B of library variants over the bench's 16 C5m queries: per-variant sums of kernel ms
# (join / other / filter) and wall ms.  usage: bash tools/ab_sum.sh lib1.so lib2.so ...
for lib in "$@"; do
  GSI_LIB=$lib timeout 900 python tools/profile_query.py --config C5m --qidx $(seq -s ' ' 0 15) --reps 2 --no-fp 2>/dev/null | python -c "
import sys, json
t = {'join': 0, 'other': 0, 'filter': 0, 'wall': 0}
for l in sys.stdin:
    if l.startswith('{'):
        d = json.loads(l)
        for k in ('join', 'other', 'filter'): t[k] += d['kernels'][k]['ms']
        t['wall'] += d['wall_ms']
print('$lib', {k: round(v, 1) for k, v in t.items()})
"
done
