# quick GPU check: selected parity tests + per-query profile of heavy C5m queries
set -x
python -m pytest tests -m gpu -x -q --timeout 900 ${TESTS:+-k "$TESTS"} 2>&1 | tail -15
timeout 900 python tools/profile_query.py --config C5m --qidx ${QIDX:-0 2 3 7 11 13 19} --reps 2 --no-fp 2>&1 | cut -c1-1200
