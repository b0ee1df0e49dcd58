#!/bin/bash
# A/B the build variants on the C5 patchy + static time-to-converge (args go to explore.py)
for v in default $(ls build/variants); do
  if [ "$v" = default ]; then lib=""; else lib=build/variants/$v/libpdd.so; fi
  echo "== $v"
  PDD_LIB=$lib python scripts/explore.py --cfg C5 "$@" 2>&1 | grep '^{' | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print(d['mode'], 'k', d['k'], 'delta', d['delta'], 't_total', d['t_total'], 'kern', d['kern_nups'], 'sweq', d['sweeps_equiv'], 'rounds', d['rounds'])"
done
