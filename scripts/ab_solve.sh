#!/bin/bash
# A/B the build variants on the C5 patchy + static time-to-converge
for v in default $(ls build/variants); do
  if [ "$v" = default ]; then lib=""; else lib=build/variants/$v/libpdd.so; fi
  echo "== $v"
  PDD_LIB=$lib python scripts/explore.py --cfg C5 --k 4 --modes patchy,static "$@" 2>&1 | tail -2 | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print(d['mode'], 't_total', d['t_total'], 'kern', d['kern_nups'], 'sweq', d['sweeps_equiv'], 'rounds', d['rounds'])"
done
