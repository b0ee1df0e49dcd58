#!/bin/bash
# A/B the in-tree lib against build/ab/<name>/libpdd.so variants on C5 (args: extra explore.py args)
# prints patchy (k=1) and static (k=4) time-to-converge and kernel node-updates/s per variant
python scripts/explore.py --cfg C5 --tol 1e-7 --modes patchy --k 1 > /dev/null 2>&1   # warm
for v in default $(ls build/ab 2>/dev/null); do
  if [ "$v" = default ]; then lib=""; else lib=build/ab/$v/libpdd.so; fi
  for rep in 1 2; do
  for mk in "patchy 1" "static 4"; do set -- $mk
    PDD_LIB=$lib python scripts/explore.py --cfg ${CFG:-C5} --tol 1e-7 --modes $1 --k $2 2>&1 | grep '^{' | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print('$v', d['mode'], 'k', d['k'], 't_total', d['t_total'], 't_sweep', d['t_sweep'], 'kern', d['kern_nups'], 'sweq', d['sweeps_equiv'], 'rounds', d['rounds'])"
  done; done
done
