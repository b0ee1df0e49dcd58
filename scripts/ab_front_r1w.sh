#!/bin/bash
# A/B of the patchy front step (PDD_DSCALE x 6 cells) on the 32 x 64 path-3 tiles, C5 and C4
for cfg in C5 C4; do
  for ds in 0.67 0.83 1.0 1.33 1.67; do
    for rep in 1 2; do
      echo "== $cfg dscale $ds rep $rep"
      PDD_DSCALE=$ds python scripts/explore.py --cfg $cfg --modes patchy --tol 1e-7 2>&1 | grep '^{' | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print(d['mode'], 'k', d['k'], 'delta', d['delta'], 't_total', d['t_total'], 'kern', d['kern_nups'], 'sweq', d['sweeps_equiv'], 'rounds', d['rounds'])"
    done
  done
done
