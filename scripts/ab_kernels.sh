#!/bin/bash
# A/B the sweep-kernel build variants on the C5 static solve (kernel node-updates/s)
for v in default $(ls build/variants); do
  if [ "$v" = default ]; then lib=""; else lib=build/variants/$v/libpdd.so; fi
  echo -n "$v "
  PDD_LIB=$lib python scripts/explore.py --cfg C5 --k 4 --modes static "$@" 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['kern_nups'], d['t_sweep'], d['rounds'])"
done
