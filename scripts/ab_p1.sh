#!/bin/bash
# path-1 (general stencil) variants on C3, the paper's Zermelo 800^2 and the general (l3, sigma3)
for v in default $(ls build/ab 2>/dev/null); do
  if [ "$v" = default ]; then lib=""; else lib=build/ab/$v/libpdd.so; fi
  echo "== $v"
  PDD_LIB=$lib python scripts/explore.py --cfg C3 --tol 1e-7 --modes patchy,static --max_rounds 30000 2>&1 | grep '^{' | cut -c1-200
  PDD_LIB=$lib python scripts/explore.py --paper zermelo:800:1e-9 --prec 64 --tol 1e-9 --modes patchy,static --max_rounds 30000 2>&1 | grep '^{' | cut -c1-200
  PDD_LIB=$lib python scripts/explore.py --general 3:3:2049:0.001:129 --prec 32 --tol 1e-6 --modes patchy,static --max_rounds 30000 2>&1 | grep '^{' | cut -c1-200
done
