#!/bin/bash
# r2w: 16-row tiles for the general / fp64 kernels (dev build -DPDD_TH=16) against 32 rows
out=gpurun_out/r2w_gth16.log
for lib in dev gth16; do
  echo "== C3 fp32 $lib" >> $out
  PDD_LIB=build/ab/$lib/libpdd.so timeout 300 python scripts/explore.py --cfg C3 --tol 1e-7 --schedule queue --modes patchy,patchy,static 2>&1 | grep -E '^\{|rror' >> $out
  echo "== paper zermelo 800 fp64 $lib" >> $out
  PDD_LIB=build/ab/$lib/libpdd.so timeout 300 python scripts/explore.py --paper zermelo:800:1e-9 --prec 64 --tol 1e-9 --schedule queue --modes patchy,patchy,static 2>&1 | grep -E '^\{|rror' >> $out
  echo "== paper eikonal 800 fp64 $lib" >> $out
  PDD_LIB=build/ab/$lib/libpdd.so timeout 300 python scripts/explore.py --paper eikonal:800:1e-9 --prec 64 --tol 1e-9 --schedule queue --modes patchy,patchy,static 2>&1 | grep -E '^\{|rror' >> $out
  echo "== C5@2049 fp64 $lib" >> $out
  PDD_LIB=build/ab/$lib/libpdd.so timeout 300 python scripts/explore.py --cfg C5 --n 2049 --prec 64 --tol 1e-9 --schedule queue --modes patchy,static 2>&1 | grep -E '^\{|rror' >> $out
done
