#!/bin/bash
# r2i: lean general-stencil kernel (path 4): tests with the dev build, then C3 timings against path 1
export PDD_LIB=build/ab/dev/libpdd.so
python - <<'PY' > gpurun_out/r2i_tests.log 2>&1
import os, sys, pytest
sys.path.insert(0, os.getcwd())
from paper_1502_01629_b200 import _native
_native.use_library(os.environ["PDD_LIB"])
sys.exit(pytest.main(["tests/test_gpu_lean_general.py", "-m", "gpu", "-x", "-q"]))
PY
echo "pytest rc=$?" >> gpurun_out/r2i_tests.log
out=gpurun_out/r2i_c3.log
for k in 4 1; do
  echo "== C3 kernel=$k" >> $out
  timeout 300 python scripts/explore.py --cfg C3 --tol 1e-7 --schedule queue --kernel $k --modes patchy,patchy,static 2>&1 | grep -E '^\{|rror' >> $out
done
echo "== paper zermelo 800 kernel 0 fp64" >> $out
timeout 300 python scripts/explore.py --paper zermelo:800:1e-9 --prec 64 --tol 1e-9 --schedule queue --modes patchy,static 2>&1 | grep -E '^\{|rror' >> $out
