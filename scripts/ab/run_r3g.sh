#!/bin/bash
# r3g: partial re-verification (dev build): tests on it, then timings against full verifications
export PDD_LIB=build/ab/dev/libpdd.so
python - <<'PY' > gpurun_out/r3g_tests.log 2>&1
import os, sys, pytest
sys.path.insert(0, os.getcwd())
from paper_1502_01629_b200 import _native
_native.use_library(os.environ["PDD_LIB"])
sys.exit(pytest.main(["tests/test_gpu_patches.py", "tests/test_gpu_edge_cases.py", "tests/test_gpu_lean_general.py", "tests/test_gpu_fuzzy_sparse.py",
                      "tests/test_gpu_parity.py", "-m", "gpu", "-x", "-q", "-k", "not schedules_reach"]))
PY
echo "pytest rc=$?" >> gpurun_out/r3g_tests.log
out=gpurun_out/r3g_partial.log
for cfg in C5 C4 C3 C2; do
  for v in "" "PDD_FULL_VERIFY=1"; do
    echo "== $cfg $v" >> $out
    env $v timeout 300 python scripts/explore.py --cfg $cfg --tol 1e-7 --schedule queue --modes patchy,patchy,patchy,static,static 2>&1 | grep -E '^\{|rror' >> $out
  done
done
