#!/bin/bash
# verification of a build (r4p: coarse fast path + strip synthesis): GPU test-suite, smoke, bench
timeout 3000 python -m pytest tests -m gpu -x -q -rs --durations=8 -s > gpurun_out/r4p_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r4p_pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r4p_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r4p_smoke.log
timeout 1200 python bench.py > gpurun_out/r4p_bench.json 2> gpurun_out/r4p_bench.err; echo "bench rc=$?" >> gpurun_out/r4p_bench.err
for cfg in C5 C4 C3 C2; do for lib in ""; do
  PDD_LIB=$lib timeout 300 python scripts/ab/canon_ab.py --cfg $cfg 2>&1 | grep -E '^\{|rror' >> gpurun_out/r4p_canon_ab.log
done; done
