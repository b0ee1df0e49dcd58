#!/bin/bash
# r2k: product build: C4 target check, full GPU suite, smoke, bench
out=gpurun_out/r2k_misc.log
for w in 0 888 666 444; do
  echo "== C4 queue_target=$w" >> $out
  timeout 300 python scripts/explore.py --cfg C4 --tol 1e-7 --schedule queue --modes patchy,patchy --qt $w 2>&1 | grep -E '^\{|rror' >> $out
done
timeout 2400 python -m pytest tests -m gpu -x -q -rs --durations=10 -s > gpurun_out/r2k_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2k_pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2k_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r2k_smoke.log
timeout 900 python bench.py > gpurun_out/r2k_bench.json 2> gpurun_out/r2k_bench.err
