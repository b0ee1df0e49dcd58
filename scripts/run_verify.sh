#!/bin/bash
# verification of a build (r3k: 16-row general tiles + three path-3 geometries): GPU test-suite, smoke, bench
timeout 3000 python -m pytest tests -m gpu -x -q -rs --durations=8 -s > gpurun_out/r3k_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r3k_pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r3k_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r3k_smoke.log
timeout 1200 python bench.py > gpurun_out/r3k_bench.json 2> gpurun_out/r3k_bench.err; echo "bench rc=$?" >> gpurun_out/r3k_bench.err
