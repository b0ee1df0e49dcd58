#!/bin/bash
# round-2 baseline at HEAD: gpu tests, smoke, bench, launch list, one ncu capture of the patchy round
python -m pytest tests -m gpu -x -q > gpurun_out/r2a_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2a_pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2a_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r2a_smoke.log
python bench.py > gpurun_out/r2a_bench.json 2> gpurun_out/r2a_bench.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2a_launches.csv \
    python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu --no-static --no-others > gpurun_out/r2a_ncu_list.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_sweep_dyn --launch-skip 150 --launch-count 1 \
    -o gpurun_out/prof_r2a_patchy -f python scripts/profile_sweep.py --mode patchy --k 1 --rounds 200 > gpurun_out/r2a_ncu_p.log 2>&1
