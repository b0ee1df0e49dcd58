#!/bin/bash
# round-1 verification of HEAD (path-3 tile per schedule: 32x64 patchy, 16x128 static on C4/C5): gpu tests, smoke, then the r1r profile set
# sweep kernel in a mid-solve patchy round (k=1) and a static round (k=4), node-updates of those rounds
set -x
python -m pytest tests -m gpu -x -q > gpurun_out/r1v_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r1v_pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r1v_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r1v_smoke.log
python bench.py > gpurun_out/r1v_bench.json 2> gpurun_out/r1v_bench.err
PDD_TRACE=1 python scripts/round_nu.py --mode patchy --k 1 --round 151 > gpurun_out/r1v_nu_patchy.json 2>/dev/null
PDD_TRACE=1 python scripts/round_nu.py --mode static --k 4 --round 101 > gpurun_out/r1v_nu_static.json 2>/dev/null
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r1v_launches.csv \
    python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu --no-static --no-others > gpurun_out/r1v_ncu_list.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_sweep_dyn --launch-skip 150 --launch-count 1 \
    -o gpurun_out/prof_r1v_patchy -f python scripts/profile_sweep.py --mode patchy --k 1 --rounds 200 > gpurun_out/r1v_ncu_p.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_sweep_dyn --launch-skip 100 --launch-count 1 \
    -o gpurun_out/prof_r1v_static -f python scripts/profile_sweep.py --mode static --k 4 --rounds 120 > gpurun_out/r1v_ncu_s.log 2>&1
