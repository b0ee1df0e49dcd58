#!/bin/bash
# round-1 profile set: bench line, ncu launch list of a short bench, ncu --set full of the sweep
# kernel in a mid-solve patchy round and a static round (C5)
set -x
python bench.py > gpurun_out/r1l_bench.json 2> gpurun_out/r1l_bench.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r1l_launches.csv \
    python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu --no-static > gpurun_out/r1l_ncu_list.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_sweep_dyn --launch-skip 150 --launch-count 1 \
    -o gpurun_out/prof_r1l_patchy -f python scripts/profile_sweep.py --mode patchy --k 1 --rounds 200 > gpurun_out/r1l_ncu_p.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_sweep_dyn --launch-skip 100 --launch-count 1 \
    -o gpurun_out/prof_r1l_static -f python scripts/profile_sweep.py --mode static --k 4 --rounds 120 > gpurun_out/r1l_ncu_s.log 2>&1
