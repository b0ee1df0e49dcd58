#!/bin/bash
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r3b_launches.csv \
    python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-static --no-others --no-accuracy-run > gpurun_out/r3b_ncu_list.log 2>&1
python scripts/launch_summary.py gpurun_out/r3b_launches.csv > gpurun_out/r3b_launches_summary.txt 2>&1
rm -f gpurun_out/r3b_launches.csv
