#!/bin/bash
# r4n (final build; r4b was the build before the rewrites): ncu --set full of a mid-solve coarse sweep (launch 150 of 377) and of the synthesis kernel on C5 (product build)
for k in k_coarse_sweep_tiles:150 k_synthesize_rt_s:0; do
  name=${k%%:*}; skip=${k#*:}
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:$name --launch-skip $skip --launch-count 1 \
      -o /tmp/prof_r4n_$name -f python scripts/ab/canon_ab.py --cfg C5 > gpurun_out/r4n_ncu_$name.log 2>&1
  python scripts/ncu_summary.py /tmp/prof_r4n_$name.ncu-rep gpurun_out/r4n_${name}_ncu_summary.txt > /dev/null 2>&1
  ncu -i /tmp/prof_r4n_$name.ncu-rep --page raw --csv > gpurun_out/r4n_${name}_raw.csv 2>/dev/null
  ncu -i /tmp/prof_r4n_$name.ncu-rep --page source --csv > gpurun_out/r4n_${name}_source.csv 2>/dev/null
done
