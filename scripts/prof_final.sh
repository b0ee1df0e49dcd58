#!/bin/bash
# final-build profile set (r4i): bench, launch list, one ncu --set full capture of the work-queue sweep kernel (C5 patchy
# path 3, C3 patchy path 4); the .ncu-rep files stay on the box, their summaries come back
timeout 1200 python bench.py > gpurun_out/r4i_bench.json 2> gpurun_out/r4i_bench.err; echo "bench rc=$?" >> gpurun_out/r4i_bench.err
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r4i_launches.csv \
    python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-static --no-others --no-accuracy-run > gpurun_out/r4i_ncu_list.log 2>&1
python scripts/launch_summary.py gpurun_out/r4i_launches.csv > gpurun_out/r4i_launches_summary.txt 2>&1
rm -f gpurun_out/r4i_launches.csv
for cfg in C5 C3; do
  timeout 1800 ncu --set full --import-source on --clock-control none -k regex:k_sweep_queue --launch-skip 0 --launch-count 1 \
      -o /tmp/prof_r4i_queue_$cfg -f python scripts/explore.py --cfg $cfg --tol 1e-7 --schedule queue --modes patchy > gpurun_out/r4i_ncu_q_$cfg.log 2>&1
  python scripts/ncu_summary.py /tmp/prof_r4i_queue_$cfg.ncu-rep gpurun_out/r4i_sweep_queue_${cfg}_ncu_summary.txt > /dev/null 2>&1
  ncu -i /tmp/prof_r4i_queue_$cfg.ncu-rep --page raw --csv > gpurun_out/r4i_sweep_queue_${cfg}_raw.csv 2>/dev/null
done
