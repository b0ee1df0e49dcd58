#!/bin/bash
# compute-sanitizer on the C2 patchy + static pipeline (work queue): one tool per call
# usage: sanitize.sh memcheck|synccheck|racecheck
tool=${1:-memcheck}
timeout 3000 compute-sanitizer --tool $tool --log-file gpurun_out/sanitize_$tool.log \
    python scripts/explore.py --cfg C2 --tol 1e-7 --schedule queue --modes patchy,static > gpurun_out/sanitize_${tool}_run.log 2>&1
echo "rc=$?" >> gpurun_out/sanitize_${tool}_run.log
tail -5 gpurun_out/sanitize_$tool.log >> gpurun_out/sanitize_${tool}_run.log
