#!/bin/bash
# r2n: GPU tests on the checked build (own bounds checks), then one full-size C5 + C3 solve on it
timeout 3000 python scripts/run_checked.py > gpurun_out/r2n_checked_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2n_checked_tests.log
timeout 1200 python scripts/run_checked.py tests/test_gpu_fullsize.py -m gpu -q -x -k "C3 or C4" > gpurun_out/r2n_checked_fullsize.log 2>&1; echo "rc=$?" >> gpurun_out/r2n_checked_fullsize.log
