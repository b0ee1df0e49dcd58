#!/bin/bash
# GPU tests on the checked build (own bounds checks), then the full-size C3 / C4 solves on it
timeout 3000 python scripts/run_checked.py > gpurun_out/r3c_checked_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r3c_checked_tests.log
timeout 1200 python scripts/run_checked.py tests/test_gpu_fullsize.py -m gpu -q -x -k "C3 or C4" > gpurun_out/r3c_checked_fullsize.log 2>&1; echo "rc=$?" >> gpurun_out/r3c_checked_fullsize.log
