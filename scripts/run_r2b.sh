#!/bin/bash
# round-2 verification of the per-patch / full-size parity commit: the whole GPU suite
timeout 2400 python -m pytest tests -m gpu -x -q -rs --durations=15 -s > gpurun_out/r2b_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2b_pytest_gpu.log
