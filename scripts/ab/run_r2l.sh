#!/bin/bash
timeout 1500 python -m pytest tests/test_gpu_fuzzy_sparse.py tests/test_gpu_general.py -m gpu -x -q -s > gpurun_out/r2l_fuzzy_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2l_fuzzy_tests.log
timeout 1200 python scripts/fuzzy_sparse_fullsize.py C5 4 1e-2 > gpurun_out/r2l_fuzzy_c5.json 2> gpurun_out/r2l_fuzzy_c5.err
