#!/bin/bash
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
AIWC_VERBOSE=1 timeout 600 python tools/fit_once.py c4 1000 3 > gpurun_out/l16.log 2>&1
AIWC_VERBOSE=1 AIWC_LIB=build/variants/c_f0bb2f7/libaiwc_cuda.so timeout 600 python tools/fit_once.py c4 1000 3 > gpurun_out/l16_base.log 2>&1
