#!/bin/bash
# GPU tests + C4 1000-tree timing of register-budget variants (build/variants/*).
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python tools/fit_once.py c4 1000 3 > gpurun_out/minb_default.log 2>&1
for v in ${VARIANTS:-m333 m444}; do
  AIWC_LIB=build/variants/$v/libaiwc_cuda.so timeout 600 python tools/fit_once.py c4 1000 3 > gpurun_out/minb_$v.log 2>&1
done
