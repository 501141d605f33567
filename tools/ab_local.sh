#!/bin/bash
# A/B of the wide grower's local mode on C4 (1000 trees) + the GPU tests.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for lm in ${LMS:-0 2048}; do
  AIWC_LOCAL_MAX=$lm timeout 600 python tools/fit_once.py c4 1000 3 > gpurun_out/ab_$lm.log 2>&1
  echo "rc=$?" >> gpurun_out/ab_$lm.log
done
