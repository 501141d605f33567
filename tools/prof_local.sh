#!/bin/bash
# GPU tests + A/B of local mode + ncu launch lists (1 lane, 148 C4 trees) per mode.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for lm in ${LMS:-0 2048}; do
  AIWC_LOCAL_MAX=$lm timeout 600 python tools/fit_once.py c4 1000 3 > gpurun_out/ab_$lm.log 2>&1
  echo "rc=$?" >> gpurun_out/ab_$lm.log
  AIWC_LOCAL_MAX=$lm AIWC_WIDE_LANES=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none \
    --csv --log-file gpurun_out/launch_$lm.csv python tools/fit_once.py c4 148 > gpurun_out/ncu_$lm.log 2>&1
  echo "ncu rc=$?" >> gpurun_out/ncu_$lm.log
done
