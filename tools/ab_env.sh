#!/bin/bash
# A/B of environment knob settings on the C4 1000-tree fit (+ optional GPU tests first).
#   VARS="AIWC_LWIN=0 AIWC_LWIN=4" [TESTS=1] bash tools/ab_env.sh
mkdir -p gpurun_out
if [ -n "$TESTS" ]; then
  timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
  echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
fi
for r in 1 2; do
  for v in ${VARS}; do
    echo "== $v" >> gpurun_out/ab_env.log
    env $v timeout 600 python tools/fit_once.py c4 1000 2 >> gpurun_out/ab_env.log 2>&1
  done
done
