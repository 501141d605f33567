#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for r in 1 2; do
  for v in base head; do
    if [ $v = base ]; then L=build/variants/c_f0bb2f7/libaiwc_cuda.so; else L=paper_1811_00156_b200/libaiwc_cuda.so; fi
    AIWC_VERBOSE=1 AIWC_LIB=$L timeout 600 python tools/fit_once.py c4 1000 1 >> gpurun_out/bis3_$v.log 2>&1
  done
done
