#!/bin/bash
mkdir -p gpurun_out
for v in c_e9f2b2f; do
  L=build/variants/$v/libaiwc_cuda.so
  AIWC_LIB=$L AIWC_WIDE_LANES=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none \
    --csv --log-file gpurun_out/launch_$v.csv python tools/fit_once.py c4 148 > gpurun_out/ncu_$v.log 2>&1
  AIWC_LIB=$L AIWC_WIDE_LANES=1 timeout 600 python tools/fit_once.py c4 148 2 > gpurun_out/l1_$v.log 2>&1
done
AIWC_LIB=build/variants/c_f0bb2f7/libaiwc_cuda.so AIWC_WIDE_LANES=1 timeout 600 python tools/fit_once.py c4 148 2 > gpurun_out/l1_base2.log 2>&1
