#!/bin/bash
# C4 1000-tree timing of library variants (build/variants/*), default first.
mkdir -p gpurun_out
timeout 600 python tools/fit_once.py c4 1000 3 > gpurun_out/bis_default.log 2>&1
for v in ${VARIANTS}; do
  AIWC_LIB=build/variants/$v/libaiwc_cuda.so timeout 600 python tools/fit_once.py c4 1000 3 > gpurun_out/bis_$v.log 2>&1
done
AIWC_WIDE_LANES=1 timeout 600 python tools/fit_once.py c4 500 2 > gpurun_out/bis_default_l1.log 2>&1
AIWC_WIDE_LANES=1 AIWC_LIB=build/variants/c_f0bb2f7/libaiwc_cuda.so timeout 600 python tools/fit_once.py c4 500 2 > gpurun_out/bis_base_l1.log 2>&1
