#!/bin/bash
mkdir -p gpurun_out
for r in 1 2; do
  for v in base head head3; do
    L=paper_1811_00156_b200/libaiwc_cuda.so; X=""
    if [ $v = base ]; then L=build/variants/c_f0bb2f7/libaiwc_cuda.so; fi
    if [ $v = head3 ]; then X="AIWC_WIDE_PER_SM=3"; fi
    env $X AIWC_VERBOSE=1 AIWC_LIB=$L timeout 600 python tools/fit_once.py c4 1000 1 >> gpurun_out/bis4_$v.log 2>&1
  done
done
