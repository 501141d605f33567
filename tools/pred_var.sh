#!/bin/bash
mkdir -p gpurun_out
for v in p512_2 p256_4; do
AIWC_LIB=build/variants/$v/libaiwc_cuda.so timeout 300 python tools/predict_once.py 100000000 2 > gpurun_out/pred_$v.log 2>&1
done
timeout 300 python tools/predict_once.py 100000000 2 > gpurun_out/pred_plain.log 2>&1
