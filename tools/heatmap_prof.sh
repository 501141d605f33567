#!/bin/bash
mkdir -p gpurun_out
for w in 20000 5000; do
AIWC_BATCH_WINDOW_US=$w AIWC_VERBOSE=1 timeout 300 oracle/_ref/dropin_test heatmap > gpurun_out/hm_batched_$w.json 2> gpurun_out/hm_batched_$w.err
done
AIWC_FIT_BATCH=0 timeout 300 oracle/_ref/dropin_test heatmap > gpurun_out/hm_serial.json 2> gpurun_out/hm_serial.err
