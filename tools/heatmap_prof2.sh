#!/bin/bash
mkdir -p gpurun_out
AIWC_PROFILE_PHASES=1 AIWC_VERBOSE=1 timeout 300 oracle/_ref/dropin_test heatmap > gpurun_out/hm_b.json 2> gpurun_out/hm_b.err
AIWC_FIT_BATCH=0 AIWC_PROFILE_PHASES=1 timeout 300 oracle/_ref/dropin_test heatmap > gpurun_out/hm_s.json 2> gpurun_out/hm_s.err
