#!/bin/bash
mkdir -p gpurun_out
AIWC_VERBOSE=1 timeout 600 python tools/fit_once.py c4 1000 3 > gpurun_out/l16.log 2>&1
AIWC_WIDE_LANES=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launch_l16.csv python tools/fit_once.py c4 148 > gpurun_out/ncu_l16.log 2>&1
