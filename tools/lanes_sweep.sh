#!/bin/bash
mkdir -p gpurun_out
for L in 4 6 8 3; do
  AIWC_WIDE_LANES=$L AIWC_VERBOSE=1 timeout 600 python tools/fit_once.py c4 1000 3 > gpurun_out/lanes_$L.log 2>&1
done
