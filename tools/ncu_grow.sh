#!/bin/bash
# Plain run, then one ncu --set full capture of the big grower kernels at a few levels.
mkdir -p gpurun_out
AIWC_WIDE_LANES=1 timeout 600 python tools/fit_once.py c4 148 > gpurun_out/plain.log 2>&1 && \
AIWC_WIDE_LANES=1 timeout 1500 ncu --set full --clock-control none --import-source on \
  -k regex:"${KREGEX:-w_chains_warp|w_route|w_lwarp}" --launch-skip ${SKIP:-12} --launch-count ${COUNT:-6} \
  -f -o gpurun_out/${OUT:-grow_full} python tools/fit_once.py c4 148 > gpurun_out/grow_ncu.log 2>&1
echo "ncu rc=$?" >> gpurun_out/grow_ncu.log
