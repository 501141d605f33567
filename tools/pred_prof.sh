#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q -k "predict or pins or rank or c1 or import or narrow or dropin or gather" > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python tools/predict_once.py 100000000 3 > gpurun_out/pred_plain.log 2>&1
AIWC_PRED_NODE8=1 timeout 300 python tools/predict_once.py 100000000 3 > gpurun_out/pred_node8.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:predict_chunk_kernel \
  --launch-skip 2 --launch-count 1 -f -o gpurun_out/pred python tools/predict_once.py 20000000 1 > gpurun_out/pred_ncu.log 2>&1
echo "ncu rc=$?" >> gpurun_out/pred_ncu.log
