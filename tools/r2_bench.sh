#!/bin/bash
# Round-2 measurement: gpu tests, smoke, default bench (CPU arm included), launch list of a
# 296-tree C4 fit (4 lanes), ncu of the C5 predict kernel.
mkdir -p gpurun_out
nvidia-smi > gpurun_out/smi.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/smoke.log
AIWC_VERBOSE=1 timeout 1500 python bench.py ${BENCH_ARGS} > gpurun_out/bench.json 2> gpurun_out/bench.err
echo "bench rc=$?" >> gpurun_out/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_r2.csv python tools/fit_once.py c4 296 > gpurun_out/launches_r2.log 2>&1
echo "ncu rc=$?" >> gpurun_out/launches_r2.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:predict_chunk_kernel \
  --launch-skip 2 --launch-count 1 -f -o gpurun_out/pred python tools/predict_once.py 20000000 1 > gpurun_out/pred_ncu.log 2>&1
echo "ncu rc=$?" >> gpurun_out/pred_ncu.log
