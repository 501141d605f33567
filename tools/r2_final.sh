#!/bin/bash
# Round-2 final measurement: gpu tests, smoke, default bench (CPU arm included),
# gloo N=2 functional bench, ncu full capture of the top grower kernels.
mkdir -p gpurun_out
nvidia-smi > gpurun_out/smi.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 1800 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
echo "bench rc=$?" >> gpurun_out/bench.err
bash tools/gloo_bench.sh
AIWC_WIDE_LANES=1 timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:"w_chains_warp|w_lwarp|w_route|w_chains_grp" --launch-skip 40 --launch-count 8 \
  -f -o gpurun_out/grow_full python tools/fit_once.py c4 148 > gpurun_out/grow_ncu.log 2>&1
echo "ncu rc=$?" >> gpurun_out/grow_ncu.log
