#!/bin/bash
# GPU-box round check: gpu tests, bench, launch list, one full ncu capture.
mkdir -p gpurun_out
nvidia-smi > gpurun_out/smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py ${BENCH_ARGS:---steps 3 --warmup 3} > gpurun_out/bench.json 2> gpurun_out/bench.err
echo "bench rc=$?" >> gpurun_out/bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches.csv python tools/fit_once.py c4 296 > gpurun_out/ncu_launch.log 2>&1
echo "ncu launch rc=$?" >> gpurun_out/ncu_launch.log
timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:"${NCU_KERNELS:-w_chains_warp|w_ltree|w_pay|w_route|w_chains_lane}" --launch-skip ${NCU_SKIP:-150} -c ${NCU_COUNT:-10} \
  -f -o gpurun_out/full python tools/fit_once.py c4 296 > gpurun_out/ncu_full.log 2>&1
echo "ncu full rc=$?" >> gpurun_out/ncu_full.log
