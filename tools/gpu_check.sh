#!/bin/bash
# GPU-box round check: gpu tests, smoke, bench, launch list + DRAM traffic of a 148-tree
# single-lane fit, one full ncu capture of the top kernels.
mkdir -p gpurun_out
nvidia-smi > gpurun_out/smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 1200 python bench.py ${BENCH_ARGS} > gpurun_out/bench.json 2> gpurun_out/bench.err
echo "bench rc=$?" >> gpurun_out/bench.err
AIWC_WIDE_LANES=1 timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
  --clock-control none --csv --log-file gpurun_out/traffic.csv python tools/fit_once.py c4 148 \
  > gpurun_out/traffic_fit.log 2>&1
echo "ncu traffic rc=$?" >> gpurun_out/traffic_fit.log
AIWC_WIDE_LANES=1 timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:"${NCU_KERNELS:-w_chains_warp|w_lwarp|w_chains_grp|w_route|w_chains_lane|w_pay}" \
  --launch-skip ${NCU_SKIP:-40} --launch-count ${NCU_COUNT:-12} \
  -f -o gpurun_out/full python tools/fit_once.py c4 148 > gpurun_out/ncu_full.log 2>&1
echo "ncu full rc=$?" >> gpurun_out/ncu_full.log
