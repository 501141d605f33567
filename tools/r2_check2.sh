#!/bin/bash
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
AIWC_BENCH_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 2 --steps 1 --warmup 1 --skip-cpu \
  --skip-predict --skip-grid --trees-per-gpu 60 --strong-steps 1 > gpurun_out/bench_gloo2.json 2> gpurun_out/bench_gloo2.err
echo "rc=$?" >> gpurun_out/bench_gloo2.err
timeout 900 python bench.py --steps 5 --warmup 3 --skip-cpu > gpurun_out/bench.json 2> gpurun_out/bench.err
echo "bench rc=$?" >> gpurun_out/bench.err
