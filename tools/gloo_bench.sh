#!/bin/bash
mkdir -p gpurun_out
AIWC_BENCH_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 2 --steps 1 --warmup 1 --skip-cpu \
  --skip-predict --trees-per-gpu 60 --strong-steps 1 --grid-cells 4 --grid-sample-only > gpurun_out/bench_gloo2.json 2> gpurun_out/bench_gloo2.err
echo "rc=$?" >> gpurun_out/bench_gloo2.err
