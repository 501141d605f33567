#!/bin/bash
# small-table knob A/B: C2 batches (tools/grid_batch.py) and C3 evaluate (tools/loko_once.py)
mkdir -p gpurun_out
for v in ${VARS}; do
  echo "== $v" >> gpurun_out/small_ab.log
  env $v timeout 300 python tools/grid_batch.py >> gpurun_out/small_ab.log 2>&1
  env $v timeout 300 python tools/loko_once.py 2>&1 | tail -2 >> gpurun_out/small_ab.log
done
