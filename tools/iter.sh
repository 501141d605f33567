#!/bin/bash
# quick GPU iteration: parity subset, C4 fit timing, optional launch list
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "${TESTS:-wide or both or c4 or c1_500}" 2>&1 | tail -n 5
timeout 300 python tools/fit_once.py c4 1000 3 2>&1 | tail -n 3
if [ -n "$PROFILE" ]; then
  timeout 800 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_it.csv python tools/fit_once.py c4 296 > gpurun_out/ncu_it.log 2>&1
  python tools/launch_share.py gpurun_out/launches_it.csv | head -n 14
fi
