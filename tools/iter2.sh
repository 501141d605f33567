#!/bin/bash
# GPU iteration: parity subset, per-level kernel profile (1 lane, 148 trees), C4 timing
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "${TESTS:-wide or both or c4 or c1_500}" 2>&1 | tail -n 2
AIWC_WIDE_LANES=1 timeout 800 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/lv.csv python tools/fit_once.py c4 148 > /dev/null 2>&1
python tools/per_level.py gpurun_out/lv.csv | awk 'NR==1 || NR<=5 || NR%8==0 || /sum/'
timeout 300 python tools/fit_once.py c4 1000 3 2>&1 | tail -n 2
