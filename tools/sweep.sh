#!/bin/bash
# env sweep of the wide grower on C4 (T trees)
T=${T:-1000}
for cfg in "${@}"; do
  echo "== $cfg"
  env $cfg timeout 300 python tools/fit_once.py c4 $T 2 2>&1 | tail -n 1
done
