#!/bin/bash
# heatmap_scan drop-in timing (serial vs batched) for library variants swapped into place
mkdir -p gpurun_out
cp paper_1811_00156_b200/libaiwc_cuda.so /tmp/lib_cur.so
for r in 1 2; do
  for v in cur ${VARIANTS}; do
    if [ $v = cur ]; then cp /tmp/lib_cur.so paper_1811_00156_b200/libaiwc_cuda.so;
    else cp build/variants/$v/libaiwc_cuda.so paper_1811_00156_b200/libaiwc_cuda.so; fi
    for m in serial batched; do
      if [ $m = serial ]; then E="AIWC_FIT_BATCH=0"; else E="X=1"; fi
      echo "== $v $m $(env $E timeout 600 oracle/_ref/dropin_test heatmap 2>/dev/null | tail -1 | python -c 'import json,sys; print(json.loads(sys.stdin.read())["seconds"])')" >> gpurun_out/heatmap_ab.log
    done
  done
done
cp /tmp/lib_cur.so paper_1811_00156_b200/libaiwc_cuda.so
