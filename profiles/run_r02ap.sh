#!/bin/bash
# ncu --set full of one 4M-block evict(64) through the fused kernel (source-level stalls)
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_evict_fused -s 2 -c 1 \
  -o gpurun_out/evict_fused_4M python bench_kv.py --only evict > gpurun_out/ncu_evict.log 2>&1
echo rc=$?
tail -3 gpurun_out/ncu_evict.log
