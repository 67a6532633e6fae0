#!/bin/bash
# round-2 ncu --set full of the continuation attention at the bench shape (one warm launch of the configs[1] step)
mkdir -p gpurun_out
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:'^k_continuation_attention$' -s 40 -c 1 \
    -o gpurun_out/r2_attention -f python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-trace --no-dense --no-pool-roofline \
    > gpurun_out/ncu_attn_r2.log 2>&1; echo rc=$?
grep -E "PROF|WARNING" gpurun_out/ncu_attn_r2.log | tail -3
