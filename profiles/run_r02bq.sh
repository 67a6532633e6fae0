#!/bin/bash
# ncu --set full of one warm CTA-pair attention launch of the configs[1] step
mkdir -p gpurun_out
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:'k_continuation_attention_pair' -s 40 -c 1 \
    -o gpurun_out/attn_pair -f python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-trace --no-dense --no-pool-roofline \
    > gpurun_out/ncu_attn_pair.log 2>&1; echo rc=$?
grep -E "PROF|WARNING|ERROR" gpurun_out/ncu_attn_pair.log | tail -3
