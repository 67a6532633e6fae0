#!/bin/bash
# CTA-pair attention with P released in one part per tile (SB_ATTN_PSPLIT=1) vs two parts vs the 1-CTA kernel
mkdir -p gpurun_out
timeout 300 env SB_ATTN_PAIR=1 SB_ATTN_PSPLIT=1 python -m pytest tests/test_attention_gpu.py -x -q -k "matches_fp32 or bench_shape" > gpurun_out/p1_test.log 2>&1; echo p1_test_rc=$?; tail -1 gpurun_out/p1_test.log
for arm in p1 p2 one p1 p2 one; do
  unset SB_ATTN_PAIR SB_ATTN_PSPLIT
  case $arm in p1) export SB_ATTN_PAIR=1 SB_ATTN_PSPLIT=1;; p2) export SB_ATTN_PAIR=1;; esac
  timeout 600 python bench.py --no-trace --no-pool-roofline --no-cpu-baseline --no-dense > gpurun_out/h_$arm.json 2> gpurun_out/h_$arm.err
  python -c "
import json;d=json.loads(open('gpurun_out/h_$arm.json').read().strip().splitlines()[-1])
print('$arm', round(d['value']), 'attn_frac', round(d['roofline']['frac'],4), d['clocks']['sm_mhz'])"
done
