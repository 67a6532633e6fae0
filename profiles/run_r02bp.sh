#!/bin/bash
# CTA-pair attention: attention tests (pair default), engine/model tests, then the configs[1] headline A/B (pair vs 1-CTA)
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_attention_gpu.py -x -q -k "not one_cta" > gpurun_out/attn_test.log 2>&1; echo attn_test_rc=$?
tail -25 gpurun_out/attn_test.log
if grep -q " passed" gpurun_out/attn_test.log && ! grep -q "failed\|error" gpurun_out/attn_test.log; then
  timeout 600 python -m pytest tests/test_engine_gpu.py tests/test_model_gpu.py -x -q > gpurun_out/engine_test.log 2>&1; echo engine_test_rc=$?
  tail -3 gpurun_out/engine_test.log
  for arm in pair one pair one; do
    unset SB_ATTN_PAIR; if [ $arm = one ]; then export SB_ATTN_PAIR=0; fi
    timeout 600 python bench.py --no-trace --no-pool-roofline --no-cpu-baseline --no-dense > gpurun_out/head_$arm.json 2> gpurun_out/head_$arm.err
    python -c "
import json;d=json.loads(open('gpurun_out/head_$arm.json').read().strip().splitlines()[-1])
print('$arm', round(d['value']), round(d['e2e']['value']), 'attn_frac', round(d['roofline']['frac'],4), d['clocks']['sm_mhz'], d['clocks'].get('power_w'))"
  done
fi
