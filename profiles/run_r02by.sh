#!/bin/bash
# after the shared-softmax refactor (both attention kernels call one device function): attention tests
# (1-CTA default + the pair arm in a subprocess), engine / model tests, the headline line
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_attention_gpu.py tests/test_engine_gpu.py tests/test_model_gpu.py -x -q > gpurun_out/attn_test.log 2>&1; echo attn_test_rc=$?
tail -2 gpurun_out/attn_test.log
for arm in one pair one; do
  unset SB_ATTN_PAIR; if [ $arm = pair ]; then export SB_ATTN_PAIR=1; fi
  timeout 600 python bench.py --no-trace --no-pool-roofline --no-cpu-baseline --no-dense > gpurun_out/head_$arm.json 2> gpurun_out/head_$arm.err
  python -c "
import json;d=json.loads(open('gpurun_out/head_$arm.json').read().strip().splitlines()[-1])
print('$arm', round(d['value']), round(d['e2e']['value']), 'attn_frac', round(d['roofline']['frac'],4), d['clocks']['sm_mhz'])"
done
