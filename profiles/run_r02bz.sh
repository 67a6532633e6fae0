#!/bin/bash
# configs[2] (long cached prefixes, 1024-token suffixes): CTA-pair vs 1-CTA attention, alternating
mkdir -p gpurun_out
for arm in one pair one pair; do
  unset SB_ATTN_PAIR; if [ $arm = pair ]; then export SB_ATTN_PAIR=1; fi
  timeout 600 python bench.py --no-trace --no-pool-roofline --no-cpu-baseline > gpurun_out/d_$arm.json 2> gpurun_out/d_$arm.err
  python -c "
import json;d=json.loads(open('gpurun_out/d_$arm.json').read().strip().splitlines()[-1]);fm=d['full_model']
print('$arm', 'dense', round(fm['tokens_per_s']), 'attn_ms', round(fm['attention_ms_per_step'],2), 'attn_tflops', round(fm['attention_tflops']), 'headline', round(d['value']), d['clocks']['sm_mhz'])"
done
