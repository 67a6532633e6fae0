#!/bin/bash
# CTA-pair attention variants (P release granularity, MMA-issuer spin vs suspended wait) vs the 1-CTA kernel, alternating
mkdir -p gpurun_out
run() {  # name, env...
  local name=$1; shift
  env "$@" timeout 600 python bench.py --no-trace --no-pool-roofline --no-cpu-baseline --no-dense > gpurun_out/v_$name.json 2> gpurun_out/v_$name.err
  python -c "
import json;d=json.loads(open('gpurun_out/v_$name.json').read().strip().splitlines()[-1])
print('$name', round(d['value']), 'attn_frac', round(d['roofline']['frac'],4), d['clocks']['sm_mhz'], d['clocks'].get('power_w'))"
}
for rep in 1 2; do
  run p4s SB_ATTN_PAIR=1
  run p2s SB_ATTN_PSPLIT=2
  run p4spin SB_ATTN_SPIN=1
  run p2spin SB_ATTN_PSPLIT=2 SB_ATTN_SPIN=1
  run one SB_ATTN_PAIR=0
done
