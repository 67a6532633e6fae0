#!/bin/bash
# persistent attention kernel (SB_ATTN_PERSIST=1): parity first, then alternating A/B of the configs[1] step
SB_ATTN_PERSIST=1 timeout 600 python -m pytest -q -x -m gpu tests/test_attention_gpu.py tests/test_engine_gpu.py 2>&1 | tail -3
echo "persist tests rc=$?"
for rep in 1 2; do for v in 0 1; do
SB_ATTN_PERSIST=$v timeout 600 python bench.py --no-trace --no-pool-roofline --no-dense --no-cpu-baseline > gpurun_out/bench_p$v.json 2>/dev/null
python -c "
import json; d=json.loads([x for x in open('gpurun_out/bench_p$v.json') if x.startswith('{')][-1]); print('persist=$v', round(d['value']), d['clocks']['sm_mhz'], round(d['roofline']['frac'],4), round(d['roofline'].get('kernel_ms', 0) or 0, 3), d['roofline'].get('library_reference',{}).get('tflops'))"
done; done
