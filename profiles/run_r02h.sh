#!/bin/bash
mkdir -p gpurun_out
timeout 900 python bench.py --no-trace --no-pool-roofline > gpurun_out/bench_fast.json 2> gpurun_out/bench_fast.err; echo bench_rc=$?
python - <<'PY'
import json
l=[x for x in open('gpurun_out/bench_fast.json') if x.startswith('{')][-1]
d=json.loads(l)
print(d['value'], d['e2e'], d['gpu_launches'], d['ms_per_step'])
print(json.dumps(d['pool']))
print(json.dumps(d['roofline'])[:400])
PY
