#!/bin/bash
timeout 900 python bench.py --no-trace --no-dense --no-cpu-baseline > gpurun_out/bench_pr.json 2> gpurun_out/bench_pr.err; echo rc=$?
python -c "
import json; d=json.loads([x for x in open('gpurun_out/bench_pr.json') if x.startswith('{')][-1])
print(round(d['value']))
for r in d['roofline_pool']['rows']: print(r['kernel'][:70], r.get('config','')[:45], round(r.get('seconds',0)*1e6,1), round(r.get('frac',0),3), r.get('error',''))"
