#!/bin/bash
# final check of the round's code: GPU suite, smoke, full bench line
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?
tail -2 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?
tail -1 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench_rc=$?
python -c "
import json;d=json.loads(open('gpurun_out/bench.json').read().strip().splitlines()[-1]);fm=d['full_model']
print('value',round(d['value']),'e2e',round(d['e2e']['value']),'attn',round(d['roofline']['frac'],4),d['clocks']['sm_mhz'],'full_model',round(fm['tokens_per_s']),'gemm',[round(r['frac'],3) for r in fm['gemm_roofline']['rows']])"
