#!/bin/bash
# end-of-round check after the GEMM / pair-attention work: GPU suite, smoke, full bench line, reference arm
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?
tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench_rc=$?
python -c "
import json;d=json.loads(open('gpurun_out/bench.json').read().strip().splitlines()[-1]);fm=d['full_model']
print('value',round(d['value']),'e2e',round(d['e2e']['value']),'attn',round(d['roofline']['frac'],4),d['clocks'],'full_model',round(fm['tokens_per_s']),'launches',d.get('gpu_launches'))"
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref_rc=$?
tail -c 600 gpurun_out/bench_ref.json
