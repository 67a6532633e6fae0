#!/bin/bash
# round-2 evidence after the fused evict kernel: smoke, bench (both arms)
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?
timeout 1200 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench_rc=$?
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref_rc=$?
