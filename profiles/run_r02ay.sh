#!/bin/bash
# end-of-round evidence: GPU suite, smoke, bench (both arms), ncu of the fused evict kernel at 4M blocks
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?
tail -2 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?
timeout 1200 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench_rc=$?
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref_rc=$?
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_evict_fused -s 2 -c 1 \
  -o gpurun_out/evict_fused_4M_v3 -f python bench_kv.py --only evict > gpurun_out/ncu_evict2.log 2>&1; echo ncu_rc=$?
