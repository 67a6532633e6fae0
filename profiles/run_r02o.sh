#!/bin/bash
# Round-2 bench line after the parallel op programs / probe / prefix-hash overlap
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench_rc=$?
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref_rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/launches_step.csv \
   python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-dense --no-trace --no-pool-roofline > gpurun_out/ncu_bench.log 2>&1; echo ncu_rc=$?
