#!/bin/bash
# final round-2 evidence: ncu of the lookup kernel, bench (both arms), smoke
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"^k_probe_rows3" -s 3 -c 1 \
    -o gpurun_out/r2_probe3 -f python bench_kv.py --only probe_big > gpurun_out/ncu_probe3.log 2>&1; echo rc=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?
timeout 1200 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench_rc=$?
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref_rc=$?
