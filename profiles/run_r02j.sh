#!/bin/bash
# ncu --set full of the pool kernels at their largest bench_kv configs (round 2 baseline)
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"^k_probe_rows" -s 3 -c 1 \
    -o gpurun_out/r2_probe -f python bench_kv.py --only probe_big > gpurun_out/ncu_probe.log 2>&1; echo rc=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_score|k_select_coop" -s 24 -c 2 \
    -o gpurun_out/r2_evict -f python bench_kv.py --only evict > gpurun_out/ncu_evict.log 2>&1; echo rc=$?
ls -la gpurun_out/*.ncu-rep
