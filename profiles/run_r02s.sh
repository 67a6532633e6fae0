#!/bin/bash
# ncu --set full of the two-phase lookup (4M pool) and of the chain hash at its throughput config
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"^k_probe_rows2" -s 3 -c 1 \
    -o gpurun_out/r2_probe2 -f python bench_kv.py --only probe_big > gpurun_out/ncu_probe2.log 2>&1; echo rc=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"^k_chain_hash16" -s 60 -c 1 \
    -o gpurun_out/r2_hash -f python bench_kv.py --only hash > gpurun_out/ncu_hash.log 2>&1; echo rc=$?
