#!/bin/bash
# Round-1 final pool-kernel evidence: one `ncu --set full` capture per kernel at
# its largest bench_kv configuration, + bench_kv.py.
mkdir -p gpurun_out
timeout 900 python bench_kv.py > gpurun_out/bench_kv.jsonl 2> gpurun_out/bench_kv.err; echo benchkv_rc=$?
# chain hash: 262144 x 512 config = launches 92..114 (5th config), take the 2nd
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"^k_chain_hash16" -s 93 -c 1 \
    -o gpurun_out/pool_hash -f python bench_kv.py --only hash > gpurun_out/ncu_hash.log 2>&1; echo rc=$?
# lookup: 4096 x 8192 tokens over a 4M-block pool (skip warm-ups)
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"^k_probe_rows" -s 4 -c 1 \
    -o gpurun_out/pool_probe -f python bench_kv.py --only probe_big > gpurun_out/ncu_probe.log 2>&1; echo rc=$?
# scoring: 16M-block pool; fill = 8192 inserts (one k_score each), then evict warm-up
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"^k_score" -s 8194 -c 1 \
    -o gpurun_out/pool_score -f python bench_kv.py --only evict_big > gpurun_out/ncu_score.log 2>&1; echo rc=$?
ls gpurun_out
