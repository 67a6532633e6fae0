#!/bin/bash
# Pool kernels after the 32 B index slot / 2-lane probe / direct-append scorer:
# GPU parity tests, bench_kv.py, and ncu --set full of k_probe_rows and k_score (4M-block pool).
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pt.log 2>&1; echo pytest_rc=$?; tail -3 gpurun_out/pt.log
timeout 600 python bench_kv.py > gpurun_out/bench_kv.jsonl 2> gpurun_out/bench_kv.err; echo benchkv_rc=$?; cat gpurun_out/bench_kv.jsonl
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"^k_probe_rows" -s 5 -c 1 \
    -o gpurun_out/probe_v5 -f python bench_kv.py --only probe > gpurun_out/ncu_probe.log 2>&1; echo ncu_probe_rc=$?
# k_score launches: 1M pool 2 x 11, then the 4M pool's fill inserts use k_score too -> select by the last launches
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"^k_score" -s 2051 -c 1 \
    -o gpurun_out/score_v5 -f python bench_kv.py --only evict > gpurun_out/ncu_score.log 2>&1; echo ncu_score_rc=$?
