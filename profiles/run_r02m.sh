#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_kvcache_gpu.py -x -q > gpurun_out/pytest_pick.log 2>&1; echo pytest_rc=$?
tail -2 gpurun_out/pytest_pick.log
timeout 600 python bench_kv.py --only evict_small,evict,evict_big 2>/dev/null > gpurun_out/kv_evict2.jsonl; echo kv=$?
SB_PICK=2 timeout 600 python bench_kv.py --only evict 2>&1 | grep "k_pick:" | tail -3
