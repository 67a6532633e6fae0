#!/bin/bash
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?
tail -2 gpurun_out/pytest_gpu.log
timeout 600 python bench_kv.py --only probe,probe_big,evict_small,evict 2>/dev/null > gpurun_out/kv_v6.jsonl; echo kv=$?
