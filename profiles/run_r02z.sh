#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_kvcache_gpu.py tests/test_engine_gpu.py tests/test_program_fastpath_gpu.py tests/test_dropin_gpu.py -x -q > gpurun_out/pytest_sel.log 2>&1; echo pytest_rc=$?
tail -2 gpurun_out/pytest_sel.log
timeout 300 python bench_engine_ops.py
timeout 900 python bench_kv.py --only probe,evict_small,evict,evict_big 2>/dev/null > gpurun_out/kv_sel.jsonl; echo kv=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ops_launches_sel.csv \
   python bench_engine_ops.py --steps 2 --warmup 1 > gpurun_out/ops_ncu.log 2>&1; echo ncu_rc=$?
