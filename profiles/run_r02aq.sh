#!/bin/bash
# fused evict kernel: full GPU suite, sanitizers over the cooperative-scorer tests, bench_kv
mkdir -p gpurun_out/sanitizer
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?
tail -2 gpurun_out/pytest_gpu.log
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_kvcache_gpu.py -q -k "cooperative or in_place or evict_everything" > gpurun_out/sanitizer/memcheck_evict_fused.log 2>&1; echo memcheck_rc=$?
tail -2 gpurun_out/sanitizer/memcheck_evict_fused.log
timeout 900 compute-sanitizer --tool racecheck --print-limit 20 python -m pytest tests/test_kvcache_gpu.py -q -k "cooperative or evict_everything" > gpurun_out/sanitizer/racecheck_evict_fused.log 2>&1; echo racecheck_rc=$?
tail -2 gpurun_out/sanitizer/racecheck_evict_fused.log
timeout 900 compute-sanitizer --tool synccheck --print-limit 20 python -m pytest tests/test_kvcache_gpu.py -q -k "cooperative or evict_everything" > gpurun_out/sanitizer/synccheck_evict_fused.log 2>&1; echo synccheck_rc=$?
tail -2 gpurun_out/sanitizer/synccheck_evict_fused.log
timeout 900 python bench_kv.py 2>/dev/null > gpurun_out/bench_kv_v7.jsonl; echo kv=$?
