#!/bin/bash
# compute-sanitizer over the round-2 kernels (parallel op programs, two-phase lookup), + bench_kv with ceilings
mkdir -p gpurun_out/sanitizer
SB_PROG_FAST=1 timeout 1500 compute-sanitizer --tool memcheck --print-limit 20 python tests/fastpath_diff.py > gpurun_out/sanitizer/memcheck_fastpath.log 2>&1; echo memcheck_rc=$?
tail -3 gpurun_out/sanitizer/memcheck_fastpath.log
timeout 1200 compute-sanitizer --tool racecheck --print-limit 20 python -m pytest tests/test_engine_gpu.py -q -k "steps_match_oracle" > gpurun_out/sanitizer/racecheck_engine.log 2>&1; echo racecheck_rc=$?
tail -3 gpurun_out/sanitizer/racecheck_engine.log
timeout 1200 compute-sanitizer --tool racecheck --print-limit 20 python -m pytest tests/test_kvcache_gpu.py -q -k "batch or lookup" > gpurun_out/sanitizer/racecheck_lookup.log 2>&1; echo racecheck2_rc=$?
tail -3 gpurun_out/sanitizer/racecheck_lookup.log
timeout 900 python bench_kv.py --only probe,probe_big,evict_small,evict,evict_big,append 2>/dev/null > gpurun_out/kv_v7.jsonl; echo kv=$?
