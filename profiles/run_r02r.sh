#!/bin/bash
# compute-sanitizer memcheck over the pool / engine / drop-in paths and the parallel op-program differential run
mkdir -p gpurun_out/sanitizer
SB_PROG_FAST=1 timeout 1500 compute-sanitizer --tool memcheck --print-limit 20 python tests/fastpath_diff.py > gpurun_out/sanitizer/memcheck_fastpath.log 2>&1; echo memcheck_rc=$?
tail -1 gpurun_out/sanitizer/memcheck_fastpath.log
timeout 2400 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_kvcache_gpu.py tests/test_engine_gpu.py tests/test_engine_lifecycle_gpu.py tests/test_hash_gpu.py -q > gpurun_out/sanitizer/memcheck_pool_engine.log 2>&1; echo memcheck2_rc=$?
tail -2 gpurun_out/sanitizer/memcheck_pool_engine.log
