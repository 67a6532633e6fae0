#!/bin/bash
# compute-sanitizer over the reworked cooperative select (staging, filters, early exit, in-place path)
mkdir -p gpurun_out/sanitizer
timeout 1200 compute-sanitizer --tool racecheck --print-limit 20 python -m pytest tests/test_kvcache_gpu.py -q -k "cooperative_scorer or beyond_shared" > gpurun_out/sanitizer/racecheck_select_v2.log 2>&1; echo racecheck_rc=$?
tail -2 gpurun_out/sanitizer/racecheck_select_v2.log
timeout 1200 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_kvcache_gpu.py -q -k "cooperative or beyond_shared or evict_everything or insert_batch_on" > gpurun_out/sanitizer/memcheck_select_v2.log 2>&1; echo memcheck_rc=$?
tail -2 gpurun_out/sanitizer/memcheck_select_v2.log
timeout 1200 compute-sanitizer --tool synccheck --print-limit 20 python -m pytest tests/test_kvcache_gpu.py -q -k "cooperative or beyond_shared" > gpurun_out/sanitizer/synccheck_select_v2.log 2>&1; echo synccheck_rc=$?
tail -2 gpurun_out/sanitizer/synccheck_select_v2.log
timeout 1200 compute-sanitizer --tool racecheck --print-limit 20 python -m pytest tests/test_kvcache_gpu.py -q -k "keys_in_place" > gpurun_out/sanitizer/racecheck_select_inplace.log 2>&1; echo racecheck2_rc=$?
tail -2 gpurun_out/sanitizer/racecheck_select_inplace.log
