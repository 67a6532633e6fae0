#!/bin/bash
# rank step with 16 B shared loads: pool parity tests, then evict rows + the phase stamps
mkdir -p gpurun_out
timeout 1500 python -m pytest -q -x -m gpu tests/test_kvcache_gpu.py tests/test_program_fastpath_gpu.py tests/test_engine_gpu.py > gpurun_out/pool_test.log 2>&1; echo pool_test_rc=$?
tail -1 gpurun_out/pool_test.log
for r in 1 2; do timeout 300 python bench_kv.py --only evict_small,evict,evict_big 2>/dev/null | python -c "
import sys,json
for l in sys.stdin:
    r=json.loads(l); print(f\"{r['config'][:60]:60s} {r['seconds']*1e6:8.1f}us frac {r['frac']:.3f}\")"; done
SB_SELECT_PROF=1 timeout 300 python bench_kv.py --only evict > /dev/null 2> gpurun_out/kv_prof.err
grep "SB_SELECT_PROF mode" gpurun_out/kv_prof.err | tail -2
