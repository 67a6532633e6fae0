#!/bin/bash
# per-CTA top-K select path: pool / engine / op-program parity tests, then evict rooflines A/B (SB_LOCAL_TOPK=1 vs 0)
mkdir -p gpurun_out
timeout 1500 python -m pytest -q -x -m gpu tests/test_kvcache_gpu.py tests/test_program_fastpath_gpu.py tests/test_engine_gpu.py tests/test_engine_lifecycle_gpu.py > gpurun_out/pool_test.log 2>&1; echo pool_test_rc=$?
tail -3 gpurun_out/pool_test.log
for arm in 1 0 1 0; do
  SB_LOCAL_TOPK=$arm timeout 300 python bench_kv.py --only evict_small,evict,evict_big 2>/dev/null | python -c "
import sys,json
for l in sys.stdin:
    r=json.loads(l); print('topk=$arm', f\"{r['config'][:60]:60s} {r['seconds']*1e6:8.1f}us frac {r['frac']:.3f}\")"
done
