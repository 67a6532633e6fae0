#!/bin/bash
# first radix pass histogrammed while scoring (window predicted from the previous select)
timeout 1500 python -m pytest -q -x -m gpu tests/test_kvcache_gpu.py tests/test_engine_gpu.py tests/test_program_fastpath_gpu.py 2>&1 | tail -2
timeout 300 python bench_kv.py --only evict_small,evict,probe,evict_big 2>/dev/null | python -c "
import sys,json
for l in sys.stdin:
    r=json.loads(l)
    if 'evict' in r['kernel'] or 'score' in r['kernel']: print(f\"  {r['kernel'][:20]:20s} {r['config'][5:13]:8s} {r['config'][-10:]:10s} {r['seconds']*1e6:7.1f}us frac {r['frac']:.3f} api {r['api_seconds']*1e6:6.1f}\")"
SB_SELECT_PROF=1 timeout 300 python bench_kv.py --only evict,evict_big > /dev/null 2> gpurun_out/sel_prof_pred.err
grep "SB_SELECT_PROF " gpurun_out/sel_prof_pred.err | awk 'NR%4==0' | tail -8 | cut -c1-300
