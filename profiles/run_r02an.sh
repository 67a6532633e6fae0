#!/bin/bash
# fused evict kernel: pool parity tests, then evict rows fused vs three kernels, phase times
timeout 900 python -m pytest -q -x -m gpu tests/test_kvcache_gpu.py tests/test_program_fastpath_gpu.py tests/test_engine_gpu.py tests/test_engine_lifecycle_gpu.py 2>&1 | tail -3
for f in 0 1; do echo "fused=$f"; SB_EVICT_FUSED=$f timeout 300 python bench_kv.py --only evict_small,evict,probe,evict_big 2>/dev/null | python -c "
import sys,json
for l in sys.stdin:
    r=json.loads(l)
    if 'evict' in r['kernel'] or 'score' in r['kernel']: print(f\"  {r['kernel'][:20]:20s} {r['config'][5:13]:8s} {r['config'][-10:]:10s} {r['seconds']*1e6:7.1f}us frac {r['frac']:.3f} api {r['api_seconds']*1e6:6.1f} {r.get('parts_us','')}\")"; done
for f in 0 1; do SB_EVICT_FUSED=$f SB_SELECT_PROF=1 timeout 300 python bench_kv.py --only evict > /dev/null 2> gpurun_out/sel_prof_f$f.err
echo "prof fused=$f"; grep SB_SELECT_PROF gpurun_out/sel_prof_f$f.err | awk 'NR%3==0' | head -8; done
