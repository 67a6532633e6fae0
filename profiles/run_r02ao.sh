#!/bin/bash
# L2 eviction-priority hints for the evict kernels: 0 none, 1 metadata evict_first, 2 + keys evict_last
for h in 0 1 2; do echo "l2hint=$h"
SB_SCORE_L2HINT=$h SB_SELECT_PROF=1 timeout 300 python bench_kv.py --only evict > /dev/null 2> gpurun_out/sel_prof_h$h.err
grep "SB_SELECT_PROF " gpurun_out/sel_prof_h$h.err | awk 'NR%4==0' | tail -2 | cut -c1-330
SB_SCORE_L2HINT=$h timeout 300 python bench_kv.py --only evict_small,evict,probe,evict_big 2>/dev/null | python -c "
import sys,json
for l in sys.stdin:
    r=json.loads(l)
    if 'evict' in r['kernel'] or 'score' in r['kernel']: print(f\"  {r['kernel'][:20]:20s} {r['config'][5:13]:8s} {r['config'][-10:]:10s} {r['seconds']*1e6:7.1f}us frac {r['frac']:.3f} api {r['api_seconds']*1e6:6.1f}\")"
done
