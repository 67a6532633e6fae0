#!/bin/bash
# early-exit bound of the cooperative select (SB_RANK_EARLY): evict rows for 6144 / 3072 / 2048 / 1024, alternating
mkdir -p gpurun_out
for rep in 1 2; do for v in 6144 3072 2048 1024; do
  SB_RANK_EARLY=$v timeout 300 python bench_kv.py --only evict_small,evict,evict_big 2>/dev/null | python -c "
import sys,json
for l in sys.stdin:
    r=json.loads(l); print('early=$v', f\"{r['config'][:58]:58s} {r['seconds']*1e6:8.1f}us frac {r['frac']:.3f}\")"
done; done
