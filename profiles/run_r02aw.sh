#!/bin/bash
# chain hash: where the per-lane latency kernel beats the staged one (SB_HASH_LAT_MAX sweep)
for m in 2048 8192 1000000; do echo "lat_max=$m"
SB_HASH_LAT_MAX=$m timeout 300 python bench_kv.py --only hash 2>/dev/null | python -c "
import sys,json
for l in sys.stdin:
    r=json.loads(l); print(f\"  {r['kernel'][:18]:18s} {r['config']:28s} {r['seconds']*1e6:8.1f}us frac {r['frac']:.3f}\")"
done
