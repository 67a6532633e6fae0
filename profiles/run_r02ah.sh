#!/bin/bash
for c in 16384 100000000; do echo coop_min=$c; SB_COOP_MIN_CAP=$c timeout 300 python bench_kv.py --only evict_small 2>/dev/null | python -c "
import sys,json
for l in sys.stdin:
    r=json.loads(l); print(f\"  {r['kernel'][:30]:30s} {r['config'][-12:]:12s} {r['seconds']*1e6:7.1f}us api {r['api_seconds']*1e6:7.1f}us\")"; done
