#!/bin/bash
timeout 900 python -m pytest tests/test_hash_gpu.py tests/test_engine_gpu.py tests/test_kvcache_gpu.py -x -q 2>&1 | tail -1
for m in 0 2048; do echo lat_max=$m; SB_HASH_LAT_MAX=$m timeout 600 python bench_kv.py --only hash 2>/dev/null | python -c "
import sys,json
for l in sys.stdin:
    r=json.loads(l); print(f\"  {r['config']:28s} {r['frac']:.4f} {r['seconds']*1e6:8.1f}us\")"; SB_HASH_LAT_MAX=$m timeout 300 python bench_engine_ops.py; done
