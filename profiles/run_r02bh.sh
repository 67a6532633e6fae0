#!/bin/bash
timeout 600 python -m pytest -q -x -m gpu tests/test_hash_gpu.py 2>&1 | tail -1
for r in 1 2; do timeout 300 python bench_kv.py --only hash 2>/dev/null | python -c "
import sys,json
for l in sys.stdin:
    r=json.loads(l); print(f\"  {r['kernel'][:18]:18s} {r['config']:28s} {r['seconds']*1e6:8.1f}us frac {r['frac']:.3f}\")"; done
