#!/bin/bash
timeout 600 python -c "
import json, bench
print(json.dumps(bench.run_toy(0), indent=1))
" 2>&1 | tail -60
