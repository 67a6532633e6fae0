#!/bin/bash
timeout 1800 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
timeout 300 python bench_engine_ops.py
timeout 900 python bench.py --no-trace --no-pool-roofline --no-dense --no-cpu-baseline > gpurun_out/bench_l.json 2>/dev/null; echo bench_rc=$?
python -c "
import json; d=json.loads([x for x in open('gpurun_out/bench_l.json') if x.startswith('{')][-1]); print(d['value'], d['gpu_launches'], d['pool']['ms_per_step'], d['pool']['share_of_step'])"
