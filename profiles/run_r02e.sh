#!/bin/bash
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ops_launches_fast.csv \
   python bench_engine_ops.py --steps 2 --warmup 1 > gpurun_out/ops_ncu.log 2>&1; echo ncu_rc=$?
