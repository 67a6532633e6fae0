#!/bin/bash
# Profiling recipe used for profiles/ (run under gpurun on one B200).
set -x
mkdir -p gpurun_out
# 1) launch list of one warm bench step (cold-cache, serialised: compare shares)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 1500 -c 1600 --csv \
    --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 2 --no-cpu-baseline \
    > gpurun_out/ncu_bench.log 2>&1
# 2) full section set of the attention kernel (2 launches) and the pool kernels
timeout 900 ncu --set full --clock-control none --import-source on -k regex:continuation -s 40 -c 1 \
    -o gpurun_out/prof_attention python bench.py --steps 1 --warmup 1 --no-cpu-baseline \
    > gpurun_out/ncu_attn.log 2>&1
