#!/bin/bash
# round-1 measurement batch: GPU tests, bench, pool-kernel rooflines, ncu of attention
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?
tail -1 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 3 --warmup 3 > gpurun_out/bench5.json 2> gpurun_out/bench5.err; echo bench_rc=$?
timeout 600 python bench_kv.py > gpurun_out/bench_kv.jsonl 2> gpurun_out/bench_kv.err; echo benchkv_rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:continuation -s 40 -c 1 \
    -o gpurun_out/prof_attention_v2 python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_attn2.log 2>&1
echo ncu_rc=$?
