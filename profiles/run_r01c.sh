#!/bin/bash
# round-1 v3 evidence: full ncu of the current attention kernel + pool kernels at scale
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:continuation -s 40 -c 1 \
    -o gpurun_out/prof_attention_v3 python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_attn3.log 2>&1
echo ncu_attn_rc=$?
timeout 600 python bench_kv.py > gpurun_out/bench_kv2.jsonl 2> gpurun_out/bench_kv2.err; echo benchkv_rc=$?
timeout 900 ncu --set full --clock-control none -k regex:"k_select_coop|k_probe_batch|k_chain_hash" -c 6 \
    -o gpurun_out/prof_pool python bench_kv.py > gpurun_out/ncu_pool.log 2>&1
echo ncu_pool_rc=$?
