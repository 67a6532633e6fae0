#!/bin/bash
# Round-1 pool-kernel evidence: GPU tests of the pool, bench_kv.py (CUPTI kernel
# times), and one `ncu --set full` capture each of the hash, lookup and scoring
# kernels (launch indices select the largest configuration of each).
set -x
python -m pytest tests -x -q -m gpu -k "kvcache or engine or dropin or replay" > gpurun_out/pt.log 2>&1; tail -3 gpurun_out/pt.log
python bench_kv.py > gpurun_out/bench_kv.jsonl 2> gpurun_out/bench_kv.err; cat gpurun_out/bench_kv.jsonl
for spec in "k_chain_hash16 70" "k_probe_batch 5" "k_score 5"; do
  set -- $spec
  ncu --set full --clock-control none --import-source on -k regex:"^$1" --launch-skip $2 --launch-count 1 \
      -o gpurun_out/pool_$1 -f python bench_kv.py > gpurun_out/ncu_$1.log 2>&1
done
ls -la gpurun_out
