#!/bin/bash
# Pool-kernel evidence: bench_kv.py (CUPTI kernel times) + one `ncu --set full`
# capture each of the hash, lookup and scoring kernels at their largest config.
mkdir -p gpurun_out
timeout 600 python bench_kv.py > gpurun_out/bench_kv.jsonl 2> gpurun_out/bench_kv.err; echo benchkv_rc=$?
# launch indices: chain hash = config 4 (262144 x 128), 2nd launch; probe 5th; score = 2M pool (skip the 1M pool's 22)
for spec in "k_chain_hash16 70" "k_probe_batch 5" "k_score 27"; do
  set -- $spec
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"^$1" -s $2 -c 1 \
      -o gpurun_out/pool_$1 -f python bench_kv.py > gpurun_out/ncu_$1.log 2>&1
  echo ncu_$1_rc=$?
done
ls -la gpurun_out
