#!/bin/bash
# Pool kernels at scale: probe variants (positions per lane pair), 4M/16M-pool scoring, large hash batch.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu -k "kvcache or engine or dropin or replay" > gpurun_out/pt.log 2>&1; echo pytest_rc=$?; tail -2 gpurun_out/pt.log
for per in 1 2 4; do
  echo "probe_per=$per"
  SB_PROBE_PER=$per timeout 600 python bench_kv.py --only probe,probe_big 2> /dev/null | grep -v '"k_score\|evict total'
done
timeout 900 python bench_kv.py --only hash,evict,evict_big 2> gpurun_out/bkv.err
