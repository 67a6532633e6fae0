#!/bin/bash
# Pool-side profiling: engine op programs (phase counters + launch list) and
# the pool-kernel rooflines under the write-only vs write+read L2 flush.
mkdir -p gpurun_out
SB_PROG_PROFILE=1 timeout 300 python bench_engine_ops.py > gpurun_out/engine_ops.json 2> gpurun_out/engine_ops.err; echo ops_rc=$?
cat gpurun_out/engine_ops.json; grep SB_PROG gpurun_out/engine_ops.err
timeout 300 python bench_engine_ops.py > gpurun_out/engine_ops_noprof.json 2>&1; cat gpurun_out/engine_ops_noprof.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ops_launches.csv \
   python bench_engine_ops.py --steps 2 --warmup 1 > gpurun_out/ops_ncu.log 2>&1; echo ncu_rc=$?
SB_FLUSH=write timeout 600 python bench_kv.py --only probe_big,evict_small,evict > gpurun_out/kv_write.jsonl 2>/dev/null; echo kvw=$?
SB_FLUSH=writeread timeout 600 python bench_kv.py --only probe_big,evict_small,evict > gpurun_out/kv_wr.jsonl 2>/dev/null; echo kvwr=$?
