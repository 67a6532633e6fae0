#!/bin/bash
# the torchrun / NCCL path of bench.py at world size 1 (the only NCCL world one GPU allows):
# process-group init, the max-over-ranks timing reductions and the trace all_gather over NCCL
mkdir -p gpurun_out
NCCL_DEBUG=INFO timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29541 \
   bench.py --gpus 1 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_nccl1.json 2> gpurun_out/bench_nccl1.err; echo nccl1_rc=$?
tail -c 600 gpurun_out/bench_nccl1.json; echo; grep -E "NCCL INFO (Using|comm|Channel 00|NVLS|Init COMPLETE)" gpurun_out/bench_nccl1.err | head -8
grep -i -E "error|traceback" gpurun_out/bench_nccl1.err | head -5
