#!/bin/bash
# functional check of the N>1 path of bench.py on one GPU: two ranks sharing it, gloo for the statistics
# reduction and gathers (NCCL refuses two ranks on one device); the numbers are NOT a scaling measurement
mkdir -p gpurun_out
SB_DIST_BACKEND=gloo timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 \
  bench.py --gpus 2 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_n2.json 2> gpurun_out/bench_n2.err; echo n2_rc=$?
tail -c 1500 gpurun_out/bench_n2.json
grep -iE "error|traceback" gpurun_out/bench_n2.err | head -5
SB_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29534 \
  bench.py --impl reference --gpus 2 --steps 2 --warmup 3 > gpurun_out/bench_ref_n2.json 2> gpurun_out/bench_ref_n2.err; echo ref_n2_rc=$?
tail -c 400 gpurun_out/bench_ref_n2.json
