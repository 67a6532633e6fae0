#!/bin/bash
# the N>1 bench path (two ranks sharing the one GPU, gloo for the statistics collectives)
mkdir -p gpurun_out
SB_DIST_BACKEND=gloo timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 \
   bench.py --gpus 2 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_n2.json 2> gpurun_out/bench_n2.err; echo n2_rc=$?
tail -c 1500 gpurun_out/bench_n2.json; tail -5 gpurun_out/bench_n2.err
