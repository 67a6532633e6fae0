#!/bin/bash
# Parallel op-program path: differential test, engine parity tests, engine-ops timing.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_program_fastpath_gpu.py tests/test_engine_gpu.py tests/test_engine_lifecycle_gpu.py tests/test_kvcache_gpu.py -x -q > gpurun_out/pytest_fast.log 2>&1; echo pytest_rc=$?
tail -30 gpurun_out/pytest_fast.log
SB_PROG_PROFILE=1 timeout 300 python bench_engine_ops.py > gpurun_out/engine_ops.json 2> gpurun_out/engine_ops.err; echo ops_rc=$?
cat gpurun_out/engine_ops.json; grep SB_PROG gpurun_out/engine_ops.err
timeout 300 python bench_engine_ops.py; SB_PROG_FAST=0 timeout 300 python bench_engine_ops.py
