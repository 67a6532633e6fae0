#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_program_fastpath_gpu.py tests/test_engine_gpu.py tests/test_engine_lifecycle_gpu.py -x -q > gpurun_out/pytest_fast.log 2>&1; echo pytest_rc=$?
tail -2 gpurun_out/pytest_fast.log
SB_PROG_PROFILE=1 timeout 300 python bench_engine_ops.py 2>&1 | grep -E "ms_per_step|parallel path"
