#!/bin/bash
# op programs at the engine's pool size (27K blocks): one-CTA k_select vs the fused cooperative kernel
for rep in 1 2; do for c in 65536 16384; do echo "prog_coop_min=$c"; SB_PROG_COOP_MIN_CAP=$c timeout 300 python bench_engine_ops.py 2>/dev/null | tail -1; done; done
SB_PROG_COOP_MIN_CAP=16384 timeout 900 python -m pytest -q -x -m gpu tests/test_engine_gpu.py tests/test_engine_lifecycle_gpu.py tests/test_program_fastpath_gpu.py 2>&1 | tail -2
