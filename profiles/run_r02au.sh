#!/bin/bash
# new pool parity tests (large-K cooperative evict, op programs on a cooperative pool, the three-kernel path), NCCL collectives
timeout 1500 python -m pytest -q -x -m gpu tests/test_kvcache_gpu.py tests/test_multirank_nccl_gpu.py 2>&1 | tail -4
