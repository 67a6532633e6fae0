#!/bin/bash
# select-path coverage: keys read in place at 16M blocks, K above the rank buffer, the three-kernel path
timeout 1500 python -m pytest -q -x -m gpu tests/test_kvcache_gpu.py -k "in_place or beyond_shared or three_kernel or cooperative" 2>&1 | tail -3
