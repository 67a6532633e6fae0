#!/bin/bash
# tcgen05 projection GEMM: numerics vs torch fp32, then timing vs cuBLAS at the configs[2] shapes
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gemm_gpu.py -x -q > gpurun_out/gemm_test.log 2>&1; echo gemm_test_rc=$?
tail -25 gpurun_out/gemm_test.log
timeout 300 python bench_gemm.py > gpurun_out/bench_gemm.jsonl 2>&1; echo bench_gemm_rc=$?
cat gpurun_out/bench_gemm.jsonl | tail -12
