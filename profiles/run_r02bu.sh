#!/bin/bash
# compute-sanitizer over the new kernels: the projections' GEMM (both kernels, every epilogue) and the CTA-pair attention
mkdir -p gpurun_out/sanitizer
K="not llama and not one_cta and not 14336 and not 128256 and not 6144"
timeout 1200 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gemm_gpu.py -q -k "$K" > gpurun_out/sanitizer/memcheck_gemm.log 2>&1; echo memcheck_gemm_rc=$?
tail -2 gpurun_out/sanitizer/memcheck_gemm.log
SB_GEMM_PAIR=0 timeout 1200 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gemm_gpu.py -q -k "$K" > gpurun_out/sanitizer/memcheck_gemm_1cta.log 2>&1; echo memcheck_gemm1_rc=$?
tail -2 gpurun_out/sanitizer/memcheck_gemm_1cta.log
timeout 1200 compute-sanitizer --tool racecheck --print-limit 20 python -m pytest tests/test_gemm_gpu.py -q -k "$K" > gpurun_out/sanitizer/racecheck_gemm.log 2>&1; echo racecheck_gemm_rc=$?
tail -2 gpurun_out/sanitizer/racecheck_gemm.log
timeout 1200 compute-sanitizer --tool synccheck --print-limit 20 python -m pytest tests/test_gemm_gpu.py -q -k "$K" > gpurun_out/sanitizer/synccheck_gemm.log 2>&1; echo synccheck_gemm_rc=$?
tail -2 gpurun_out/sanitizer/synccheck_gemm.log
SB_ATTN_PAIR=1 timeout 1500 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_attention_gpu.py -q -k "matches_fp32 and not f32 and not 32768" > gpurun_out/sanitizer/memcheck_attn_pair.log 2>&1; echo memcheck_attn_pair_rc=$?
tail -2 gpurun_out/sanitizer/memcheck_attn_pair.log
SB_ATTN_PAIR=1 timeout 1500 compute-sanitizer --tool racecheck --print-limit 20 python -m pytest tests/test_attention_gpu.py -q -k "matches_fp32 and not f32 and not 32768" > gpurun_out/sanitizer/racecheck_attn_pair.log 2>&1; echo racecheck_attn_pair_rc=$?
tail -2 gpurun_out/sanitizer/racecheck_attn_pair.log
