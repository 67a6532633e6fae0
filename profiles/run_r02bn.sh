#!/bin/bash
# CTA-pair GEMM: tests (both kernels), timing vs cuBLAS, full-model A/B
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gemm_gpu.py -x -q -k "not one_cta" > gpurun_out/gemm_test.log 2>&1; echo gemm_test_rc=$?
tail -15 gpurun_out/gemm_test.log
timeout 300 python -m pytest tests/test_gemm_gpu.py -x -q -k "one_cta" > gpurun_out/gemm_test1.log 2>&1; echo gemm_test1_rc=$?
tail -3 gpurun_out/gemm_test1.log
timeout 300 python bench_gemm.py > gpurun_out/bench_gemm.jsonl 2>&1; echo bench_gemm_rc=$?
cat gpurun_out/bench_gemm.jsonl | tail -6
SB_GEMM_PAIR=0 timeout 300 python bench_gemm.py --ours-only > gpurun_out/bench_gemm_1cta.jsonl 2>&1
cat gpurun_out/bench_gemm_1cta.jsonl | tail -6
timeout 600 python -m pytest tests/test_model_gpu.py -x -q > gpurun_out/model_test.log 2>&1; echo model_test_rc=$?
tail -2 gpurun_out/model_test.log
for arm in ours cublas ours1cta; do
  unset SB_GEMM_CUBLAS SB_GEMM_PAIR
  if [ $arm = cublas ]; then export SB_GEMM_CUBLAS=1; fi
  if [ $arm = ours1cta ]; then export SB_GEMM_PAIR=0; fi
  timeout 600 python bench.py --no-trace --no-pool-roofline --no-cpu-baseline > gpurun_out/dense_$arm.json 2> gpurun_out/dense_$arm.err
  python -c "
import json;d=json.loads(open('gpurun_out/dense_$arm.json').read().strip().splitlines()[-1]);fm=d['full_model']
print('$arm', round(fm['tokens_per_s']), round(fm['ms_per_step'],2), 'attn_ms', round(fm['attention_ms_per_step'],2), 'rest_tflops', round(fm['rest_tflops']), d['clocks']['sm_mhz'], 'headline', round(d['value']))"
done
