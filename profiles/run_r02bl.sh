#!/bin/bash
# configs[2] with the tcgen05 GEMM: model tests, then the full-model step, ours vs the cuBLAS A/B arm (alternating)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_model_gpu.py tests/test_gemm_gpu.py -x -q > gpurun_out/model_test.log 2>&1; echo model_test_rc=$?
tail -3 gpurun_out/model_test.log
for arm in ours cublas ours cublas; do
  if [ $arm = cublas ]; then export SB_GEMM_CUBLAS=1; else unset SB_GEMM_CUBLAS; fi
  timeout 600 python bench.py --no-trace --no-pool-roofline --no-cpu-baseline > gpurun_out/dense_$arm.json 2> gpurun_out/dense_$arm.err
  python -c "
import json;d=json.loads(open('gpurun_out/dense_$arm.json').read().strip().splitlines()[-1]);fm=d['full_model']
print('$arm', round(fm['tokens_per_s']), round(fm['ms_per_step'],2), 'attn_ms', round(fm['attention_ms_per_step'],2), 'rest_tflops', round(fm['rest_tflops']), d['clocks']['sm_mhz'], 'headline', round(d['value']))"
done
