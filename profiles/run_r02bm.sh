#!/bin/bash
# GEMM with the banded tile raster: tests, timing vs cuBLAS, ncu of the QKV-shape launch, full-model A/B
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gemm_gpu.py -x -q > gpurun_out/gemm_test.log 2>&1; echo gemm_test_rc=$?
tail -2 gpurun_out/gemm_test.log
timeout 300 python bench_gemm.py > gpurun_out/bench_gemm.jsonl 2>&1; echo bench_gemm_rc=$?
cat gpurun_out/bench_gemm.jsonl | tail -6
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_gemm -c 1 -o gpurun_out/gemm_qkv -f \
  python bench_gemm.py --only qkv --iters 1 --ours-only > gpurun_out/ncu_gemm.log 2>&1; echo ncu_rc=$?
for arm in ours cublas; do
  if [ $arm = cublas ]; then export SB_GEMM_CUBLAS=1; else unset SB_GEMM_CUBLAS; fi
  timeout 600 python bench.py --no-trace --no-pool-roofline --no-cpu-baseline > gpurun_out/dense_$arm.json 2> gpurun_out/dense_$arm.err
  python -c "
import json;d=json.loads(open('gpurun_out/dense_$arm.json').read().strip().splitlines()[-1]);fm=d['full_model']
print('$arm', round(fm['tokens_per_s']), round(fm['ms_per_step'],2), 'attn_ms', round(fm['attention_ms_per_step'],2), 'rest_tflops', round(fm['rest_tflops']), d['clocks']['sm_mhz'], 'headline', round(d['value']))"
done
