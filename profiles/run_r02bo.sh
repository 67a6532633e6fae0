#!/bin/bash
# configs[2] line with the GEMM roofline block; ncu of the CTA-pair GEMM (QKV and down shapes)
mkdir -p gpurun_out
timeout 600 python bench.py --no-trace --no-pool-roofline --no-cpu-baseline > gpurun_out/dense.json 2> gpurun_out/dense.err; echo dense_rc=$?
python -c "
import json;d=json.loads(open('gpurun_out/dense.json').read().strip().splitlines()[-1]);fm=d['full_model']
print(round(fm['tokens_per_s']), d['clocks']['sm_mhz']); print(json.dumps(fm['gemm_roofline'],indent=0))"
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_gemm_pair -c 1 -o gpurun_out/gemm_pair_qkv -f \
  python bench_gemm.py --only qkv --iters 1 --ours-only > gpurun_out/ncu_gemm_pair.log 2>&1; echo ncu_rc=$?
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_gemm_pair -c 1 -o gpurun_out/gemm_pair_down -f \
  python bench_gemm.py --only down+res --iters 1 --ours-only > gpurun_out/ncu_gemm_pair2.log 2>&1; echo ncu2_rc=$?
