#!/bin/bash
# GEMM with the k-adaptive raster band: tests, timing (down projection), ncu DRAM bytes of the down launch
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gemm_gpu.py -x -q > gpurun_out/gemm_test.log 2>&1; echo gemm_test_rc=$?
tail -2 gpurun_out/gemm_test.log
for r in 1 2; do timeout 300 python bench_gemm.py --ours-only > gpurun_out/bench_gemm_band_$r.jsonl 2>&1; cat gpurun_out/bench_gemm_band_$r.jsonl; done
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:k_gemm_pair -c 1 \
  python bench_gemm.py --only down+res --iters 1 --ours-only > gpurun_out/ncu_gemm_down_band.log 2>&1; echo ncu_rc=$?
grep -E "dram__bytes|duration|tensor" gpurun_out/ncu_gemm_down_band.log
