#!/bin/bash
# 1-CTA vs CTA-pair attention on a uniform problem, with the SM clock sampled during each run
mkdir -p gpurun_out
for arm in 0 1 0 1; do
  nvidia-smi --query-gpu=clocks.sm,power.draw --format=csv,noheader,nounits -lms 200 > gpurun_out/clk_$arm.txt &
  SMI=$!
  SB_ATTN_PAIR=$arm timeout 300 python profiles/attn_uniform_ab.py > gpurun_out/uni_$arm.json 2> gpurun_out/uni_$arm.err
  kill $SMI
  python -c "
import json,statistics
d=json.loads(open('gpurun_out/uni_$arm.json').read().strip().splitlines()[-1])
c=[float(l.split(',')[0]) for l in open('gpurun_out/clk_$arm.txt') if l.strip()]
c=c[len(c)//4:]
print('pair=$arm', round(d['ms'],3), 'ms', round(d['tflops']), 'TFLOP/s', 'sm_mhz', statistics.median(c) if c else None, 'tflop_per_ghz', round(d['tflops']/(statistics.median(c)/1000),1) if c else None)"
done
