"""Kernel-time breakdown of the configs[2] full-model measurement (bench.run_dense)
under torch.profiler (CUPTI kernel records; timing diagnostic only, never a bench
value).  Prints the top kernels by total device time."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from torch.profiler import ProfilerActivity, profile

import bench

args = argparse.Namespace(steps=2, warmup=3)
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    bench.run_dense(args, 0, 1, 0)
    torch.cuda.synchronize()
rows = []
for e in prof.key_averages():
    t = getattr(e, "device_time_total", None) or getattr(e, "cuda_time_total", 0)
    if t > 0:
        rows.append((t, e.count, e.key))
rows.sort(reverse=True)
tot = sum(r[0] for r in rows)
for t, c, k in rows[:25]:
    print(f"{t / 1e3:10.2f} ms {100 * t / tot:6.2f} % {c:7d}  {k[:110]}")
