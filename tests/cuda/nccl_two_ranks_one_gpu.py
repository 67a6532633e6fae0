"""Can two ranks share one GPU over NCCL here? (manual probe)"""
import os
import torch
import torch.distributed as dist

dist.init_process_group("nccl")
r = dist.get_rank()
torch.cuda.set_device(0)
x = torch.full((4,), float(r + 1), device="cuda")
dist.all_reduce(x)
print("rank", r, "all_reduce ->", x.tolist(), flush=True)
dist.destroy_process_group()
