"""Standalone repro of tests/test_engine_gpu.py (pool smaller than one step's
suffix blocks) for compute-sanitizer runs."""
import sys

sys.path.insert(0, ".")
import numpy as np
import torch

from paper_2601_12967_b200 import workload as W
from paper_2601_12967_b200.engine import ContinuationEngine, ModelShape

n_req, slack = int(sys.argv[1]), float(sys.argv[2])
reqs = W.agentic_continuation_batch(n_req, sys_len=256, seed=3)
pre = sum(r.prefix_len // 16 for r in reqs) - (n_req - 1) * 16
suf = sum((r.suffix_len + 15) // 16 for r in reqs)
cap = pre + int(slack * suf) + 1
eng = ContinuationEngine(ModelShape(2, 8, 2, 128), cap, policy=1)
handles = [eng.submit_partial_prefill(r.prefix_tokens, r.prefix_tags, now=0) for r in reqs]
batch = eng.make_batch(handles, [r.suffix_len for r in reqs])
for step in range(3):
    suffix = np.concatenate([W.fresh_suffix_tokens(r, step) for r in reqs]).view(np.int64)
    batch.stage_suffix_device(torch.from_numpy(suffix).cuda())
    batch.run(10 + step, seed=step)
    torch.cuda.synchronize()
    print("step", step, "status", batch.status.cpu().tolist(), flush=True)
