"""Continuation attention on a uniform problem (every sequence q_len suffix
tokens over a `prefix`-token cached prefix, Llama-3-8B heads; q_len a
multiple of 4 query tiles so CTA-pair quads are always full): back-to-back
launches for ~`seconds`, CUDA events, TFLOP/s of the median launch.  Run once
per SB_ATTN_PAIR setting (read at library load) to compare the 1-CTA and the
CTA-pair kernels without causal-extent or empty-slot effects."""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_12967_b200.attention import attention_work_list, continuation_attention

ap = argparse.ArgumentParser()
ap.add_argument("--seqs", type=int, default=64)
ap.add_argument("--q", type=int, default=1024)
ap.add_argument("--prefix", type=int, default=4096)
ap.add_argument("--seconds", type=float, default=6.0)
a = ap.parse_args()
hq, hkv = 32, 8
q_lens = [a.q] * a.seqs
kv_lens = [a.prefix + a.q] * a.seqs
nblk = [(k + 15) // 16 for k in kv_lens]
g = torch.Generator(device="cuda").manual_seed(0)
kp = torch.randn(sum(nblk), hkv, 16, 128, device="cuda", generator=g, dtype=torch.bfloat16)
vp = torch.randn(sum(nblk), hkv, 16, 128, device="cuda", generator=g, dtype=torch.bfloat16)
q = torch.randn(sum(q_lens), hq, 128, device="cuda", generator=g, dtype=torch.bfloat16)
table = torch.arange(sum(nblk), dtype=torch.int32, device="cuda").view(a.seqs, -1)
q_off = torch.tensor(np.cumsum([0] + q_lens), dtype=torch.int32, device="cuda")
kvl = torch.tensor(kv_lens, dtype=torch.int32, device="cuda")
work = torch.from_numpy(attention_work_list(q_lens, kv_lens, hq, hkv)).cuda()
out = torch.empty_like(q)
flops = sum(4 * 128 * hq * sum(p + i + 1 for i in range(ql)) for p, ql in zip([a.prefix] * a.seqs, q_lens))
for _ in range(3):
    continuation_attention(q, kp, vp, q_off, kvl, table, a.q, out=out, work=work)
torch.cuda.synchronize()
ts = []
t_end = time.time() + a.seconds
while time.time() < t_end:
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    continuation_attention(q, kp, vp, q_off, kvl, table, a.q, out=out, work=work)
    e1.record()
    e1.synchronize()
    ts.append(e0.elapsed_time(e1))
ms = float(np.median(ts))
print(json.dumps({"pair": os.environ.get("SB_ATTN_PAIR", "0"), "ms": ms, "tflops": flops / (ms * 1e-3) / 1e12,
                  "launches": len(ts), "seqs": a.seqs, "q": a.q, "prefix": a.prefix}))
