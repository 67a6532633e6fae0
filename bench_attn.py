"""Micro-benchmark of the continuation-prefill attention kernel alone, on the
bench step's configs[1] shapes (64 requests' suffix tokens over their cached
prefixes, Llama-3-8B heads), CUDA-event timed per launch.

    python bench_attn.py [--launches N]
"""
from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)


def setup(n_requests: int = 64, flashinfer: bool = False):
    """The configs[1] step's attention problem on synthetic paged KV:
    (q, k_pool, v_pool, q_off, kv_lens, table, work, out, run_ours, run_fi)
    with run_fi = flashinfer's trtllm-gen paged context kernel on the same
    tensors (None when flashinfer is absent or not requested)."""
    import torch
    from paper_2601_12967_b200 import workload as W
    from paper_2601_12967_b200.attention import attention_work_list, continuation_attention

    reqs = W.agentic_continuation_batch(n_requests, seed=1)
    hq, hkv = 32, 8
    q_lens = [r.suffix_len for r in reqs]
    kv_lens = [r.prefix_len + r.suffix_len for r in reqs]
    nblk = [(k + 15) // 16 for k in kv_lens]
    n_pages = sum(nblk)
    g = torch.Generator(device="cuda").manual_seed(0)
    kp = torch.randn(n_pages, hkv, 16, 128, device="cuda", generator=g, dtype=torch.bfloat16)
    vp = torch.randn(n_pages, hkv, 16, 128, device="cuda", generator=g, dtype=torch.bfloat16)
    q = torch.randn(sum(q_lens), hq, 128, device="cuda", generator=g, dtype=torch.bfloat16)
    perm = torch.randperm(n_pages, device="cuda", generator=g).to(torch.int32)
    table = torch.full((len(reqs), max(nblk)), -1, dtype=torch.int32, device="cuda")
    o = 0
    for i, n in enumerate(nblk):
        table[i, :n] = perm[o:o + n]
        o += n
    q_off = torch.tensor(np.cumsum([0] + q_lens), dtype=torch.int32, device="cuda")
    kvl = torch.tensor(kv_lens, dtype=torch.int32, device="cuda")
    work = torch.from_numpy(attention_work_list(q_lens, kv_lens, hq, hkv)).cuda()
    out = torch.empty_like(q)

    def run_ours():
        continuation_attention(q, kp, vp, q_off, kvl, table, max(q_lens), out=out, work=work)
        return out

    run_fi = None
    if flashinfer:
        try:
            import flashinfer.prefill as FP

            ws = torch.zeros(256 << 20, dtype=torch.uint8, device="cuda")
            seq_lens = torch.tensor(kv_lens, dtype=torch.int32, device="cuda")
            cum_kv = torch.tensor(np.cumsum([0] + kv_lens), dtype=torch.int32, device="cuda")
            fo = torch.empty_like(q)

            def run_fi():
                FP.trtllm_batch_context_with_kv_cache(q, (kp, vp), ws, table, seq_lens, max(q_lens), max(kv_lens),
                                                      1.0 / np.sqrt(128), 1.0, len(reqs), q_off, cum_kv, out=fo,
                                                      kv_layout="HND", causal=True)
                return fo
        except Exception:
            run_fi = None
    return q, kp, vp, q_off, kvl, table, work, out, run_ours, run_fi


def measure(n_requests: int = 64, launches: int = 6, flashinfer: bool = False) -> dict:
    """Our kernel (and optionally flashinfer's trtllm-gen kernel) on the same
    synthetic paged KV / queries of the configs[1] step."""
    import torch
    from paper_2601_12967_b200 import workload as W
    from paper_2601_12967_b200.attention import attention_flops

    reqs = W.agentic_continuation_batch(n_requests, seed=1)
    q_lens = [r.suffix_len for r in reqs]
    kv_lens = [r.prefix_len + r.suffix_len for r in reqs]
    flops = attention_flops(q_lens, kv_lens, 32)
    q, kp, vp, q_off, kvl, table, work, out, run_ours, run_fi = setup(n_requests, flashinfer)
    if flashinfer and run_fi is None:
        raise RuntimeError("flashinfer trtllm-gen kernel unavailable")

    def timed(fn, n):
        ts = []
        for _ in range(n):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            fn()
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        return ts

    # warm both, then alternate rounds so both kernels see the same clock /
    # power-cap state (short single runs of either are boost-clock biased)
    for fn in (run_ours, run_fi):
        if fn is not None:
            timed(fn, 4)
    ts, fts = [], []
    for _ in range(3):
        ts += timed(run_ours, launches)
        if run_fi is not None:
            fts += timed(run_fi, launches)
    ms = float(np.median(ts))
    fi = None
    if run_fi is not None:
        fms = float(np.median(fts))
        fi = {"kernel": "flashinfer trtllm_batch_context_with_kv_cache (trtllm-gen cubin)", "ms": fms,
              "tflops": flops / fms / 1e9,
              "max_abs_diff_vs_ours": float((run_fi().float() - run_ours().float()).abs().max()),
              "max_abs_out": float(out.float().abs().max())}
    res = {"kernel": "k_continuation_attention", "ms": ms, "tflops": flops / ms / 1e9, "flops": flops,
           "checksum": float(out.float().abs().mean()), "flashinfer": fi}
    del kp, vp, q, out
    torch.cuda.empty_cache()
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--launches", type=int, default=6)
    ap.add_argument("--requests", type=int, default=64)
    ap.add_argument("--flashinfer", action="store_true",
                    help="also time flashinfer's trtllm-gen paged context kernel (library reference point)")
    args = ap.parse_args()
    print(json.dumps(measure(args.requests, args.launches, args.flashinfer)))


if __name__ == "__main__":
    main()
