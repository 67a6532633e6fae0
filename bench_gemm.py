"""Projection GEMM timing (csrc/gemm.cu vs cuBLAS through torch) at the
configs[2] Llama-3-8B shapes: QKV, O (+residual), gate/up (+SwiGLU), down
(+residual) for `rows` suffix tokens, and the LM head over 64 last tokens.
CUDA events on the launching stream, L2 flushed between launches, median of
`--iters`.  One JSON line per shape: ours / cuBLAS µs and TFLOP/s (SwiGLU
counts the 2n-column GEMM; cuBLAS's line adds the separate SwiGLU kernel
only when --with-elementwise)."""
import argparse
import ctypes as C
import json

import torch
import torch.nn.functional as F

from paper_2601_12967_b200 import _lib


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rows", type=int, default=8192)
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--only", default="", help="comma-separated shape names")
    ap.add_argument("--ours-only", action="store_true")
    a = ap.parse_args()
    L = _lib.lib()
    st = torch.cuda.current_stream()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    T = a.rows
    shapes = [("qkv", T, 6144, 4096, 0), ("o+res", T, 4096, 4096, 1), ("gate_up+swiglu", T, 14336, 4096, 3),
              ("down+res", T, 4096, 14336, 1), ("lm_head", 64, 128256, 4096, 2)]
    for name, rows, n, k, mode in shapes:
        if a.only and name not in a.only.split(","):
            continue
        wr = 2 * n if mode == 3 else n
        x = (torch.randn(rows, k, device="cuda") * 0.5).to(torch.bfloat16)
        w = (torch.randn(wr, k, device="cuda") / k ** 0.5).to(torch.bfloat16)
        y = torch.zeros(rows, n, device="cuda", dtype=torch.float32 if mode == 2 else torch.bfloat16)
        gu = torch.empty(rows, wr, device="cuda", dtype=torch.bfloat16)

        def ours():
            _lib.check(L.sb_gemm_bf16(C.c_void_p(x.data_ptr()), C.c_void_p(w.data_ptr()), C.c_void_p(y.data_ptr()),
                                      rows, n, k, mode, C.c_void_p(st.cuda_stream)))

        def blas():
            if mode == 3:
                torch.matmul(x, w.T, out=gu)
                F.silu(gu[:, :n]) * gu[:, n:]
            elif mode == 1:
                y.addmm_(x, w.T)
            elif mode == 2:
                torch.matmul(x, w.T).float()
            else:
                torch.matmul(x, w.T, out=y)

        res = {}
        for tag, fn in (("ours", ours),) + ((("cublas", blas),) if not a.ours_only else ()):
            for _ in range(3):
                fn()
            ts = []
            for _ in range(a.iters):
                flush.zero_()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                fn()
                e1.record()
                e1.synchronize()
                ts.append(e0.elapsed_time(e1) * 1e3)
            ts.sort()
            us = ts[len(ts) // 2]
            res[tag] = {"us": round(us, 2), "tflops": round(2.0 * rows * wr * k / (us * 1e-6) / 1e12, 1)}
        if "cublas" in res:
            res["speedup"] = round(res["cublas"]["us"] / res["ours"]["us"], 3)
        print(json.dumps({"shape": name, "rows": rows, "n": n, "k": k, **res}), flush=True)


if __name__ == "__main__":
    main()
