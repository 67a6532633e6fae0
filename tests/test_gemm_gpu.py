"""GPU numerics of the projections' GEMM (csrc/gemm.cu: tcgen05 + TMA,
persistent, fused epilogues) through the C-ABI `sb_gemm_bf16`, against a
torch fp32 matmul of the same bf16 operands.

Tolerance: max |Y - Y_ref| <= 1e-2 * max |Y_ref| (max-norm relative, no
absolute floor) for the bf16 outputs; 1e-5 relative for the fp32 output
(fp32 accumulation in both, only the summation order differs).  Shapes cover
ragged rows (not a multiple of the 128-row tile), n not a multiple of the
256-column tile, k not a multiple of the 64-wide stage, more tiles than SMs
(the persistent loop and both TMEM accumulators), and the configs[2]
Llama-3-8B projection shapes (QKV 6144 x 4096, O 4096 x 4096, gate/up 2 x
14336 x 4096, down 4096 x 14336, LM head 128256 x 4096)."""
import ctypes as C

import pytest

pytestmark = pytest.mark.gpu

STORE, ADD, F32, SWIGLU = 0, 1, 2, 3


def _gemm(x, w, y, rows, n, k, mode):
    import torch

    from paper_2601_12967_b200 import _lib

    L = _lib.lib()
    st = torch.cuda.current_stream().cuda_stream
    _lib.check(L.sb_gemm_bf16(C.c_void_p(x.data_ptr()), C.c_void_p(w.data_ptr()), C.c_void_p(y.data_ptr()), rows, n,
                              k, mode, C.c_void_p(st)), "sb_gemm_bf16")
    torch.cuda.synchronize()


def _operands(rows, n, k, seed, w_rows=None):
    import torch

    g = torch.Generator(device="cuda").manual_seed(seed)
    x = (torch.randn(rows, k, device="cuda", generator=g) * 0.5).to(torch.bfloat16)
    w = (torch.randn(w_rows or n, k, device="cuda", generator=g) / k ** 0.5).to(torch.bfloat16)
    return x, w


def _rel(y, ref):
    return ((y.float() - ref).abs().max() / ref.abs().max()).item()


@pytest.mark.parametrize("rows,n,k", [(1, 8, 8), (37, 1000, 512), (128, 256, 64), (300, 520, 200), (1024, 3072, 1024),
                                      (2000, 6144, 4096)])
def test_store_bf16(rows, n, k):
    import torch

    x, w = _operands(rows, n, k, 1)
    y = torch.full((rows, n), float("nan"), device="cuda", dtype=torch.bfloat16)
    _gemm(x, w, y, rows, n, k, STORE)
    ref = x.float() @ w.float().T
    assert torch.isfinite(y.float()).all()
    err = _rel(y, ref)
    assert err <= 1e-2, err


@pytest.mark.parametrize("rows,n,k", [(37, 512, 512), (777, 4096, 4096), (300, 4096, 14336)])
def test_residual_add(rows, n, k):
    import torch

    x, w = _operands(rows, n, k, 2)
    y0 = torch.randn(rows, n, device="cuda").to(torch.bfloat16)
    y = y0.clone()
    _gemm(x, w, y, rows, n, k, ADD)
    ref = y0.float() + x.float() @ w.float().T
    err = _rel(y, ref)
    assert err <= 1e-2, err


@pytest.mark.parametrize("rows,n,k", [(1, 1000, 512), (64, 128256, 4096), (130, 776, 96)])
def test_store_f32(rows, n, k):
    import torch

    x, w = _operands(rows, n, k, 3)
    y = torch.full((rows, n), float("nan"), device="cuda", dtype=torch.float32)
    _gemm(x, w, y, rows, n, k, F32)
    ref = x.double() @ w.double().T
    assert torch.isfinite(y).all()
    err = ((y.double() - ref).abs().max() / ref.abs().max()).item()
    assert err <= 1e-5, err


@pytest.mark.parametrize("rows,dff,k", [(5, 1024, 512), (333, 1000, 256), (1500, 14336, 4096)])
def test_swiglu(rows, dff, k):
    import torch
    import torch.nn.functional as F

    x, w = _operands(rows, dff, k, 4, w_rows=2 * dff)
    y = torch.full((rows, dff), float("nan"), device="cuda", dtype=torch.bfloat16)
    _gemm(x, w, y, rows, dff, k, SWIGLU)
    gu = x.float() @ w.float().T
    ref = F.silu(gu[:, :dff]) * gu[:, dff:]
    assert torch.isfinite(y.float()).all()
    err = _rel(y, ref)
    assert err <= 1e-2, err


def test_columns_beyond_n_untouched():
    """The epilogue masks rows >= rows and columns >= n: a guard band around
    the output keeps its sentinel."""
    import torch

    rows, n, k = 100, 264, 128
    x, w = _operands(rows, n, k, 5)
    out = torch.full((rows * n + 4096,), 7.0, device="cuda", dtype=torch.bfloat16)
    _gemm(x, w, out, rows, n, k, STORE)
    assert (out[rows * n:] == 7.0).all()
    ref = x.float() @ w.float().T
    assert _rel(out[:rows * n].view(rows, n), ref) <= 1e-2


def test_unsupported_shape_is_an_error():
    import torch

    from paper_2601_12967_b200 import _lib, errors

    x, w = _operands(16, 16, 16, 6)
    y = torch.empty(16, 16, device="cuda", dtype=torch.bfloat16)
    with pytest.raises(errors.Unsupported):
        _gemm(x, w, y, 16, 16, 12, STORE)  # k not a multiple of 8
    with pytest.raises(ValueError):
        _gemm(x, w, y, 16, 16, 16, 9)  # unknown mode
    y2 = torch.empty(16 * 16 + 1, device="cuda", dtype=torch.bfloat16)[1:]  # 2-byte offset
    with pytest.raises(errors.Unsupported):
        _gemm(x, w, y2, 16, 16, 16, STORE)
    del _lib


def test_one_cta_kernel_at_every_shape():
    """Rows above 128 run on the CTA-pair kernel; the same tests with
    SB_GEMM_PAIR=0 put every shape through the 1-CTA kernel."""
    import os
    import subprocess
    import sys

    env = dict(os.environ, SB_GEMM_PAIR="0")
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", os.path.abspath(__file__), "-k",
                        "not one_cta_kernel"], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
