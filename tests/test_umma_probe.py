"""Hardware check of the tcgen05/TMA operand layouts used by the attention
kernel (tests/cuda/probe_umma.cu) against a torch fp32 reference."""
import ctypes
import os
import subprocess

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
SO = os.path.join(HERE, "cuda", "_build", "libprobe_umma.so")


def build_probe():
    src = os.path.join(HERE, "cuda", "probe_umma.cu")
    if os.path.exists(SO) and os.path.getmtime(SO) >= os.path.getmtime(src):
        return SO
    os.makedirs(os.path.dirname(SO), exist_ok=True)
    subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17", "-shared",
                    "-Xcompiler", "-fPIC", src, "-o", SO], check=True)
    return SO


@pytest.mark.gpu
def test_umma_qk_and_pv_layouts():
    import torch

    lib = ctypes.CDLL(build_probe())
    g = torch.Generator(device="cpu").manual_seed(0)
    q = torch.randn(128, 128, generator=g).to(torch.bfloat16).cuda()
    k = torch.randn(128, 128, generator=g).to(torch.bfloat16).cuda()
    v = torch.randn(128, 128, generator=g).to(torch.bfloat16).cuda()
    s = torch.zeros(128, 128, device="cuda")
    o = torch.zeros(128, 128, device="cuda")
    rc = lib.probe_umma(ctypes.c_void_p(q.data_ptr()), ctypes.c_void_p(k.data_ptr()), ctypes.c_void_p(v.data_ptr()),
                        ctypes.c_void_p(s.data_ptr()), ctypes.c_void_p(o.data_ptr()))
    assert rc == 0
    s_ref = q.float() @ k.float().T
    torch.testing.assert_close(s, s_ref, rtol=1e-3, atol=1e-2)
    p = s_ref.to(torch.bfloat16).float()
    o_ref = p @ v.float()
    torch.testing.assert_close(o, o_ref, rtol=2e-2, atol=2e-1)
