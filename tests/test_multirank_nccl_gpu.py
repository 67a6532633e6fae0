"""The two collectives of the multi-GPU bench over NCCL: the statistics
reduction (bench.reduce_over_ranks) and the gather of per-request trace
metrics (bench.gather_rows).  One GPU allows an NCCL world of one rank only
(NCCL rejects two ranks on one device), so this checks the device, dtype and
backend handling of those calls on NCCL; the world-size-2 semantics are
tests/test_multirank_stats.py (gloo)."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CODE = r"""
import socket, numpy as np, torch, torch.distributed as dist
s = socket.socket(); s.bind(("127.0.0.1", 0)); port = s.getsockname()[1]; s.close()
torch.cuda.set_device(0)
dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1)
assert dist.get_backend() == "nccl"
import bench
mx, sm = bench.reduce_over_ranks([3.5, 7.0, 1.0], device=torch.device("cuda", 0))
assert mx == [3.5, 7.0, 1.0] and sm == [3.5, 7.0, 1.0], (mx, sm)
rows = np.arange(24, dtype=np.float64).reshape(6, 4)
out = bench.gather_rows(rows, 1, dev=torch.device("cuda", 0))
assert out.shape == rows.shape and np.array_equal(out, rows)
dist.destroy_process_group()
print("NCCL_OK")
"""


@pytest.mark.gpu
def test_bench_collectives_over_nccl():
    r = subprocess.run([sys.executable, "-c", CODE], cwd=ROOT, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and "NCCL_OK" in r.stdout, r.stdout[-2000:] + r.stderr[-4000:]
