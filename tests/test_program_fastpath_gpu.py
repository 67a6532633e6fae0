"""The op programs' parallel path (csrc/pool_batch.cuh) decides and applies a
whole program of engine ops across the GPU when it can prove the result
equals the sequential program's; otherwise the one-CTA program runs.  Both
must give identical results on every workload: tests/fastpath_diff.py is run
with the parallel path off (SB_PROG_FAST=0) and on, and every observable
(hits, pin outcomes, statuses, chains, the full pool dump after every step /
op, evictions) must agree.  The parallel path must actually be taken on the
engine's batched steps (tests/test_engine_gpu.py checks the same steps
against the reference itself)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(fast: str) -> dict:
    env = dict(os.environ, SB_PROG_FAST=fast)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "fastpath_diff.py")], env=env,
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    return json.loads(r.stdout.strip().splitlines()[-1])


@pytest.mark.gpu
def test_parallel_program_path_equals_sequential():
    seq = _run("0")
    par = _run("1")
    for k in ("configs1", "ragged", "percall", "inserts", "single"):
        assert len(seq[k]) == len(par[k])
        for i, (a, b) in enumerate(zip(seq[k], par[k])):
            assert a == b, (k, i)
    # the sequential run never takes the parallel path; the parallel run does,
    # on every configs[1]-style batch whose pool holds a step (slack >= 1:
    # the 0.6 / 0.8 pools run into CacheFull, which only the program handles)
    assert all(s["parallel"] == 0 for s in seq["stats"]["configs1"])
    for i in (0, 1, 3):
        s = par["stats"]["configs1"][i]
        assert s["parallel"] >= s["programs"] - 2, par["stats"]
    taken = sum(s["parallel"] for g in par["stats"].values() for s in g)
    total = sum(s["programs"] for g in par["stats"].values() for s in g)
    assert taken > 0.3 * total, (taken, total)
