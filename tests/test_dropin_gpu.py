"""Drop-in check: the UNMODIFIED reference engine + orchestrator (compiled from
/root/reference into oracle/_ref) replays agent traces with its KvCache served
by the B200 block pool (integration/agentsim_kvcache_b200.cpp over the C-ABI).
Every per-request FTR, end-to-end latency, hit count and the eviction total
must equal the pure reference run — the pool changes where the cache lives,
not one decision."""
import ctypes as C
import os

import numpy as np
import pytest

from oracle import oracle as O

SMALL = [320.0, 48.0, 24.0, 48.0, 0.5, 0.3, 0.45, 0.0]
MEDIUM = [2400.0, 300.0, 60.0, 200.0, 0.2, 0.0, 0.0, 0.0]


def _have_b200_lib():
    return os.path.exists(os.path.join(O.REF_DIR, "libagentsim_b200.so"))


@pytest.mark.gpu
@pytest.mark.skipif(not _have_b200_lib(), reason="oracle/_ref/libagentsim_b200.so not built")
@pytest.mark.parametrize("preset", [0, 1, 2])
@pytest.mark.parametrize("cap,n,gen", [(96, 5, SMALL), (4096, 5, SMALL), (1500, 12, MEDIUM)])
def test_reference_engine_on_b200_pool_is_identical(preset, cap, n, gen):
    ref = O.ref_run_trace(n, 7, preset, cap, 16, gen=gen)
    got = O.ref_run_trace(n, 7, preset, cap, 16, gen=gen, b200=True)
    for k, name in enumerate(["ftr", "e2e", "hit_tokens", "prompt_tokens"]):
        assert np.array_equal(ref[k], got[k]), (name, ref[k], got[k])
    assert ref[4] == got[4], ("evictions", ref[4], got[4])


@pytest.mark.gpu
@pytest.mark.skipif(not _have_b200_lib(), reason="oracle/_ref/libagentsim_b200.so not built")
def test_paper_scenarios_pass_on_b200_pool():
    buf = C.create_string_buffer(1 << 16)
    assert O.b200_lib().refrun_scenarios(buf, len(buf)) == 1, buf.value.decode()
    hits = np.zeros(3, np.int64)
    for tiered, expect0 in ((0, 0), (1, 512)):
        assert O.b200_lib().refrun_thrashing(tiered, hits.ctypes.data_as(O.I64P)) == 0
        assert hits[0] == expect0


@pytest.mark.gpu
def test_bench_trace_shard_on_b200_pool_is_identical():
    """The bench's configs[3] generator (trace_gen default workload, seed 1,
    an 8192-block pool) through the drop-in library the bench uses
    (integration/_build/libagentsim_b200.so via dropin.py) vs the pure
    reference simulator: every request's FTR, hits and the eviction total.
    (Long enough that the binding's residency mirror, fed by
    sb_kv_last_evicted after every insert, decides admissions.)"""
    from paper_2601_12967_b200 import dropin as D

    ref_lib = os.path.join(O.REF_DIR, "libagentsim_ref.so")
    if not os.path.exists(ref_lib):
        pytest.skip("oracle/_ref not built")
    for preset in ("sutradhara", "baseline"):
        ref = D.run_shard(32, 1, preset, 8192, shard=0, n_shards=1, lib_path=ref_lib)
        got = D.run_shard(32, 1, preset, 8192, shard=0, n_shards=1)
        assert np.array_equal(ref.ftr_ms, got.ftr_ms), preset
        assert np.array_equal(ref.hit_tokens, got.hit_tokens), preset
        assert ref.evictions == got.evictions, (preset, ref.evictions, got.evictions)
