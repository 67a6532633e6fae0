"""The B200 trace replay (csrc/replay.cu) against the reference simulator
(oracle/_ref, compiled from /root/reference): identical per-request FTR,
end-to-end time, prefix-hit tokens and eviction totals on the same
generated agent traces, for all three presets and several pool sizes."""
import numpy as np
import pytest

from oracle import oracle as O

SMALL = [320.0, 48.0, 24.0, 48.0, 0.5, 0.3, 0.45, 0.0]
MEDIUM = [2400.0, 300.0, 60.0, 200.0, 0.2, 0.0, 0.0, 0.0]
PRESETS = ["baseline", "baseline_sched", "sutradhara"]


@pytest.mark.gpu
@pytest.mark.parametrize("preset", [0, 1, 2])
@pytest.mark.parametrize("cap,n,gen,workload", [(96, 5, SMALL, None), (4096, 6, SMALL, None),
                                                 (1500, 12, MEDIUM, None), (2500, 8, MEDIUM, "tool_heavy")])
def test_replay_matches_reference(preset, cap, n, gen, workload):
    from paper_2601_12967_b200.replay import replay

    ref = O.ref_run_trace(n, 7, preset, cap, 16, gen=gen, workload=workload)
    got = replay(n, 7, PRESETS[preset], cap, 16, workload=workload or "default", gen=gen)
    assert np.array_equal(got.ftr_ms, ref[0]), (got.ftr_ms, ref[0])
    assert np.array_equal(got.e2e_ms, ref[1])
    assert np.array_equal(got.hit_tokens, ref[2])
    assert np.array_equal(got.prompt_tokens, ref[3])
    assert got.evictions == ref[4]
