"""GPU parity of the batched engine step (engine.py ContinuationBatch, one op
program per transition) with the reference engine's KV lifecycle, restated by
oracle/engine_oracle.py (pinned against the reference Engine itself in
tests/test_engine_scripts.py) over the reference's own KvCache (oracle/_ref)
when built, else the C restatement.

One step = n new agentic calls at `now`: admission lookups of the prefixes,
pin_partial, extend with fresh tool outputs, complete_prefill (hint-aware
eviction under pool pressure), finish_decode with one response token.
Checked after every step: lookup hits, pin outcomes, complete statuses, the
chains the continuation attended over, the full audit dump and the eviction
count."""
import os

import numpy as np
import pytest

from oracle import oracle as O
from oracle.engine_oracle import EngineOracle


def _cache(bs, cap, policy):
    if os.path.exists(os.path.join(O.REF_DIR, "libagentsim_ref.so")):
        return O.RefCache(bs, cap, policy)
    return O.OracleCache(bs, cap, policy)


def run_and_check(eng, reqs, cap, policy, steps, sys_len, now0=10, keys=None):
    import torch
    from paper_2601_12967_b200 import workload as W

    n = len(reqs)
    keys = keys if keys is not None else [1000 + i for i in range(n)]
    batch = eng.make_batch([r.prefix_tokens for r in reqs], [r.prefix_tags for r in reqs],
                           [r.suffix_len for r in reqs], stream_keys=keys)
    oc = _cache(16, cap, policy)
    eo = EngineOracle(oc, 16)
    for step in range(steps):
        now = now0 + step
        sfx = [W.fresh_suffix_tokens(r, step) for r in reqs]
        batch.stage_suffix_device(torch.from_numpy(np.concatenate(sfx).view(np.int64)).cuda())
        batch.run(now, seed=step)
        torch.cuda.synchronize()
        calls = [eo.submit(r.prefix_tokens, r.prefix_tags, now, partial=True) for r in reqs]
        exp_hits = [eo.cached(c) for c in calls]
        exp_pin = [eo.prefill_done(c, now) for c in calls]
        for c, r, s in zip(calls, reqs, sfx):
            eo.extend(c, s, [(0, len(s), 1)], now)
        for c in calls:
            assert eo.prefill_done(c, now) == 3
        exp_chain = [list(eo.calls[c].chain) for c in calls]
        for i, c in enumerate(calls):
            eo.finish(c, np.array([O.decode_token(keys[i], 0)], np.uint64), now)
        hits, status, got = batch.results()
        assert hits.tolist() == exp_hits, step
        assert batch.pin_outcomes().tolist() == exp_pin, step
        assert (status == 0).all(), step
        for i, ids in enumerate(exp_chain):
            a, b = batch.blk_off_h[i], batch.blk_off_h[i + 1]
            assert got[a:b].tolist() == ids, (step, i)
        assert eng.cache.dump() == oc.dump(), step
        assert eng.cache.total_evicted() == oc.total_evicted(), step
    eng.cache.audit()
    return batch


@pytest.mark.gpu
@pytest.mark.parametrize("n_req,slack,policy", [(6, 1.25, 1), (12, 1.0, 1), (12, 1.0, 0)])
def test_engine_steps_match_oracle(n_req, slack, policy):
    from paper_2601_12967_b200 import workload as W
    from paper_2601_12967_b200.engine import ContinuationEngine, ModelShape

    reqs = W.agentic_continuation_batch(n_req, sys_len=256, seed=3)
    bs = 16
    pre = sum(r.prefix_len // bs for r in reqs) - (n_req - 1) * (256 // bs)
    suf = sum((r.suffix_len + bs - 1) // bs for r in reqs) + n_req
    cap = pre + int(slack * suf) + 1
    eng = ContinuationEngine(ModelShape(n_layers=2, n_q_heads=8, n_kv_heads=2, head_dim=128), cap, policy=policy)
    run_and_check(eng, reqs, cap, policy, steps=4, sys_len=256)


@pytest.mark.gpu
def test_engine_steps_match_reference_at_bench_shape():
    """The configs[1] bench step itself: bench.py's 64 requests, its
    capacity_for() pool (27K blocks, ~5.5K evictions per step), 3 steps,
    checked against the reference's own KvCache (oracle/_ref) under the
    engine lifecycle after every step."""
    import bench
    from paper_2601_12967_b200.engine import ContinuationEngine, ModelShape

    reqs = bench.setup_workload(0, 64)
    _, _, cap = bench.capacity_for(reqs)
    eng = ContinuationEngine(ModelShape(n_layers=1, n_q_heads=8, n_kv_heads=2, head_dim=128), cap, policy=1)
    run_and_check(eng, reqs, cap, 1, steps=3, sys_len=2048)
    assert eng.cache.total_evicted() > 5000
    st = eng.cache.program_stats()  # the batched programs ran on the parallel path (pool_batch.cuh)
    assert st["parallel"] >= 2 * 3, st
