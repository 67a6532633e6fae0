"""GPU parity of the batched continuation-prefill step (engine.py) with the
reference semantics: per step, the batched admission lookups must return the
oracle's hit lengths, the batched inserts the oracle's block ids (in batch
order, sequential semantics), and the pool's audit dump must equal the
oracle's after every step — under pool pressure with evictions."""
import numpy as np
import pytest

from oracle import oracle as O


def _workload(n):
    from paper_2601_12967_b200 import workload as W

    return W.agentic_continuation_batch(n, sys_len=256, seed=3)


@pytest.mark.gpu
@pytest.mark.parametrize("n_req,slack", [(6, 1.25), (12, 0.6)])
def test_engine_steps_match_oracle(n_req, slack):
    import torch
    from paper_2601_12967_b200 import workload as W
    from paper_2601_12967_b200.engine import ContinuationEngine, ModelShape

    reqs = _workload(n_req)
    bs = 16
    pre = sum(r.prefix_len // bs for r in reqs) - (n_req - 1) * (256 // bs)
    suf = sum((r.suffix_len + bs - 1) // bs for r in reqs)
    cap = pre + int(slack * suf) + 1
    shape = ModelShape(n_layers=2, n_q_heads=8, n_kv_heads=2, head_dim=128)
    eng = ContinuationEngine(shape, cap, policy=1)
    oc = O.OracleCache(bs, cap, 1)
    handles = []
    for r in reqs:
        handles.append(eng.submit_partial_prefill(r.prefix_tokens, r.prefix_tags, now=0))
        st, ids = oc.insert(r.prefix_tokens, r.prefix_tags, 0)
        assert st == 0 and ids == handles[-1].block_ids
        assert oc.set_reuse_priority(ids, 1, 4) == 0
    assert eng.cache.dump() == oc.dump()
    batch = eng.make_batch(handles, [r.suffix_len for r in reqs])
    for step in range(4):
        now = 10 + step
        suffix = np.concatenate([W.fresh_suffix_tokens(r, step) for r in reqs]).view(np.int64)
        batch.stage_suffix_device(torch.from_numpy(suffix).cuda())
        batch.run(now, seed=step)
        torch.cuda.synchronize()
        exp_hits, exp_ids, exp_st = [], [], []
        prompts = []
        for r in reqs:
            toks = np.concatenate([r.prefix_tokens, W.fresh_suffix_tokens(r, step)])
            prompts.append(toks)
            exp_hits.append(oc.lookup_prefix(toks, now))
        for r, toks in zip(reqs, prompts):
            st, ids = oc.insert(toks, list(r.prefix_tags) + [(r.prefix_len, len(toks), 1)], now)
            exp_st.append(st)
            exp_ids.append(ids)
        for st, ids in zip(exp_st, exp_ids):
            if st == 0:
                assert oc.release(ids) == 0
        hits, status, got = batch.results()
        assert hits.tolist() == exp_hits, step
        assert status.tolist() == exp_st, step
        for i, ids in enumerate(exp_ids):
            if exp_st[i] == 0:
                a, b = batch.blk_off_h[i], batch.blk_off_h[i + 1]
                assert got[a:b].tolist() == ids, (step, i)
        assert eng.cache.dump() == oc.dump(), step
        assert eng.cache.total_evicted() == oc.total_evicted(), step
    eng.cache.audit()
