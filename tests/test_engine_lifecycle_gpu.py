"""The B200 engine's per-call lifecycle (sb_engine_*: submit_call /
submit_partial_prefill / prefill_done (pin_partial or complete_prefill) /
extend_prefill / abandon_partial / finish_decode) replays the reference
Engine's event lists (tests/engine_scripts.py, recorded by oracle/ref_engine.cpp
from the UNMODIFIED engine.cpp) with byte-identical pool dumps after every
event: the paper's overlap scenario (scenarios.cpp:193-240, proven equal to
the orchestrator-driven run in tests/test_engine_scripts.py) and overlapping
partials over a shared system prompt with shared pin counts, abandons before
and after the pin, a pin failure and restored tiers deciding later evictions
(engine.cpp:234-322), under the tiered and the LRU policy."""
import gzip
import json
import os

import pytest

from tests import engine_scripts as S
from tests.engine_replay import replay

GOLD = os.path.join(os.path.dirname(__file__), "golden")


@pytest.mark.gpu
@pytest.mark.parametrize("name", list(S.SCRIPTS))
def test_engine_lifecycle_matches_reference(name):
    from paper_2601_12967_b200.engine import ContinuationEngine, ModelShape

    with gzip.open(os.path.join(GOLD, f"engine_{name}.jsonl.gz"), "rt") as f:
        events = [json.loads(x) for x in f.read().splitlines()]
    script = S.SCRIPTS[name]()
    eng = ContinuationEngine(ModelShape(n_layers=1, n_q_heads=2, n_kv_heads=1, head_dim=128), script.capacity,
                             policy=script.policy)
    n = replay(eng, eng.cache, script, events)
    assert n >= 5
    eng.cache.audit()


@pytest.mark.gpu
def test_engine_lifecycle_errors():
    """StaleHandle / InvalidState as the reference raises them
    (engine.cpp:131-133, 187-197, 226-231, 234-240)."""
    import numpy as np
    from paper_2601_12967_b200 import errors as E
    from paper_2601_12967_b200.engine import ContinuationEngine, ModelShape

    eng = ContinuationEngine(ModelShape(1, 2, 1, 128), 64, policy=1)
    p, t = S.prompt((S.SYS, 40, 5))
    with pytest.raises(E.InvalidState):
        eng.submit_partial_prefill(np.zeros(0, np.uint64), [], now=0)
    with pytest.raises(E.InvalidState):
        eng.submit_call(p, [(0, 10, 3)], 3, now=0)   # tags do not cover the prompt
    c = eng.submit_call(p, t, 3, now=0)
    with pytest.raises(E.StaleHandle):
        eng.extend_prefill(c, p[:3], [(0, 3, 1)], 2, now=1)  # not a partial
    with pytest.raises(E.StaleHandle):
        eng.abandon_partial(c)
    h = eng.submit_partial_prefill(p, t, now=1)
    with pytest.raises(E.InvalidState):
        eng.extend_prefill(h, p[:3], [(0, 3, 1)], 0, now=1)  # decode_length < 1
    assert eng.prefill_done(h, now=2) == eng.PINNED
    eng.abandon_partial(h)
    with pytest.raises(E.StaleHandle):
        eng.abandon_partial(h)
    with pytest.raises(E.StaleHandle):
        eng.extend_prefill(999, p[:3], [(0, 3, 1)], 2, now=1)
    with pytest.raises(E.InvalidState):
        eng.finish_decode(c, p[:1], now=3)  # still queued
    assert eng.prefill_done(c, now=3) == eng.COMPLETED
    eng.finish_decode(c, p[:2], now=4)
    eng.cache.audit()
