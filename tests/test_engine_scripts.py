"""CPU checks of the engine-lifecycle parity infrastructure (no GPU):

* the scripted overlap scenario reproduces the reference orchestrator's run
  of scenarios.cpp:193-240 at the KvCache boundary (identical op log and
  dump digests), so replaying the script IS replaying the scenario;
* the EngineOracle restatement (oracle/engine_oracle.py) replays every
  script's reference event list with byte-identical pool dumps — it is
  pinned against the reference engine before it checks batched steps;
* the event lists equal the committed golden fixtures (tests/golden/engine_*),
  which is what the GPU tests replay when the reference library is absent.
"""
import gzip
import json
import os

import pytest

from oracle import oracle as O
from oracle.engine_oracle import EngineOracle
from tests import engine_scripts as S
from tests.engine_replay import OracleSurface, replay

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _ref_available():
    return os.path.exists(os.path.join(O.REF_DIR, "libagentsim_ref.so"))


needs_ref = pytest.mark.skipif(not _ref_available(), reason="oracle/_ref not built")


@needs_ref
def test_overlap_script_is_the_reference_scenario():
    _, _, log = S.run_reference(S.overlap_script(), kvlog=True)
    _, ftr, olog = O.ref_overlap_scenario(True, kvlog=True)

    def ops(text):
        rows = [json.loads(x) for x in text.splitlines()]
        return [(r["op"], r.get("now"), r.get("dump_fnv"), r.get("status")) for r in rows if r["op"] != "audit"]

    assert ops(log) == ops(olog)
    assert ftr > 0


@needs_ref
@pytest.mark.parametrize("name", list(S.SCRIPTS))
def test_engine_oracle_replays_reference_events(name):
    script = S.SCRIPTS[name]()
    events, _, _ = S.run_reference(script)
    cache = O.RefCache(script.block_size, script.capacity, script.policy)
    n = replay(OracleSurface(EngineOracle(cache, script.block_size), cache), cache, script, events)
    assert n >= 5


@needs_ref
@pytest.mark.parametrize("name", list(S.SCRIPTS))
def test_golden_engine_events_current(name):
    with gzip.open(os.path.join(GOLD, f"engine_{name}.jsonl.gz"), "rt") as f:
        gold = [json.loads(x) for x in f.read().splitlines()]
    events, _, _ = S.run_reference(S.SCRIPTS[name]())
    assert events == gold


@pytest.mark.parametrize("name", list(S.SCRIPTS))
def test_engine_oracle_replays_golden_events(name):
    """Without the reference library: the C restatement under the same engine
    bookkeeping reproduces the committed golden dumps."""
    with gzip.open(os.path.join(GOLD, f"engine_{name}.jsonl.gz"), "rt") as f:
        gold = [json.loads(x) for x in f.read().splitlines()]
    script = S.SCRIPTS[name]()
    cache = O.OracleCache(script.block_size, script.capacity, script.policy)
    assert replay(OracleSurface(EngineOracle(cache, script.block_size), cache), cache, script, gold) >= 5
