"""Pins the CPU oracle (oracle/kvcache_oracle.c) against golden vectors produced
by the reference itself (tests/golden, oracle/gen_golden.py).  CPU only."""
import json
import os

import numpy as np
import pytest

from oracle import oracle as O
from tests import oplog

GOLDEN = oplog.GOLDEN


def test_hash_vectors():
    hv = json.load(open(os.path.join(GOLDEN, "hashes.json")))
    assert str(O.root_hash()) == hv["root"]
    for s in hv["sections"]:
        got = O.materialize(s["tag"], s["len"], int(s["key"]), s["src"])
        assert [str(int(x)) for x in got] == s["tokens"]
    for d in hv["decode"]:
        assert str(O.decode_token(int(d["key"]), d["index"])) == d["token"]
    for c in hv["chains"]:
        toks = np.array([int(x) for x in c["tokens"]], dtype=np.uint64)
        assert str(O.chain_hash(int(c["parent"]), toks)) == c["hash"]


@pytest.mark.parametrize("name", oplog.golden_logs())
def test_oracle_replays_reference_oplog(name):
    errs = oplog.replay(oplog.load(name), lambda bs, cap, pol: O.OracleCache(bs, cap, pol))
    assert not errs, "\n".join(errs)


def test_thrashing_scenario_directions():
    man = json.load(open(os.path.join(GOLDEN, "manifest.json")))
    # Fig. 5/7 (scenarios.cpp:98-112): LRU loses R1's context, tiered keeps it.
    assert man["oplog_thrashing_lru.jsonl.gz"]["it2_hits"][0] == 0
    assert man["oplog_thrashing_tiered.jsonl.gz"]["it2_hits"] == [512, 512, 512]


def test_oracle_edge_cases():
    c = O.OracleCache(16, 4, 1)
    assert c.lookup_prefix(np.zeros(0, np.uint64), 0) == 0
    st, ids = c.insert(np.zeros(0, np.uint64), [], 0)
    assert st == 0 and ids == []
    t = O.materialize(0, 33, 5)
    st, ids = c.insert(t, [(0, 33, 3)], 1)
    assert st == 0 and len(ids) == 3  # ceiling division, last block holds 1 token
    assert c.lookup_prefix(t, 2) == 32  # partial block never hits
    st, ids2 = c.insert(t, [(0, 33, 3)], 3)
    assert ids2 == ids  # dedup
    assert c.set_reuse_priority(ids, 1, -1) == 0
    st, _ = c.insert(O.materialize(1, 40, 9), [(0, 40, 0)], 4)
    assert st == 1  # CacheFull: all resident blocks pinned/referenced
    assert c.release([999]) == 2
