"""Replays a reference engine event list (tests/engine_scripts.py) through an
engine with the B200 engine's call surface — the product ContinuationEngine
or the CPU EngineOracle — comparing the pool dump after every event that
carries one (test infrastructure)."""
from __future__ import annotations

import numpy as np

from oracle import oracle as O


class OracleSurface:
    """EngineOracle behind the ContinuationEngine method names."""

    def __init__(self, eo, cache):
        self.eo, self.cache = eo, cache

    def submit_call(self, tokens, tags, decode_length, now):
        return self.eo.submit(tokens, tags, now, partial=False)

    def submit_partial_prefill(self, tokens, tags, now):
        return self.eo.submit(tokens, tags, now, partial=True)

    def cached_at_submit(self, cid):
        return self.eo.cached(cid)

    def prefill_done(self, cid, now):
        return self.eo.prefill_done(cid, now)

    def extend_prefill(self, cid, suffix, tags, decode_length, now):
        return self.eo.extend(cid, suffix, tags, now)

    def abandon_partial(self, cid):
        self.eo.abandon(cid)

    def finish_decode(self, cid, response, now):
        self.eo.finish(cid, response, now)


def replay(engine, cache, script, events):
    """engine: ContinuationEngine-like; cache: its pool (has .dump()).
    Returns the number of dumps compared."""
    actions = iter(script.actions)
    ids = {}          # reference call id -> engine call id
    keys = {}         # reference call id -> decode stream key
    done_at_extend = set()
    compared = 0
    for ev in events:
        kind, rc, t = ev["ev"], ev["call"], ev["t"]
        if kind in ("submit_call", "submit_partial", "extend", "abandon"):
            at, akind, a = next(actions)
            assert akind == kind and at == t, (akind, kind, at, t)
            if kind == "submit_call":
                ids[rc] = engine.submit_call(a["tokens"], a["tags"], a["decode"], now=t)
                keys[rc] = a["key"]
            elif kind == "submit_partial":
                ids[rc] = engine.submit_partial_prefill(a["tokens"], a["tags"], now=t)
                keys[rc] = a["key"]
            elif kind == "extend":
                if engine.extend_prefill(ids[rc], a["tokens"], a["tags"], a["decode"], now=t):
                    done_at_extend.add(rc)
            else:
                engine.abandon_partial(ids[rc])
            if "cached" in ev:
                assert engine.cached_at_submit(ids[rc]) == ev["cached"], (ev, engine.cached_at_submit(ids[rc]))
        elif kind in ("pin", "pin_failed"):
            out = engine.prefill_done(ids[rc], now=t)
            assert out == (1 if kind == "pin" else 2), (kind, out)
        elif kind == "complete":
            if rc in done_at_extend:
                done_at_extend.discard(rc)
            else:
                assert engine.prefill_done(ids[rc], now=t) == 3
        elif kind == "finish":
            resp = np.array([O.decode_token(keys[rc], i) for i in range(ev["emitted"])], np.uint64)
            engine.finish_decode(ids[rc], resp, now=t)
        else:
            raise AssertionError(kind)
        if ev.get("dump") is not None:
            got = cache.dump()
            assert got == ev["dump"], f"dump differs after {kind} of call {rc} at t={t}"
            compared += 1
    return compared
