"""TEST INFRASTRUCTURE ONLY — a restatement of the reference engine's KV
lifecycle bookkeeping over a KvCache checker (``RefCache``: the reference's
own kv_cache.cpp through oracle/_ref, or ``OracleCache``: the C restatement).

Follows /root/reference/proj/src/engine.cpp line by line:
  submit_call / submit_partial_prefill   :128-182  (admission lookup)
  extend_prefill                         :184-223
  abandon_partial                        :234-248
  pin_partial                            :250-286
  release_partial_pins                   :288-303
  complete_prefill                       :305-322
  finish_decode                          :324-347
without the event loop: the caller says when a call's prefill is done
(``prefill_done``), exactly what the B200 engine's C-ABI exposes.  It is
pinned against the reference Engine itself on scripted runs
(tests/test_engine_scripts.py), then used to check batched engine steps whose
transition order (all calls of a step at one virtual time, one transition
kind after the other) the reference event loop cannot produce.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Dict, List, Optional

import numpy as np

PARTIAL_PREFILL, USER_QUERY, RESPONSE = 4, 2, 0
QUEUED, PREFILLING, AWAITING, DECODING, DONE, ABORTED = range(6)
PINNED, PIN_FAILED, COMPLETED = 1, 2, 3


@dataclass
class _Call:
    partial: bool
    prompt: np.ndarray
    tags: list
    cached: int = 0
    state: int = QUEUED
    ext: bool = False
    chain: List[int] = field(default_factory=list)
    pinned: List[int] = field(default_factory=list)


class EngineOracle:
    def __init__(self, cache, block_size: int = 16):
        self.c = cache
        self.bs = block_size
        self.calls: Dict[int, _Call] = {}
        self.next_id = 1
        self.pin_counts: Dict[int, int] = {}   # engine.hpp:187
        self.real_tags: Dict[int, int] = {}    # engine.hpp:188

    # engine.cpp:128-182
    def submit(self, tokens, tags, now: int, partial: bool) -> int:
        cid = self.next_id
        self.next_id += 1
        t = np.ascontiguousarray(tokens, np.uint64)
        self.calls[cid] = _Call(partial, t, list(tags), cached=self.c.lookup_prefix(t, now))
        return cid

    def cached(self, cid: int) -> int:
        return self.calls[cid].cached

    # engine.cpp:184-223 (the tag shift of :203-205)
    def extend(self, cid: int, suffix, tags, now: int) -> bool:
        call = self.calls[cid]
        p = len(call.prompt)
        call.ext = True
        call.prompt = np.concatenate([call.prompt, np.ascontiguousarray(suffix, np.uint64)])
        call.tags = call.tags + [(b + p, e + p, tg) for b, e, tg in tags]
        if call.state == AWAITING:
            if len(suffix) == 0:
                self.prefill_done(cid, now)
                return True
            call.state = PREFILLING
        return False

    # engine.cpp:234-248
    def abandon(self, cid: int):
        call = self.calls[cid]
        self._release_pins(call)
        if call.chain:
            assert self.c.release(call.chain) == 0
            call.chain = []
        call.state = ABORTED

    # engine.cpp:305-322 with pin_partial (:250-286)
    def prefill_done(self, cid: int, now: int) -> int:
        call = self.calls[cid]
        if call.partial and not call.ext:
            n = len(call.prompt)
            st, ids = self.c.insert(call.prompt, [(0, n, PARTIAL_PREFILL)], now)
            if st == 1:  # CacheFull
                call.state = ABORTED
                return PIN_FAILED
            assert st == 0, st
            call.chain = list(ids)

            def tag_at(pos):  # engine.cpp:267-272
                for b, e, tg in call.tags:
                    if b <= pos < e:
                        return tg
                return USER_QUERY

            for i, bid in enumerate(ids):
                cnt = self.pin_counts.get(bid, 0)
                self.pin_counts[bid] = cnt + 1
                if cnt == 0:
                    cur = self.c.block(bid)[1]["tag"]
                    self.real_tags[bid] = cur if cur != PARTIAL_PREFILL else tag_at(i * self.bs)
                assert self.c.set_reuse_priority([bid], 1, PARTIAL_PREFILL) == 0
            call.pinned = list(ids)
            call.state = AWAITING
            return PINNED
        old = call.chain
        call.chain = []
        st, ids = self.c.insert(call.prompt, call.tags, now)
        if st == 0:
            call.chain = list(ids)
        else:
            assert st == 1, st  # CacheFull: proceed uncached
        if call.pinned:
            self._release_pins(call)
        if old:
            assert self.c.release(old) == 0
        call.state = DECODING
        return COMPLETED

    # engine.cpp:288-303
    def _release_pins(self, call: _Call):
        for bid in call.pinned:
            if bid not in self.pin_counts:
                continue
            self.pin_counts[bid] -= 1
            if self.pin_counts[bid] > 0:
                continue
            del self.pin_counts[bid]
            if self.c.contains(bid):
                assert self.c.set_reuse_priority([bid], 0, -1) == 0
                if bid in self.real_tags:
                    assert self.c.set_tag(bid, self.real_tags[bid]) == 0
            self.real_tags.pop(bid, None)
        call.pinned = []

    # engine.cpp:324-347
    def finish(self, cid: int, response, now: int):
        call = self.calls[cid]
        resp = np.ascontiguousarray(response, np.uint64)
        full = np.concatenate([call.prompt, resp])
        n = len(call.prompt)
        st, ids = self.c.insert(full, list(call.tags) + [(n, n + len(resp), RESPONSE)], now)
        if st == 0:
            assert self.c.release(ids) == 0
        else:
            assert st == 1, st
        if call.chain:
            assert self.c.release(call.chain) == 0
            call.chain = []
        call.state = DONE
