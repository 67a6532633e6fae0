"""Synthetic agentic workloads (host side, numpy).

Token identity follows the reference exactly: a section's tokens are
``splitmix64(section_seed + position)`` with the seed derived from
(tag, content_key, src_iteration) as in src/trace.cpp:50-78, so prefix
sharing behaves as in the reference simulator.

``agentic_continuation_batch`` builds the bench workload of BASELINE.json
configs[1]: 64 concurrent agentic requests with 4-8 tool iterations and a
shared 2K-token system prefix, each caught at the moment its tool outputs
arrive (the continuation prefill of prompt splitting, paper §4.2).
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import List, Tuple

import numpy as np

GOLDEN = np.uint64(0x9E3779B97F4A7C15)
M1 = np.uint64(0xBF58476D1CE4E5B9)
M2 = np.uint64(0x94D049BB133111EB)
SALT = [np.uint64(0x53595354454D5052), np.uint64(0x555345525155455A), np.uint64(0x544F4F4C4F555450),
        np.uint64(0x48495354F52590AA)]
# SectionTag order (trace.hpp:18) -> KvTag (orchestrator.cpp:95-103)
SYS, USER, TOOL, HIST = 0, 1, 2, 3
SECTION_TO_KVTAG = {SYS: 3, USER: 2, TOOL: 1, HIST: 5}


def splitmix64(x):
    x = np.asarray(x, dtype=np.uint64)
    with np.errstate(over="ignore"):
        x = x + GOLDEN
        z = (x ^ (x >> np.uint64(30))) * M1
        z = (z ^ (z >> np.uint64(27))) * M2
    return z ^ (z >> np.uint64(31))


def hash_combine(seed, value):
    seed = np.uint64(seed)
    with np.errstate(over="ignore"):
        mixed = np.uint64(value) + GOLDEN + (seed << np.uint64(6)) + (seed >> np.uint64(2))
    return splitmix64(seed ^ mixed)


def materialize(tag: int, length: int, key: int, src_iter: int = -1) -> np.ndarray:
    seed = splitmix64(np.uint64(key) ^ SALT[tag])
    if tag == TOOL:
        seed = hash_combine(seed, np.uint64(src_iter & 0xFFFFFFFFFFFFFFFF))
    with np.errstate(over="ignore"):
        return splitmix64(np.uint64(seed) + np.arange(length, dtype=np.uint64))


@dataclass
class Section:
    tag: int
    length: int
    key: int
    src_iter: int = -1


def build_prompt(sections: List[Section]) -> Tuple[np.ndarray, List[Tuple[int, int, int]]]:
    toks, tags, pos = [], [], 0
    for s in sections:
        t = materialize(s.tag, s.length, s.key, s.src_iter)
        if s.length:
            toks.append(t)
            tags.append((pos, pos + s.length, SECTION_TO_KVTAG[s.tag]))
            pos += s.length
    return (np.concatenate(toks) if toks else np.zeros(0, np.uint64)), tags


@dataclass
class ContinuationRequest:
    request_id: int
    iterations: int
    iteration: int  # the iteration whose prompt is being extended
    prefix: List[Section]  # tool-independent slice (already prefilled, pinned)
    suffix: List[Section]  # tool outputs of the previous iteration
    prefix_tokens: np.ndarray = field(default=None)
    prefix_tags: list = field(default=None)

    @property
    def prefix_len(self):
        return sum(s.length for s in self.prefix)

    @property
    def suffix_len(self):
        return sum(s.length for s in self.suffix)


SYSTEM_KEY = 0x5157E3


def agentic_continuation_batch(n_requests: int = 64, sys_len: int = 2048, seed: int = 1) -> List[ContinuationRequest]:
    """Deterministic configs[1] workload; all section lengths are multiples of
    16 so the tool-independent prefix ends on a KV-block boundary."""
    reqs = []
    for r in range(n_requests):
        iters = 4 + r % 5                      # 4..8 tool iterations
        it = 1 + (r * 7) % (iters - 1)         # continuation of iteration `it`
        user = Section(USER, 16 * (16 + (r * 37) % 48), 1000 * seed + r)
        hist = Section(HIST, 16 * (32 + (r * 53) % 96), 2000 * seed + r)
        outputs = []
        for i in range(it):
            fan = 1 + (r + i) % 3
            outputs.append([Section(TOOL, 16 * (20 + (r * 11 + i * 7 + j * 5) % 60), 3000 * seed + 97 * r + 7 * i + j, i)
                            for j in range(fan)])
        prefix = [Section(SYS, sys_len, SYSTEM_KEY), user, hist] + [s for o in outputs[:-1] for s in o]
        suffix = outputs[-1]
        req = ContinuationRequest(r, iters, it, prefix, suffix)
        req.prefix_tokens, req.prefix_tags = build_prompt(prefix)
        reqs.append(req)
    return reqs


def fresh_suffix_tokens(req: ContinuationRequest, step: int) -> np.ndarray:
    """New tool outputs for `step` (same lengths, new content), so every timed
    step inserts and evicts real blocks."""
    secs = [Section(s.tag, s.length, s.key ^ (0x9E37 * (step + 1)), s.src_iter) for s in req.suffix]
    return build_prompt(secs)[0]


def long_prefix_continuation_batch(n_requests: int = 8, prefix_min: int = 8192, prefix_max: int = 32768,
                                   suffix_len: int = 1024, sys_len: int = 2048,
                                   seed: int = 1) -> List[ContinuationRequest]:
    """BASELINE.json configs[2]: continuation prefill of `suffix_len` tool-output
    tokens over 8K-32K-token cached prefixes (shared system prompt + history),
    prefix lengths evenly spread and rounded to the 16-token block."""
    reqs = []
    for r in range(n_requests):
        frac = r / max(1, n_requests - 1)
        plen = 16 * int(round((prefix_min + frac * (prefix_max - prefix_min)) / 16))
        prefix = [Section(SYS, sys_len, SYSTEM_KEY), Section(HIST, plen - sys_len, 5000 * seed + r)]
        suffix = [Section(TOOL, suffix_len, 6000 * seed + r, 0)]
        req = ContinuationRequest(r, 2, 1, prefix, suffix)
        req.prefix_tokens, req.prefix_tags = build_prompt(prefix)
        reqs.append(req)
    return reqs
