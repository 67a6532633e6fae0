"""Engine-boundary scripts for the lifecycle parity tests (test
infrastructure).

A script is a list of actions ``(time, kind, args)`` issued at virtual times
to an engine — the calls the reference orchestrator makes on
``agentsim::Engine`` (orchestrator.cpp:225-259, 383-427).  ``run_reference``
plays a script through the UNMODIFIED reference engine (oracle.RefEngine) and
returns its event list: every action and every engine-internal KV transition
(pin / pin_failed / complete / finish) with the pool dump right after it.
The B200 engine replays the same event list (tests/test_engine_lifecycle_gpu.py).
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import List, Tuple

import numpy as np

from oracle import oracle as O

SYS, USER, TOOL, HIST = 0, 1, 2, 3
KVTAG = {SYS: 3, USER: 2, TOOL: 1, HIST: 5}  # SectionTag -> KvTag (orchestrator.cpp build_prompt)


def prompt(*sections) -> Tuple[np.ndarray, list]:
    """sections: (section_tag, length, content_key[, src_iteration])."""
    toks, tags, pos = [], [], 0
    for s in sections:
        tag, length, key = s[:3]
        src = s[3] if len(s) > 3 else -1
        if length == 0:
            continue
        toks.append(O.materialize(tag, length, key, src))
        tags.append((pos, pos + length, KVTAG[tag]))
        pos += length
    return (np.concatenate(toks) if toks else np.zeros(0, np.uint64)), tags


@dataclass
class Script:
    block_size: int = 16
    capacity: int = 4096
    policy: int = 0
    sched: int = 0
    actions: List[tuple] = field(default_factory=list)  # (t, kind, dict)


def overlap_script() -> Script:
    """scenarios.cpp:193-240 (overlap timeline, split + stream) at the engine
    boundary: R1 iteration 0 is a full call (1536-token system prompt + 512
    user tokens, 30 decode tokens); when its decode completes with the tool
    still running (t=764, after the tool was dispatched at token 10) the
    orchestrator submits iteration 1's tool-independent slice (a new
    2048-token system prompt) as a partial prefill; the tool returns at t=846
    and its 512 output tokens extend the partial before the prefix prefill is
    done.  Times are those of the reference run's timeline; the test checks
    that this script reproduces the orchestrator run's KvCache op log exactly."""
    s = Script(capacity=4096, policy=0)
    p0, t0 = prompt((SYS, 1536, 41), (USER, 512, 42))
    p1, t1 = prompt((SYS, 2048, 44))
    sfx, ts = prompt((TOOL, 512, 43, 0))
    k0, k1 = O.stream_key("R1", 0), O.stream_key("R1", 1)
    s.actions = [(0, "submit_call", dict(name="it0", tokens=p0, tags=t0, decode=30, key=k0)),
                 (764, "submit_partial", dict(name="it1", tokens=p1, tags=t1, key=k1)),
                 (846, "extend", dict(name="it1", tokens=sfx, tags=ts, decode=10))]
    return s


def pin_abandon_script(policy: int = 1, capacity: int = 160) -> Script:
    """Overlapping partial prefills over a shared system prompt, pinned at the
    PARTIAL_PREFILL tier with shared pin counts (engine.cpp:250-286), one
    abandoned while the other still holds the shared blocks (real tags restored
    only for blocks whose count drops to zero, engine.cpp:288-303), an abandon
    before the pin, an extension completing over the pinned prefix
    (engine.cpp:305-322), a pin failure in a pool too small for the prefix
    (CacheFull -> on_pin_failed), and enough later traffic that the restored
    tiers decide the eviction order."""
    s = Script(capacity=capacity, policy=policy)
    sysp = (SYS, 512, 7)
    a, ta = prompt(sysp, (USER, 160, 11), (HIST, 96, 12))
    b, tb = prompt(sysp, (USER, 208, 21))
    c, tc = prompt(sysp, (USER, 64, 31), (HIST, 48, 32))
    d, td = prompt((SYS, 400, 8), (USER, 100, 41))          # never pinned: abandoned while queued
    e, te = prompt((SYS, 2400, 9))                          # larger than the pool: pin fails
    f, tf = prompt((USER, 256, 51), (TOOL, 300, 52, 0))     # later full call, forces evictions
    g, tg = prompt(sysp, (USER, 160, 11), (HIST, 96, 12), (TOOL, 77, 61, 0))  # re-uses A's prefix
    sa, tsa = prompt((TOOL, 90, 71, 0))
    sb, tsb = prompt((TOOL, 33, 72, 0))
    s.actions = [
        (0, "submit_partial", dict(name="A", tokens=a, tags=ta, key=101)),
        (5, "submit_partial", dict(name="B", tokens=b, tags=tb, key=102)),
        (200, "submit_partial", dict(name="C", tokens=c, tags=tc, key=103)),
        (210, "submit_partial", dict(name="D", tokens=d, tags=td, key=104)),
        (211, "abandon", dict(name="D")),
        (400, "abandon", dict(name="A")),
        (420, "extend", dict(name="B", tokens=sb, tags=tsb, decode=3)),
        (430, "submit_partial", dict(name="E", tokens=e, tags=te, key=105)),
        (700, "extend", dict(name="C", tokens=sa, tags=tsa, decode=2)),
        (900, "submit_call", dict(name="F", tokens=f, tags=tf, decode=4, key=106)),
        (1400, "submit_call", dict(name="G", tokens=g, tags=tg, decode=2, key=107)),
    ]
    return s


def run_reference(script: Script, kvlog: bool = False):
    """Plays the script through the reference engine; returns (events, names,
    oplog) where names maps the script's call names to engine call ids."""
    eng = O.RefEngine(script.block_size, script.capacity, script.policy, script.sched, kvlog=kvlog)
    names = {}
    for t, kind, a in script.actions:
        eng.run(t)
        if kind == "submit_call":
            names[a["name"]] = eng.submit_call(a["tokens"], a["tags"], a["decode"], a["key"])
        elif kind == "submit_partial":
            names[a["name"]] = eng.submit_partial(a["tokens"], a["tags"], a["key"])
        elif kind == "extend":
            st = eng.extend(names[a["name"]], a["tokens"], a["tags"], a["decode"])
            assert st == 0, st
        elif kind == "abandon":
            st = eng.abandon(names[a["name"]])
            assert st == 0, st
    eng.run(-1)
    ev = eng.events()
    log = eng.oplog() if kvlog else None
    eng.close()
    return ev, names, log


SCRIPTS = {
    "overlap": overlap_script,
    "pin_abandon_tiered": lambda: pin_abandon_script(policy=1),
    "pin_abandon_lru": lambda: pin_abandon_script(policy=0),
}
