"""Replays a golden KvCache op log (tests/golden/oplog_*.jsonl.gz, produced by
the reference itself — see oracle/gen_golden.py) against any cache object with
the reference's call surface and reports every divergence.

The cache factory receives (block_size, capacity, policy).  Methods used:
lookup_prefix, insert, evict, set_reuse_priority, set_tag, release, touch,
block, dump, audit, total_evicted.  Status codes follow
include/sutradhara_b200.h.
"""
from __future__ import annotations

import base64
import gzip
import json
import os
from typing import Callable, List

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def fnv(s: str) -> str:
    from oracle import oracle as O  # C implementation of FNV-1a (test infrastructure)

    return str(O.fnv1a(s))


def load(name: str) -> List[dict]:
    with gzip.open(os.path.join(GOLDEN, name), "rt") as f:
        return [json.loads(line) for line in f if line.strip()]


def golden_logs(prefix: str = "oplog_") -> List[str]:
    return sorted(n for n in os.listdir(GOLDEN) if n.startswith(prefix) and n.endswith(".jsonl.gz"))


def tokens_of(rec: dict) -> np.ndarray:
    return np.frombuffer(base64.b64decode(rec["tokens"]), dtype=np.uint64).copy()


def replay(ops: List[dict], factory: Callable, check_dump: bool = True, max_errors: int = 5) -> List[str]:
    errs: List[str] = []
    cache = None

    def bad(i, what):
        errs.append(f"op#{i} {ops[i]['op']}: {what}")

    for i, r in enumerate(ops):
        op = r["op"]
        if op == "create":
            cache = factory(r["block_size"], r["capacity"], r["policy"])
            continue
        if op == "lookup":
            got = cache.lookup_prefix(tokens_of(r), r["now"])
            if got != r["ret"]:
                bad(i, f"hit {got} != {r['ret']}")
        elif op == "insert":
            tags = [tuple(t) for t in r["tags"]]
            st, ids = cache.insert(tokens_of(r), tags, r["now"])
            if st != r["status"]:
                bad(i, f"status {st} != {r['status']}")
            elif st == 0 and list(ids) != list(r["ids"]):
                bad(i, f"ids {list(ids)[:8]}.. != {r['ids'][:8]}..")
        elif op == "evict":
            st, ids = cache.evict(r["needed"])
            if list(ids) != list(r["ret"]):
                bad(i, f"evicted {list(ids)[:8]} != {r['ret'][:8]}")
        elif op == "set_priority":
            st = cache.set_reuse_priority(r["ids"], r["pinned"], r["tier"])
            if st != r["status"]:
                bad(i, f"status {st} != {r['status']}")
        elif op == "set_tag":
            st = cache.set_tag(r["id"], r["tag"])
            if st != r["status"]:
                bad(i, f"status {st} != {r['status']}")
        elif op == "release":
            st = cache.release(r["ids"])
            if st != r["status"]:
                bad(i, f"status {st} != {r['status']}")
        elif op == "touch":
            st = cache.touch(r["ids"], r["now"])
            if st != r["status"]:
                bad(i, f"status {st} != {r['status']}")
        elif op == "block":
            st, info = cache.block(r["id"])
            if st != r["status"]:
                bad(i, f"status {st} != {r['status']}")
            elif st == 0:
                for k in ("tag", "tier", "ref", "pinned", "ntok", "last"):
                    if info[k] != r[k]:
                        bad(i, f"{k} {info[k]} != {r[k]}")
                if str(info["chain"]) != r["chain"] or str(info["parent"]) != r["parent"]:
                    bad(i, "chain/parent hash mismatch")
            continue
        elif op == "audit":
            st = cache.audit()
            if st != r["status"]:
                bad(i, f"audit {st} != {r['status']}")
            continue
        elif op == "final":
            d = cache.dump()
            if d != r["dump"]:
                bad(i, "final dump differs")
            if cache.total_evicted() != r["total_evicted"]:
                bad(i, f"total_evicted {cache.total_evicted()} != {r['total_evicted']}")
            continue
        if check_dump and "dump_fnv" in r:
            if fnv(cache.dump()) != r["dump_fnv"]:
                bad(i, "cache state (dump digest) differs")
        if len(errs) >= max_errors:
            break
    if cache is not None and hasattr(cache, "close"):
        cache.close()
    return errs


class StatusAdapter:
    """Wraps the product's exception-raising KvCache into the status-code call
    surface the op-log replayer uses."""

    def __init__(self, cache):
        self.c = cache

    def _st(self, fn, *a):
        from paper_2601_12967_b200 import errors

        try:
            return 0, fn(*a)
        except Exception as e:  # map back to the C-ABI status codes
            for cls, code in errors.STATUS_OF.items():
                if type(e) is cls:
                    return code, None
            raise

    def lookup_prefix(self, t, now):
        return self.c.lookup_prefix(t, now)

    def insert(self, t, tags, now):
        st, ids = self._st(self.c.insert, t, tags, now)
        return st, ids or []

    def evict(self, needed):
        st, ids = self._st(self.c.evict, needed)
        return st, ids or []

    def set_reuse_priority(self, ids, pinned, tier):
        return self._st(self.c.set_reuse_priority, ids, None if pinned < 0 else bool(pinned),
                        None if tier < 0 else tier)[0]

    def set_tag(self, bid, tag):
        return self._st(self.c.set_tag, bid, tag)[0]

    def release(self, ids):
        return self._st(self.c.release, ids)[0]

    def touch(self, ids, now):
        return self._st(self.c.touch, ids, now)[0]

    def block(self, bid):
        st, b = self._st(self.c.block, bid)
        if st:
            return st, None
        return 0, dict(tag=b.tag, tier=b.tier, ref=b.ref_count, pinned=int(b.pinned), ntok=len(b.tokens),
                       last=b.last_used, chain=b.chain_hash, parent=b.parent_hash, tokens=b.tokens)

    def dump(self):
        return self.c.dump()

    def audit(self):
        return self._st(self.c.audit)[0]

    def total_evicted(self):
        return self.c.total_evicted()

    def close(self):
        self.c.close()
