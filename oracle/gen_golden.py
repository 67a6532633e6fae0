"""TEST INFRASTRUCTURE ONLY — generates tests/golden/ from the reference itself.

Run in the build container (needs oracle/_ref, built from /root/reference by
``make -C oracle ref``):

    python oracle/gen_golden.py

Fixtures written (all produced by the UNMODIFIED reference code):

* ``oplog_*.jsonl.gz`` — every KvCache call the reference engine/orchestrator
  makes while replaying a trace (recorded by oracle/ref_kvlog.cpp): inputs,
  return values, status and an FNV-1a digest of the cache's audit dump after
  the call.  Sources: the paper's thrashing scenario (scenarios.cpp:45-85)
  under LRU and tiered eviction, and small generated agent traces under the
  three presets (runner.cpp:120-135).
* ``oplog_fuzz_*.jsonl.gz`` — seeded random op sequences (insert / lookup /
  evict / release / set_priority / set_tag / touch incl. error paths:
  CacheFull, UnknownBlock, ZeroRefRelease, bad tag ranges, partial blocks)
  applied to the reference KvCache through oracle/ref_capi.cpp.
* ``hashes.json`` — materialize_tokens / decode_token / kv_chain_hash vectors.
* ``runs.json`` — per-request FTR / hit tokens of small reference replays.
"""
from __future__ import annotations

import base64
import gzip
import json
import os
import random
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path[0] = os.path.dirname(HERE)
from oracle import oracle as O  # noqa: E402

OUT = os.path.join(os.path.dirname(HERE), "tests", "golden")

# small-prompt generator overrides: [prompt_median, tool_out_median,
# decode_inter_median, decode_final_median, qps, depth_p, fanout_p, ratio_scale]
SMALL_GEN = [320.0, 48.0, 24.0, 48.0, 0.5, 0.3, 0.45, 0.0]


def fnv(s: str) -> str:
    h = 0xCBF29CE484222325
    for ch in s.encode():
        h ^= ch
        h = (h * 0x100000001B3) & 0xFFFFFFFFFFFFFFFF
    return str(h)


def write_gz(name: str, text: str):
    with gzip.open(os.path.join(OUT, name), "wt") as f:
        f.write(text)


def b64(tokens: np.ndarray) -> str:
    return base64.b64encode(np.ascontiguousarray(tokens, np.uint64).tobytes()).decode()


def fuzz_log(seed: int, block_size: int, capacity: int, policy: int, n_ops: int) -> str:
    """Random op sequence on the reference KvCache (exercises error paths)."""
    rng = random.Random(seed)
    c = O.RefCache(block_size, capacity, policy)
    lines = [json.dumps({"op": "create", "block_size": block_size, "capacity": capacity, "policy": policy})]
    # a small library of token streams sharing prefixes (system prompts)
    pools = [O.materialize(0, rng.randint(8, 6 * block_size), 1000 + k) for k in range(4)]
    held: list = []
    now = 0
    for _ in range(n_ops):
        now += rng.randint(0, 3)
        r = rng.random()
        if r < 0.40:
            base = pools[rng.randrange(len(pools))]
            tail = O.materialize(rng.randrange(4), rng.randint(0, 4 * block_size), rng.randrange(12), rng.randint(-1, 3))
            toks = np.concatenate([base[: rng.randint(0, len(base))], tail])
            if rng.random() < 0.08:
                toks = toks[:0]
            n = len(toks)
            cuts = sorted(rng.sample(range(1, n), min(rng.randint(0, 3), max(n - 1, 0)))) if n > 1 else []
            bounds = [0] + cuts + [n]
            tags = [[bounds[i], bounds[i + 1], rng.randrange(6)] for i in range(len(bounds) - 1)]
            if n == 0:
                tags = []
            if rng.random() < 0.04 and tags:
                tags[-1][1] += 1  # invalid coverage -> CacheError
            st, ids = c.insert(toks, [tuple(t) for t in tags], now)
            if st == 0 and ids:
                held.append(ids)
            lines.append(json.dumps({"op": "insert", "now": now, "tokens": b64(toks), "tags": tags,
                                     "status": st, "ids": ids, "dump_fnv": fnv(c.dump())}))
        elif r < 0.60:
            base = pools[rng.randrange(len(pools))]
            tail = O.materialize(rng.randrange(4), rng.randint(0, 3 * block_size), rng.randrange(12), rng.randint(-1, 3))
            toks = np.concatenate([base[: rng.randint(0, len(base))], tail])
            hit = c.lookup_prefix(toks, now)
            lines.append(json.dumps({"op": "lookup", "now": now, "tokens": b64(toks), "ret": hit, "status": 0,
                                     "dump_fnv": fnv(c.dump())}))
        elif r < 0.78:
            if held and rng.random() < 0.9:
                ids = held.pop(rng.randrange(len(held)))
            else:
                ids = [rng.randrange(capacity) for _ in range(rng.randint(1, 3))]
            if rng.random() < 0.05 and ids:
                ids = ids + ids[:1]  # duplicate id in one release call
            st = c.release(ids)
            lines.append(json.dumps({"op": "release", "ids": ids, "status": st, "dump_fnv": fnv(c.dump())}))
        elif r < 0.86:
            needed = rng.randint(0, max(1, capacity // 3))
            st, ids = c.evict(needed)
            lines.append(json.dumps({"op": "evict", "needed": needed, "ret": ids, "status": st,
                                     "dump_fnv": fnv(c.dump())}))
        elif r < 0.94:
            ids = [rng.randrange(capacity) for _ in range(rng.randint(1, 4))]
            pin = rng.choice([-1, 0, 1])
            tier = rng.choice([-1, -1, 0, 1, 2, 3, 4, 5])
            st = c.set_reuse_priority(ids, pin, tier)
            lines.append(json.dumps({"op": "set_priority", "ids": ids, "pinned": pin, "tier": tier, "status": st,
                                     "dump_fnv": fnv(c.dump())}))
        elif r < 0.97:
            bid, tag = rng.randrange(capacity), rng.randrange(6)
            st = c.set_tag(bid, tag)
            lines.append(json.dumps({"op": "set_tag", "id": bid, "tag": tag, "status": st, "dump_fnv": fnv(c.dump())}))
        else:
            ids = [rng.randrange(capacity) for _ in range(rng.randint(1, 4))]
            st = c.touch(ids, now)
            lines.append(json.dumps({"op": "touch", "ids": ids, "now": now, "status": st, "dump_fnv": fnv(c.dump())}))
    lines.append(json.dumps({"op": "final", "dump": c.dump(), "total_evicted": c.total_evicted(),
                             "audit": c.audit()}))
    c.close()
    return "\n".join(lines) + "\n"


def main():
    os.makedirs(OUT, exist_ok=True)
    O.build_ref()
    manifest = {}

    # 1. the paper's thrashing scenario (Fig. 5/7) under both policies
    for tiered in (0, 1):
        hits, log = O.kvlog_thrashing(tiered)
        name = f"oplog_thrashing_{'tiered' if tiered else 'lru'}.jsonl.gz"
        write_gz(name, log)
        manifest[name] = {"source": "scenarios.cpp:45-85 thrashing_trace", "it2_hits": hits,
                          "ops": len(log.splitlines())}

    # 2. small generated agent traces under the three presets
    runs = {}
    for preset, pname in ((0, "baseline"), (1, "baseline_sched"), (2, "sutradhara")):
        for cap in (96, 4096):
            r = O.ref_run_trace(5, 7, preset, cap, 16, gen=SMALL_GEN, kvlog=True)
            ftr, e2e, hit, prm, ev, _wall, log = r
            name = f"oplog_trace_{pname}_cap{cap}.jsonl.gz"
            write_gz(name, log)
            manifest[name] = {"source": "trace_gen.cpp + orchestrator.cpp replay", "preset": pname,
                              "capacity": cap, "requests": 5, "seed": 7, "gen": SMALL_GEN,
                              "ops": len(log.splitlines())}
            runs[f"{pname}_cap{cap}"] = {"ftr": ftr.tolist(), "e2e": e2e.tolist(), "hit": hit.tolist(),
                                         "prompt": prm.tolist(), "evictions": ev}

    # 3. fuzzed op sequences with error paths, both policies, two block sizes
    for seed, bs, cap, pol in ((1, 16, 24, 1), (2, 16, 24, 0), (3, 4, 40, 1), (4, 16, 64, 1), (5, 8, 12, 0)):
        name = f"oplog_fuzz_s{seed}_bs{bs}_cap{cap}_p{pol}.jsonl.gz"
        log = fuzz_log(seed, bs, cap, pol, 700)
        write_gz(name, log)
        manifest[name] = {"source": "random ops on kv_cache.cpp via ref_capi", "seed": seed, "ops": 700}

    # 4. hashing vectors
    L = O.ref()
    hv = {"root": str(int(L.ref_root_hash())), "sections": [], "decode": [], "chains": []}
    import ctypes as C
    for tag, length, key, src in ((0, 37, 7, -1), (1, 16, 8, -1), (2, 21, 99, 0), (2, 21, 99, 1), (3, 5, 2**63 + 5, -1), (0, 0, 1, -1)):
        out = np.zeros(max(length, 1), np.uint64)
        L.ref_materialize(tag, length, key, src, out.ctypes.data_as(C.POINTER(C.c_uint64)))
        hv["sections"].append({"tag": tag, "len": length, "key": str(key), "src": src,
                               "tokens": [str(int(x)) for x in out[:length]]})
    for key, idx in ((0, 0), (12345, 3), (2**64 - 1, 77)):
        hv["decode"].append({"key": str(key), "index": idx, "token": str(int(L.ref_decode_token(key, idx)))})
    rng = np.random.default_rng(5)
    for n in (0, 1, 15, 16, 17, 100):
        toks = rng.integers(0, 2**63, n, dtype=np.uint64)
        parent = int(L.ref_root_hash())
        h = int(L.ref_chain_hash(parent, toks.ctypes.data_as(C.POINTER(C.c_uint64)), n))
        hv["chains"].append({"parent": str(parent), "tokens": [str(int(x)) for x in toks], "hash": str(h)})
    with open(os.path.join(OUT, "hashes.json"), "w") as f:
        json.dump(hv, f, indent=1)
    with open(os.path.join(OUT, "runs.json"), "w") as f:
        json.dump(runs, f, indent=1)
    with open(os.path.join(OUT, "manifest.json"), "w") as f:
        json.dump(manifest, f, indent=1)
    print(json.dumps(manifest, indent=1))
    engine_events()


def engine_events():
    """Golden engine event lists: the reference engine (oracle/ref_engine.cpp)
    driven by the scripts of tests/engine_scripts.py."""
    import sys

    sys.path.insert(0, os.path.dirname(HERE))
    from tests import engine_scripts as S

    for name, mk in S.SCRIPTS.items():
        ev, _, _ = S.run_reference(mk())
        write_gz(f"engine_{name}.jsonl.gz", "\n".join(json.dumps(e) for e in ev) + "\n")


if __name__ == "__main__":
    main()
