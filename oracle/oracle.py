"""TEST INFRASTRUCTURE ONLY — ctypes front-end of the CPU oracle.

Two checkers live here:

* ``OracleCache`` — the plain-C restatement (oracle/kvcache_oracle.c) of the
  reference KvCache (/root/reference/proj/src/kv_cache.cpp:23-281) and its
  hashing (include/agentsim/common.hpp:136-145, src/trace.cpp:50-83).
* ``RefCache`` / ``ref_*`` — the reference itself compiled from its own sources
  into oracle/_ref/ by oracle/Makefile (see oracle/ref_capi.cpp).

Only tests/, ``__graft_entry__.smoke()`` and bench.py's cpu_baseline /
reference legs may import this module.  The product package never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import threading
from typing import List, Optional, Sequence, Tuple

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
BUILD = os.path.join(HERE, "_build")
REF_DIR = os.path.join(HERE, "_ref")

_lock = threading.Lock()
_lib = None
_ref = None
_kvlog = None

U64P = C.POINTER(C.c_uint64)
I64P = C.POINTER(C.c_int64)
I32P = C.POINTER(C.c_int32)

STATUS_NAMES = {0: "ok", 1: "CacheFull", 2: "UnknownBlock", 3: "ZeroRefRelease", 4: "CacheError", 5: "ConfigError"}


def build_oracle() -> str:
    path = os.path.join(BUILD, "libkvoracle.so")
    src = os.path.join(HERE, "kvcache_oracle.c")
    if not os.path.exists(path) or os.path.getmtime(path) < os.path.getmtime(src):
        subprocess.run(["make", "-C", HERE, "liboracle"], check=True, capture_output=True)
    return path


def build_ref() -> bool:
    """Compile oracle/_ref from /root/reference (only possible in the build container)."""
    if not os.path.isdir("/root/reference/proj/src"):
        return os.path.exists(os.path.join(REF_DIR, "libagentsim_ref.so"))
    subprocess.run(["make", "-C", HERE, "-j8", "ref"], check=True, capture_output=True)
    if os.path.exists(os.path.join(os.path.dirname(HERE), "paper_2601_12967_b200", "_build", "libsutradhara_b200.so")):
        subprocess.run(["make", "-C", HERE, "-j8", "b200"], check=True, capture_output=True)
    return True


def _u64(a: np.ndarray):
    return a.ctypes.data_as(U64P)


def _i32(a: np.ndarray):
    return a.ctypes.data_as(I32P)


def _i64(a: np.ndarray):
    return a.ctypes.data_as(I64P)


def lib():
    global _lib
    with _lock:
        if _lib is None:
            L = C.CDLL(build_oracle())
            L.oc_splitmix64.restype = C.c_uint64
            L.oc_splitmix64.argtypes = [C.c_uint64]
            L.oc_hash_combine.restype = C.c_uint64
            L.oc_hash_combine.argtypes = [C.c_uint64, C.c_uint64]
            L.oc_root_hash.restype = C.c_uint64
            L.oc_chain_hash.restype = C.c_uint64
            L.oc_chain_hash.argtypes = [C.c_uint64, U64P, C.c_int64]
            L.oc_materialize.argtypes = [C.c_int, C.c_int64, C.c_uint64, C.c_int32, U64P]
            L.oc_decode_token.restype = C.c_uint64
            L.oc_decode_token.argtypes = [C.c_uint64, C.c_int64]
            L.oc_create.restype = C.c_void_p
            L.oc_create.argtypes = [C.c_int64, C.c_int64, C.c_int]
            L.oc_destroy.argtypes = [C.c_void_p]
            L.oc_lookup_prefix.restype = C.c_int64
            L.oc_lookup_prefix.argtypes = [C.c_void_p, U64P, C.c_int64, C.c_int64]
            L.oc_insert.argtypes = [C.c_void_p, U64P, C.c_int64, I64P, C.c_int64, C.c_int64, I32P, I64P]
            L.oc_evict.restype = C.c_int64
            L.oc_evict.argtypes = [C.c_void_p, C.c_int64, I32P]
            L.oc_set_priority.argtypes = [C.c_void_p, I32P, C.c_int64, C.c_int, C.c_int]
            L.oc_set_tag.argtypes = [C.c_void_p, C.c_int32, C.c_int]
            L.oc_release.argtypes = [C.c_void_p, I32P, C.c_int64]
            L.oc_touch.argtypes = [C.c_void_p, I32P, C.c_int64, C.c_int64]
            L.oc_resident.restype = C.c_int64
            L.oc_resident.argtypes = [C.c_void_p]
            L.oc_total_evicted.restype = C.c_uint64
            L.oc_total_evicted.argtypes = [C.c_void_p]
            L.oc_contains.argtypes = [C.c_void_p, C.c_int32]
            L.oc_block_info.argtypes = [C.c_void_p, C.c_int32, I64P, U64P, U64P]
            L.oc_dump.restype = C.c_int64
            L.oc_dump.argtypes = [C.c_void_p, C.c_char_p, C.c_int64]
            L.oc_audit.argtypes = [C.c_void_p]
            L.oc_fnv1a.restype = C.c_uint64
            L.oc_fnv1a.argtypes = [C.c_char_p, C.c_int64]
            _lib = L
    return _lib


# ----------------------------------------------------------------- hashing
def fnv1a(text: str) -> int:
    b = text.encode()
    return int(lib().oc_fnv1a(b, len(b)))


def splitmix64(x: int) -> int:
    return int(lib().oc_splitmix64(x & 0xFFFFFFFFFFFFFFFF))


def root_hash() -> int:
    return int(lib().oc_root_hash())


def chain_hash(parent: int, tokens: np.ndarray) -> int:
    t = np.ascontiguousarray(tokens, dtype=np.uint64)
    return int(lib().oc_chain_hash(parent, _u64(t), len(t)))


def block_hashes(tokens: np.ndarray, block_size: int, parent: Optional[int] = None) -> np.ndarray:
    """Chain hash of every block (last one partial) of a token sequence."""
    t = np.ascontiguousarray(tokens, dtype=np.uint64)
    out = []
    h = root_hash() if parent is None else parent
    for pos in range(0, len(t), block_size):
        h = chain_hash(h, t[pos:pos + block_size])
        out.append(h)
    return np.array(out, dtype=np.uint64)


def materialize(tag: int, length: int, key: int, src_iter: int = -1) -> np.ndarray:
    out = np.zeros(max(length, 0), dtype=np.uint64)
    if length > 0:
        lib().oc_materialize(tag, length, key & 0xFFFFFFFFFFFFFFFF, src_iter, _u64(out))
    return out


def decode_token(stream_key: int, index: int) -> int:
    return int(lib().oc_decode_token(stream_key & 0xFFFFFFFFFFFFFFFF, index))


# ----------------------------------------------------------------- caches
def _tags_arr(tags: Sequence[Tuple[int, int, int]]) -> np.ndarray:
    return np.array([v for r in tags for v in r], dtype=np.int64).reshape(-1) if tags else np.zeros(0, np.int64)


class OracleCache:
    """The C restatement, with the same call surface as the product's KvCache."""

    def __init__(self, block_size: int, capacity: int, policy: int):
        self.block_size = block_size
        self.capacity = capacity
        self.policy = policy
        self._h = lib().oc_create(block_size, capacity, policy)
        if not self._h:
            raise ValueError("bad cache config")

    def close(self):
        if self._h:
            lib().oc_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def lookup_prefix(self, tokens, now: int) -> int:
        t = np.ascontiguousarray(tokens, dtype=np.uint64)
        return int(lib().oc_lookup_prefix(self._h, _u64(t), len(t), now))

    def insert(self, tokens, tags, now: int):
        t = np.ascontiguousarray(tokens, dtype=np.uint64)
        tg = _tags_arr(tags)
        out = np.zeros(len(t) // self.block_size + 2, dtype=np.int32)
        n = C.c_int64(0)
        st = lib().oc_insert(self._h, _u64(t), len(t), _i64(tg), len(tags), now, _i32(out), C.byref(n))
        return st, out[: n.value].tolist()

    def evict(self, needed: int):
        out = np.zeros(max(needed, 1), dtype=np.int32)
        n = lib().oc_evict(self._h, needed, _i32(out))
        return 0, out[:n].tolist()

    def set_reuse_priority(self, ids, pinned: int = -1, tier: int = -1) -> int:
        a = np.ascontiguousarray(ids, dtype=np.int32)
        return int(lib().oc_set_priority(self._h, _i32(a), len(a), pinned, tier))

    def set_tag(self, block_id: int, tag: int) -> int:
        return int(lib().oc_set_tag(self._h, block_id, tag))

    def release(self, ids) -> int:
        a = np.ascontiguousarray(ids, dtype=np.int32)
        return int(lib().oc_release(self._h, _i32(a), len(a)))

    def touch(self, ids, now: int) -> int:
        a = np.ascontiguousarray(ids, dtype=np.int32)
        return int(lib().oc_touch(self._h, _i32(a), len(a), now))

    def resident_blocks(self) -> int:
        return int(lib().oc_resident(self._h))

    def total_evicted(self) -> int:
        return int(lib().oc_total_evicted(self._h))

    def contains(self, block_id: int) -> bool:
        return bool(lib().oc_contains(self._h, block_id))

    def block(self, block_id: int):
        f = np.zeros(6, np.int64)
        h = np.zeros(2, np.uint64)
        toks = np.zeros(self.block_size, np.uint64)
        st = lib().oc_block_info(self._h, block_id, _i64(f), _u64(h), _u64(toks))
        if st:
            return st, None
        return 0, dict(tag=int(f[0]), tier=int(f[1]), ref=int(f[2]), pinned=int(f[3]), ntok=int(f[4]),
                       last=int(f[5]), chain=int(h[0]), parent=int(h[1]), tokens=toks[: int(f[4])].copy())

    def dump(self) -> str:
        n = lib().oc_dump(self._h, None, 0)
        buf = C.create_string_buffer(int(n) + 1)
        lib().oc_dump(self._h, buf, n + 1)
        return buf.value.decode()

    def audit(self) -> int:
        return int(lib().oc_audit(self._h))


# ------------------------------------------------------------- reference
def _load_ref(name: str):
    path = os.path.join(REF_DIR, name)
    if not os.path.exists(path):
        raise FileNotFoundError(f"{path} missing: run `make -C oracle ref` in the build container")
    return C.CDLL(path, mode=C.RTLD_LOCAL)


def _declare_ref(L, p: str):
    getattr(L, p + "root_hash").restype = C.c_uint64
    getattr(L, p + "chain_hash").restype = C.c_uint64
    getattr(L, p + "chain_hash").argtypes = [C.c_uint64, U64P, C.c_int64]
    getattr(L, p + "materialize").argtypes = [C.c_int32, C.c_int64, C.c_uint64, C.c_int32, U64P]
    getattr(L, p + "decode_token").restype = C.c_uint64
    getattr(L, p + "decode_token").argtypes = [C.c_uint64, C.c_int64]
    getattr(L, p + "kv_create").argtypes = [C.c_int64, C.c_int64, C.c_int32, C.POINTER(C.c_void_p)]
    getattr(L, p + "kv_destroy").argtypes = [C.c_void_p]
    getattr(L, p + "kv_lookup").argtypes = [C.c_void_p, U64P, C.c_int64, C.c_int64, I64P]
    getattr(L, p + "kv_insert").argtypes = [C.c_void_p, U64P, C.c_int64, I64P, C.c_int64, C.c_int64, I32P, I64P]
    getattr(L, p + "kv_evict").argtypes = [C.c_void_p, C.c_int64, I32P, I64P]
    getattr(L, p + "kv_set_priority").argtypes = [C.c_void_p, I32P, C.c_int64, C.c_int32, C.c_int32]
    getattr(L, p + "kv_set_tag").argtypes = [C.c_void_p, C.c_int32, C.c_int32]
    getattr(L, p + "kv_release").argtypes = [C.c_void_p, I32P, C.c_int64]
    getattr(L, p + "kv_touch").argtypes = [C.c_void_p, I32P, C.c_int64, C.c_int64]
    getattr(L, p + "kv_resident").restype = C.c_int64
    getattr(L, p + "kv_resident").argtypes = [C.c_void_p]
    getattr(L, p + "kv_total_evicted").restype = C.c_uint64
    getattr(L, p + "kv_total_evicted").argtypes = [C.c_void_p]
    getattr(L, p + "kv_contains").argtypes = [C.c_void_p, C.c_int32]
    getattr(L, p + "kv_block").argtypes = [C.c_void_p, C.c_int32, I64P, U64P, U64P]
    getattr(L, p + "kv_dump").restype = C.c_int64
    getattr(L, p + "kv_dump").argtypes = [C.c_void_p, C.c_char_p, C.c_int64]
    getattr(L, p + "kv_audit").argtypes = [C.c_void_p]
    getattr(L, p + "last_error").restype = C.c_char_p


def ref():
    global _ref
    with _lock:
        if _ref is None:
            L = _load_ref("libagentsim_ref.so")
            _declare_ref(L, "ref_")
            L.refrun_generate_and_run.argtypes = [C.c_char_p, C.POINTER(C.c_double), C.c_int32, C.c_uint64,
                                                  C.c_int32, C.c_int64, C.c_int64, I64P, I64P, I64P, I64P,
                                                  U64P, C.POINTER(C.c_double)]
            L.refrun_scenarios.argtypes = [C.c_char_p, C.c_int64]
            L.refrun_thrashing.argtypes = [C.c_int32, I64P]
            L.refrun_last_error.restype = C.c_char_p
            _ref = L
    return _ref


_b200 = None


def b200_lib():
    """Reference engine/orchestrator linked against the B200 block pool."""
    global _b200
    with _lock:
        if _b200 is None:
            L = _load_ref("libagentsim_b200.so")
            L.refrun_generate_and_run.argtypes = [C.c_char_p, C.POINTER(C.c_double), C.c_int32, C.c_uint64,
                                                  C.c_int32, C.c_int64, C.c_int64, I64P, I64P, I64P, I64P,
                                                  U64P, C.POINTER(C.c_double)]
            L.refrun_scenarios.argtypes = [C.c_char_p, C.c_int64]
            L.refrun_thrashing.argtypes = [C.c_int32, I64P]
            L.refrun_last_error.restype = C.c_char_p
            _b200 = L
    return _b200


def kvlog_lib():
    global _kvlog
    with _lock:
        if _kvlog is None:
            L = _load_ref("libagentsim_kvlog.so")
            L.kvlog_take.restype = C.c_int64
            L.kvlog_take.argtypes = [C.c_char_p, C.c_int64]
            L.kvlog_enable.argtypes = [C.c_int]
            L.refrun_last_error.restype = C.c_char_p
            L.refrun_generate_and_run.argtypes = [C.c_char_p, C.POINTER(C.c_double), C.c_int32, C.c_uint64,
                                                  C.c_int32, C.c_int64, C.c_int64, I64P, I64P, I64P, I64P,
                                                  U64P, C.POINTER(C.c_double)]
            L.refrun_scenarios.argtypes = [C.c_char_p, C.c_int64]
            L.refrun_thrashing.argtypes = [C.c_int32, I64P]
            _kvlog = L
    return _kvlog


class RefCache:
    """The reference's own KvCache through oracle/ref_capi.cpp."""

    def __init__(self, block_size: int, capacity: int, policy: int):
        self.L = ref()
        self.block_size = block_size
        h = C.c_void_p()
        st = self.L.ref_kv_create(block_size, capacity, policy, C.byref(h))
        if st:
            raise ValueError(self.L.ref_last_error().decode())
        self._h = h

    def close(self):
        if self._h:
            self.L.ref_kv_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def lookup_prefix(self, tokens, now):
        t = np.ascontiguousarray(tokens, dtype=np.uint64)
        hit = C.c_int64(0)
        self.L.ref_kv_lookup(self._h, _u64(t), len(t), now, C.byref(hit))
        return hit.value

    def insert(self, tokens, tags, now):
        t = np.ascontiguousarray(tokens, dtype=np.uint64)
        tg = _tags_arr(tags)
        out = np.zeros(len(t) // self.block_size + 2, np.int32)
        n = C.c_int64(0)
        st = self.L.ref_kv_insert(self._h, _u64(t), len(t), _i64(tg), len(tags), now, _i32(out), C.byref(n))
        return st, out[: n.value].tolist()

    def evict(self, needed):
        out = np.zeros(max(needed, 1), np.int32)
        n = C.c_int64(0)
        st = self.L.ref_kv_evict(self._h, needed, _i32(out), C.byref(n))
        return st, out[: n.value].tolist()

    def set_reuse_priority(self, ids, pinned=-1, tier=-1):
        a = np.ascontiguousarray(ids, np.int32)
        return self.L.ref_kv_set_priority(self._h, _i32(a), len(a), pinned, tier)

    def set_tag(self, block_id, tag):
        return self.L.ref_kv_set_tag(self._h, block_id, tag)

    def release(self, ids):
        a = np.ascontiguousarray(ids, np.int32)
        return self.L.ref_kv_release(self._h, _i32(a), len(a))

    def touch(self, ids, now):
        a = np.ascontiguousarray(ids, np.int32)
        return self.L.ref_kv_touch(self._h, _i32(a), len(a), now)

    def resident_blocks(self):
        return int(self.L.ref_kv_resident(self._h))

    def total_evicted(self):
        return int(self.L.ref_kv_total_evicted(self._h))

    def contains(self, block_id):
        return bool(self.L.ref_kv_contains(self._h, block_id))

    def block(self, block_id):
        f = np.zeros(6, np.int64)
        h = np.zeros(2, np.uint64)
        toks = np.zeros(self.block_size, np.uint64)
        st = self.L.ref_kv_block(self._h, block_id, _i64(f), _u64(h), _u64(toks))
        if st:
            return st, None
        return 0, dict(tag=int(f[0]), tier=int(f[1]), ref=int(f[2]), pinned=int(f[3]), ntok=int(f[4]),
                       last=int(f[5]), chain=int(h[0]), parent=int(h[1]), tokens=toks[: int(f[4])].copy())

    def dump(self):
        n = self.L.ref_kv_dump(self._h, None, 0)
        buf = C.create_string_buffer(int(n) + 1)
        self.L.ref_kv_dump(self._h, buf, n + 1)
        return buf.value.decode()

    def audit(self):
        return int(self.L.ref_kv_audit(self._h))


def ref_run_trace(n_requests: int, seed: int, preset: int, capacity: int, block_size: int = 16,
                  workload: Optional[str] = None, gen: Optional[Sequence[float]] = None, kvlog: bool = False,
                  b200: bool = False):
    """Generate + replay a trace in the reference simulator (b200=True: with
    its KvCache served by the B200 block pool through the C-ABI).

    Returns (ftr, e2e, hit_tokens, prompt_tokens, evictions, wall_s[, oplog]).
    """
    L = kvlog_lib() if kvlog else (b200_lib() if b200 else ref())
    g = (C.c_double * 8)(*(list(gen) + [0.0] * (8 - len(gen)))) if gen is not None else None
    ftr = np.zeros(n_requests, np.int64)
    e2e = np.zeros(n_requests, np.int64)
    hit = np.zeros(n_requests, np.int64)
    prm = np.zeros(n_requests, np.int64)
    ev = C.c_uint64(0)
    wall = C.c_double(0)
    if kvlog:
        L.kvlog_take(None, 0)
        _drain_kvlog(L)
    st = L.refrun_generate_and_run(workload.encode() if workload else None, g, n_requests, seed, preset,
                                   capacity, block_size, _i64(ftr), _i64(e2e), _i64(hit), _i64(prm),
                                   C.byref(ev), C.byref(wall))
    if st:
        raise RuntimeError("reference run failed: " + L.refrun_last_error().decode(errors="replace"))
    res = (ftr, e2e, hit, prm, int(ev.value), float(wall.value))
    if kvlog:
        res = res + (_drain_kvlog(L),)
    return res


def _drain_kvlog(L) -> str:
    n = L.kvlog_take(None, 0)
    buf = C.create_string_buffer(int(n) + 1)
    L.kvlog_take(buf, n + 1)
    return buf.value.decode()


def kvlog_thrashing(tiered: int) -> Tuple[List[int], str]:
    L = kvlog_lib()
    _drain_kvlog(L)
    hits = np.zeros(3, np.int64)
    st = L.refrun_thrashing(tiered, _i64(hits))
    if st:
        raise RuntimeError("thrashing scenario failed")
    return hits.tolist(), _drain_kvlog(L)


# ------------------------------------------------- reference engine (scripted)
def _declare_refeng(L):
    L.refeng_last_error.restype = C.c_char_p
    L.refeng_create.restype = C.c_void_p
    L.refeng_create.argtypes = [C.c_int64, C.c_int64, C.c_int32, C.c_int32, C.POINTER(C.c_double)]
    L.refeng_destroy.argtypes = [C.c_void_p]
    L.refeng_now.restype = C.c_int64
    L.refeng_now.argtypes = [C.c_void_p]
    L.refeng_submit_call.argtypes = [C.c_void_p, U64P, C.c_int64, I64P, C.c_int64, C.c_int64, C.c_uint64, I64P]
    L.refeng_submit_partial.argtypes = [C.c_void_p, U64P, C.c_int64, I64P, C.c_int64, C.c_uint64, I64P]
    L.refeng_extend.argtypes = [C.c_void_p, C.c_int64, U64P, C.c_int64, I64P, C.c_int64, C.c_int64]
    L.refeng_abandon.argtypes = [C.c_void_p, C.c_int64]
    L.refeng_run.argtypes = [C.c_void_p, C.c_int64]
    L.refeng_events.restype = C.c_int64
    L.refeng_events.argtypes = [C.c_void_p, C.c_char_p, C.c_int64]
    L.refeng_overlap_scenario.restype = C.c_int64
    L.refeng_overlap_scenario.argtypes = [C.c_int32, C.c_char_p, C.c_int64, I64P]
    L.refeng_stream_key.restype = C.c_uint64
    L.refeng_stream_key.argtypes = [C.c_char_p, C.c_uint64]


def _kvlog_drain(L) -> str:
    """Returns and clears the recording cache's op log."""
    n = L.kvlog_take(None, 0)
    buf = C.create_string_buffer(n + 1)
    L.kvlog_take(buf, n + 1)
    return buf.value.decode()


def stream_key(request_id: str, iteration: int) -> int:
    """Orchestrator::decode_stream_key (orchestrator.cpp:179-181)."""
    L = ref()
    if not hasattr(L, "_refeng"):
        _declare_refeng(L)
        L._refeng = True
    return int(L.refeng_stream_key(request_id.encode(), iteration))


class RefEngine:
    """The UNMODIFIED reference Engine (engine.cpp) driven by a script of
    engine-boundary actions at chosen virtual times (oracle/ref_engine.cpp).
    ``events()`` returns every action and engine-internal KV transition
    (pin / pin_failed / complete / finish) with the pool dump after it.
    With ``kvlog=True`` the run goes through the recording cache and
    ``oplog()`` returns its KvCache op log."""

    def __init__(self, block_size: int, capacity: int, policy: int, sched: int = 0, cost=None, kvlog: bool = False):
        L = kvlog_lib() if kvlog else ref()
        if not hasattr(L, "_refeng"):
            _declare_refeng(L)
            L._refeng = True
        self._L = L
        self.kvlog = kvlog
        if kvlog:
            _kvlog_drain(L)
        cst = (C.c_double * 4)(*cost) if cost is not None else None
        self._h = L.refeng_create(block_size, capacity, policy, sched, cst)
        if not self._h:
            raise RuntimeError(L.refeng_last_error().decode())

    def _chk(self, st):
        if st:
            raise RuntimeError(f"reference engine status {st}: {self._L.refeng_last_error().decode()}")

    @staticmethod
    def _tags(tags):
        a = np.array([[int(b), int(e), int(t)] for b, e, t in tags], dtype=np.int64).reshape(-1, 3)
        return np.ascontiguousarray(a)

    def run(self, until: int = -1):
        self._chk(self._L.refeng_run(self._h, until))

    def now(self) -> int:
        return int(self._L.refeng_now(self._h))

    def submit_call(self, tokens, tags, decode_length: int, key: int) -> int:
        t, g, out = np.ascontiguousarray(tokens, np.uint64), self._tags(tags), C.c_int64()
        self._chk(self._L.refeng_submit_call(self._h, _u64(t), len(t), _i64(g), len(g), decode_length, key,
                                             C.byref(out)))
        return out.value

    def submit_partial(self, tokens, tags, key: int) -> int:
        t, g, out = np.ascontiguousarray(tokens, np.uint64), self._tags(tags), C.c_int64()
        self._chk(self._L.refeng_submit_partial(self._h, _u64(t), len(t), _i64(g), len(g), key, C.byref(out)))
        return out.value

    def extend(self, call: int, tokens, tags, decode_length: int) -> int:
        t, g = np.ascontiguousarray(tokens, np.uint64), self._tags(tags)
        return self._L.refeng_extend(self._h, call, _u64(t), len(t), _i64(g), len(g), decode_length)

    def abandon(self, call: int) -> int:
        return self._L.refeng_abandon(self._h, call)

    def events(self):
        import json

        n = self._L.refeng_events(self._h, None, 0)
        buf = C.create_string_buffer(n + 1)
        self._L.refeng_events(self._h, buf, n + 1)
        return [json.loads(x) for x in buf.value.decode().splitlines()]

    def oplog(self) -> str:
        return _kvlog_drain(self._L)

    def close(self):
        if getattr(self, "_h", None):
            self._L.refeng_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def ref_overlap_scenario(split: bool, kvlog: bool = False):
    """scenarios.cpp:193-240 through the reference orchestrator: (timeline
    text, FTR of R1, KvCache op log when kvlog)."""
    L = kvlog_lib() if kvlog else ref()
    if not hasattr(L, "_refeng"):
        _declare_refeng(L)
        L._refeng = True
    if kvlog:
        _kvlog_drain(L)
    buf, ftr = C.create_string_buffer(1 << 20), C.c_int64()
    n = L.refeng_overlap_scenario(1 if split else 0, buf, 1 << 20, C.byref(ftr))
    if n < 0:
        raise RuntimeError(L.refeng_last_error().decode())
    log = _kvlog_drain(L) if kvlog else None
    return buf.value.decode(), ftr.value, log
