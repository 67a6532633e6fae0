"""Host-side mirror of the reference's ``agentsim::KvCache``
(/root/reference/proj/include/agentsim/kv_cache.hpp:70-128), backed by the
device-resident block pool in csrc/kv_pool.cu through the C-ABI.

Same method names, argument meaning and error behaviour as the reference:
``insert`` raises CacheFull after reproducing the reference's rollback,
``release`` raises UnknownBlock / ZeroRefRelease, ``set_reuse_priority`` is
all-or-nothing, ``touch`` applies up to the first unknown id, and so on.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import List, Optional, Sequence, Tuple

import numpy as np

from . import _lib
from .errors import CacheError, CacheFull, UnknownBlock, ZeroRefRelease  # noqa: F401 (re-export)

# KvTag (kv_cache.hpp:21-28) and EvictionPolicy (kv_cache.hpp:36)
RESPONSE, TOOL_OUTPUT, USER_QUERY, SYSTEM_PROMPT, PARTIAL_PREFILL, HISTORY = range(6)
LRU, TIERED = 0, 1
TAG_NAMES = ["response", "tool_output", "user_query", "system_prompt", "partial_prefill", "history"]


def eviction_tier(tag: int) -> int:
    """kv_cache.cpp:23-33."""
    return (0, 1, 2, 3, 4, 2)[tag]


def kv_root_hash() -> int:
    return int(_lib.lib().sb_kv_root_hash())


def kv_chain_hash(parent: int, tokens) -> int:
    t = np.ascontiguousarray(tokens, dtype=np.uint64)
    return int(_lib.lib().sb_kv_chain_hash_host(parent, t.ctypes.data_as(_lib.U64P), len(t)))


@dataclass
class CacheConfig:
    block_size: int = 16
    capacity_blocks: int = 4096
    policy: int = LRU


@dataclass
class KvBlock:
    block_id: int
    chain_hash: int
    parent_hash: int
    tag: int
    tier: int
    ref_count: int
    last_used: int
    pinned: bool
    tokens: np.ndarray


def _tag_array(tags: Sequence[Tuple[int, int, int]]):
    arr = (_lib.TagRange * max(len(tags), 1))()
    for i, (b, e, t) in enumerate(tags):
        arr[i].begin, arr[i].end, arr[i].tag = int(b), int(e), int(t)
    return arr


class KvCache:
    """Paged, prefix-indexed KV block pool with tiered (hint-aware) or LRU eviction."""

    def __init__(self, config: CacheConfig = CacheConfig(), device: int = 0):
        self.config = config
        L = _lib.lib()
        h = C.c_void_p()
        _lib.check(L.sb_kv_create(config.block_size, config.capacity_blocks, config.policy, device, C.byref(h)),
                   "KvCache")
        self._h = h
        self._L = L

    # -- lifetime
    def close(self):
        if getattr(self, "_h", None):
            if getattr(self, "_owner", True):
                self._L.sb_kv_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def handle(self):
        return self._h

    # -- reference API
    def lookup_prefix(self, tokens, now: int) -> int:
        t = np.ascontiguousarray(tokens, dtype=np.uint64)
        hit = C.c_int64(0)
        _lib.check(self._L.sb_kv_lookup_prefix(self._h, t.ctypes.data_as(_lib.U64P), len(t), now, C.byref(hit)),
                   "lookup_prefix")
        return hit.value

    def insert(self, tokens, tags: Sequence[Tuple[int, int, int]], now: int) -> List[int]:
        t = np.ascontiguousarray(tokens, dtype=np.uint64)
        bs = self.config.block_size
        out = np.zeros((len(t) + bs - 1) // bs + 1, dtype=np.int32)
        n = C.c_int64(0)
        st = self._L.sb_kv_insert(self._h, t.ctypes.data_as(_lib.U64P), len(t), _tag_array(tags), len(tags), now,
                                  out.ctypes.data_as(_lib.I32P), C.byref(n))
        _lib.check(st, "insert")
        return out[: n.value].tolist()

    def evict(self, needed: int) -> List[int]:
        out = np.zeros(max(needed, 1), dtype=np.int32)
        n = C.c_int64(0)
        _lib.check(self._L.sb_kv_evict(self._h, needed, out.ctypes.data_as(_lib.I32P), C.byref(n)), "evict")
        return out[: n.value].tolist()

    def set_reuse_priority(self, ids, pinned: Optional[bool] = None, tier_override: Optional[int] = None):
        a = np.ascontiguousarray(ids, dtype=np.int32)
        pin = -1 if pinned is None else int(bool(pinned))
        tier = -1 if tier_override is None else int(tier_override)
        _lib.check(self._L.sb_kv_set_reuse_priority(self._h, a.ctypes.data_as(_lib.I32P), len(a), pin, tier),
                   "set_reuse_priority")

    def set_tag(self, block_id: int, tag: int):
        _lib.check(self._L.sb_kv_set_tag(self._h, block_id, tag), "set_tag")

    def release(self, ids):
        a = np.ascontiguousarray(ids, dtype=np.int32)
        _lib.check(self._L.sb_kv_release(self._h, a.ctypes.data_as(_lib.I32P), len(a)), "release")

    def touch(self, ids, now: int):
        a = np.ascontiguousarray(ids, dtype=np.int32)
        _lib.check(self._L.sb_kv_touch(self._h, a.ctypes.data_as(_lib.I32P), len(a), now), "touch")

    def resident_blocks(self) -> int:
        return int(self._L.sb_kv_resident_blocks(self._h))

    def capacity_blocks(self) -> int:
        return int(self._L.sb_kv_capacity_blocks(self._h))

    def free_blocks(self) -> int:
        return int(self._L.sb_kv_free_blocks(self._h))

    def total_evicted(self) -> int:
        return int(self._L.sb_kv_total_evicted(self._h))

    def contains(self, block_id: int) -> bool:
        return bool(self._L.sb_kv_contains(self._h, block_id))

    def block(self, block_id: int) -> KvBlock:
        info = _lib.BlockInfo()
        toks = np.zeros(self.config.block_size, dtype=np.uint64)
        _lib.check(self._L.sb_kv_block(self._h, block_id, C.byref(info), toks.ctypes.data_as(_lib.U64P)), "block")
        return KvBlock(info.block_id, info.chain_hash, info.parent_hash, info.tag, info.tier, info.ref_count,
                       info.last_used, bool(info.pinned), toks[: info.n_tokens].copy())

    def blocks(self, block_ids) -> list:
        """Batched contains()/block() metadata: one device round trip; None
        for an id that is not resident (block() would raise for it)."""
        ids = np.ascontiguousarray(block_ids, dtype=np.int32)
        infos = (_lib.BlockInfo * max(len(ids), 1))()
        _lib.check(self._L.sb_kv_blocks(self._h, ids.ctypes.data_as(_lib.I32P), len(ids), infos), "blocks")
        return [None if b.n_tokens == 0 else
                KvBlock(b.block_id, b.chain_hash, b.parent_hash, b.tag, b.tier, b.ref_count, b.last_used,
                        bool(b.pinned), None) for b in infos[: len(ids)]]

    def audit(self):
        _lib.check(self._L.sb_kv_audit(self._h), "audit")

    def dump(self) -> str:
        n = C.c_int64(0)
        _lib.check(self._L.sb_kv_dump(self._h, None, 0, C.byref(n)), "dump")
        buf = C.create_string_buffer(n.value + 1)
        _lib.check(self._L.sb_kv_dump(self._h, buf, n.value + 1, C.byref(n)), "dump")
        return buf.value.decode()

    def stats(self) -> dict:
        out = (C.c_uint64 * 6)()
        _lib.check(self._L.sb_kv_stats(self._h, out), "stats")
        keys = ["lookups", "hit_tokens", "looked_up_tokens", "inserted_blocks", "evicted_blocks", "cache_full"]
        return dict(zip(keys, [int(x) for x in out]))

    def last_evicted(self) -> list:
        """Block ids the last insert / evict evicted, in eviction order (sb_kv_last_evicted)."""
        n = C.c_int64(0)
        _lib.check(self._L.sb_kv_last_evicted(self._h, None, 0, C.byref(n)), "last_evicted")
        out = np.zeros(max(n.value, 1), dtype=np.int32)
        _lib.check(self._L.sb_kv_last_evicted(self._h, out.ctypes.data_as(_lib.I32P), n.value, C.byref(n)),
                   "last_evicted")
        return out[: n.value].tolist()

    def program_stats(self) -> dict:
        """Op programs run on this pool and how many the parallel path applied."""
        out = (C.c_uint64 * 2)()
        _lib.check(self._L.sb_kv_program_stats(self._h, out), "program_stats")
        return {"programs": int(out[0]), "parallel": int(out[1])}
