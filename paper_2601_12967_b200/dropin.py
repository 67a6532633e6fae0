"""The drop-in: the reference simulator's UNMODIFIED engine and orchestrator
(/root/reference/proj/src) running on the B200 block pool, i.e. with its
KvCache implemented by integration/agentsim_kvcache_b200.cpp over the C-ABI
(every admission lookup, partial-prefill pin, completion insert with
hint-aware eviction and release is a device op).  Built by
integration/Makefile into integration/_build/libagentsim_b200.so, which loads
the product library paper_2601_12967_b200/_build/libsutradhara_b200.so.

``run_shard`` replays shard ``shard`` of ``n_shards`` (request i -> shard
i mod n) of ONE synthetic agent trace (trace_gen.cpp:96-193) under a run
preset (runner.cpp:120-153) and returns the per-request metrics, including
the FTR breakdown (metrics.cpp:104-129).  The pool lives on SB_DEVICE /
LOCAL_RANK (the binding's configuration)."""
from __future__ import annotations

import ctypes as C
import os
import threading
from dataclasses import dataclass
from typing import Optional, Sequence

import numpy as np

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
DROPIN_LIB = os.path.join(ROOT, "integration", "_build", "libagentsim_b200.so")
PRESETS = {"baseline": 0, "baseline_sched": 1, "sutradhara": 2}

_lock = threading.Lock()
_libs = {}

I64P = C.POINTER(C.c_int64)


def load(path: str = DROPIN_LIB):
    with _lock:
        if path not in _libs:
            if not os.path.exists(path):
                raise RuntimeError(f"{path} missing — build it with `make -C integration` (needs the reference "
                                   "sources; the built library travels with the tree)")
            L = C.CDLL(path)
            L.agentsim_run_last_error.restype = C.c_char_p
            L.agentsim_run_shard.restype = C.c_int64
            L.agentsim_run_shard.argtypes = [C.c_char_p, C.POINTER(C.c_double), C.c_int32, C.c_uint64, C.c_int32,
                                             C.c_int32, C.c_int64, C.c_int64, C.POINTER(C.c_double), C.c_int32, C.c_int32,
                                             I64P, I64P, I64P, I64P, I64P, I64P, I64P, I64P,
                                             C.POINTER(C.c_uint64), C.POINTER(C.c_double)]
            L.agentsim_thrashing.restype = C.c_int
            L.agentsim_thrashing.argtypes = [C.c_int32, I64P, C.POINTER(C.c_double), C.POINTER(C.c_uint64)]
            _libs[path] = L
    return _libs[path]


@dataclass
class ShardResult:
    ftr_ms: np.ndarray
    e2e_ms: np.ndarray
    hit_tokens: np.ndarray
    prompt_tokens: np.ndarray
    tool_ms: np.ndarray      # FTR breakdown: critical (non-overlapped) tool time
    wait_ms: np.ndarray
    prefill_ms: np.ndarray
    decode_ms: np.ndarray
    evictions: int
    wall_s: float


def run_shard(n_requests: int, seed: int, preset: str, capacity: int, block_size: int = 16,
              workload: Optional[str] = "default", gen: Optional[Sequence[float]] = None,
              cost: Optional[Sequence[float]] = None, shard: int = 0, n_shards: int = 1,
              kv_tiering: int = -1, lib_path: str = DROPIN_LIB) -> ShardResult:
    L = load(lib_path)
    n = n_requests
    arrs = [np.zeros(n, np.int64) for _ in range(8)]
    ev, wall = C.c_uint64(), C.c_double()
    g = (C.c_double * 8)(*gen) if gen is not None else None
    cst = (C.c_double * 4)(*cost) if cost is not None else None
    k = L.agentsim_run_shard(workload.encode() if workload else None, g, n, seed, PRESETS[preset], kv_tiering,
                             capacity, block_size, cst, shard, n_shards, *[a.ctypes.data_as(I64P) for a in arrs],
                             C.byref(ev), C.byref(wall))
    if k < 0:
        raise RuntimeError(L.agentsim_run_last_error().decode())
    a = [x[:k] for x in arrs]
    return ShardResult(*a, evictions=int(ev.value), wall_s=wall.value)


def thrashing(tiered: bool, lib_path: str = DROPIN_LIB):
    """scenarios.cpp:45-85 under LRU / hint-aware eviction: (iteration-2 hit
    tokens per request, run hit rate, evictions)."""
    L = load(lib_path)
    hits = np.zeros(8, np.int64)
    hr, ev = C.c_double(), C.c_uint64()
    k = L.agentsim_thrashing(1 if tiered else 0, hits.ctypes.data_as(I64P), C.byref(hr), C.byref(ev))
    if k < 0:
        raise RuntimeError(L.agentsim_run_last_error().decode())
    return hits[:k].tolist(), hr.value, int(ev.value)

