"""Agentic-trace replay on the B200 block pool (csrc/replay.cu): per-request
FTR / end-to-end time / prefix hits under the reference's engine and
orchestrator timing rules, with every KV decision made by the device pool.

``cost`` overrides the engine cost model (reference defaults: 0.05 ms per
prefill token, 20 ms per decode token, 2 ms batch overhead, chunk 256); a
B200-calibrated replay sets ``prefill_ms_per_token`` from the measured
continuation-prefill throughput."""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Optional, Sequence

import numpy as np

from . import _lib

PRESETS = {"baseline": 0, "baseline_sched": 1, "sutradhara": 2}


@dataclass
class ReplayResult:
    ftr_ms: np.ndarray
    e2e_ms: np.ndarray
    hit_tokens: np.ndarray
    prompt_tokens: np.ndarray
    evictions: int

    @property
    def hit_rate(self) -> float:
        return float(self.hit_tokens.sum()) / max(1.0, float(self.prompt_tokens.sum()))

    def p50(self, values=None) -> float:
        """Nearest-rank median (metrics.cpp:136-151)."""
        v = np.sort(self.ftr_ms if values is None else values)
        return float(v[max(1, int(np.ceil(0.5 * len(v)))) - 1])


def replay(n_requests: int, seed: int = 1, preset: str = "sutradhara", capacity_blocks: int = 8192,
           block_size: int = 16, workload: str = "default", gen: Optional[Sequence[float]] = None,
           cost: Optional[Sequence[float]] = None, device: int = 0) -> ReplayResult:
    out = [np.zeros(n_requests, np.int64) for _ in range(4)]
    ev = C.c_uint64(0)
    g = (C.c_double * 8)(*(list(gen) + [0.0] * (8 - len(gen)))) if gen is not None else None
    cst = (C.c_double * 4)(*cost) if cost is not None else None
    st = _lib.lib().sb_replay_generated(workload.encode(), g, n_requests, seed, PRESETS[preset], capacity_blocks,
                                        block_size, cst, device, *(o.ctypes.data_as(_lib.I64P) for o in out),
                                        C.byref(ev))
    _lib.check(st, "replay")
    return ReplayResult(out[0], out[1], out[2], out[3], int(ev.value))
