"""Tool-aware split prefill on one B200: the engine side of Sutradhara's
prompt splitting (paper §4.2) over the device block pool and the
continuation-prefill attention kernel.

Mirrors the reference engine's continuation API
(/root/reference/proj/include/agentsim/engine.hpp:110-135):

* ``submit_partial_prefill`` — insert the tool-independent prefix into the
  block pool and pin it at the PARTIAL_PREFILL tier (Engine::pin_partial,
  engine.cpp:250-286).  Its KV pages are produced by the (untimed) eager
  prefill while the tool runs.
* ``extend_prefill_batch`` — the hot path: for a batch of continuations,
  chain-hash the full prompts, look up the cached prefix (the admission
  lookup of engine.cpp:170), insert the prompt (hits on the pinned prefix,
  new blocks for the tool outputs, hint-aware eviction under pool pressure:
  Engine::complete_prefill, engine.cpp:305-322), scatter the suffix K/V into
  the new pages and run the continuation attention layer by layer; the
  call's block references are released at the end (engine.cpp:343-346).
* ``abandon_partial`` — unpin (engine.cpp:234-248).

All device work is issued on one CUDA stream with no host round trip; torch
only provides device memory.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass
from typing import List, Optional, Sequence

import numpy as np

import os

from . import _lib
from .kv_cache import PARTIAL_PREFILL, TIERED, TOOL_OUTPUT, CacheConfig, KvCache


@dataclass
class ModelShape:
    n_layers: int = 32
    n_q_heads: int = 32
    n_kv_heads: int = 8
    head_dim: int = 128

    @property
    def kv_bytes_per_token(self) -> int:  # K + V, all layers, bf16
        return 2 * self.n_layers * self.n_kv_heads * self.head_dim * 2


_DEBUG = os.environ.get("SB_DEBUG", "0") == "1"

LLAMA3_8B = ModelShape(32, 32, 8, 128)
TOY_2L_256 = ModelShape(2, 2, 1, 128)  # configs[0]: 2 layers, d_model = 2 x 128


def _p(t):
    return C.c_void_p(t.data_ptr())


@dataclass
class PartialHandle:
    """ContinuationHandle (engine.hpp:72) + the pinned prefix it owns."""
    call_id: int
    tokens: np.ndarray
    tags: list
    block_ids: List[int]


class ContinuationEngine:
    def __init__(self, shape: ModelShape, capacity_blocks: int, policy: int = TIERED, block_size: int = 16,
                 device: int = 0, seed: int = 0):
        import torch

        assert block_size == 16, "KV pages are 16 tokens"
        self.shape = shape
        self.bs = block_size
        self.device = torch.device("cuda", device)
        self.cache = KvCache(CacheConfig(block_size, capacity_blocks, policy), device)
        self.capacity = capacity_blocks
        L = _lib.lib()
        self._L = L
        # one K and one V page pool per layer: [pages, kv_heads, 16, head_dim] bf16
        shp = (capacity_blocks, shape.n_kv_heads, block_size, shape.head_dim)
        self.k_pools = [torch.empty(shp, dtype=torch.bfloat16, device=self.device) for _ in range(shape.n_layers)]
        self.v_pools = [torch.empty(shp, dtype=torch.bfloat16, device=self.device) for _ in range(shape.n_layers)]
        stream = self._stream()
        for li in range(shape.n_layers):
            # stand-in for the KV the eager prefill wrote (random-init model)
            _lib.check(L.sb_fill_random_bf16(_p(self.k_pools[li]), self.k_pools[li].numel(), seed * 131 + 2 * li, 1.0,
                                             stream))
            _lib.check(L.sb_fill_random_bf16(_p(self.v_pools[li]), self.v_pools[li].numel(), seed * 131 + 2 * li + 1,
                                             1.0, stream))
        self._next_call = 1

    def _stream(self):
        import torch

        return C.c_void_p(torch.cuda.current_stream(self.device).cuda_stream)

    # ---------------------------------------------------------------- API
    def submit_partial_prefill(self, prefix_tokens: np.ndarray, tags, now: int) -> PartialHandle:
        ids = self.cache.insert(prefix_tokens, tags, now)
        self.cache.set_reuse_priority(ids, pinned=True, tier_override=PARTIAL_PREFILL)
        h = PartialHandle(self._next_call, prefix_tokens, list(tags), ids)
        self._next_call += 1
        return h

    def abandon_partial(self, handle: PartialHandle):
        self.cache.set_reuse_priority(handle.block_ids, pinned=False)
        self.cache.release(handle.block_ids)

    def make_batch(self, handles: Sequence[PartialHandle], suffix_lens: Sequence[int]) -> "ContinuationBatch":
        return ContinuationBatch(self, list(handles), list(suffix_lens))


class ContinuationBatch:
    """Static device layout of one batch of continuations (prefix + suffix per
    request); ``run`` executes one extend_prefill step for new suffix tokens."""

    def __init__(self, eng: ContinuationEngine, handles: List[PartialHandle], suffix_lens: List[int]):
        import torch

        self.eng = eng
        dev = eng.device
        bs = eng.bs
        self.n = len(handles)
        self.prefix_lens = [len(h.tokens) for h in handles]
        for pl in self.prefix_lens:
            assert pl % bs == 0, "tool-independent prefix must end on a block boundary"
        self.suffix_lens = list(suffix_lens)
        self.full_lens = [p + s for p, s in zip(self.prefix_lens, self.suffix_lens)]
        self.seq_off_h = np.cumsum([0] + self.full_lens).astype(np.int64)
        self.blk_off_h = np.cumsum([0] + [(n + bs - 1) // bs for n in self.full_lens]).astype(np.int64)
        self.total_blocks = int(self.blk_off_h[-1])
        self.max_blocks = int(max((n + bs - 1) // bs for n in self.full_lens))
        self.total_q = int(sum(self.suffix_lens))
        self.max_q = int(max(self.suffix_lens))
        # packed prompt tokens; prefixes are static, suffix slots rewritten per step
        toks = np.zeros(int(self.seq_off_h[-1]), dtype=np.uint64)
        tag_list, tag_off = [], [0]
        for i, h in enumerate(handles):
            a = int(self.seq_off_h[i])
            toks[a:a + len(h.tokens)] = h.tokens
            tg = [tuple(t) for t in h.tags] + [(self.prefix_lens[i], self.full_lens[i], TOOL_OUTPUT)]
            tag_list += tg
            tag_off.append(len(tag_list))
        self.tokens = torch.from_numpy(toks.view(np.int64)).to(dev)
        self.seq_off = torch.from_numpy(self.seq_off_h).to(dev)
        self.blk_off = torch.from_numpy(self.blk_off_h).to(dev)
        tag_arr = (_lib.TagRange * len(tag_list))()
        for i, (b, e, t) in enumerate(tag_list):
            tag_arr[i].begin, tag_arr[i].end, tag_arr[i].tag = b, e, t
        self.tags = torch.frombuffer(bytearray(tag_arr), dtype=torch.uint8).to(dev)
        self.tag_off = torch.tensor(tag_off, dtype=torch.int64, device=dev)
        self.hashes = torch.empty(self.total_blocks, dtype=torch.int64, device=dev)
        self.ids = torch.empty(self.total_blocks, dtype=torch.int32, device=dev)
        self.status = torch.empty(self.n, dtype=torch.int32, device=dev)
        self.hits = torch.empty(self.n, dtype=torch.int64, device=dev)
        self.table = torch.empty((self.n, self.max_blocks), dtype=torch.int32, device=dev)
        self.q_off = torch.tensor(np.cumsum([0] + self.suffix_lens), dtype=torch.int32, device=dev)
        self.kv_lens = torch.tensor(self.full_lens, dtype=torch.int32, device=dev)
        sh = eng.shape
        self.q = torch.empty((self.total_q, sh.n_q_heads, sh.head_dim), dtype=torch.bfloat16, device=dev)
        self.k_new = torch.empty((self.total_q, sh.n_kv_heads, sh.head_dim), dtype=torch.bfloat16, device=dev)
        self.v_new = torch.empty_like(self.k_new)
        self.out = torch.empty_like(self.q)
        # suffix slots: (offset in packed tokens, length, offset in packed suffix)
        so = np.cumsum([0] + self.suffix_lens)
        self.slots = [(int(self.seq_off_h[i]) + self.prefix_lens[i], self.suffix_lens[i], int(so[i]))
                      for i in range(self.n)]
        self.suffix_dev = torch.empty(self.total_q, dtype=torch.int64, device=dev)
        self.scale = 1.0 / math.sqrt(sh.head_dim)
        from .attention import attention_work_list

        w = attention_work_list(self.suffix_lens, self.full_lens, sh.n_q_heads, sh.n_kv_heads)
        self.work = torch.from_numpy(w.copy()).to(dev)
        self.n_work = int(w.shape[0])
        self.launches_per_step = None

    def stage_suffix_host(self, host_suffix) -> int:
        """H2D of this step's suffix tokens (pinned host tensor [total_q] int64)
        into their prompt slots.  Returns bytes copied."""
        self.suffix_dev.copy_(host_suffix, non_blocking=True)
        return self._scatter_suffix()

    def stage_suffix_device(self, dev_suffix) -> int:
        self.suffix_dev.copy_(dev_suffix)
        return self._scatter_suffix()

    def _scatter_suffix(self) -> int:
        for (a, n, s) in self.slots:
            self.tokens[a:a + n].copy_(self.suffix_dev[s:s + n], non_blocking=True)
        return self.total_q * 8

    def run(self, now: int, seed: int, attn_events: Optional[list] = None) -> int:
        """One continuation-prefill step.  Returns the number of library kernel
        launches issued."""
        import torch

        eng, L = self.eng, self.eng._L
        st = eng._stream()
        h_blk = self.blk_off_h.ctypes.data_as(_lib.I64P)
        launches = 0
        # 1. chain hashes of every block of every prompt (sequential fold per
        #    sequence, all sequences in parallel)
        _lib.check(L.sb_chain_hash_batch(_p(self.tokens), _p(self.seq_off), _p(self.blk_off), None, self.n, eng.bs,
                                         _p(self.hashes), st), "chain_hash")
        launches += 1
        # 2. admission lookup of the cached prefix (engine.cpp:170)
        _lib.check(L.sb_kv_lookup_prefix_batch(eng.cache.handle, _p(self.tokens), _p(self.seq_off), _p(self.blk_off),
                                               h_blk, _p(self.hashes), self.n, now, _p(self.hits), st), "lookup")
        launches += 3
        # 3. insert the full prompt: prefix hits, new tool-output blocks,
        #    hint-aware eviction (engine.cpp:305-322)
        _lib.check(L.sb_kv_insert_batch(eng.cache.handle, _p(self.tokens), _p(self.seq_off), _p(self.tags),
                                        _p(self.tag_off), _p(self.blk_off), h_blk, _p(self.hashes), self.n, now,
                                        _p(self.ids), _p(self.status), st), "insert")
        launches += 5 * self.n
        _lib.check(L.sb_build_block_table(_p(self.ids), _p(self.blk_off), self.n, self.max_blocks, _p(self.table), st))
        launches += 1
        if _DEBUG:
            torch.cuda.synchronize()
            tb = self.table.cpu().numpy()
            bad = np.argwhere((tb < -1) | (tb >= eng.capacity))
            assert len(bad) == 0, f"block table out of range at {bad[:5].tolist()}: {tb[tuple(bad[0])]}"
            stt = self.status.cpu().numpy()
            for i in range(self.n):
                nb = int(self.blk_off_h[i + 1] - self.blk_off_h[i])
                row = tb[i, :nb]
                assert (row >= 0).all() if stt[i] == 0 else (row == -1).all(), (i, stt[i], row[:8])
        # 4. per layer: projections (random-init stand-in), KV append, attention
        sh = eng.shape
        for li in range(sh.n_layers):
            base = (seed * 1000003 + li) * 3
            _lib.check(L.sb_fill_random_bf16(_p(self.q), self.q.numel(), base, 1.0, st))
            _lib.check(L.sb_fill_random_bf16(_p(self.k_new), self.k_new.numel(), base + 1, 1.0, st))
            _lib.check(L.sb_fill_random_bf16(_p(self.v_new), self.v_new.numel(), base + 2, 1.0, st))
            _lib.check(L.sb_kv_append(_p(self.k_new), _p(self.v_new), _p(eng.k_pools[li]), _p(eng.v_pools[li]),
                                      _p(self.q_off), _p(self.kv_lens), _p(self.table), self.n, self.max_blocks,
                                      sh.n_kv_heads, sh.head_dim, eng.bs, st), "kv_append")
            ev = None
            if attn_events is not None:
                ev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                ev[0].record()
            _lib.check(L.sb_continuation_attention(_p(self.q), _p(eng.k_pools[li]), _p(eng.v_pools[li]), _p(self.out),
                                                   _p(self.q_off), _p(self.kv_lens), _p(self.table), self.n,
                                                   self.max_blocks, self.max_q, self.total_q, sh.n_q_heads,
                                                   sh.n_kv_heads, sh.head_dim, eng.bs, eng.capacity,
                                                   C.c_float(self.scale), _p(self.work), self.n_work, st),
                       "attention")
            if ev is not None:
                ev[1].record()
                attn_events.append(ev)
            launches += 5
        # 5. drop the call's block references (engine.cpp:343-346)
        _lib.check(L.sb_kv_release_batch(eng.cache.handle, _p(self.ids), self.total_blocks, None, st), "release")
        launches += 3
        self.launches_per_step = launches
        return launches

    def attention_flops(self) -> float:
        from .attention import attention_flops

        return attention_flops(self.suffix_lens, self.full_lens, self.eng.shape.n_q_heads, self.eng.shape.head_dim)
