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


@dataclass
class DenseShape:
    """Dense layers of a Llama-3-style decoder around the paged attention."""
    n_layers: int = 32
    d_model: int = 4096
    n_q_heads: int = 32
    n_kv_heads: int = 8
    d_ff: int = 14336
    vocab: int = 128256
    rope_theta: float = 500000.0


LLAMA3_8B_DENSE = DenseShape()


class DenseModel:
    """Binding of ``sb_model`` (csrc/model.cu): seeded random-init bf16
    weights of a Llama-3-shaped decoder; attach it to a ContinuationBatch to
    run the real layers (QKV/O/MLP GEMMs on cuBLAS, RMSNorm/RoPE/SwiGLU and
    the paged attention in our kernels) instead of the stand-in projections."""

    def __init__(self, shape: DenseShape, seed: int = 0, device: int = 0):
        self.shape = shape
        self._L = _lib.lib()
        h = C.c_void_p()
        _lib.check(self._L.sb_model_create(shape.n_layers, shape.d_model, shape.n_q_heads, shape.n_kv_heads,
                                           shape.d_ff, shape.vocab, shape.rope_theta, seed, device, C.byref(h)),
                   "model")
        self._h = h

    def weight(self, layer: int, which: int):
        """(device pointer, element count) of a bf16 weight (see sb_model_weight)."""
        ptr, n = C.c_void_p(), C.c_int64()
        _lib.check(self._L.sb_model_weight(self._h, layer, which, C.byref(ptr), C.byref(n)), "weight")
        return ptr.value, n.value

    def close(self):
        if getattr(self, "_h", None):
            self._L.sb_model_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
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
    """Binding of the C++ continuation engine (csrc/engine.cu, ``sb_engine_*``)."""

    def __init__(self, shape: ModelShape, capacity_blocks: int, policy: int = TIERED, block_size: int = 16,
                 device: int = 0, seed: int = 0):
        assert block_size == 16, "KV pages are 16 tokens"
        self.shape = shape
        self.bs = block_size
        self.capacity = capacity_blocks
        self.device_index = device
        self._L = _lib.lib()
        h = C.c_void_p()
        _lib.check(self._L.sb_engine_create(shape.n_layers, shape.n_q_heads, shape.n_kv_heads, shape.head_dim,
                                            capacity_blocks, policy, device, seed, C.byref(h)), "engine")
        self._h = h
        self.cache = KvCache.__new__(KvCache)  # non-owning view of the engine's pool
        self.cache.config = CacheConfig(block_size, capacity_blocks, policy)
        self.cache._h = C.c_void_p(self._L.sb_engine_cache(h))
        self.cache._L = self._L
        self.cache._owner = False

    def close(self):
        if getattr(self, "_h", None):
            self.cache._h = None
            self._L.sb_engine_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def k_pool(self, layer: int):
        return self._L.sb_engine_k_pool(self._h, layer)

    def v_pool(self, layer: int):
        return self._L.sb_engine_v_pool(self._h, layer)

    # ---------------------------------------------------------------- API
    def submit_partial_prefill(self, prefix_tokens: np.ndarray, tags, now: int) -> PartialHandle:
        t = np.ascontiguousarray(prefix_tokens, dtype=np.uint64)
        arr = (_lib.TagRange * max(len(tags), 1))()
        for i, (b, e, tg) in enumerate(tags):
            arr[i].begin, arr[i].end, arr[i].tag = int(b), int(e), int(tg)
        hid = C.c_int32(0)
        _lib.check(self._L.sb_engine_submit_partial(self._h, t.ctypes.data_as(_lib.U64P), len(t), arr, len(tags), now,
                                                    C.byref(hid)), "submit_partial_prefill")
        ids = np.zeros((len(t) + 15) // 16, dtype=np.int32)
        n = C.c_int64(0)
        _lib.check(self._L.sb_engine_partial_blocks(self._h, hid.value, ids.ctypes.data_as(_lib.I32P), len(ids),
                                                    C.byref(n)))
        return PartialHandle(hid.value, t, list(tags), ids[: n.value].tolist())

    def prefill_partials(self, handles: Sequence[PartialHandle], model: "DenseModel"):
        """Run the model over the uncached part of each partial prefix (the
        prefill that overlaps the tool call), writing its K/V into the pinned
        pages (``sb_engine_prefill_partials``)."""
        hid = np.array([h.call_id for h in handles], dtype=np.int32)
        _lib.check(self._L.sb_engine_prefill_partials(self._h, model._h, hid.ctypes.data_as(_lib.I32P), len(hid),
                                                      ContinuationBatch._stream()), "prefill_partials")

    def cached_at_submit(self, handle: PartialHandle) -> int:
        n = C.c_int64(0)
        _lib.check(self._L.sb_engine_partial_cached(self._h, handle.call_id, C.byref(n)), "partial_cached")
        return n.value

    def abandon_partial(self, handle: PartialHandle):
        _lib.check(self._L.sb_engine_abandon_partial(self._h, handle.call_id), "abandon_partial")

    def make_batch(self, handles: Sequence[PartialHandle], suffix_lens: Sequence[int]) -> "ContinuationBatch":
        return ContinuationBatch(self, list(handles), list(suffix_lens))


class ContinuationBatch:
    """A batch of extend_prefill continuations (``sb_batch_*``)."""

    def __init__(self, eng: ContinuationEngine, handles: List[PartialHandle], suffix_lens: List[int]):
        self.eng = eng
        self._L = eng._L
        self.n = len(handles)
        hid = np.array([h.call_id for h in handles], dtype=np.int32)
        sl = np.array(suffix_lens, dtype=np.int64)
        h = C.c_void_p()
        _lib.check(self._L.sb_batch_create(eng._h, hid.ctypes.data_as(_lib.I32P), sl.ctypes.data_as(_lib.I64P),
                                           self.n, C.byref(h)), "batch")
        self._h = h
        self.prefix_lens = [len(x.tokens) for x in handles]
        self.suffix_lens = list(suffix_lens)
        self.full_lens = [p + s for p, s in zip(self.prefix_lens, self.suffix_lens)]
        self.blk_off_h = np.cumsum([0] + [(n + 15) // 16 for n in self.full_lens]).astype(np.int64)
        tq, tb, pt, fl, out = C.c_int64(), C.c_int64(), C.c_int64(), C.c_double(), C.c_void_p()
        self._L.sb_batch_info(h, C.byref(tq), C.byref(tb), C.byref(pt), C.byref(fl), C.byref(out))
        self.total_q, self.total_blocks, self.prompt_tokens = tq.value, tb.value, pt.value
        self._flops = fl.value
        self.out_ptr = out.value
        self.launches_per_step = None

    def close(self):
        if getattr(self, "_h", None):
            self._L.sb_batch_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @staticmethod
    def _stream():
        import torch

        return C.c_void_p(torch.cuda.current_stream().cuda_stream)

    def stage_suffix_host(self, host_suffix) -> int:
        """H2D of this step's suffix tokens (pinned host tensor/array [total_q])."""
        ptr = host_suffix.data_ptr() if hasattr(host_suffix, "data_ptr") else host_suffix.ctypes.data
        _lib.check(self._L.sb_batch_stage_suffix(self._h, C.c_void_p(ptr), 0, self._stream()), "stage_suffix")
        return self.total_q * 8

    def stage_suffix_device(self, dev_suffix) -> int:
        _lib.check(self._L.sb_batch_stage_suffix(self._h, C.c_void_p(dev_suffix.data_ptr()), 1, self._stream()),
                   "stage_suffix")
        return 0

    def run(self, now: int, seed: int, time_attention: bool = False) -> int:
        n = C.c_int32(0)
        _lib.check(self._L.sb_batch_run(self._h, now, seed, int(time_attention), self._stream(), C.byref(n)), "run")
        self.launches_per_step = n.value
        return n.value

    def attention_ms(self) -> List[float]:
        out = (C.c_float * self.eng.shape.n_layers)()
        _lib.check(self._L.sb_batch_attention_ms(self._h, out))
        return list(out)

    def results(self):
        hits = np.zeros(self.n, np.int64)
        st = np.zeros(self.n, np.int32)
        ids = np.zeros(self.total_blocks, np.int32)
        _lib.check(self._L.sb_batch_results(self._h, hits.ctypes.data_as(_lib.I64P), st.ctypes.data_as(_lib.I32P),
                                            ids.ctypes.data_as(_lib.I32P), self._stream()))
        return hits, st, ids

    def output_sample(self, host_buf, n_rows: int = 1) -> int:
        """Async D2H of the last n_rows query rows of the last layer's attention
        output into a pinned host buffer; returns bytes copied."""
        sh = self.eng.shape
        nbytes = n_rows * sh.n_q_heads * sh.head_dim * 2
        _lib.check(self._L.sb_batch_copy_output(self._h, self.total_q - n_rows, n_rows, C.c_void_p(host_buf.data_ptr()),
                                                self._stream()), "copy_output")
        return nbytes

    def attention_flops(self) -> float:
        return self._flops

    def set_model(self, model: Optional["DenseModel"]):
        """Run the real dense layers around the attention (None: stand-ins)."""
        self._model = model  # keep the weights alive while attached
        _lib.check(self._L.sb_batch_set_model(self._h, model._h if model is not None else None), "set_model")

    def model_result(self, logits: bool = False):
        """Greedy next token per sequence (and fp32 last-token logits)."""
        nxt = np.zeros(self.n, np.int32)
        lg = np.zeros((self.n, self._model.shape.vocab), np.float32) if logits else None
        _lib.check(self._L.sb_batch_model_result(self._h, nxt.ctypes.data_as(_lib.I32P),
                                                 lg.ctypes.data_as(C.POINTER(C.c_float)) if logits else None,
                                                 self._stream()), "model_result")
        return (nxt, lg) if logits else nxt

    def dense_flops(self) -> float:
        f = C.c_double()
        self._L.sb_batch_dense_flops(self._h, C.byref(f))
        return f.value
