"""Tool-aware split prefill on one B200: the engine side of Sutradhara's
prompt splitting (paper §4.2) over the device block pool and the
continuation-prefill attention kernel.

Mirrors the reference engine's call lifecycle
(/root/reference/proj/include/agentsim/engine.hpp:104-111, src/engine.cpp):

* ``submit_call`` / ``submit_partial_prefill`` — admission lookup of the
  prompt (engine.cpp:128-182);
* ``prefill_done`` — Engine::complete_prefill (engine.cpp:305-322): a partial
  not yet extended is pinned at PARTIAL_PREFILL with shared pin counts and
  remembered real tags (pin_partial, engine.cpp:250-286), else the prompt is
  inserted, the pins released (engine.cpp:288-303) and the old refs dropped;
* ``extend_prefill`` (engine.cpp:184-223), ``abandon_partial``
  (engine.cpp:234-248), ``finish_decode`` (engine.cpp:324-347).

Every KV transition is one op of the block pool's device op program.  The
hot path is ``ContinuationBatch``: one ``run`` is the whole lifecycle of a
batch of agentic continuations (admission lookups, pins, extension,
complete with hint-aware eviction, per layer KV append + tcgen05 attention,
finish), each transition one op program over the batch.
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


class ContinuationEngine:
    """Binding of the C++ continuation engine (csrc/engine.cu, ``sb_engine_*``)."""

    # agentsim::CallState (engine.hpp:35)
    QUEUED, PREFILLING, AWAITING_EXTENSION, DECODING, DONE, ABORTED = range(6)
    PINNED, PIN_FAILED, COMPLETED = 1, 2, 3

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

    @staticmethod
    def _tags(tags):
        arr = (_lib.TagRange * max(len(tags), 1))()
        for i, (b, e, tg) in enumerate(tags):
            arr[i].begin, arr[i].end, arr[i].tag = int(b), int(e), int(tg)
        return arr

    # ------------------------------------------------------------ lifecycle
    def submit_call(self, tokens, tags, decode_length: int, now: int) -> int:
        t = np.ascontiguousarray(tokens, dtype=np.uint64)
        out = C.c_int32(0)
        _lib.check(self._L.sb_engine_submit_call(self._h, t.ctypes.data_as(_lib.U64P), len(t), self._tags(tags),
                                                 len(tags), decode_length, now, C.byref(out)), "submit_call")
        return out.value

    def submit_partial_prefill(self, prefix_tokens, tags, now: int) -> int:
        t = np.ascontiguousarray(prefix_tokens, dtype=np.uint64)
        out = C.c_int32(0)
        _lib.check(self._L.sb_engine_submit_partial(self._h, t.ctypes.data_as(_lib.U64P), len(t), self._tags(tags),
                                                    len(tags), now, C.byref(out)), "submit_partial_prefill")
        return out.value

    def prefill_done(self, call: int, now: int) -> int:
        """The call's prefill finished: pin (partial) or complete.  Returns
        PINNED / PIN_FAILED / COMPLETED."""
        out = C.c_int32(0)
        _lib.check(self._L.sb_engine_prefill_done(self._h, call, now, C.byref(out)), "prefill_done")
        return out.value

    def extend_prefill(self, call: int, suffix, tags, decode_length: int, now: int) -> bool:
        t = np.ascontiguousarray(suffix, dtype=np.uint64)
        done = C.c_int32(0)
        _lib.check(self._L.sb_engine_extend(self._h, call, t.ctypes.data_as(_lib.U64P), len(t), self._tags(tags),
                                            len(tags), decode_length, now, C.byref(done)), "extend_prefill")
        return bool(done.value)

    def abandon_partial(self, call: int):
        _lib.check(self._L.sb_engine_abandon_partial(self._h, call), "abandon_partial")

    def finish_decode(self, call: int, response, now: int):
        t = np.ascontiguousarray(response, dtype=np.uint64)
        _lib.check(self._L.sb_engine_finish(self._h, call, t.ctypes.data_as(_lib.U64P), len(t), now), "finish_decode")

    def call_info(self, call: int) -> dict:
        st, cached, prompt, nc, npn = C.c_int32(), C.c_int64(), C.c_int64(), C.c_int32(), C.c_int32()
        _lib.check(self._L.sb_engine_call_info(self._h, call, C.byref(st), C.byref(cached), C.byref(prompt),
                                               C.byref(nc), C.byref(npn)), "call_info")
        return {"state": st.value, "cached_prefix": cached.value, "prompt_tokens": prompt.value,
                "n_chain": nc.value, "n_pinned": npn.value}

    def call_blocks(self, call: int, pinned: bool = False) -> List[int]:
        info = self.call_info(call)
        n = info["n_pinned" if pinned else "n_chain"]
        out = np.zeros(max(n, 1), np.int32)
        got = C.c_int64(0)
        _lib.check(self._L.sb_engine_call_blocks(self._h, call, int(pinned), out.ctypes.data_as(_lib.I32P), len(out),
                                                 C.byref(got)))
        return out[: got.value].tolist()

    def cached_at_submit(self, call: int) -> int:
        return self.call_info(call)["cached_prefix"]

    def prefill_partials(self, calls: Sequence[int], model: "DenseModel"):
        """Run the model over the uncached part of each pinned partial prefix
        (the prefill that overlaps the tool call), writing its K/V into the
        pinned pages (``sb_engine_prefill_partials``)."""
        hid = np.array(list(calls), dtype=np.int32)
        _lib.check(self._L.sb_engine_prefill_partials(self._h, model._h, hid.ctypes.data_as(_lib.I32P), len(hid),
                                                      ContinuationBatch._stream()), "prefill_partials")

    def make_batch(self, prefixes: Sequence[np.ndarray], prefix_tags: Sequence[list], suffix_lens: Sequence[int],
                   stream_keys: Optional[Sequence[int]] = None) -> "ContinuationBatch":
        return ContinuationBatch(self, list(prefixes), list(prefix_tags), list(suffix_lens), stream_keys)


class ContinuationBatch:
    """A batch of agentic continuations run through the engine lifecycle per
    step (``sb_batch_*``): slot i has a fixed tool-independent prefix and a
    fixed tool-output length; every ``run`` is n new calls."""

    def __init__(self, eng: ContinuationEngine, prefixes, prefix_tags, suffix_lens, stream_keys=None):
        self.eng = eng
        self._L = eng._L
        self.n = len(prefixes)
        toks = np.ascontiguousarray(np.concatenate([np.asarray(p, np.uint64) for p in prefixes]), dtype=np.uint64)
        off = np.cumsum([0] + [len(p) for p in prefixes]).astype(np.int64)
        flat = [t for tg in prefix_tags for t in tg]
        toff = np.cumsum([0] + [len(tg) for tg in prefix_tags]).astype(np.int64)
        sl = np.array(suffix_lens, dtype=np.int64)
        keys = np.array(stream_keys, dtype=np.uint64) if stream_keys is not None else None
        h = C.c_void_p()
        _lib.check(self._L.sb_batch_create(eng._h, self.n, toks.ctypes.data_as(_lib.U64P), off.ctypes.data_as(_lib.I64P),
                                           ContinuationEngine._tags(flat), toff.ctypes.data_as(_lib.I64P),
                                           sl.ctypes.data_as(_lib.I64P),
                                           keys.ctypes.data_as(_lib.U64P) if keys is not None else None, C.byref(h)),
                   "batch")
        self._h = h
        self.prefix_lens = [len(p) for p in prefixes]
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

    def run(self, now: int, seed: int = 0, time_attention: bool = False) -> int:
        n = C.c_int32(0)
        _lib.check(self._L.sb_batch_run(self._h, now, seed, int(time_attention), self._stream(), C.byref(n)), "run")
        self.launches_per_step = n.value
        return n.value

    def attention_ms(self) -> List[float]:
        out = (C.c_float * self.eng.shape.n_layers)()
        _lib.check(self._L.sb_batch_attention_ms(self._h, out))
        return list(out)

    def pool_ms(self) -> List[float]:
        """Pool-side phases of the last timed run: [submit + pin, extend +
        complete, finish] in ms (CUDA events on the batch's stream)."""
        out = (C.c_float * 3)()
        _lib.check(self._L.sb_batch_pool_ms(self._h, out))
        return list(out)

    def results(self):
        """(admission hits [n], complete statuses [n], chains the continuation
        attended over [total_blocks] laid out by blk_off_h)."""
        hits = np.zeros(self.n, np.int64)
        st = np.zeros(self.n, np.int32)
        ids = np.zeros(self.total_blocks, np.int32)
        _lib.check(self._L.sb_batch_results(self._h, hits.ctypes.data_as(_lib.I64P), st.ctypes.data_as(_lib.I32P),
                                            ids.ctypes.data_as(_lib.I32P), self._stream()))
        return hits, st, ids

    def pin_outcomes(self) -> np.ndarray:
        out = np.zeros(self.n, np.int32)
        _lib.check(self._L.sb_batch_pin_outcomes(self._h, out.ctypes.data_as(_lib.I32P)))
        return out

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
