"""Continuation-prefill attention over the paged KV pool (csrc/attention.cu).

The suffix tokens of each sequence (the tool-output segment spliced by
``extend_prefill``, /root/reference/proj/src/engine.cpp:184-223) attend to the
sequence's cached prefix pages plus causally to themselves.  torch is used
only to hold device memory; the compute is the sm_100a kernel.

Layouts (bf16):
  q, out            [total_q, n_q_heads, 128]  (suffix tokens, packed)
  k_pool, v_pool    [n_pool_blocks, n_kv_heads, 16, 128]
  q_offsets         int32 [n_seqs + 1]  token offsets into q
  kv_lens           int32 [n_seqs]      prefix + suffix length
  block_table       int32 [n_seqs, max_blocks]  pool page of key positions
"""
from __future__ import annotations

import ctypes as C
import math
from typing import Optional

from . import _lib


def _ptr(t):
    return C.c_void_p(t.data_ptr())


def _stream_ptr(stream):
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


def attention_work_list(q_lens, kv_lens, n_q_heads: int, n_kv_heads: int):
    """LPT-ordered work items (host int32 array [n, 2]) for continuation_attention."""
    import numpy as np

    qo = np.cumsum([0] + list(q_lens)).astype(np.int32)
    kl = np.asarray(kv_lens, dtype=np.int32)
    tpt = 128 // (n_q_heads // n_kv_heads)
    cap = int(sum(-(-q // (2 * tpt)) for q in q_lens)) * n_kv_heads + 1
    out = np.zeros(2 * cap, dtype=np.int32)
    n = C.c_int32(0)
    _lib.check(_lib.lib().sb_attention_work_list(qo.ctypes.data_as(_lib.I32P), kl.ctypes.data_as(_lib.I32P), len(q_lens),
                                                 n_q_heads, n_kv_heads, out.ctypes.data_as(_lib.I32P), cap, C.byref(n)),
               "attention_work_list")
    return out[: 2 * n.value].reshape(-1, 2)


def continuation_attention(q, k_pool, v_pool, q_offsets, kv_lens, block_table, max_q_len: int,
                           softmax_scale: Optional[float] = None, out=None, stream=None, work=None):
    """work: optional device int32 tensor from attention_work_list (LPT order)."""
    import torch

    assert q.is_contiguous() and k_pool.is_contiguous() and v_pool.is_contiguous()
    if q.dtype == torch.float32:  # fp32 contract (CUDA-core kernel, 1e-5 of an fp32 reference)
        assert k_pool.dtype == torch.float32 and v_pool.dtype == torch.float32
        total_q, n_q_heads, head_dim = q.shape
        n_blocks, n_kv_heads, page, _ = k_pool.shape
        out = torch.empty_like(q) if out is None else out
        scale = 1.0 / math.sqrt(head_dim) if softmax_scale is None else softmax_scale
        _lib.check(_lib.lib().sb_continuation_attention_f32(
            _ptr(q), _ptr(k_pool), _ptr(v_pool), _ptr(out), _ptr(q_offsets), _ptr(kv_lens), _ptr(block_table),
            kv_lens.numel(), block_table.shape[1], total_q, n_q_heads, n_kv_heads, head_dim, page,
            C.c_float(scale), _stream_ptr(stream)), "continuation_attention_f32")
        return out
    assert q.dtype == torch.bfloat16 and k_pool.dtype == torch.bfloat16 and v_pool.dtype == torch.bfloat16
    total_q, n_q_heads, head_dim = q.shape
    n_blocks, n_kv_heads, page, hd2 = k_pool.shape
    assert hd2 == head_dim and tuple(v_pool.shape) == tuple(k_pool.shape)
    if out is None:
        out = torch.empty_like(q)
    if softmax_scale is None:
        softmax_scale = 1.0 / math.sqrt(head_dim)
    n_seqs = kv_lens.numel()
    st = _lib.lib().sb_continuation_attention(
        _ptr(q), _ptr(k_pool), _ptr(v_pool), _ptr(out), _ptr(q_offsets), _ptr(kv_lens), _ptr(block_table), n_seqs,
        block_table.shape[1], max_q_len, total_q, n_q_heads, n_kv_heads, head_dim, page, n_blocks,
        C.c_float(softmax_scale), _ptr(work) if work is not None else None,
        int(work.shape[0]) if work is not None else 0, _stream_ptr(stream))
    _lib.check(st, "continuation_attention")
    return out


def kv_append(k_new, v_new, k_pool, v_pool, q_offsets, kv_lens, block_table, stream=None):
    n_blocks, n_kv_heads, page, head_dim = k_pool.shape
    st = _lib.lib().sb_kv_append(_ptr(k_new), _ptr(v_new), _ptr(k_pool), _ptr(v_pool), _ptr(q_offsets), _ptr(kv_lens),
                                 _ptr(block_table), kv_lens.numel(), block_table.shape[1], n_kv_heads, head_dim, page,
                                 _stream_ptr(stream))
    _lib.check(st, "kv_append")


def attention_flops(q_lens, kv_lens, n_q_heads: int, head_dim: int = 128) -> float:
    """Algorithmic FLOPs: 4 * head_dim * n_q_heads * sum over queries of the
    number of keys each query attends to (QK^T and PV, causal suffix)."""
    total = 0
    for ql, kl in zip(q_lens, kv_lens):
        prefix = kl - ql
        total += ql * prefix + ql * (ql + 1) // 2
    return 4.0 * head_dim * n_q_heads * total
