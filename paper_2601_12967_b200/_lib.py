"""Loader for the in-tree sm_100a library (paper_2601_12967_b200/_build).

No fallback: if the CUDA library is missing the import of any op fails
loudly with the command that builds it."""
from __future__ import annotations

import ctypes as C
import os
import threading

from . import errors

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(PKG, "_build", "libsutradhara_b200.so")

_lock = threading.Lock()
_lib = None

U64P = C.POINTER(C.c_uint64)
I64P = C.POINTER(C.c_int64)
I32P = C.POINTER(C.c_int32)
VP = C.c_void_p


class TagRange(C.Structure):
    _fields_ = [("begin", C.c_int64), ("end", C.c_int64), ("tag", C.c_int32), ("_pad", C.c_int32)]


class BlockInfo(C.Structure):
    _fields_ = [("block_id", C.c_int32), ("tag", C.c_int32), ("tier", C.c_int32), ("ref_count", C.c_int32),
                ("last_used", C.c_int64), ("chain_hash", C.c_uint64), ("parent_hash", C.c_uint64),
                ("pinned", C.c_int32), ("n_tokens", C.c_int32)]


# name -> (restype, argtypes); mirrors include/sutradhara_b200.h
SIGNATURES = {
    "sb_last_error": (C.c_char_p, []),
    "sb_version": (C.c_char_p, []),
    "sb_kv_root_hash": (C.c_uint64, []),
    "sb_kv_chain_hash_host": (C.c_uint64, [C.c_uint64, U64P, C.c_int64]),
    "sb_chain_hash_batch": (C.c_int, [VP, VP, VP, VP, C.c_int32, C.c_int64, VP, VP]),
    "sb_chain_hash_segments": (C.c_int, [VP, VP, VP, VP, C.c_int32, C.c_int64, VP, VP]),
    "sb_materialize_tokens": (C.c_int, [C.c_int32, C.c_int64, C.c_uint64, C.c_int32, VP, VP]),
    "sb_decode_tokens": (C.c_int, [C.c_uint64, C.c_int64, C.c_int64, VP, VP]),
    "sb_kv_create": (C.c_int, [C.c_int64, C.c_int64, C.c_int32, C.c_int32, C.POINTER(VP)]),
    "sb_kv_destroy": (None, [VP]),
    "sb_kv_lookup_prefix": (C.c_int, [VP, U64P, C.c_int64, C.c_int64, I64P]),
    "sb_kv_insert": (C.c_int, [VP, U64P, C.c_int64, C.POINTER(TagRange), C.c_int64, C.c_int64, I32P, I64P]),
    "sb_kv_evict": (C.c_int, [VP, C.c_int64, I32P, I64P]),
    "sb_kv_set_reuse_priority": (C.c_int, [VP, I32P, C.c_int64, C.c_int32, C.c_int32]),
    "sb_kv_set_tag": (C.c_int, [VP, C.c_int32, C.c_int32]),
    "sb_kv_release": (C.c_int, [VP, I32P, C.c_int64]),
    "sb_kv_touch": (C.c_int, [VP, I32P, C.c_int64, C.c_int64]),
    "sb_kv_block_size": (C.c_int64, [VP]),
    "sb_kv_resident_blocks": (C.c_int64, [VP]),
    "sb_kv_capacity_blocks": (C.c_int64, [VP]),
    "sb_kv_free_blocks": (C.c_int64, [VP]),
    "sb_kv_total_evicted": (C.c_uint64, [VP]),
    "sb_kv_policy": (C.c_int32, [VP]),
    "sb_kv_contains": (C.c_int, [VP, C.c_int32]),
    "sb_kv_last_evicted": (C.c_int, [VP, I32P, C.c_int64, I64P]),
    "sb_kv_resident_ids": (C.c_int, [VP, I32P, I64P]),
    "sb_kv_block": (C.c_int, [VP, C.c_int32, C.POINTER(BlockInfo), U64P]),
    "sb_kv_blocks": (C.c_int, [VP, I32P, C.c_int64, C.POINTER(BlockInfo)]),
    "sb_kv_audit": (C.c_int, [VP]),
    "sb_kv_dump": (C.c_int, [VP, C.c_char_p, C.c_int64, I64P]),
    "sb_kv_lookup_prefix_batch": (C.c_int, [VP, VP, VP, VP, VP, VP, C.c_int32, C.c_int64, VP, VP]),
    "sb_kv_insert_batch": (C.c_int, [VP, VP, VP, VP, VP, VP, VP, VP, C.c_int32, C.c_int64, VP, VP, VP]),
    "sb_kv_release_batch": (C.c_int, [VP, VP, C.c_int64, VP, VP]),
    "sb_kv_stats": (C.c_int, [VP, U64P]),
    "sb_kv_program_stats": (C.c_int, [VP, U64P]),
    "sb_continuation_attention": (C.c_int, [VP, VP, VP, VP, VP, VP, VP, C.c_int32, C.c_int32, C.c_int32, C.c_int32,
                                            C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int64, C.c_float, VP,
                                            C.c_int32, VP]),
    "sb_continuation_attention_f32": (C.c_int, [VP, VP, VP, VP, VP, VP, VP, C.c_int32, C.c_int32, C.c_int32, C.c_int32,
                                                C.c_int32, C.c_int32, C.c_int32, C.c_float, VP]),
    "sb_attention_work_list": (C.c_int, [I32P, I32P, C.c_int32, C.c_int32, C.c_int32, I32P, C.c_int32, I32P]),
    "sb_build_block_table": (C.c_int, [VP, VP, C.c_int32, C.c_int32, VP, VP]),
    "sb_kv_gather_chain_hashes": (C.c_int, [VP, VP, VP, C.c_int64, VP, VP]),
    "sb_fill_random_bf16": (C.c_int, [VP, C.c_int64, C.c_uint64, C.c_float, VP]),
    "sb_engine_create": (C.c_int, [C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int64, C.c_int32, C.c_int32,
                                   C.c_uint64, C.POINTER(VP)]),
    "sb_engine_destroy": (None, [VP]),
    "sb_engine_cache": (VP, [VP]),
    "sb_engine_k_pool": (VP, [VP, C.c_int32]),
    "sb_engine_v_pool": (VP, [VP, C.c_int32]),
    "sb_engine_submit_call": (C.c_int, [VP, U64P, C.c_int64, C.POINTER(TagRange), C.c_int64, C.c_int64, C.c_int64,
                                        I32P]),
    "sb_engine_submit_partial": (C.c_int, [VP, U64P, C.c_int64, C.POINTER(TagRange), C.c_int64, C.c_int64, I32P]),
    "sb_engine_prefill_done": (C.c_int, [VP, C.c_int32, C.c_int64, I32P]),
    "sb_engine_extend": (C.c_int, [VP, C.c_int32, U64P, C.c_int64, C.POINTER(TagRange), C.c_int64, C.c_int64,
                                   C.c_int64, I32P]),
    "sb_engine_abandon_partial": (C.c_int, [VP, C.c_int32]),
    "sb_engine_finish": (C.c_int, [VP, C.c_int32, U64P, C.c_int64, C.c_int64]),
    "sb_engine_call_info": (C.c_int, [VP, C.c_int32, I32P, I64P, I64P, I32P, I32P]),
    "sb_engine_call_blocks": (C.c_int, [VP, C.c_int32, C.c_int32, I32P, C.c_int64, I64P]),
    "sb_engine_partial_blocks": (C.c_int, [VP, C.c_int32, I32P, C.c_int64, I64P]),
    "sb_batch_create": (C.c_int, [VP, C.c_int32, U64P, I64P, C.POINTER(TagRange), I64P, I64P, U64P, C.POINTER(VP)]),
    "sb_batch_pin_outcomes": (C.c_int, [VP, I32P]),
    "sb_batch_destroy": (None, [VP]),
    "sb_batch_stage_suffix": (C.c_int, [VP, VP, C.c_int32, VP]),
    "sb_batch_run": (C.c_int, [VP, C.c_int64, C.c_uint64, C.c_int32, VP, I32P]),
    "sb_batch_attention_ms": (C.c_int, [VP, C.POINTER(C.c_float)]),
    "sb_batch_pool_ms": (C.c_int, [VP, C.POINTER(C.c_float)]),
    "sb_batch_results": (C.c_int, [VP, I64P, I32P, I32P, VP]),
    "sb_batch_copy_output": (C.c_int, [VP, C.c_int64, C.c_int64, VP, VP]),
    "sb_batch_info": (C.c_int, [VP, I64P, I64P, I64P, C.POINTER(C.c_double), C.POINTER(VP)]),
    "sb_kv_append": (C.c_int, [VP, VP, VP, VP, VP, VP, VP, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int32, VP]),
    "sb_gemm_bf16": (C.c_int, [VP, VP, VP, C.c_int64, C.c_int64, C.c_int64, C.c_int32, VP]),
    "sb_model_create": (C.c_int, [C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int64, C.c_float,
                                  C.c_uint64, C.c_int32, C.POINTER(VP)]),
    "sb_model_destroy": (None, [VP]),
    "sb_model_shape": (None, [VP, I32P, I32P, I32P]),
    "sb_model_vocab": (None, [VP, I64P]),
    "sb_model_weight": (C.c_int, [VP, C.c_int32, C.c_int32, C.POINTER(VP), I64P]),
    "sb_batch_set_model": (C.c_int, [VP, VP]),
    "sb_engine_prefill_partials": (C.c_int, [VP, VP, I32P, C.c_int32, VP]),
    "sb_engine_partial_cached": (C.c_int, [VP, C.c_int32, I64P]),
    "sb_batch_model_result": (C.c_int, [VP, I32P, C.POINTER(C.c_float), VP]),
    "sb_batch_dense_flops": (C.c_int, [VP, C.POINTER(C.c_double)]),
}


def lib():
    """The loaded library (raises if it was not built)."""
    global _lib
    with _lock:
        if _lib is None:
            path = os.environ.get("SB_LIB_PATH", LIB_PATH)  # A/B runs load an alternative build
            if not os.path.exists(path):
                raise RuntimeError(f"{path} missing — build it with `python -m paper_2601_12967_b200.build` "
                                   "(no CPU fallback exists)")
            L = C.CDLL(path)
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(L, name)
                fn.restype = res
                fn.argtypes = args
            _lib = L
    return _lib


def check(status: int, what: str = ""):
    if status != 0:
        msg = lib().sb_last_error().decode(errors="replace")
        raise errors.from_status(status, f"{what}: {msg}" if what else msg)
