"""Roofline micro-benchmarks of the block-pool kernels (HBM side of the hot
path): chain hashing, batched prefix lookup, hint-aware eviction scoring and
the KV append, each timed with CUDA events on its stream and reported as
algorithmic GB/s against the measured HBM copy bandwidth.

    python bench_kv.py            # one JSON line per kernel/config

Algorithmic bytes per unit:
  chain hash     8 B read per token + 8 B written per block
  lookup         per full block position: 128 B query tokens + 128 B stored
                 tokens + 24 B index slot (chain hash, parent, id, ntok) + 8 B
                 chain hash of the position
  evict scoring  per pool block: ntok/ref/pinned(+exclusion mark)/tag (16 B) + last (8 B)
  kv append      per token and layer: 2 x H_kv x 128 x 2 B read + same written
"""
from __future__ import annotations

import ctypes as C
import json
import re
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    return json.load(open(p)) if os.path.exists(p) else {"hbm_gbs": 6650.0}


_FLUSH = None


_CLEAN = None


def flush_l2():
    """Overwrite a buffer twice the size of L2 so the next launch reads HBM,
    then read a second buffer of the same size so the lines L2 holds are
    clean: the write-back of the flush's dirty lines is not charged to the
    kernel that follows (SB_FLUSH=write keeps the write-only flush)."""
    import torch

    global _FLUSH, _CLEAN
    if os.environ.get("SB_FLUSH") == "none":  # diagnostics only: warm L2
        return
    if _FLUSH is None:
        _FLUSH = torch.empty(64 << 20, dtype=torch.int32, device="cuda")
        _CLEAN = torch.ones(64 << 20, dtype=torch.int32, device="cuda")
    _FLUSH.fill_(1)
    if os.environ.get("SB_FLUSH", "writeread") != "write":
        _CLEAN.max()


def timed(fn, reps=10, warm=3, kernels=(), flush=False):
    """Median CUDA-event time of fn() and, via the CUDA profiler (CUPTI
    activity records, no replay), the mean device duration of each kernel
    whose name contains one of `kernels`."""
    import torch
    from torch.profiler import ProfilerActivity, profile

    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
    for a, b in ev:
        if flush:
            flush_l2()
        a.record()
        fn()
        b.record()
    torch.cuda.synchronize()
    api = float(np.median([a.elapsed_time(b) for a, b in ev])) * 1e-3
    dev = {}
    if kernels:
        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            for _ in range(reps):
                if flush:
                    flush_l2()
                fn()
            torch.cuda.synchronize()
        # the device span of one call: first matched kernel's start to the last
        # one's end (launch gaps between a call's kernels included); calls are
        # separated by the L2 flush
        try:
            evs = sorted((e.time_range.start, e.time_range.end) for e in prof.events()
                         if e.device_type.name == "CUDA" and any(re.search(r"\b" + k + r"\b", e.name) for k in kernels))
        except AttributeError:
            evs = []
        spans, cur = [], None
        for a, b in evs:
            if cur and a - cur[1] < 20:  # us
                cur[1] = max(cur[1], b)
            else:
                if cur:
                    spans.append(cur[1] - cur[0])
                cur = [a, b]
        if cur:
            spans.append(cur[1] - cur[0])
        if spans:
            dev["span"] = [float(np.median(spans)) * 1e-6, 1]
        for e in prof.key_averages():
            for k in kernels:
                if re.search(r"\b" + k + r"\b", e.key) and e.count:  # k_select must not match k_select_coop
                    d = dev.setdefault(k, [0.0, 0])
                    d[0] += e.device_time_total * 1e-6
                    d[1] += e.count
        dev = {k: v[0] / v[1] for k, v in dev.items()}
    return api, dev


ROWS = []  # every emitted row (bench.py collects them as roofline_pool)
QUIET = False


def emit(kernel, config, bytes_, api_s, dev_s, hbm, launches=1, parts=None, note=None):
    """frac uses the kernel's own device time when the profiler saw it."""
    sec = dev_s * launches if dev_s else api_s
    gbs = bytes_ / sec / 1e9
    row = {"kernel": kernel, "config": config, "seconds": sec, "api_seconds": api_s,
           "timing": "kernel (CUPTI)" if dev_s else "api (CUDA events)", "algorithmic_bytes": bytes_,
           "achieved_gbs": gbs, "peak_gbs": hbm, "frac": gbs / hbm}
    if parts:
        row["parts_us"] = {k: round(v * 1e6, 2) for k, v in parts.items() if v}
    if note:
        row["note"] = note
    ROWS.append(row)
    if not QUIET:
        print(json.dumps(row), flush=True)


def fill_pool(L, cache, dev, n_seqs, toks, st):
    """Insert n_seqs random prompts of toks tokens (one SYSTEM tag range each),
    then release them: every block resident with ref 0 (an eviction candidate)."""
    import torch
    from paper_2601_12967_b200 import _lib

    p = lambda t: C.c_void_p(t.data_ptr())
    n = n_seqs * toks
    tokens = torch.randint(0, 2**62, (n,), dtype=torch.int64, device=dev)
    seq_off = torch.arange(0, n + 1, toks, dtype=torch.int64, device=dev)
    blk_off = torch.arange(0, n // 16 + 1, toks // 16, dtype=torch.int64, device=dev)
    blk_off_h = np.arange(0, n // 16 + 1, toks // 16, dtype=np.int64)
    tags = (_lib.TagRange * n_seqs)()
    for i in range(n_seqs):
        tags[i].begin, tags[i].end, tags[i].tag = 0, toks, 3
    tag_dev = torch.frombuffer(bytearray(tags), dtype=torch.uint8).to(dev)
    tag_off = torch.arange(n_seqs + 1, dtype=torch.int64, device=dev)
    ids = torch.empty(n // 16, dtype=torch.int32, device=dev)
    status = torch.empty(n_seqs, dtype=torch.int32, device=dev)
    _lib.check(L.sb_kv_insert_batch(cache.handle, p(tokens), p(seq_off), p(tag_dev), p(tag_off), p(blk_off),
                                    blk_off_h.ctypes.data_as(_lib.I64P), None, n_seqs, 1, p(ids), p(status), st))
    _lib.check(L.sb_kv_release_batch(cache.handle, p(ids), n // 16, None, st))
    torch.cuda.synchronize()


def evict_bench(L, cache, cap, hbm):
    from paper_2601_12967_b200 import _lib

    for needed in (64, 4096):
        def ev():
            out = np.zeros(needed, dtype=np.int32)
            k = C.c_int64(0)
            L.sb_kv_evict(cache.handle, needed, out.ctypes.data_as(_lib.I32P), C.byref(k))
        res = cache.resident_blocks()
        names = ("k_plan", "k_score", "k_select_coop", "k_evict_fused", "k_select")
        api, kt = timed(ev, reps=5, warm=1, kernels=names, flush=True)
        cfg = f"pool {cap} blocks, ~{res} resident (all candidates), evict {needed}"
        # scoring: 24 B of metadata read per pool block (ntok/ref/pinned/tag + last) + one 8 B key per candidate
        if kt.get("k_score"):
            emit("k_score (hint-aware eviction scoring)", cfg, cap * 24 + res * 8, api, kt.get("k_score"), hbm)
        # evict total = the device span of one evict (first kernel start to last
        # kernel end, launch gaps included); parts = per-kernel durations
        tot = kt.get("span") or sum(kt.get(k, 0.0) for k in names)
        label = ("evict total (k_evict_fused: scoring + select, one cooperative launch)" if kt.get("k_evict_fused")
                 else "evict total (k_plan + k_score + k_select_coop)")
        emit(label, cfg, cap * 24 + res * 8, api, tot or None, hbm, parts={k: kt.get(k) for k in names},
             note="device span of the evict's kernels incl. launch gaps" if kt.get("span") else None)


def main(only=None):
    import argparse

    import torch
    from paper_2601_12967_b200 import _lib
    from paper_2601_12967_b200.kv_cache import CacheConfig, KvCache

    if only is None:
        ap = argparse.ArgumentParser()
        ap.add_argument("--only", default="hash,probe,probe_big,evict_small,evict,evict_big,append")
        only = ap.parse_args().only
    only = set(only.split(","))
    L = _lib.lib()
    hbm = float(peaks()["hbm_gbs"])
    dev = torch.device("cuda")
    p = lambda t: C.c_void_p(t.data_ptr())
    st = C.c_void_p(torch.cuda.current_stream().cuda_stream)

    # ---- chain hashing: latency-bound per sequence, throughput over sequences
    for n_seqs, toks in ((64, 8192), (4096, 1024), (65536, 512), (262144, 128), (262144, 512)) if "hash" in only else ():
        n = n_seqs * toks
        tokens = torch.randint(0, 2**62, (n,), dtype=torch.int64, device=dev)
        seq_off = torch.arange(0, n + 1, toks, dtype=torch.int64, device=dev)
        blk_off = torch.arange(0, n // 16 + 1, toks // 16, dtype=torch.int64, device=dev)
        out = torch.empty(n // 16, dtype=torch.int64, device=dev)
        names = ("k_chain_hash16", "k_chain_hash_lat")  # the latency kernel takes <= 2048 sequences
        api, kt = timed(lambda: L.sb_chain_hash_batch(p(tokens), p(seq_off), p(blk_off), None, n_seqs, 16, p(out), st),
                         kernels=names, flush=True)
        kn = next((k for k in names if kt.get(k)), names[0])
        emit(kn, f"{n_seqs} seqs x {toks} tokens", 8 * n + 8 * (n // 16), api,
             kt.get(kn), hbm,
             note="one dependent 64-bit splitmix chain per sequence (~90 clk per token): fewer sequences than "
                  "resident lanes are latency bound, many sequences ALU-pipe bound" if n_seqs < 65536 else None)
        del tokens

    if "probe" in only:
        probe_bench(L, dev, st, hbm, 1 << 20, 1024, 8192, evict=True)
    if "probe_big" in only:
        probe_bench(L, dev, st, hbm, 1 << 22, 4096, 8192, evict=False)
    # ---- eviction at pool scale: evict() = k_plan + k_score (HBM pass) + k_select_coop
    if "evict_small" in only:  # the engine step's pool size class (27K blocks)
        cache3 = KvCache(CacheConfig(16, 1 << 15, 1))
        fill_pool(L, cache3, dev, 28, 16384, st)
        evict_bench(L, cache3, 1 << 15, hbm)
        del cache3
    for big, n_fill in ((1 << 22, 2048), (1 << 24, 8192)):
        if ("evict" if big == 1 << 22 else "evict_big") in only:
            cache2 = KvCache(CacheConfig(16, big, 1))
            fill_pool(L, cache2, dev, n_fill, 16384, st)
            evict_bench(L, cache2, big, hbm)
            del cache2
    if "append" in only:
        append_bench(L, dev, st, hbm)


def probe_bench(L, dev, st, hbm, cap, n_seqs, toks, evict):
    import torch
    from paper_2601_12967_b200 import _lib
    from paper_2601_12967_b200.kv_cache import CacheConfig, KvCache

    p = lambda t: C.c_void_p(t.data_ptr())
    # ---- batched lookup over a populated pool (all-hit prefixes)
    cache = KvCache(CacheConfig(16, cap, 1))
    n = n_seqs * toks
    host = np.random.default_rng(0).integers(0, 2**62, n, dtype=np.int64)
    tokens = torch.from_numpy(host).to(dev)
    seq_off = torch.arange(0, n + 1, toks, dtype=torch.int64, device=dev)
    blk_off = torch.arange(0, n // 16 + 1, toks // 16, dtype=torch.int64, device=dev)
    blk_off_h = np.arange(0, n // 16 + 1, toks // 16, dtype=np.int64)
    tags = (_lib.TagRange * n_seqs)()
    for i in range(n_seqs):
        tags[i].begin, tags[i].end, tags[i].tag = 0, toks, 3
    tag_dev = torch.frombuffer(bytearray(tags), dtype=torch.uint8).to(dev)
    tag_off = torch.arange(n_seqs + 1, dtype=torch.int64, device=dev)
    ids = torch.empty(n // 16, dtype=torch.int32, device=dev)
    status = torch.empty(n_seqs, dtype=torch.int32, device=dev)
    hashes = torch.empty(n // 16, dtype=torch.int64, device=dev)
    L.sb_chain_hash_batch(p(tokens), p(seq_off), p(blk_off), None, n_seqs, 16, p(hashes), st)
    _lib.check(L.sb_kv_insert_batch(cache.handle, p(tokens), p(seq_off), p(tag_dev), p(tag_off), p(blk_off),
                                    blk_off_h.ctypes.data_as(_lib.I64P), p(hashes), n_seqs, 1, p(ids), p(status), st))
    _lib.check(L.sb_kv_release_batch(cache.handle, p(ids), n // 16, None, st))
    torch.cuda.synchronize()
    hits = torch.empty(n_seqs, dtype=torch.int64, device=dev)
    names = ("k_probe_rows3", "k_probe_rows2", "k_probe_rows")  # SB_PROBE_PER selects the variant
    api, kt = timed(lambda: L.sb_kv_lookup_prefix_batch(cache.handle, p(tokens), p(seq_off), p(blk_off),
                                                         blk_off_h.ctypes.data_as(_lib.I64P), p(hashes), n_seqs, 2,
                                                         p(hits), st), kernels=names, flush=True)
    assert int(hits.sum()) == n
    kn = next((k for k in names if kt.get(k)), names[0])
    emit(kn, f"{n_seqs} seqs x {toks} tokens, pool {cap} blocks, all hit",
         (n // 16) * (128 + 128 + 24 + 8), api, kt.get(kn), hbm)

    if evict:
        evict_bench(L, cache, cap, hbm)
    del cache


def append_bench(L, dev, st, hbm):
    import torch

    p = lambda t: C.c_void_p(t.data_ptr())
    # ---- KV append (Llama-3-8B kv heads), one layer
    tok_n, hkv, pages = 98896, 8, 27281
    kp = torch.empty(pages, hkv, 16, 128, dtype=torch.bfloat16, device=dev)
    vp = torch.empty_like(kp)
    k_new = torch.randn(tok_n, hkv, 128, device=dev).to(torch.bfloat16)
    v_new = torch.randn_like(k_new)
    q_off = torch.tensor([0, tok_n], dtype=torch.int32, device=dev)
    kv_len = torch.tensor([tok_n], dtype=torch.int32, device=dev)
    table = torch.randperm(pages, device=dev)[: (tok_n + 15) // 16].to(torch.int32).reshape(1, -1).contiguous()
    api, kt = timed(lambda: L.sb_kv_append(p(k_new), p(v_new), p(kp), p(vp), p(q_off), p(kv_len), p(table), 1,
                                            table.shape[1], hkv, 128, 16, st), kernels=("k_kv_append",), flush=True)
    emit("k_kv_append", f"{tok_n} tokens x {hkv} kv heads", 2 * 2 * tok_n * hkv * 128 * 2, api,
         kt.get("k_kv_append"), hbm)


if __name__ == "__main__":
    main()
