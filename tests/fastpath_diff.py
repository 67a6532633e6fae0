"""Differential harness of the op programs' parallel path (csrc/pool_batch.cuh)
against the sequential one-CTA program (csrc/pool_program.cuh).

    SB_PROG_FAST=0|1 python tests/fastpath_diff.py

Runs batched engine steps (configs[1]-style and ragged random batches under
pool pressure, both eviction policies) and random per-call engine
sequences, and prints ONE JSON object: every observable result per step / op
(admission hits, pin outcomes, statuses, the chains, a digest of the full
pool dump, the eviction count) plus the pool's program statistics.  The
test (tests/test_program_fastpath_gpu.py) runs it with the parallel path on
and off and requires identical results."""
import hashlib
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

SHAPE = None


def digest(s: str) -> str:
    return hashlib.sha256(s.encode()).hexdigest()[:16]


def batch_run(reqs_prefix, reqs_tags, suffix_lens, suffix_fn, cap, policy, steps, keys):
    import torch
    from paper_2601_12967_b200.engine import ContinuationEngine

    eng = ContinuationEngine(SHAPE, cap, policy=policy)
    batch = eng.make_batch(reqs_prefix, reqs_tags, suffix_lens, stream_keys=keys)
    out = []
    for step in range(steps):
        sfx = np.concatenate([suffix_fn(i, step) for i in range(len(reqs_prefix))]).view(np.int64)
        batch.stage_suffix_device(torch.from_numpy(sfx).cuda())
        rec = {}
        try:
            batch.run(10 + step, seed=step)
            torch.cuda.synchronize()
            hits, status, got = batch.results()
            rec = {"hits": hits.tolist(), "pin": batch.pin_outcomes().tolist(), "status": status.tolist(),
                   "chains": digest(",".join(map(str, got.tolist())))}
        except Exception as e:  # CacheFull inside a step is reported, the pool state still compared
            rec = {"error": type(e).__name__ + ":" + str(e)[:60]}
        rec["dump"] = digest(eng.cache.dump())
        rec["evicted"] = eng.cache.total_evicted()
        out.append(rec)
    eng.cache.audit()
    st = eng.cache.program_stats()
    del batch
    eng.close()
    return out, st


def configs1_batches():
    from paper_2601_12967_b200 import workload as W

    res, stats = [], []
    for n_req, sys_len, seed, slack, policy in ((12, 256, 3, 1.0, 1), (12, 256, 3, 1.0, 0), (24, 128, 5, 0.6, 1),
                                                (8, 512, 7, 1.25, 1), (16, 64, 9, 0.8, 0)):
        reqs = W.agentic_continuation_batch(n_req, sys_len=sys_len, seed=seed)
        pre = sum(r.prefix_len // 16 for r in reqs) - (n_req - 1) * (sys_len // 16)
        suf = sum((r.suffix_len + 15) // 16 for r in reqs) + n_req
        cap = pre + int(slack * suf) + 1
        r, st = batch_run([q.prefix_tokens for q in reqs], [q.prefix_tags for q in reqs], [q.suffix_len for q in reqs],
                          lambda i, s: W.fresh_suffix_tokens(reqs[i], s), cap, policy, 4,
                          [1000 + i for i in range(n_req)])
        res.append(r)
        stats.append(st)
    return res, stats


def ragged_batches():
    """Prefixes and suffixes of any length (partial blocks), shared system
    prompts of ragged length, some requests duplicating another's prefix
    (shared blocks; identical fresh content across ops forces the fallback),
    random tag ranges, tight pools."""
    res, stats = [], []
    for seed in range(6):
        rng = np.random.default_rng(100 + seed)
        n = int(rng.integers(3, 20))
        sys_tok = rng.integers(1, 2**62, int(rng.integers(1, 300)), dtype=np.uint64)
        prefixes, tags, slen = [], [], []
        for i in range(n):
            if i and rng.random() < 0.25:
                j = int(rng.integers(0, i))
                prefixes.append(prefixes[j].copy())
                tags.append(list(tags[j]))
            else:
                own = rng.integers(1, 2**62, int(rng.integers(1, 400)), dtype=np.uint64)
                p = np.concatenate([sys_tok, own])
                cut = sorted(set([len(sys_tok)] + [int(x) for x in rng.integers(1, len(p), 2)]))
                bounds = [0] + [c for c in cut if 0 < c < len(p)] + [len(p)]
                tags.append([(bounds[k], bounds[k + 1], int(rng.choice([1, 2, 3, 5]))) for k in range(len(bounds) - 1)])
                prefixes.append(p)
            slen.append(int(rng.integers(1, 200)))
        same_sfx = rng.random() < 0.3  # identical tool outputs across requests: duplicate new blocks
        blocks = sum((len(p) + s + 16) // 16 for p, s in zip(prefixes, slen))
        cap = max(int(blocks * float(rng.uniform(0.7, 1.3))), max((len(p) + s) // 16 + 4 for p, s in zip(prefixes, slen)))
        policy = int(seed % 2)

        def sfx(i, s, slen=slen, seed=seed, same=same_sfx):
            r2 = np.random.default_rng(10_000 * seed + 7 * s + (0 if same else i))
            return r2.integers(1, 2**62, slen[i], dtype=np.uint64)

        r, st = batch_run(prefixes, tags, slen, sfx, cap, policy, 4, [7 + i for i in range(n)])
        res.append(r)
        stats.append(st)
    return res, stats


def insert_batches():
    """sb_kv_insert_batch programs (PK_INSERT ops) under pressure: batches of
    prompts sharing prefixes (hits on blocks that are eviction candidates,
    misses that evict), random tag ranges (some invalid: CacheError), releases
    of random earlier inserts between batches, tight pools, both policies."""
    import ctypes as C
    import torch
    from paper_2601_12967_b200 import _lib
    from paper_2601_12967_b200.kv_cache import CacheConfig, KvCache

    L = _lib.lib()
    p = lambda t: C.c_void_p(t.data_ptr())
    dev = torch.device("cuda")
    out_all, stats = [], []
    for seed in range(5):
        rng = np.random.default_rng(700 + seed)
        cap = int(rng.integers(60, 400))
        cache = KvCache(CacheConfig(16, cap, int(seed % 2)))
        bases = [rng.integers(1, 2**62, int(rng.integers(16, 300)), dtype=np.uint64) for _ in range(4)]
        held, out = [], []
        for rnd in range(8):
            n = int(rng.integers(2, 12))
            seqs, tags = [], []
            for _ in range(n):
                b = bases[int(rng.integers(0, len(bases)))]
                tail = rng.integers(1, 2**62, int(rng.integers(0, 120)), dtype=np.uint64)
                s_ = np.concatenate([b[: int(rng.integers(1, len(b) + 1))], tail])
                seqs.append(s_)
                cut = int(rng.integers(0, len(s_) + 1))
                if rng.random() < 0.1:  # a gap: CacheError for this sequence
                    tags.append([(0, max(cut - 1, 0), 1), (cut, len(s_), 2)])
                else:
                    tags.append([(0, cut, int(rng.integers(6))), (cut, len(s_), int(rng.integers(6)))])
            tok = torch.from_numpy(np.concatenate(seqs).view(np.int64)).to(dev)
            off = torch.tensor(np.cumsum([0] + [len(x) for x in seqs]), dtype=torch.int64, device=dev)
            blk = torch.tensor(np.cumsum([0] + [(len(x) + 15) // 16 for x in seqs]), dtype=torch.int64, device=dev)
            flat = [r for t in tags for r in t]
            tarr = (_lib.TagRange * len(flat))()
            for i, (b_, e_, g_) in enumerate(flat):
                tarr[i].begin, tarr[i].end, tarr[i].tag = b_, e_, g_
            tag_dev = torch.frombuffer(bytearray(tarr), dtype=torch.uint8).to(dev)
            tag_off = torch.tensor(np.cumsum([0] + [len(t) for t in tags]), dtype=torch.int64, device=dev)
            ids = torch.full((int(blk[-1]),), -1, dtype=torch.int32, device=dev)
            status = torch.zeros(n, dtype=torch.int32, device=dev)
            _lib.check(L.sb_kv_insert_batch(cache.handle, p(tok), p(off), p(tag_dev), p(tag_off), p(blk), None, None,
                                            n, 10 + rnd, p(ids), p(status), None))
            torch.cuda.synchronize()
            st, idl, b = status.cpu().tolist(), ids.cpu().tolist(), blk.cpu().tolist()
            for i in range(n):
                if st[i] == 0:
                    held.append(idl[b[i]:b[i + 1]])
            rel = []
            for _ in range(int(rng.integers(0, len(held) + 1))):  # release random held inserts
                rel.append(held.pop(int(rng.integers(0, len(held)))))
            for r in rel:
                cache.release(r)
            out.append([st, digest(",".join(map(str, idl))), digest(cache.dump()), cache.total_evicted()])
        out_all.append(out)
        stats.append(cache.program_stats())
    return out_all, stats


def single_inserts():
    """Per-call KvCache.insert (one PK_INSERT op per program) under pressure,
    with releases in between: status, ids and the evicted ids the call
    reports (sb_kv_last_evicted — the drop-in binding's residency mirror
    consumes them)."""
    from paper_2601_12967_b200.kv_cache import CacheConfig, KvCache

    out_all = []
    for seed in range(3):
        rng = np.random.default_rng(900 + seed)
        cache = KvCache(CacheConfig(16, int(rng.integers(40, 200)), int(seed % 2)))
        bases = [rng.integers(1, 2**62, int(rng.integers(16, 400)), dtype=np.uint64) for _ in range(3)]
        held, out = [], []
        for k in range(60):
            b = bases[int(rng.integers(0, len(bases)))]
            t = np.concatenate([b[: int(rng.integers(1, len(b) + 1))],
                                rng.integers(1, 2**62, int(rng.integers(0, 200)), dtype=np.uint64)])
            try:
                ids = cache.insert(t, [(0, len(t), int(rng.integers(6)))], 5 + k)
                held.append(ids)
                rec = [list(map(int, ids)), cache.last_evicted()]
            except Exception as e:
                rec = ["E:" + type(e).__name__]
            if held and rng.random() < 0.6:
                cache.release(held.pop(int(rng.integers(0, len(held)))))
            rec.append(digest(cache.dump()))
            out.append(rec)
        out_all.append(out)
    return out_all


def percall_sequences():
    """Random interleavings of the per-call engine API (one op per program)."""
    from paper_2601_12967_b200.engine import ContinuationEngine

    out_all, stats = [], []
    for seed in range(4):
        rng = np.random.default_rng(500 + seed)
        segs = [rng.integers(1, 2**62, int(rng.integers(5, 90)), dtype=np.uint64) for _ in range(8)]
        cap = int(rng.integers(20, 60))
        eng = ContinuationEngine(SHAPE, cap, policy=int(seed % 2))
        live, partial, out = [], [], []
        for step in range(120):
            now = 10 + step // 3
            kind = rng.integers(0, 5)
            rec = [int(kind)]
            try:
                if kind == 0 or not (live or partial):
                    toks = np.concatenate([segs[int(k)] for k in rng.integers(0, len(segs), int(rng.integers(1, 4)))])
                    tg = [(0, len(toks), int(rng.choice([1, 2, 3])))]
                    if rng.random() < 0.5:
                        c = eng.submit_partial_prefill(toks, tg, now)
                        partial.append(c)
                    else:
                        c = eng.submit_call(toks, tg, 1, now)
                        live.append(c)
                    rec += [c, eng.cached_at_submit(c)]
                elif kind == 1 and (live or partial):
                    c = (live + partial)[int(rng.integers(0, len(live) + len(partial)))]
                    rec += [eng.prefill_done(c, now)]
                elif kind == 2 and partial:
                    c = partial.pop(int(rng.integers(0, len(partial))))
                    sfx = segs[int(rng.integers(0, len(segs)))][: int(rng.integers(1, 40))]
                    rec += [bool(eng.extend_prefill(c, sfx, [(0, len(sfx), 1)], 1, now))]
                    live.append(c)
                elif kind == 3 and live:
                    c = live.pop(int(rng.integers(0, len(live))))
                    eng.finish_decode(c, np.array([int(rng.integers(1, 99))], np.uint64), now)
                elif kind == 4 and partial:
                    c = partial.pop(int(rng.integers(0, len(partial))))
                    eng.abandon_partial(c)
            except Exception as e:
                rec += ["E:" + type(e).__name__]
            rec.append(digest(eng.cache.dump()))
            out.append(rec)
        out_all.append(out)
        stats.append(eng.cache.program_stats())
        eng.close()
    return out_all, stats


def main():
    global SHAPE
    from paper_2601_12967_b200.engine import ModelShape

    SHAPE = ModelShape(n_layers=1, n_q_heads=8, n_kv_heads=2, head_dim=128)
    a, sa = configs1_batches()
    b, sb = ragged_batches()
    c, sc = percall_sequences()
    d, sd = insert_batches()
    e = single_inserts()
    print(json.dumps({"configs1": a, "ragged": b, "percall": c, "inserts": d, "single": e,
                      "stats": {"configs1": sa, "ragged": sb, "percall": sc, "inserts": sd}}))


if __name__ == "__main__":
    main()
