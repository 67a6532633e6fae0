"""GPU parity of the device block pool (csrc/kv_pool.cu) with the reference:
golden op logs recorded from the reference engine + randomized large-scale
comparisons against the C oracle.  Bit-exact: hit lengths, block ids,
eviction order, statuses and the full audit dump after every op."""
import numpy as np
import pytest

from oracle import oracle as O
from tests import oplog


def product(bs, cap, pol):
    from paper_2601_12967_b200.kv_cache import CacheConfig, KvCache

    return oplog.StatusAdapter(KvCache(CacheConfig(bs, cap, pol)))


@pytest.mark.gpu
@pytest.mark.parametrize("name", oplog.golden_logs())
def test_product_replays_reference_oplog(name):
    errs = oplog.replay(oplog.load(name), product)
    assert not errs, "\n".join(errs)


def _random_workload(seed, n_ops, bs, cap, pol, long=False):
    """Engine-like traffic: shared system prompts, growing conversations,
    partial-prefill pins, releases, explicit evictions."""
    rng = np.random.default_rng(seed)
    sys_prompts = [O.materialize(0, int(rng.integers(200, 2500 if long else 600)), 100 + k) for k in range(5)]
    ops = []
    live = []
    now = 0
    for _ in range(n_ops):
        now += int(rng.integers(0, 20))
        r = rng.random()
        sp = sys_prompts[int(rng.integers(len(sys_prompts)))]
        tail = O.materialize(int(rng.integers(4)), int(rng.integers(0, 3000 if long else 400)), int(rng.integers(50)),
                             int(rng.integers(-1, 3)))
        toks = np.concatenate([sp, tail])
        if r < 0.35:
            ops.append(("lookup", toks, now))
        elif r < 0.75:
            n = len(toks)
            cut = int(rng.integers(1, n)) if n > 1 else n
            tags = [(0, cut, int(rng.integers(6))), (cut, n, int(rng.integers(6)))] if cut < n else [(0, n, 3)]
            ops.append(("insert", toks, tags, now))
        elif r < 0.9:
            ops.append(("release_one",))
        elif r < 0.95:
            ops.append(("evict", int(rng.integers(1, max(2, cap // 8)))))
        else:
            ops.append(("pin_some", int(rng.integers(0, 2))))
    return ops


def _run(cache, ops, bs):
    out = []
    live = []
    rng = np.random.default_rng(7)
    for op in ops:
        if op[0] == "lookup":
            out.append(("L", cache.lookup_prefix(op[1], op[2])))
        elif op[0] == "insert":
            st, ids = cache.insert(op[1], op[2], op[3])
            out.append(("I", st, tuple(ids)))
            if st == 0:
                live.append(ids)
        elif op[0] == "release_one":
            if live:
                ids = live.pop(int(rng.integers(len(live))))
                out.append(("R", cache.release(ids)))
        elif op[0] == "evict":
            out.append(("E", tuple(cache.evict(op[1])[1])))
        elif op[0] == "pin_some":
            if live:
                out.append(("P", cache.set_reuse_priority(live[-1][:3], op[1], -1)))
    out.append(("D", cache.dump()))
    out.append(("T", cache.total_evicted()))
    return out


@pytest.mark.gpu
@pytest.mark.parametrize("pol", [0, 1])
def test_product_matches_oracle_engine_like(pol):
    bs, cap = 16, 700
    ops = _random_workload(3 + pol, 400, bs, cap, pol)
    ref = _run(O.OracleCache(bs, cap, pol), ops, bs)
    got = _run(product(bs, cap, pol), ops, bs)
    for i, (a, b) in enumerate(zip(ref, got)):
        assert a == b, f"op {i}: oracle {str(a)[:200]} vs product {str(b)[:200]}"


@pytest.mark.gpu
def test_product_matches_oracle_large_pool_long_prompts():
    """8192-block pool (the reference's default capacity), multi-K-token prompts:
    victim lists longer than the shared-memory sort exercise the global path."""
    bs, cap = 16, 8192
    ops = _random_workload(11, 160, bs, cap, 1, long=True)
    ref = _run(O.OracleCache(bs, cap, 1), ops, bs)
    got = _run(product(bs, cap, 1), ops, bs)
    for i, (a, b) in enumerate(zip(ref, got)):
        assert a == b, f"op {i}: oracle {str(a)[:200]} vs product {str(b)[:200]}"


@pytest.mark.gpu
def test_evict_everything_sorted_order():
    bs, cap = 4, 9000  # > shared-memory sort size when evicting all
    c = product(bs, cap, 1)
    o = O.OracleCache(bs, cap, 1)
    rng = np.random.default_rng(5)
    for k in range(40):
        t = O.materialize(int(rng.integers(4)), int(rng.integers(1, 900)), k)
        tags = [(0, len(t), int(rng.integers(6)))]
        a = o.insert(t, tags, k)
        b = c.insert(t, tags, k)
        assert a == b
        if a[0] == 0:
            assert o.release(a[1]) == c.release(b[1]) == 0
    assert o.evict(cap) == c.evict(cap)
    assert o.dump() == c.dump()


@pytest.mark.gpu
def test_batch_apis_match_sequential_oracle():
    import torch
    import ctypes as C
    from paper_2601_12967_b200 import _lib
    from paper_2601_12967_b200.kv_cache import CacheConfig, KvCache

    bs, cap = 16, 600
    rng = np.random.default_rng(9)
    base = O.materialize(0, 700, 1)
    seqs = [np.concatenate([base[: int(rng.integers(0, 700))], O.materialize(2, int(rng.integers(1, 300)), k, 0)])
            for k in range(24)]
    tags = [[(0, len(s), int(rng.integers(6)))] for s in seqs]
    o = O.OracleCache(bs, cap, 1)
    exp = [o.insert(s, t, 5) for s, t in zip(seqs, tags)]
    exp_hits = [o.lookup_prefix(s, 9) for s in seqs]
    c = KvCache(CacheConfig(bs, cap, 1))
    dev = torch.device("cuda")
    tok = torch.from_numpy(np.concatenate(seqs).view(np.int64)).to(dev)
    off = torch.tensor(np.cumsum([0] + [len(s) for s in seqs]), dtype=torch.int64, device=dev)
    blk = torch.tensor(np.cumsum([0] + [(len(s) + bs - 1) // bs for s in seqs]), dtype=torch.int64, device=dev)
    tag_arr = (_lib.TagRange * len(seqs))()
    for i, t in enumerate(tags):
        tag_arr[i].begin, tag_arr[i].end, tag_arr[i].tag = t[0]
    tag_dev = torch.empty(len(seqs) * 24, dtype=torch.uint8, device=dev)
    tag_dev.copy_(torch.frombuffer(bytearray(tag_arr), dtype=torch.uint8))
    tag_off = torch.arange(len(seqs) + 1, dtype=torch.int64, device=dev)
    out_ids = torch.full((int(blk[-1]),), -1, dtype=torch.int32, device=dev)
    status = torch.zeros(len(seqs), dtype=torch.int32, device=dev)
    p = lambda t: C.c_void_p(t.data_ptr())
    _lib.check(_lib.lib().sb_kv_insert_batch(c.handle, p(tok), p(off), p(tag_dev), p(tag_off), p(blk), None, None,
                                             len(seqs), 5, p(out_ids), p(status), None))
    torch.cuda.synchronize()
    st = status.cpu().tolist()
    ids = out_ids.cpu().tolist()
    b = blk.cpu().tolist()
    for i, (est, eids) in enumerate(exp):
        assert st[i] == est, i
        if est == 0:
            assert ids[b[i]:b[i + 1]] == eids, i
    hits = torch.zeros(len(seqs), dtype=torch.int64, device=dev)
    _lib.check(_lib.lib().sb_kv_lookup_prefix_batch(c.handle, p(tok), p(off), None, None, None, len(seqs), 9, p(hits), None))
    torch.cuda.synchronize()
    assert hits.cpu().tolist() == exp_hits
    assert c.dump() == o.dump()


@pytest.mark.gpu
def test_insert_batch_on_cooperative_pool_under_pressure():
    """sb_kv_insert_batch op programs on a pool large enough (>= 64K blocks)
    for their eviction to go through the all-SM cooperative select (mode 2),
    under pressure: statuses, block ids and the dump equal sequential
    reference inserts."""
    import ctypes as C

    import torch
    from paper_2601_12967_b200 import _lib
    from paper_2601_12967_b200.kv_cache import CacheConfig, KvCache

    bs, cap = 1, 70000
    rng = np.random.default_rng(41)
    o = O.OracleCache(bs, cap, 1)
    c = KvCache(CacheConfig(bs, cap, 1))
    dev = torch.device("cuda")
    p = lambda t: C.c_void_p(t.data_ptr())
    for rnd in range(3):
        seqs = [O.materialize(int(rng.integers(4)), int(rng.integers(800, 2000)), 50 * rnd + k) for k in range(20)]
        tags = [[(0, len(s) // 2, int(rng.integers(6))), (len(s) // 2, len(s), int(rng.integers(6)))] for s in seqs]
        now = 10 + rnd
        exp = [o.insert(s, t, now) for s, t in zip(seqs, tags)]
        tok = torch.from_numpy(np.concatenate(seqs).view(np.int64)).to(dev)
        off = torch.tensor(np.cumsum([0] + [len(s) for s in seqs]), dtype=torch.int64, device=dev)
        blk = torch.tensor(np.cumsum([0] + [len(s) for s in seqs]), dtype=torch.int64, device=dev)
        tag_arr = (_lib.TagRange * (2 * len(seqs)))()
        for i, t in enumerate(tags):
            for j, (b0, e0, tg) in enumerate(t):
                tag_arr[2 * i + j].begin, tag_arr[2 * i + j].end, tag_arr[2 * i + j].tag = b0, e0, tg
        tag_dev = torch.frombuffer(bytearray(tag_arr), dtype=torch.uint8).to(dev)
        tag_off = torch.arange(0, 2 * len(seqs) + 1, 2, dtype=torch.int64, device=dev)
        out_ids = torch.full((int(blk[-1]),), -1, dtype=torch.int32, device=dev)
        status = torch.zeros(len(seqs), dtype=torch.int32, device=dev)
        _lib.check(_lib.lib().sb_kv_insert_batch(c.handle, p(tok), p(off), p(tag_dev), p(tag_off), p(blk), None,
                                                 None, len(seqs), now, p(out_ids), p(status), None))
        torch.cuda.synchronize()
        st, ids, b = status.cpu().tolist(), out_ids.cpu().tolist(), blk.cpu().tolist()
        for i, (est, eids) in enumerate(exp):
            assert st[i] == est, (rnd, i)
            if est == 0:
                assert ids[b[i]:b[i + 1]] == eids, (rnd, i)
        for i, (est, eids) in enumerate(exp):  # release two of every three inserted chains
            if est == 0 and i % 3:
                assert o.release(eids) == 0
                c.release(eids)
    assert o.dump() == c.dump()


@pytest.mark.gpu
def test_large_pool_cooperative_scorer():
    """Pools of >= 16384 blocks use the all-SM cooperative scorer
    (k_select_coop): eviction order, insert ids under pressure and the full
    dump must still equal the oracle."""
    bs, cap = 1, 70000
    c = product(bs, cap, 1)
    o = O.OracleCache(bs, cap, 1)
    rng = np.random.default_rng(21)
    live = []
    for k in range(34):
        t = O.materialize(int(rng.integers(4)), 2000, 500 + k)
        tags = [(0, 1000, int(rng.integers(6))), (1000, 2000, int(rng.integers(6)))]
        a, b = o.insert(t, tags, k), c.insert(t, tags, k)
        assert a == b, k
        live.append(a[1])
    for ids in live[::2]:
        assert o.release(ids) == c.release(ids) == 0
    for needed in (1, 777, 5000):
        assert o.evict(needed) == c.evict(needed), needed
    for k in range(2):  # inserts that must evict
        t = O.materialize(1, 3000, 900 + k)
        tags = [(0, 3000, 1)]
        assert o.insert(t, tags, 100 + k) == c.insert(t, tags, 100 + k)
    assert o.dump() == c.dump()
    assert o.total_evicted() == c.total_evicted()


@pytest.mark.gpu
def test_cooperative_evict_beyond_shared_memory_sort():
    """evict(K) with K above what the cooperative select ranks in shared
    memory (24K keys in the fused kernel, 16K in k_select_coop): CTA 0 sorts
    the winners in global memory instead.
    Every tier and several timestamps, so the radix passes run over the
    tier and last_used bits of the keys as well as the ids."""
    bs, cap = 1, 70000
    c = product(bs, cap, 1)
    o = O.OracleCache(bs, cap, 1)
    rng = np.random.default_rng(33)
    live = []
    for k in range(30):
        t = O.materialize(int(rng.integers(4)), 2200, 300 + k)
        tags = [(0, 700, int(rng.integers(6))), (700, 2200, int(rng.integers(6)))]
        now = int(rng.integers(0, 40))
        a, b = o.insert(t, tags, now), c.insert(t, tags, now)
        assert a == b, k
        live.append(a[1])
    for ids in live[::3]:
        assert o.release(ids) == c.release(ids) == 0
    for ids in live[1::3]:
        assert o.release(ids) == c.release(ids) == 0
    for needed in (30000, 3, 9000):  # 30000: above the fused kernel's 24K-key rank buffer
        assert o.evict(needed) == c.evict(needed), needed
    assert o.dump() == c.dump()


@pytest.mark.gpu
def test_cooperative_select_keys_in_place():
    """A 16M-block pool whose candidates crowd into the first score slices:
    one CTA holds more keys than shared memory, so the select reads them in
    place (compaction after pass 1, slice filters, the grid striding over the
    few live slices), for K below and above the rank-step and shared-memory
    limits."""
    bs, cap = 1, 1 << 24
    c = product(bs, cap, 1)
    o = O.OracleCache(bs, cap, 1)
    rng = np.random.default_rng(77)
    live = []
    for k in range(10):
        t = O.materialize(int(rng.integers(4)), 4000, 1200 + k)
        tags = [(0, 1300, int(rng.integers(6))), (1300, 4000, int(rng.integers(6)))]
        now = int(rng.integers(0, 20))
        a, b = o.insert(t, tags, now), c.insert(t, tags, now)
        assert a == b, k
        live.append(a[1])
    for ids in live:
        assert o.release(ids) == c.release(ids) == 0
    for needed in (64, 5000, 3, 20000, 9000):
        assert o.evict(needed) == c.evict(needed), needed
    assert o.total_evicted() == c.total_evicted()
    assert o.dump() == c.dump()


@pytest.mark.gpu
def test_three_kernel_evict_path():
    """SB_EVICT_FUSED=0 selects k_plan + k_score + k_select_coop instead of
    the fused cooperative kernel: the same parity tests through that path
    (a subprocess: the switch is read once per process)."""
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, SB_EVICT_FUSED="0")
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", "tests/test_kvcache_gpu.py", "-k",
                        "cooperative_scorer or beyond_shared_memory or in_place"], cwd=root, env=env,
                       capture_output=True, text=True, timeout=1200)
    assert r.returncode == 0 and "4 passed" in r.stdout, r.stdout[-3000:] + r.stderr[-2000:]


@pytest.mark.gpu
def test_huge_pool_keys_read_in_place():
    """Pools above ~4.1M blocks: k_select_coop cannot stage its slices' keys
    in shared memory and radix-selects them in place; victim keys carry
    23 id bits (now limited to +-2^37).  Same oracle parity bar."""
    bs, cap = 1, 4_500_000
    c = product(bs, cap, 1)
    o = O.OracleCache(bs, cap, 1)
    rng = np.random.default_rng(5)
    live = []
    for k in range(12):
        t = O.materialize(int(rng.integers(4)), 3000, 700 + k)
        tags = [(0, 1500, int(rng.integers(6))), (1500, 3000, int(rng.integers(6)))]
        a, b = o.insert(t, tags, k * 1000), c.insert(t, tags, k * 1000)
        assert a == b, k
        live.append(a[1])
    for ids in live[1::2]:
        assert o.release(ids) == c.release(ids) == 0
    for needed in (3, 2049, 9000):
        assert o.evict(needed) == c.evict(needed), needed
    assert o.dump() == c.dump()
    c.audit()


@pytest.mark.gpu
def test_time_range_guard():
    """Victim keys hold last_used in 61 - idb bits: times outside +-2^(60-idb)
    are rejected loudly (never silently wrapped) by every call that stores
    a time."""
    from paper_2601_12967_b200 import errors
    from paper_2601_12967_b200.kv_cache import CacheConfig, KvCache

    c = KvCache(CacheConfig(16, 64, 1))
    t = O.materialize(0, 32, 1)
    ids = c.insert(t, [(0, 32, 3)], (1 << 39) - 1)
    for bad in (1 << 39, -(1 << 39) - 1):
        with pytest.raises(errors.Unsupported):
            c.insert(t, [(0, 32, 3)], bad)
        with pytest.raises(errors.Unsupported):
            c.lookup_prefix(t, bad)
        with pytest.raises(errors.Unsupported):
            c.touch(ids, bad)


@pytest.mark.gpu
def test_batched_block_readback_matches_block():
    """blocks(ids) (one round trip) == contains()/block() per id, including
    out-of-range and evicted ids."""
    from paper_2601_12967_b200.kv_cache import CacheConfig, KvCache

    c = KvCache(CacheConfig(16, 96, 1))
    ids = []
    for k in range(6):
        t = O.materialize(k % 4, 100 + 37 * k, k)
        ids += list(c.insert(t, [(0, 50, k % 6), (50, len(t), (k + 2) % 6)], 10 + k))
    c.set_reuse_priority(ids[:5], pinned=True, tier_override=4)
    c.release(ids[5:20])
    c.evict(4)
    probe = list(range(-2, 99))
    got = c.blocks(probe)
    for i, b in zip(probe, got):
        if not c.contains(i):
            assert b is None, i
            continue
        ref = c.block(i)
        assert b is not None
        for f in ("block_id", "chain_hash", "parent_hash", "tag", "tier", "ref_count", "last_used", "pinned"):
            assert getattr(b, f) == getattr(ref, f), (i, f)
    assert c.blocks([]) == []


@pytest.mark.gpu
def test_batched_lookup_consecutive_id_guess_and_fallbacks():
    """The batched lookup guesses that a chain's blocks are consecutive ids
    (k_probe_rows3) and falls back to the index per position: chains built
    by interleaved growing inserts (ids strided by the number of chains),
    chains with holes re-filled after evictions, chains allocated in one
    insert (consecutive), partial hits (a differing block mid-chain) and
    partial last blocks — hit lengths and the dump equal the oracle's."""
    import ctypes as C
    import torch
    from paper_2601_12967_b200 import _lib

    bs, cap = 16, 3000
    rng = np.random.default_rng(31)
    o = O.OracleCache(bs, cap, 1)
    c = product(bs, cap, 1)
    n_chains, n_blk = 20, 40
    chains = [O.materialize(1, n_blk * bs, 900 + k) for k in range(n_chains)]
    now = 1
    for k in range(1, n_blk + 1):  # round k extends every chain by one block: ids strided by n_chains
        for ch in chains[: n_chains // 2]:
            t = ch[: k * bs]
            a, b = o.insert(t, [(0, len(t), 2)], now), c.insert(t, [(0, len(t), 2)], now)
            assert a == b
            assert o.release(a[1]) == c.release(b[1]) == 0
        now += 1
    for ch in chains[n_chains // 2:]:  # one insert per chain: consecutive ids
        a, b = o.insert(ch, [(0, len(ch), 3)], now), c.insert(ch, [(0, len(ch), 3)], now)
        assert a == b
        assert o.release(a[1]) == c.release(b[1]) == 0
    assert o.evict(150) == c.evict(150)  # holes
    for k in range(4):  # re-filled with new chains
        t = O.materialize(2, int(rng.integers(100, 900)), 7000 + k)
        a, b = o.insert(t, [(0, len(t), 1)], now), c.insert(t, [(0, len(t), 1)], now)
        assert a == b
    queries = []
    for ch in chains:
        queries.append(ch)
        q = ch.copy()
        q[int(rng.integers(0, len(q)))] ^= np.uint64(1)  # a partial hit
        queries.append(q)
        queries.append(ch[: int(rng.integers(1, len(ch)))])  # a partial last block
    exp = [o.lookup_prefix(q, now + 1) for q in queries]
    dev = torch.device("cuda")
    tok = torch.from_numpy(np.concatenate(queries).view(np.int64)).to(dev)
    off = torch.tensor(np.cumsum([0] + [len(q) for q in queries]), dtype=torch.int64, device=dev)
    hits = torch.zeros(len(queries), dtype=torch.int64, device=dev)
    p = lambda t: C.c_void_p(t.data_ptr())
    _lib.check(_lib.lib().sb_kv_lookup_prefix_batch(c.c.handle, p(tok),
                                                    p(off), None, None, None, len(queries), now + 1, p(hits), None))
    torch.cuda.synchronize()
    assert hits.cpu().tolist() == exp
    assert c.dump() == o.dump()
