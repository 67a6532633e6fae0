"""GPU chain hashing (k_chain_hash16 / k_chain_hash) against the CPU oracle:
every block's chain hash of ragged batches — single long sequences, empty
and sub-block sequences, warps mixing full and partial blocks, parent seeds."""
import ctypes as C

import numpy as np
import pytest

from oracle import oracle as O


def _gpu_hashes(seqs, bs, parents=None):
    import torch
    from paper_2601_12967_b200 import _lib

    L = _lib.lib()
    lens = [len(s) for s in seqs]
    off = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    nblk = [(n + bs - 1) // bs for n in lens]
    boff = np.concatenate([[0], np.cumsum(nblk)]).astype(np.int64)
    tok = torch.from_numpy(np.concatenate(seqs).view(np.int64) if sum(lens) else np.zeros(1, np.int64)).cuda()
    d_off, d_boff = torch.from_numpy(off).cuda(), torch.from_numpy(boff).cuda()
    out = torch.zeros(max(1, int(boff[-1])), dtype=torch.int64, device="cuda")
    par = torch.from_numpy(np.array(parents, dtype=np.uint64).view(np.int64)).cuda() if parents is not None else None
    p = lambda t: C.c_void_p(t.data_ptr()) if t is not None else None
    _lib.check(L.sb_chain_hash_batch(p(tok), p(d_off), p(d_boff), p(par), len(seqs), bs, p(out), None))
    torch.cuda.synchronize()
    h = out.cpu().numpy().view(np.uint64)
    return [h[boff[i]:boff[i + 1]].tolist() for i in range(len(seqs))]


def _cpu_hashes(seq, bs, parent):
    out, h = [], parent
    for b in range(0, len(seq), bs):
        h = O.chain_hash(h, seq[b:b + bs])
        out.append(int(h))
    return out


@pytest.mark.gpu
@pytest.mark.parametrize("bs", [16, 4])
@pytest.mark.parametrize("lens", [[8197], [0, 1, 15, 16, 17, 33], [16 * 40] * 33 + [16 * 40 + 3],
                                  [int(x) for x in np.random.default_rng(2).integers(0, 3000, 70)]])
def test_chain_hash_batch_matches_oracle(bs, lens):
    rng = np.random.default_rng(len(lens) * 31 + bs)
    seqs = [rng.integers(0, 2**63, n, dtype=np.uint64) for n in lens]
    got = _gpu_hashes(seqs, bs)
    for i, s in enumerate(seqs):
        assert got[i] == _cpu_hashes(s, bs, O.root_hash()), (i, len(s))
    parents = [int(x) for x in rng.integers(0, 2**63, len(seqs), dtype=np.uint64)]
    got = _gpu_hashes(seqs, bs, parents)
    for i, s in enumerate(seqs):
        assert got[i] == _cpu_hashes(s, bs, parents[i]), (i, len(s))


@pytest.mark.gpu
def test_chain_hash_segments_and_prefix_gather():
    """Incremental hashing: the suffix segments of prompts whose prefixes are
    cached fold from the prefix's last chain hash (sb_chain_hash_segments);
    the prefix hashes come from the pool (sb_kv_gather_chain_hashes).  Both
    must equal the oracle's full-prompt chain."""
    import torch
    from paper_2601_12967_b200 import _lib
    from paper_2601_12967_b200.kv_cache import CacheConfig, KvCache

    L = _lib.lib()
    rng = np.random.default_rng(9)
    bs = 16
    pre_lens, suf_lens = [32, 160, 16 * 37, 64], [5, 16, 700, 33]
    cache = KvCache(CacheConfig(bs, 512, 1))
    prompts, pre_ids = [], []
    for pl, sl in zip(pre_lens, suf_lens):
        t = rng.integers(0, 2**63, pl + sl, dtype=np.uint64)
        prompts.append(t)
        pre_ids.append(cache.insert(t[:pl], [(0, pl, 3)], 1))
    toks = np.concatenate(prompts)
    off = np.concatenate([[0], np.cumsum([len(t) for t in prompts])])
    nblk = [(len(t) + bs - 1) // bs for t in prompts]
    boff = np.concatenate([[0], np.cumsum(nblk)])
    seg = np.array([[off[i] + pre_lens[i], off[i + 1]] for i in range(len(prompts))], dtype=np.int64).ravel()
    segblk = np.array([boff[i] + pre_lens[i] // bs for i in range(len(prompts))], dtype=np.int64)
    ids = np.concatenate([np.array(x, dtype=np.int32) for x in pre_ids])
    pos = np.concatenate([boff[i] + np.arange(pre_lens[i] // bs) for i in range(len(prompts))]).astype(np.int64)
    last = np.array([x[-1] for x in pre_ids], dtype=np.int32)
    d = lambda a: torch.from_numpy(a).cuda()
    out = torch.zeros(int(boff[-1]), dtype=torch.int64, device="cuda")
    par = torch.zeros(len(prompts), dtype=torch.int64, device="cuda")
    p = lambda t: C.c_void_p(t.data_ptr())
    dt, dseg, dsb, dids, dpos, dlast = d(toks.view(np.int64)), d(seg), d(segblk), d(ids), d(pos), d(last)
    _lib.check(L.sb_kv_gather_chain_hashes(cache.handle, p(dids), p(dpos), len(ids), p(out), None))
    _lib.check(L.sb_kv_gather_chain_hashes(cache.handle, p(dlast), None, len(last), p(par), None))
    _lib.check(L.sb_chain_hash_segments(p(dt), p(dseg), p(dsb), p(par), len(prompts), bs, p(out), None))
    torch.cuda.synchronize()
    h = out.cpu().numpy().view(np.uint64)
    for i, t in enumerate(prompts):
        assert h[boff[i]:boff[i + 1]].tolist() == _cpu_hashes(t, bs, O.root_hash()), i
