"""GPU numerics of the dense layers around the continuation attention
(csrc/model.cu, attached to a ContinuationBatch): the engine's continuation
step — embed, per layer RMSNorm / QKV / RoPE + KV scatter into the pool pages
/ paged continuation attention / O projection / SwiGLU MLP, final norm + LM
head on each sequence's last token — against a torch fp32 restatement that
uses the same weights (read back from the device) and the same cached prefix
pages, rounding activations to bf16 where the device path stores them.

Tolerance (bf16 activations, fp32 accumulation): last-token logits within
2e-2 of the reference's max |logit|; greedy tokens equal wherever the
reference's top-2 gap exceeds that tolerance."""
import math

import numpy as np
import pytest

from oracle import oracle as O

BS = 16


def _bf(x):
    import torch

    return x.to(torch.bfloat16).float()


class _DevBuf:
    """A raw device pointer exposed through __cuda_array_interface__."""

    def __init__(self, ptr, n):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<i2", "data": (ptr, False), "version": 3}


def _dev_tensor(ptr, n, shape):
    """fp32 copy of a bf16 device buffer owned by the library."""
    import torch

    t = torch.as_tensor(_DevBuf(ptr, n), device="cuda").view(torch.bfloat16)
    return t.float().reshape(shape).clone()


def _rope(x, pos, theta):
    """x [T, H, 128] fp32, rotate-half RoPE at absolute positions pos [T]."""
    import torch

    f = torch.arange(64, dtype=torch.float64, device=x.device)
    inv = theta ** (-2.0 * f / 128.0)
    ang = pos.double()[:, None] * inv[None, :]
    c, s = torch.cos(ang).float()[:, None, :], torch.sin(ang).float()[:, None, :]
    x1, x2 = x[..., :64], x[..., 64:]
    return torch.cat([x1 * c - x2 * s, x2 * c + x1 * s], -1)


def _rms(x, w, eps=1e-5):
    return x * (x.pow(2).mean(-1, keepdim=True) + eps).rsqrt() * w


def _dense_check(ds, prefix_lens, suffix_lens, model_seed=3, eng_seed=7):
    """Run one continuation step of the dense model through the engine and
    compare last-token logits with the torch fp32 restatement."""
    import torch
    import torch.nn.functional as F
    from paper_2601_12967_b200.engine import ContinuationEngine, DenseModel, ModelShape

    hq, hkv, d, dff, vocab, nl = ds.n_q_heads, ds.n_kv_heads, ds.d_model, ds.d_ff, ds.vocab, ds.n_layers
    cap = sum((p + s + 15) // 16 for p, s in zip(prefix_lens, suffix_lens)) + 4 + len(prefix_lens)
    eng = ContinuationEngine(ModelShape(nl, hq, hkv, 128), cap, policy=1, seed=eng_seed)
    model = DenseModel(ds, seed=model_seed)
    prefixes = [O.materialize(0, p, 100 + i) for i, p in enumerate(prefix_lens)]
    batch = eng.make_batch(prefixes, [[(0, p, 3)] for p in prefix_lens], suffix_lens)
    batch.set_model(model)
    rng = np.random.default_rng(1)
    suffix = rng.integers(0, 2**62, sum(suffix_lens), dtype=np.int64)
    batch.stage_suffix_device(torch.from_numpy(suffix).cuda())
    batch.run(now=5, seed=0)
    nxt, logits = batch.model_result(logits=True)
    hits, status, ids = batch.results()
    assert (status == 0).all()

    # ---- torch restatement
    W = {}
    for l in range(nl):
        for which, shp in ((0, ((hq + 2 * hkv) * 128, d)), (1, (d, d)), (2, (2 * dff, d)), (3, (d, dff)), (4, (d,)),
                           (5, (d,))):
            ptr, n = model.weight(l, which)
            W[l, which] = _dev_tensor(ptr, n, shp)
    emb = _dev_tensor(*model.weight(-1, 0), (vocab, d))
    lm = _dev_tensor(*model.weight(-1, 1), (vocab, d))
    fnorm = _dev_tensor(*model.weight(-1, 2), (d,))
    blk = np.cumsum([0] + [(p + s + 15) // 16 for p, s in zip(prefix_lens, suffix_lens)])
    ref_logits = []
    off = 0
    for si, (p, s) in enumerate(zip(prefix_lens, suffix_lens)):
        tok = torch.from_numpy(suffix[off:off + s].view(np.uint64) % np.uint64(vocab)).long().cuda()
        off += s
        x = emb[tok]  # bf16 values already
        pos = torch.arange(p, p + s, device="cuda")
        pages = torch.from_numpy(ids[blk[si]:blk[si] + p // 16]).long().cuda()
        for l in range(nl):
            kp = _dev_tensor(eng.k_pool(l), cap * hkv * 16 * 128, (cap, hkv, 16, 128))
            vp = _dev_tensor(eng.v_pool(l), cap * hkv * 16 * 128, (cap, hkv, 16, 128))
            xn = _bf(_rms(x, W[l, 4]))
            qkv = _bf(xn @ W[l, 0].t()).reshape(s, hq + 2 * hkv, 128)
            q = _bf(_rope(qkv[:, :hq], pos, ds.rope_theta))
            k = _bf(_rope(qkv[:, hq:hq + hkv], pos, ds.rope_theta))
            v = qkv[:, hq + hkv:]
            kpre = kp[pages].permute(1, 0, 2, 3).reshape(hkv, -1, 128)  # [hkv, p, 128]
            vpre = vp[pages].permute(1, 0, 2, 3).reshape(hkv, -1, 128)
            del kp, vp
            K = torch.cat([kpre, k.permute(1, 0, 2)], 1).repeat_interleave(hq // hkv, 0)
            V = torch.cat([vpre, v.permute(1, 0, 2)], 1).repeat_interleave(hq // hkv, 0)
            sc = q.permute(1, 0, 2) @ K.transpose(1, 2) / math.sqrt(128)
            mask = torch.arange(p + s, device="cuda")[None, :] > (p + torch.arange(s, device="cuda"))[:, None]
            a = _bf((torch.softmax(sc.masked_fill(mask, float("-inf")), -1) @ V).permute(1, 0, 2).reshape(s, d))
            del K, V, sc
            x = _bf(x + a @ W[l, 1].t())
            xn = _bf(_rms(x, W[l, 5]))
            gu = _bf(xn @ W[l, 2].t())
            h = _bf(F.silu(gu[:, :dff]) * gu[:, dff:])
            x = _bf(x + h @ W[l, 3].t())
        xl = _bf(_rms(x[-1:], fnorm))
        ref_logits.append((xl @ lm.t())[0])
    ref = torch.stack(ref_logits).cpu()
    got = torch.from_numpy(logits)
    tol = 2e-2 * ref.abs().max().item()
    err = (got - ref).abs().max().item()
    print(f"dense step {ds}: max |logit err| {err:.3e} vs tol {tol:.3e} (max |logit| {ref.abs().max().item():.3f})")
    assert ref.abs().max().item() > 0
    assert err <= tol, (err, tol)
    top2 = ref.topk(2, -1).values
    for i in range(len(prefix_lens)):
        if (top2[i, 0] - top2[i, 1]).item() > 2 * tol:
            assert nxt[i] == int(ref[i].argmax()), i


@pytest.mark.gpu
@pytest.mark.parametrize("prefix_lens,suffix_lens", [([48, 96, 16], [37, 70, 1]), ([256], [130])])
def test_dense_step_matches_torch_reference(prefix_lens, suffix_lens):
    from paper_2601_12967_b200.engine import DenseShape

    ds = DenseShape(n_layers=2, d_model=512, n_q_heads=4, n_kv_heads=2, d_ff=1024, vocab=1000, rope_theta=10000.0)
    _dense_check(ds, prefix_lens, suffix_lens)


@pytest.mark.gpu
@pytest.mark.parametrize("n_layers,prefix_lens,suffix_lens", [(2, [8192], [256]), (1, [32768, 8192], [160, 96])])
def test_dense_step_at_llama3_8b_shape(n_layers, prefix_lens, suffix_lens):
    """configs[2]'s model shape: d_model 4096, 32 q / 8 kv heads, d_ff 14336,
    vocab 128256, RoPE theta 5e5, 8K and 32K cached prefixes."""
    from paper_2601_12967_b200.engine import LLAMA3_8B_DENSE, DenseShape

    ds = DenseShape(n_layers=n_layers, d_model=LLAMA3_8B_DENSE.d_model, n_q_heads=LLAMA3_8B_DENSE.n_q_heads,
                    n_kv_heads=LLAMA3_8B_DENSE.n_kv_heads, d_ff=LLAMA3_8B_DENSE.d_ff, vocab=LLAMA3_8B_DENSE.vocab,
                    rope_theta=LLAMA3_8B_DENSE.rope_theta)
    _dense_check(ds, prefix_lens, suffix_lens)


def _torch_forward_logits(tok_ids, W, emb, lm, fnorm, nl, hq, hkv, d, dff, theta):
    """Monolithic fp32 forward (bf16 rounding where the device stores) of one
    whole prompt: last-token logits."""
    import torch
    import torch.nn.functional as F

    s = len(tok_ids)
    x = emb[tok_ids]
    pos = torch.arange(0, s, device="cuda")
    mask = torch.arange(s, device="cuda")[None, :] > torch.arange(s, device="cuda")[:, None]
    for l in range(nl):
        xn = _bf(_rms(x, W[l, 4]))
        qkv = _bf(xn @ W[l, 0].t()).reshape(s, hq + 2 * hkv, 128)
        q = _bf(_rope(qkv[:, :hq], pos, theta))
        k = _bf(_rope(qkv[:, hq:hq + hkv], pos, theta))
        v = qkv[:, hq + hkv:]
        K = k.permute(1, 0, 2).repeat_interleave(hq // hkv, 0)
        V = v.permute(1, 0, 2).repeat_interleave(hq // hkv, 0)
        sc = q.permute(1, 0, 2) @ K.transpose(1, 2) / math.sqrt(128)
        a = _bf((torch.softmax(sc.masked_fill(mask, float("-inf")), -1) @ V).permute(1, 0, 2).reshape(s, d))
        x = _bf(x + a @ W[l, 1].t())
        xn = _bf(_rms(x, W[l, 5]))
        gu = _bf(xn @ W[l, 2].t())
        h = _bf(F.silu(gu[:, :dff]) * gu[:, dff:])
        x = _bf(x + h @ W[l, 3].t())
    return (_bf(_rms(x[-1:], fnorm)) @ lm.t())[0]


@pytest.mark.gpu
def test_split_prefill_equals_monolithic_prefill():
    """Prompt splitting (paper §4.2) is exact: prefill the tool-independent
    prefix (its uncached part, while the tool runs), then the continuation of
    the tool output over the cached pages, gives the same last-token logits as
    one prefill of the whole prompt.  Request B shares A's system prompt, so
    its prefix prefill starts at A's cached blocks."""
    import torch
    from paper_2601_12967_b200.engine import ContinuationEngine, DenseModel, DenseShape, ModelShape

    hq, hkv, d, dff, vocab, nl = 4, 2, 512, 1024, 1000, 2
    ds = DenseShape(n_layers=nl, d_model=d, n_q_heads=hq, n_kv_heads=hkv, d_ff=dff, vocab=vocab, rope_theta=10000.0)
    eng = ContinuationEngine(ModelShape(nl, hq, hkv, 128), 256, policy=1, seed=9)
    model = DenseModel(ds, seed=4)
    rng = np.random.default_rng(3)
    system = rng.integers(0, 2**62, 64, dtype=np.int64).view(np.uint64)
    pre_a = np.concatenate([system, rng.integers(0, 2**62, 96, dtype=np.int64).view(np.uint64)])
    pre_b = np.concatenate([system, rng.integers(0, 2**62, 80, dtype=np.int64).view(np.uint64)])
    tags_a, tags_b = [(0, 64, 3), (64, 160, 2)], [(0, 64, 3), (64, 144, 2)]
    ha = eng.submit_partial_prefill(pre_a, tags_a, now=0)
    assert eng.prefill_done(ha, now=0) == eng.PINNED      # pages of the prefix admitted
    hb = eng.submit_partial_prefill(pre_b, tags_b, now=1)
    assert eng.prefill_done(hb, now=1) == eng.PINNED
    assert eng.cached_at_submit(ha) == 0 and eng.cached_at_submit(hb) == 64
    eng.prefill_partials([ha, hb], model)          # while the tools run
    sfx = [37, 50]
    batch = eng.make_batch([pre_a, pre_b], [tags_a, tags_b], sfx)  # the tool outputs arrive
    batch.set_model(model)
    suffix = rng.integers(0, 2**62, sum(sfx), dtype=np.int64)
    batch.stage_suffix_device(torch.from_numpy(suffix).cuda())
    batch.run(now=5, seed=0)
    _, logits = batch.model_result(logits=True)
    assert (batch.results()[1] == 0).all()

    W = {}
    for l in range(nl):
        for which, shp in ((0, ((hq + 2 * hkv) * 128, d)), (1, (d, d)), (2, (2 * dff, d)), (3, (d, dff)), (4, (d,)),
                           (5, (d,))):
            W[l, which] = _dev_tensor(*model.weight(l, which), shp)
    emb = _dev_tensor(*model.weight(-1, 0), (vocab, d))
    lm = _dev_tensor(*model.weight(-1, 1), (vocab, d))
    fnorm = _dev_tensor(*model.weight(-1, 2), (d,))
    refs = []
    for pre, (o, n) in zip((pre_a, pre_b), ((0, sfx[0]), (sfx[0], sfx[1]))):
        whole = np.concatenate([pre, suffix[o:o + n].view(np.uint64)])
        ids = torch.from_numpy((whole % np.uint64(vocab)).astype(np.int64)).cuda()
        refs.append(_torch_forward_logits(ids, W, emb, lm, fnorm, nl, hq, hkv, d, dff, ds.rope_theta))
    ref = torch.stack(refs).cpu()
    got = torch.from_numpy(logits)
    tol = 2e-2 * ref.abs().max().item()
    err = (got - ref).abs().max().item()
    print(f"split vs monolithic prefill: max |logit err| {err:.3e} vs tol {tol:.3e}")
    assert err <= tol, (err, tol)

    # negative control: without the partial prefill the prefix pages hold the
    # engine's stand-in KV, and the same check must fail
    eng2 = ContinuationEngine(ModelShape(nl, hq, hkv, 128), 256, policy=1, seed=9)
    b2 = eng2.make_batch([pre_a, pre_b], [tags_a, tags_b], sfx)
    b2.set_model(model)
    b2.stage_suffix_device(torch.from_numpy(suffix).cuda())
    b2.run(now=5, seed=0)
    _, lg2 = b2.model_result(logits=True)
    assert (torch.from_numpy(lg2) - ref).abs().max().item() > tol
