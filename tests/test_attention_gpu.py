"""GPU numerics of the continuation-prefill attention kernel (csrc/attention.cu)
against a plain PyTorch fp32 reference of the same op.  Tolerance (north
star): bf16 outputs within 1e-2 relative (max-norm) of the fp32 reference."""
import math

import numpy as np
import pytest

REL_TOL_BF16 = 1e-2


def ref_attention(q, k_pool, v_pool, q_off, kv_lens, table, scale):
    """fp32 reference: gather pages, causal over the suffix, full over the prefix."""
    import torch

    dt = torch.float64 if q.dtype == torch.float64 else torch.float32
    out = torch.zeros_like(q, dtype=dt)
    n_kv = k_pool.shape[1]
    group = q.shape[1] // n_kv
    for s in range(len(kv_lens)):
        a, b = int(q_off[s]), int(q_off[s + 1])
        ql, kl = b - a, int(kv_lens[s])
        if ql == 0:
            continue
        pages = table[s, : (kl + 15) // 16].long()
        k = k_pool[pages].to(dt).permute(1, 0, 2, 3).reshape(n_kv, -1, 128)[:, :kl]  # [kvh, kl, d]
        v = v_pool[pages].to(dt).permute(1, 0, 2, 3).reshape(n_kv, -1, 128)[:, :kl]
        qs = q[a:b].to(dt).permute(1, 0, 2)  # [hq, ql, d]
        k = k.repeat_interleave(group, 0)
        v = v.repeat_interleave(group, 0)
        sc = qs @ k.transpose(1, 2) * scale  # [hq, ql, kl]
        qpos = torch.arange(kl - ql, kl, device=q.device)[:, None]
        kpos = torch.arange(kl, device=q.device)[None, :]
        sc = sc.masked_fill(kpos > qpos, float("-inf"))
        out[a:b] = (torch.softmax(sc, -1) @ v).permute(1, 0, 2)
    return out


def make_case(q_lens, prefix_lens, n_q_heads, n_kv_heads, seed=0, pool_extra=7):
    import torch

    g = torch.Generator().manual_seed(seed)
    kv_lens = [p + q for p, q in zip(prefix_lens, q_lens)]
    max_blocks = max((k + 15) // 16 for k in kv_lens)
    n_blocks = sum((k + 15) // 16 for k in kv_lens) + pool_extra
    perm = torch.randperm(n_blocks, generator=g)
    table = torch.zeros(len(q_lens), max_blocks, dtype=torch.int32)
    c = 0
    for s, k in enumerate(kv_lens):
        nb = (k + 15) // 16
        table[s, :nb] = perm[c:c + nb].int()
        c += nb
    k_pool = (torch.randn(n_blocks, n_kv_heads, 16, 128, generator=g)).to(torch.bfloat16)
    v_pool = (torch.randn(n_blocks, n_kv_heads, 16, 128, generator=g)).to(torch.bfloat16)
    q = (torch.randn(sum(q_lens), n_q_heads, 128, generator=g) * 1.5).to(torch.bfloat16)
    q_off = torch.tensor(np.cumsum([0] + list(q_lens)), dtype=torch.int32)
    return q, k_pool, v_pool, q_off, torch.tensor(kv_lens, dtype=torch.int32), table


CASES = [
    # (q_lens, prefix_lens, n_q_heads, n_kv_heads)
    ([64], [0], 4, 1),                        # single tile, no prefix
    ([32], [128], 4, 1),                      # exactly one prefix tile
    ([100, 37, 1], [300, 0, 1000], 8, 2),     # ragged, non-multiples of 16/128
    ([257, 64], [2048, 4095], 32, 8),         # Llama-3-8B heads, multi-tile
    ([130], [70], 2, 2),                      # MHA (group 1): 128 tokens per tile
    ([96, 200], [500, 33], 16, 8),            # group 2
    ([40, 17], [32768, 20000], 32, 8),        # configs[2]-long cached prefixes (2K+ pages per sequence)
    ([50, 300], [1000, 16], 64, 8),           # group 8 (Llama-3-70B heads): 16 tokens per tile
    ([20, 9], [77, 0], 16, 1),                # group 16
    ([0, 45, 0], [100, 60, 7], 8, 2),         # sequences without suffix tokens in the batch
    ([256], [256], 4, 4),                     # group 1, exactly one tile pair, block-aligned prefix
]


@pytest.mark.gpu
@pytest.mark.parametrize("case", CASES)
@pytest.mark.parametrize("use_work_list", [False, True])
def test_continuation_attention_matches_fp32(case, use_work_list):
    import torch
    from paper_2601_12967_b200.attention import attention_work_list, continuation_attention

    q_lens, prefix, hq, hkv = case
    q, kp, vp, qo, kl, tb = make_case(q_lens, prefix, hq, hkv)
    dev = torch.device("cuda")
    q, kp, vp, qo, kl, tb = (x.to(dev) for x in (q, kp, vp, qo, kl, tb))
    scale = 1.0 / math.sqrt(128)
    work = None
    if use_work_list:
        w = attention_work_list(q_lens, [p + ql for p, ql in zip(prefix, q_lens)], hq, hkv)
        work = torch.from_numpy(w.copy()).to(dev)
    out = continuation_attention(q, kp, vp, qo, kl, tb, max(q_lens), scale, work=work)
    torch.cuda.synchronize()
    ref = ref_attention(q, kp, vp, qo.cpu(), kl.cpu(), tb, scale)
    err = (out.float() - ref).abs().max().item()
    assert torch.isfinite(out.float()).all()
    rel = err / ref.abs().max().item()
    assert rel <= REL_TOL_BF16, rel


@pytest.mark.gpu
def test_kv_append_then_attend():
    """extend_prefill semantics: write the suffix K/V into pool pages, then the
    suffix queries attend over prefix + suffix."""
    import torch
    from paper_2601_12967_b200.attention import continuation_attention, kv_append

    dev = torch.device("cuda")
    q_lens, prefix = [48, 130], [200, 16]
    q, kp, vp, qo, kl, tb = (x.to(dev) for x in make_case(q_lens, prefix, 8, 2, seed=3))
    g = torch.Generator(device="cpu").manual_seed(4)
    k_new = torch.randn(sum(q_lens), 2, 128, generator=g).to(torch.bfloat16).to(dev)
    v_new = torch.randn(sum(q_lens), 2, 128, generator=g).to(torch.bfloat16).to(dev)
    kv_append(k_new, v_new, kp, vp, qo, kl, tb)
    torch.cuda.synchronize()
    # the appended rows are where the table says
    for s, (ql, pl) in enumerate(zip(q_lens, prefix)):
        for i in (0, ql - 1):
            pos = pl + i
            page = int(tb[s, pos // 16])
            tok = int(qo[s]) + i
            assert torch.equal(kp[page, :, pos % 16], k_new[tok])
            assert torch.equal(vp[page, :, pos % 16], v_new[tok])
    out = continuation_attention(q, kp, vp, qo, kl, tb, max(q_lens))
    ref = ref_attention(q, kp, vp, qo.cpu(), kl.cpu(), tb, 1 / math.sqrt(128))
    assert (out.float() - ref).abs().max().item() <= REL_TOL_BF16 * ref.abs().max().item()


@pytest.mark.gpu
def test_running_max_keeps_growing():
    """Scores that rise along the key axis force the online softmax to raise
    its running max (and lazily rescale O in TMEM) again and again."""
    import torch
    from paper_2601_12967_b200.attention import continuation_attention

    q_lens, prefix = [70, 33], [3000, 1200]
    q, kp, vp, qo, kl, tb = make_case(q_lens, prefix, 8, 2, seed=5)
    # key position p of sequence s gets dim 0 = p / 64 (bf16-exact multiples), queries dim 0 = 2:
    # the logit grows by ~0.25 nats per 16 keys -> a new max far above the old one every few tiles
    for s, k in enumerate([p + ql for p, ql in zip(prefix, q_lens)]):
        for pos in range(k):
            kp[tb[s, pos // 16], :, pos % 16, 0] = pos / 64.0
    q[:, :, 0] = 2.0
    dev = torch.device("cuda")
    q, kp, vp, qo, kl, tb = (x.to(dev) for x in (q, kp, vp, qo, kl, tb))
    out = continuation_attention(q, kp, vp, qo, kl, tb, max(q_lens))
    torch.cuda.synchronize()
    ref = ref_attention(q, kp, vp, qo.cpu(), kl.cpu(), tb, 1 / math.sqrt(128))
    assert torch.isfinite(out.float()).all()
    err = (out.float() - ref).abs().max().item()
    assert err <= REL_TOL_BF16 * ref.abs().max().item(), err


@pytest.mark.gpu
def test_attention_at_the_bench_shape():
    """The configs[1] step's attention problem itself (64 requests, 98,896
    suffix queries over 441,888 cached prefix keys, 32 q / 8 kv heads, pages
    spread over the pool): sampled sequences x every head x first / middle /
    last query rows vs the fp32 reference, max-norm relative <= 1e-2; and,
    when flashinfer's trtllm-gen paged kernel loads, the whole output against
    it within the same bound."""
    import torch
    import bench_attn

    q, kp, vp, q_off, kvl, table, work, out, run_ours, run_fi = bench_attn.setup(64, flashinfer=True)
    run_ours()
    torch.cuda.synchronize()
    n = len(kvl)
    qo = q_off.cpu().tolist()
    worst = 0.0
    for s in range(0, n, 7):
        a, b = qo[s], qo[s + 1]
        rows = sorted({a, a + 1, (a + b) // 2, b - 2, b - 1})
        kl = int(kvl[s])
        pages = table[s, : (kl + 15) // 16].long()
        k = kp[pages].float().permute(1, 0, 2, 3).reshape(8, -1, 128)[:, :kl].repeat_interleave(4, 0)
        v = vp[pages].float().permute(1, 0, 2, 3).reshape(8, -1, 128)[:, :kl].repeat_interleave(4, 0)
        for r in rows:
            qs = q[r].float()[:, None, :]                              # [32, 1, 128]
            pos = kl - (b - a) + (r - a)
            sc = (qs @ k[:, : pos + 1].transpose(1, 2)) / math.sqrt(128)
            ref = (torch.softmax(sc, -1) @ v[:, : pos + 1])[:, 0]     # [32, 128]
            rel = ((out[r].float() - ref).abs().max() / ref.abs().max()).item()
            worst = max(worst, rel)
    print(f"bench-shape attention: worst sampled max-norm relative error {worst:.2e}")
    assert worst <= REL_TOL_BF16, worst
    if run_fi is not None:
        fo = run_fi()
        torch.cuda.synchronize()
        rel = ((fo.float() - out.float()).abs().max() / out.float().abs().max()).item()
        print(f"vs trtllm-gen: max-norm relative difference {rel:.2e}")
        assert rel <= REL_TOL_BF16, rel


REL_TOL_F32 = 1e-5


@pytest.mark.gpu
@pytest.mark.parametrize("case", [([64], [0], 4, 1), ([100, 37, 1], [300, 0, 1000], 8, 2), ([33], [2000], 2, 1),
                                  ([0, 50], [10, 300], 64, 8)])
def test_continuation_attention_f32_matches_fp32(case):
    """fp32 contract (north star: 1e-5 in fp32), e.g. the toy 2-layer d=256
    model of configs[0] (2 q heads x 128)."""
    import torch
    from paper_2601_12967_b200.attention import continuation_attention

    q_lens, prefix, hq, hkv = case
    q, kp, vp, qo, kl, tb = make_case(q_lens, prefix, hq, hkv, seed=11)
    dev = torch.device("cuda")
    q, kp, vp = (x.float().to(dev) for x in (q, kp, vp))
    qo, kl, tb = (x.to(dev) for x in (qo, kl, tb))
    out = continuation_attention(q, kp, vp, qo, kl, tb, max(q_lens))
    torch.cuda.synchronize()
    # float64 reference of the same op (so the tolerance measures our fp32 error)
    ref = ref_attention(q.double(), kp.double(), vp.double(), qo.cpu(), kl.cpu(), tb, 1 / math.sqrt(128))
    err = ((out.double() - ref).abs().max() / ref.abs().max()).item()
    assert err <= REL_TOL_F32, err


@pytest.mark.gpu
def test_pair_attention_kernel():
    """The default launch is the 1-CTA kernel; the same tests with
    SB_ATTN_PAIR=1 run the CTA-pair kernel (cta_group::2, the A/B arm)."""
    import os
    import subprocess
    import sys

    env = dict(os.environ, SB_ATTN_PAIR="1")
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", os.path.abspath(__file__), "-k",
                        "not pair_attention"], env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
