"""The decode operations around the attention (toy_model.hpp:161-274, SURVEY
8(f) rank 4) on the device -- csrc/model.cu through lyc_gemv -- against plain
PyTorch fp32 references of the same ops, and a whole decode step of the toy
model (decode_engine.hpp:95-151) against an fp32 restatement that rounds at
the same points (bf16 q / cache rows / attention outputs / FFN activations)."""
import math

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.set_device(0)


def rel(a, b):
    a, b = a.double(), b.double()
    return ((a - b).abs().max() / b.abs().max().clamp_min(1e-3)).item()


def rmsnorm(x, gain, eps=1e-6):  # toy_model.hpp:161-169
    return x * torch.rsqrt((x * x).mean() + eps) * gain


def rope(v, pos, d):  # toy_model.hpp:184-194, pairs (i, i+1) per head
    v = v.double().view(-1, d).clone()
    i = torch.arange(0, d, 2, dtype=torch.float64, device=v.device)
    ang = pos * torch.pow(10000.0, -i / d)
    c, s = torch.cos(ang), torch.sin(ang)
    a, b = v[:, 0::2].clone(), v[:, 1::2].clone()
    v[:, 0::2] = a * c - b * s
    v[:, 1::2] = a * s + b * c
    return v.view(-1).float()


@pytest.mark.parametrize("M,K", [(4096, 4096), (1000, 14336), (130, 64)])
def test_gemv_modes_vs_torch(M, K):
    from paper_2602_04541_b200 import _lib as LL
    from paper_2602_04541_b200.model import gemv
    g = torch.Generator(device="cuda").manual_seed(M + K)
    w = torch.randn((M, K), generator=g, device="cuda").mul_(K ** -0.5).bfloat16()
    x = torch.randn(K, generator=g, device="cuda")
    gain = 1 + 0.1 * torch.randn(K, generator=g, device="cuda")
    wf = w.float()
    # STORE with the rmsnorm prologue (output_logits)
    y = torch.empty(M, device="cuda")
    gemv(w, x=x, gain=gain, mode=LL.GEMV_STORE, y=y)
    assert rel(y, wf @ rmsnorm(x, gain)) < 1e-4
    # RESIDUAL from a bf16 input (attn_project_residual / ffn_residual)
    xb = x.bfloat16()
    base = torch.randn(M, generator=g, device="cuda")
    y = base.clone()
    gemv(w, xb=xb, mode=LL.GEMV_RESIDUAL, y=y)
    assert rel(y, base + wf @ xb.float()) < 1e-4
    # SILU_BF16 (the FFN's W1)
    yb = torch.empty(M, dtype=torch.bfloat16, device="cuda")
    gemv(w, x=x, gain=gain, mode=LL.GEMV_SILU_BF16, yb=yb)
    ref = torch.nn.functional.silu(wf @ rmsnorm(x, gain))
    assert rel(yb.float(), ref) < 1e-2


def test_prefetch_hint_leaves_results_unchanged():
    """lyc_gemv_desc.prefetch (L2 prefetch of the next launch's weights) is a
    hint only: outputs bitwise equal with and without it."""
    from paper_2602_04541_b200 import _lib as LL
    from paper_2602_04541_b200.model import gemv
    g = torch.Generator(device="cuda").manual_seed(11)
    w = torch.randn((3000, 4096), generator=g, device="cuda").bfloat16()
    nxt = torch.randn((4096, 4096), generator=g, device="cuda").bfloat16()
    x = torch.randn(4096, generator=g, device="cuda")
    gain = torch.ones(4096, device="cuda")
    y0, y1 = torch.empty(3000, device="cuda"), torch.empty(3000, device="cuda")
    gemv(w, x=x, gain=gain, mode=LL.GEMV_STORE, y=y0)
    gemv(w, x=x, gain=gain, mode=LL.GEMV_STORE, y=y1, prefetch=nxt)
    gemv(w, x=x, gain=gain, mode=LL.GEMV_STORE, y=y1, prefetch=nxt, prefetch_bytes=1 << 20)
    torch.cuda.synchronize()
    assert torch.equal(y0, y1)


def test_next_is_gemv_flag_chain_equals_plain_chain():
    """LYC_GEMV_FLAG_NEXT_IS_GEMV only lets the next launch be scheduled
    early (it still waits for this one's completion): a dependent chain
    x -> W_o residual -> W_1 silu -> W_2 residual gives bitwise-equal results."""
    from paper_2602_04541_b200 import _lib as LL
    from paper_2602_04541_b200.model import gemv
    g = torch.Generator(device="cuda").manual_seed(12)
    D, F = 1024, 3072
    wo = torch.randn((D, D), generator=g, device="cuda").mul_(D ** -0.5).bfloat16()
    w1 = torch.randn((F, D), generator=g, device="cuda").mul_(D ** -0.5).bfloat16()
    w2 = torch.randn((D, F), generator=g, device="cuda").mul_(F ** -0.5).bfloat16()
    o = torch.randn(D, generator=g, device="cuda").bfloat16()
    gain = 1 + 0.1 * torch.randn(D, generator=g, device="cuda")
    x0 = torch.randn(D, generator=g, device="cuda")
    outs = []
    for flag in (False, True):
        x = x0.clone()
        mid = torch.empty(F, dtype=torch.bfloat16, device="cuda")
        for _ in range(3):
            gemv(wo, xb=o, mode=LL.GEMV_RESIDUAL, y=x, next_is_gemv=flag)
            gemv(w1, x=x, gain=gain, mode=LL.GEMV_SILU_BF16, yb=mid, next_is_gemv=flag)
            gemv(w2, xb=mid, mode=LL.GEMV_RESIDUAL, y=x, next_is_gemv=False)
        torch.cuda.synchronize()
        outs.append(x)
    assert torch.equal(outs[0], outs[1])


def test_qkv_rope_writes_q_and_cache_rows():
    from paper_2602_04541_b200 import _lib as LL
    from paper_2602_04541_b200.model import gemv
    nq, nkv, d, D, cap, pos = 8, 2, 64, 512, 100, 37
    g = torch.Generator(device="cuda").manual_seed(3)
    M = (nq + 2 * nkv) * d
    w = torch.randn((M, D), generator=g, device="cuda").mul_(D ** -0.5).bfloat16()
    x = torch.randn(D, generator=g, device="cuda")
    gain = 1 + 0.1 * torch.randn(D, generator=g, device="cuda")
    q = torch.empty(nq * d, dtype=torch.bfloat16, device="cuda")
    kc = torch.zeros((nkv, cap, d), dtype=torch.bfloat16, device="cuda")
    vc = torch.zeros_like(kc)
    gemv(w, x=x, gain=gain, mode=LL.GEMV_QKV_ROPE, q_out=q, k_cache=kc, v_cache=vc,
         slab_stride=cap * d, nq=nq, nkv=nkv, d=d, pos=pos)
    torch.cuda.synchronize()
    y = w.float() @ rmsnorm(x, gain)
    qr = rope(y[:nq * d], pos, d)
    kr = rope(y[nq * d:(nq + nkv) * d], pos, d).view(nkv, d)
    vr = y[(nq + nkv) * d:].view(nkv, d)
    assert rel(q.float(), qr) < 1e-2
    assert rel(kc[:, pos].float(), kr) < 1e-2
    assert rel(vc[:, pos].float(), vr) < 1e-2
    others = torch.cat([kc[:, :pos], kc[:, pos + 1:], vc[:, :pos], vc[:, pos + 1:]], 1)
    assert others.abs().max().item() == 0  # only row `pos` was written


def _reference_token(m, token, pos):
    """decode_engine.hpp:95-151 + toy_model.hpp in fp32 with full (dense)
    attention, rounding to bf16 where the device path stores bf16."""
    cfg = m.cfg
    d, nq, H, G = cfg.d_head, cfg.n_q_heads, cfg.n_kv_heads, cfg.group_size
    bf = lambda t: t.bfloat16().float()  # noqa: E731
    x = m.embedding[token].float().clone()
    K = m.k[:, 0].float().clone()
    V = m.v[:, 0].float().clone()
    for l in range(cfg.n_layers):
        y = m.wqkv[l].float() @ rmsnorm(x, m.attn_norm[l])
        q = bf(rope(y[:nq * d], pos, d)).view(nq, d)
        K[l, :, pos] = bf(rope(y[nq * d:(nq + H) * d], pos, d)).view(H, d)
        V[l, :, pos] = bf(y[(nq + H) * d:]).view(H, d)
        o = torch.empty(nq, d, device=x.device)
        for hd in range(nq):  # dense_attention (attention.hpp:50-75)
            s = K[l, hd // G, :pos + 1] @ q[hd] / math.sqrt(d)
            o[hd] = torch.softmax(s, 0) @ V[l, hd // G, :pos + 1]
        x = x + m.wo[l].float() @ bf(o).view(-1)
        mid = bf(torch.nn.functional.silu(m.w1[l].float() @ rmsnorm(x, m.ffn_norm[l])))
        x = x + m.w2[l].float() @ mid
    return m.lm_head.float() @ rmsnorm(x, m.final_norm)


def test_decode_token_full_attention_vs_fp32_reference():
    import paper_2602_04541_b200 as P
    from paper_2602_04541_b200.model import PRESETS
    cfg = P.ModelConfig(max_seq_len=512, **PRESETS["tiny"])
    m = P.DecodeModel(cfg, attention="full", seed=5)
    pos = 300
    m.fill_cache(pos)
    ref = _reference_token(m, 17, pos)
    logits = m.decode_token(17, pos).clone()
    torch.cuda.synchronize()
    assert rel(logits, ref) < 2e-2
    m.close()


def test_decode_token_hybrid_full_budget_equals_full():
    """With a budget >= the context every sparse head attends every token, so
    the hybrid step equals the dense one (decode_engine_test.cpp:184-222)."""
    import paper_2602_04541_b200 as P
    from paper_2602_04541_b200.model import PRESETS
    cfg = P.ModelConfig(max_seq_len=512, **PRESETS["tiny"])
    roles = np.ones((cfg.n_layers, cfg.n_kv_heads), np.uint8)
    roles[0] = 0
    pos = 200
    out = []
    for att in ("full", "hybrid"):
        m = P.DecodeModel(cfg, attention=att, roles=roles, policy=P.SparsityPolicy.top_k(512), seed=5)
        m.fill_cache(pos)
        out.append(m.decode_token(3, pos).clone())
        m.close()
    torch.cuda.synchronize()
    assert rel(out[1], out[0]) < 2e-2
