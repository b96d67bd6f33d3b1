"""Variable-length batches (second half): one decode step
over B independent sequences of different lengths (lyc_decoder_step_varlen).

The reference's Workload carries one seq_len (kernel_sim.hpp:126) and
DecodeEngine runs one sequence (decode_engine.hpp:95-151), so the oracle for
item b is the oracle's decode_step over item b alone at its own length: its
retrieval heads attend rows [0, len_b), select with budget(len_b), and its
sparse heads read those sets.
"""
import numpy as np
import pytest
import torch

from tests.test_gpu_decode import (BF16_TOL, FP32_TOL, _policy_weights, check_policy_set, check_set,
                                   pooled_scores, rel_err, roles_for)

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2602_04541_b200  # noqa: F401
    torch.cuda.set_device(0)


def synth(seed, NL, B, H, G, d, cap, dtype):
    g = torch.Generator().manual_seed(seed)
    q = (torch.rand((NL, B, H * G, d), generator=g) * 2 - 1).to(dtype)
    K = (torch.rand((NL, B, H, cap, d), generator=g) * 2 - 1).to(dtype)
    V = (torch.rand((NL, B, H, cap, d), generator=g) * 2 - 1).to(dtype)
    return q, K, V


def run(P, *, NL, B, H, G, d, cap, lens, dtype, roles, policy, seed, select="tokens"):
    q, K, V = synth(seed, NL, B, H, G, d, cap, dtype)
    dec = P.HybridDecoder(n_layers=NL, batch=B, n_kv_heads=H, group_size=G, d_head=d, seq_cap=cap,
                          roles=roles, policy=policy, dtype=dtype, select=select)
    qd, Kd, Vd = q.cuda(), K.cuda(), V.cuda()
    out = dec.decode_step(qd, Kd, Vd, lens)
    torch.cuda.synchronize()
    return dec, (qd, Kd, Vd), q.float().numpy(), K.float().numpy(), V.float().numpy(), \
        out.float().cpu().numpy()


@pytest.mark.parametrize("kind,value,lens", [
    ("topk", 256, [1000, 100, 257]),        # 100 < k: every row of item 1 is kept
    ("topk", 256, [64, 4096, 1]),           # one-block item, a full item, a 1-token item
    ("ratio", 0.75, [777, 2048, 130]),      # per-item budget ceil(0.25 * len)
    ("topp", 0.4, [3000, 513, 64]),         # device-count sets per item
    ("threshold", 0.002, [1500, 700, 90]),
])
def test_varlen_fp32_vs_oracle(orc, kind, value, lens):
    import paper_2602_04541_b200 as P
    NL, B, H, G, d, cap = 4, len(lens), 2, 4, 64, 4096
    roles = roles_for(NL, H, [(2, 1)])
    policy = {"topk": lambda: P.SparsityPolicy.top_k(value),
              "ratio": lambda: P.SparsityPolicy.ratio(value),
              "topp": lambda: P.SparsityPolicy.top_p(value),
              "threshold": lambda: P.SparsityPolicy.threshold(value)}[kind]()
    dec, _, q, K, V, out = run(P, NL=NL, B=B, H=H, G=G, d=d, cap=cap, lens=lens,
                               dtype=torch.float32, roles=roles, policy=policy, seed=21)
    sets = dec.token_sets()
    scale = 1 / np.sqrt(d)
    diffs = 0
    for b, L in enumerate(lens):
        kw = dict(k=value) if kind == "topk" else dict(value=value)
        r = orc.decode_step(q[:, b], K[:, b], V[:, b], roles, seq=L, scale=scale, kind=kind, **kw)
        for g in range(H):
            assert np.all(np.diff(sets[b][g]) > 0) and sets[b][g].max() < L
            if kind in ("topk", "ratio"):
                kk = min(value, L) if kind == "topk" else orc.fraction_budget(1 - value, L)
                assert len(sets[b][g]) == kk
                src = max(ll for ll in range(NL) if roles[ll, g] == 0)
                sc = pooled_scores(q[src, b], K[src, b, g], G, g, L)
                assert check_set(sets[b][g], r["sets"][g], sc, kk) == 0
            else:
                src = max(ll for ll in range(NL) if roles[ll, g] == 0)
                w = _policy_weights(q[src, b], K[src, b, g], G, g, L, scale)
                diffs += check_policy_set(sets[b][g], r["sets"][g], w, kind, value)
        if diffs == 0:
            assert rel_err(out[:, b], r["out"]) < FP32_TOL, b


def test_varlen_bf16_llama_heads_vs_oracle(orc):
    """Llama-3-8B head shapes, bf16, two items of different lengths (ragged
    last blocks), TopK 512."""
    import paper_2602_04541_b200 as P
    NL, H, G, d, cap, k = 3, 8, 4, 128, 8192, 512
    lens = [8192, 3001]
    roles = roles_for(NL, H, [(1, 3), (2, 5)])
    dec, _, q, K, V, out = run(P, NL=NL, B=2, H=H, G=G, d=d, cap=cap, lens=lens,
                               dtype=torch.bfloat16, roles=roles, policy=P.SparsityPolicy.top_k(k),
                               seed=4)
    sets = dec.token_sets()
    swaps = 0
    for b, L in enumerate(lens):
        r = orc.decode_step(q[:, b], K[:, b], V[:, b], roles, seq=L, scale=1 / np.sqrt(d),
                            kind="topk", k=k)
        assert rel_err(out[:, b], r["out"]) < BF16_TOL
        for g in range(H):
            src = max(ll for ll in range(NL) if roles[ll, g] == 0)
            sc = pooled_scores(q[src, b], K[src, b, g], G, g, L)
            swaps += check_set(sets[b][g], r["sets"][g], sc, k)
    print("tie-band swaps:", swaps)


def test_equal_lengths_match_uniform_step_bitwise():
    """Equal lengths plan exactly like decode_step(int) (the fused step kernel)."""
    import paper_2602_04541_b200 as P
    NL, B, H, G, d, cap, L = 3, 2, 4, 4, 128, 4096, 3000
    roles = roles_for(NL, H, [(1, 2)])
    q, K, V = synth(8, NL, B, H, G, d, cap, torch.bfloat16)
    qd, Kd, Vd = q.cuda(), K.cuda(), V.cuda()
    mk = lambda: P.HybridDecoder(n_layers=NL, batch=B, n_kv_heads=H, group_size=G, d_head=d,  # noqa: E731
                                 seq_cap=cap, roles=roles, policy=P.SparsityPolicy.top_k(256),
                                 dtype=torch.bfloat16)
    d1, d2 = mk(), mk()
    o1 = d1.decode_step(qd, Kd, Vd, L)
    o2 = d2.decode_step(qd, Kd, Vd, [L] * B)
    torch.cuda.synchronize()
    assert torch.equal(o1, o2)
    # and a varlen step followed by a uniform one re-plans (no stale plan)
    d2.decode_step(qd, Kd, Vd, [L, 1200])
    o3 = d2.decode_step(qd, Kd, Vd, L)
    torch.cuda.synchronize()
    assert torch.equal(o1, o3)


def test_varlen_items_independent():
    """Item b's outputs do not depend on the other items' lengths."""
    import paper_2602_04541_b200 as P
    NL, B, H, G, d, cap = 3, 3, 2, 4, 64, 2048
    roles = roles_for(NL, H, [(1, 0)])
    q, K, V = synth(12, NL, B, H, G, d, cap, torch.float32)
    qd, Kd, Vd = q.cuda(), K.cuda(), V.cuda()
    dec = P.HybridDecoder(n_layers=NL, batch=B, n_kv_heads=H, group_size=G, d_head=d, seq_cap=cap,
                          roles=roles, policy=P.SparsityPolicy.top_k(128), dtype=torch.float32)
    a = dec.decode_step(qd, Kd, Vd, [900, 2000, 333]).clone()
    b = dec.decode_step(qd, Kd, Vd, [900, 50, 1777]).clone()
    torch.cuda.synchronize()
    assert torch.allclose(a[:, 0], b[:, 0], rtol=1e-6, atol=1e-6)


def test_varlen_errors():
    import paper_2602_04541_b200 as P
    NL, B, H, G, d, cap = 2, 2, 2, 2, 64, 512
    roles = roles_for(NL, H, [])
    q, K, V = synth(1, NL, B, H, G, d, cap, torch.float32)
    qd, Kd, Vd = q.cuda(), K.cuda(), V.cuda()
    dec = P.HybridDecoder(n_layers=NL, batch=B, n_kv_heads=H, group_size=G, d_head=d, seq_cap=cap,
                          roles=roles, policy=P.SparsityPolicy.top_k(16), dtype=torch.float32)
    with pytest.raises(P.InvalidArgument):
        dec.decode_step(qd, Kd, Vd, [100, 0])
    with pytest.raises(P.InvalidArgument):
        dec.decode_step(qd, Kd, Vd, [100, cap + 1])
    with pytest.raises(ValueError):
        dec.decode_step(qd, Kd, Vd, [100])


@pytest.mark.parametrize("select,k", [("tokens", 512), ("blocks", 1024)])
def test_varlen_fused_equals_per_item_decoders(select, k):
    """bf16 ragged batches run on the fused step kernel (per-row budgets, the
    padded tail of shorter rows masked out of the selection): every item's
    sets equal those of a batch-1 decoder at its own length, and its outputs
    agree within bf16 rounding (the split-KV partition differs)."""
    import paper_2602_04541_b200 as P
    NL, H, G, d, cap = 4, 8, 4, 128, 8192
    lens = [5000, 8192, 777]
    roles = roles_for(NL, H, [(1, 3), (2, 5), (3, 0)])
    B = len(lens)
    q, K, V = synth(31, NL, B, H, G, d, cap, torch.bfloat16)
    qd, Kd, Vd = q.cuda(), K.cuda(), V.cuda()
    mk = lambda b: P.HybridDecoder(n_layers=NL, batch=b, n_kv_heads=H, group_size=G,  # noqa: E731
                                   d_head=d, seq_cap=cap, roles=roles,
                                   policy=P.SparsityPolicy.top_k(k), dtype=torch.bfloat16,
                                   select=select)
    dec = mk(B)
    out = dec.decode_step(qd, Kd, Vd, lens)
    torch.cuda.synchronize()
    assert dec.fused
    sets = dec.token_sets()
    for b, L in enumerate(lens):
        one = mk(1)
        o1 = one.decode_step(qd[:, b:b + 1].contiguous(), Kd[:, b:b + 1].contiguous(),
                             Vd[:, b:b + 1].contiguous(), L)
        torch.cuda.synchronize()
        s1 = one.token_sets()[0]
        for g in range(H):
            assert np.array_equal(sets[b][g], s1[g]), (b, g)
        assert rel_err(out[:, b].float().cpu().numpy(), o1[:, 0].float().cpu().numpy()) < 1e-2


def test_varlen_graph_capture_replay():
    """lyc_decoder_capture_varlen: a replay of the captured ragged step equals
    the eager step bitwise (fused kernel, bf16)."""
    import paper_2602_04541_b200 as P
    NL, B, H, G, d, cap = 3, 3, 8, 4, 128, 4096
    lens = [4096, 1500, 2900]
    roles = roles_for(NL, H, [(1, 3), (2, 5)])
    q, K, V = synth(17, NL, B, H, G, d, cap, torch.bfloat16)
    qd, Kd, Vd = q.cuda(), K.cuda(), V.cuda()
    dec = P.HybridDecoder(n_layers=NL, batch=B, n_kv_heads=H, group_size=G, d_head=d, seq_cap=cap,
                          roles=roles, policy=P.SparsityPolicy.top_k(512), dtype=torch.bfloat16)
    eager = dec.decode_step(qd, Kd, Vd, lens).clone()
    sets = dec.token_sets()
    out = torch.zeros_like(qd)
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        dec.capture(qd, Kd, Vd, lens, out, stream=st)
        dec.replay(stream=st)
        dec.replay(stream=st)
    st.synchronize()
    assert torch.equal(out, eager)
    s2 = dec.token_sets()
    assert all(np.array_equal(a, b) for ra, rb in zip(sets, s2) for a, b in zip(ra, rb))
