"""Device KV write path (kv_cache.hpp:14-69) through the C-ABI lyc_kv_write:
append + commit_row row by row, window overwrite, errors, and a decode step
over the appended cache equal (bitwise) to one over the same rows written by
torch."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2602_04541_b200  # noqa: F401
    torch.cuda.set_device(0)


@pytest.mark.parametrize("dtype,d", [(torch.bfloat16, 128), (torch.float32, 64)])
def test_append_commit_overwrite(dtype, d):
    import paper_2602_04541_b200 as P
    NL, B, H, cap, T = 3, 2, 4, 96, 80
    kv = P.KvCache(n_layers=NL, batch=B, n_kv_heads=H, d_head=d, seq_cap=cap, dtype=dtype)
    g = torch.Generator(device="cuda").manual_seed(1)
    K = torch.rand((T, NL, B, H, d), generator=g, device="cuda").to(dtype)
    V = torch.rand((T, NL, B, H, d), generator=g, device="cuda").to(dtype)
    for t in range(T):  # decode order: every layer appends, then the row commits
        for l in range(NL):
            kv.append(l, K[t, l], V[t, l])
        kv.commit_row()
    assert kv.length == T
    ref_k = torch.zeros_like(kv.k)
    ref_v = torch.zeros_like(kv.v)
    ref_k[:, :, :, :T] = K.permute(1, 2, 3, 0, 4)
    ref_v[:, :, :, :T] = V.permute(1, 2, 3, 0, 4)
    torch.cuda.synchronize()
    assert torch.equal(kv.k, ref_k) and torch.equal(kv.v, ref_v)
    # cache correction: rewrite the trailing W rows of layer 1 (kv_cache.hpp:34-42)
    W = 16
    wk = torch.rand((B, H, W, d), generator=g, device="cuda").to(dtype)
    wv = torch.rand((B, H, W, d), generator=g, device="cuda").to(dtype)
    kv.overwrite(1, T - W, wk, wv)
    ref_k[1, :, :, T - W:T] = wk
    ref_v[1, :, :, T - W:T] = wv
    # single-row overwrite
    kv.overwrite(2, 5, K[0, 0], V[0, 0])
    ref_k[2, :, :, 5] = K[0, 0]
    ref_v[2, :, :, 5] = V[0, 0]
    torch.cuda.synchronize()
    assert torch.equal(kv.k, ref_k) and torch.equal(kv.v, ref_v)
    with pytest.raises(P.InvalidArgument):
        kv.overwrite(0, T - 2, wk, wv)  # beyond the committed length


def test_write_errors():
    import paper_2602_04541_b200 as P
    from paper_2602_04541_b200 import _lib
    import ctypes as C
    kv = P.KvCache(n_layers=2, batch=1, n_kv_heads=2, d_head=64, seq_cap=8, dtype=torch.bfloat16)
    rows = torch.zeros((1, 2, 64), dtype=torch.bfloat16, device="cuda")
    lib = _lib.lib()
    with pytest.raises(P.InvalidArgument):  # layer out of range
        _lib.check(lib.lyc_kv_write(kv.k.data_ptr(), kv.v.data_ptr(), C.byref(kv._lay), 2, 0, 1,
                                    rows.data_ptr(), rows.data_ptr(), None))
    with pytest.raises(P.InvalidArgument):  # beyond seq_cap
        _lib.check(lib.lyc_kv_write(kv.k.data_ptr(), kv.v.data_ptr(), C.byref(kv._lay), 0, 8, 1,
                                    rows.data_ptr(), rows.data_ptr(), None))
    for _ in range(8):
        for l in range(2):
            kv.append(l, rows, rows)
        kv.commit_row()
    with pytest.raises(P.InvalidArgument):  # full
        kv.append(0, rows, rows)


def test_decode_over_appended_cache_matches_prefilled():
    """The decoder reads the cache the write path built: same outputs and
    sets as over a cache filled by torch (bitwise)."""
    import paper_2602_04541_b200 as P
    NL, B, H, G, d, seq = 2, 1, 8, 4, 128, 4096
    roles = np.ones((NL, H), dtype=np.uint8)
    roles[0] = 0
    roles[1, 2] = 0
    g = torch.Generator(device="cuda").manual_seed(7)
    K = (torch.rand((NL, B, H, seq, d), generator=g, device="cuda") * 2 - 1).to(torch.bfloat16)
    V = (torch.rand((NL, B, H, seq, d), generator=g, device="cuda") * 2 - 1).to(torch.bfloat16)
    q = (torch.rand((NL, B, H * G, d), generator=g, device="cuda") * 2 - 1).to(torch.bfloat16)
    kv = P.KvCache(n_layers=NL, batch=B, n_kv_heads=H, d_head=d, seq_cap=seq, dtype=torch.bfloat16)
    # a prompt cache adopted in one window write per layer, then 3 decoded rows
    for l in range(NL):
        kv._write(l, 0, K[l, :, :, : seq - 3], V[l, :, :, : seq - 3])
    kv.length = seq - 3
    for t in range(seq - 3, seq):
        for l in range(NL):
            kv.append(l, K[l, :, :, t], V[l, :, :, t])
        kv.commit_row()
    dec = P.HybridDecoder(n_layers=NL, batch=B, n_kv_heads=H, group_size=G, d_head=d,
                          seq_cap=seq, roles=roles, policy=P.SparsityPolicy.top_k(256),
                          dtype=torch.bfloat16)
    out_a = dec.decode_step(q, kv.k, kv.v, seq)
    sets_a = dec.token_sets()
    out_b = dec.decode_step(q, K, V, seq)
    sets_b = dec.token_sets()
    torch.cuda.synchronize()
    assert torch.equal(out_a, out_b)
    assert all(np.array_equal(a, b) for a, b in zip(sets_a[0], sets_b[0]))


@pytest.mark.parametrize("d,G,W,start,dtype", [(128, 4, 32, 3000, torch.bfloat16),
                                                (64, 8, 16, 1000, torch.bfloat16),
                                                (128, 4, 5, 70, torch.bfloat16),
                                                (128, 4, 64, 3977, torch.bfloat16),
                                                (64, 8, 32, 1, torch.bfloat16),
                                                (128, 1, 3, 4000, torch.bfloat16),
                                                (64, 4, 8, 500, torch.float32)])
def test_correction_attention_vs_oracle(orc, d, G, W, start, dtype):
    """decode_engine.hpp:164-204 attention part: after the window's rows are
    rewritten, window position i attends keys [0, start + i] (dense,
    attention.hpp:50-75) -- checked per (b, position, q head) against the
    oracle's f64 dense_attention; bf16 tolerance 2e-2."""
    import paper_2602_04541_b200 as P
    NL, B, H, cap = 2, 2, 2, 4096
    Hq = H * G
    g = torch.Generator(device="cuda").manual_seed(11)
    kv = P.KvCache(n_layers=NL, batch=B, n_kv_heads=H, d_head=d, seq_cap=cap, dtype=dtype)
    kv.k.uniform_(-1, 1, generator=g)
    kv.v.uniform_(-1, 1, generator=g)
    kv.length = start + W
    wk = (torch.rand((B, H, W, d), generator=g, device="cuda") * 2 - 1).to(dtype)
    wv = (torch.rand((B, H, W, d), generator=g, device="cuda") * 2 - 1).to(dtype)
    kv.overwrite(1, start, wk, wv)  # the rewritten window rows (kv_cache.hpp:34-42)
    q = (torch.rand((B, W, Hq, d), generator=g, device="cuda") * 2 - 1).to(dtype)
    out = P.correction_attention(kv.k, kv.v, 1, q, start)
    torch.cuda.synchronize()
    Kn = kv.k[1].float().cpu().numpy()
    Vn = kv.v[1].float().cpu().numpy()
    qn = q.float().cpu().numpy()
    on = out.float().cpu().numpy()
    scale = 1 / np.sqrt(d)
    worst = 0.0
    for b in range(B):
        for i in range(W):
            p = start + i
            for hd in range(Hq):
                ref, _ = orc.dense_attention(qn[b, i, hd], Kn[b, hd // G, : p + 1],
                                             Vn[b, hd // G, : p + 1], scale)
                worst = max(worst, np.abs(on[b, i, hd] - ref).max() / max(np.abs(ref).max(), 1e-3))
    assert worst < (2e-2 if dtype == torch.bfloat16 else 1e-5), worst


@pytest.mark.parametrize("dtype,d,G,H,B,L,policy,select", [
    (torch.float32, 64, 4, 2, 1, 4096, ("topk", 256), "tokens"),
    (torch.bfloat16, 128, 4, 8, 2, 5000, ("topk", 512), "tokens"),
    (torch.bfloat16, 128, 4, 4, 1, 3000, ("ratio", 0.9), "tokens"),
    (torch.float32, 64, 4, 2, 1, 2000, ("topp", 0.5), "tokens"),
    (torch.float32, 64, 4, 2, 1, 2000, ("threshold", 0.001), "tokens"),
    (torch.bfloat16, 128, 4, 4, 2, 6000, ("topk", 1024), "blocks"),
])
def test_refresh_sets_vs_oracle(orc, dtype, d, G, H, B, L, policy, select):
    """decode_engine.hpp:190-197: after correction, each KV head's set is
    select_tokens(policy, dense_attention(pooled q of the last window
    position, K[:len]).weights) -- the device refresh against the oracle
    (sets exact except documented fp ties; block mode: the composed
    block-max top-k of the oracle)."""
    import paper_2602_04541_b200 as P
    from tests.test_gpu_decode import check_policy_set, check_set
    NL, cap, layer = 2, L + 64, 1
    kind, val = policy
    pol = {"topk": lambda: P.SparsityPolicy.top_k(val), "ratio": lambda: P.SparsityPolicy.ratio(val),
           "topp": lambda: P.SparsityPolicy.top_p(val),
           "threshold": lambda: P.SparsityPolicy.threshold(val)}[kind]()
    roles = np.ones((NL, H), np.uint8)
    roles[0] = 0
    dec = P.HybridDecoder(n_layers=NL, batch=B, n_kv_heads=H, group_size=G, d_head=d, seq_cap=cap,
                          roles=roles, policy=pol, dtype=dtype, select=select)
    g = torch.Generator(device="cuda").manual_seed(21)
    K = (torch.rand((NL, B, H, cap, d), generator=g, device="cuda") * 2 - 1).to(dtype)
    q = (torch.rand((B, H * G, d), generator=g, device="cuda") * 2 - 1).to(dtype)
    dec.refresh_sets(layer, q, K, L)
    torch.cuda.synchronize()
    sets = dec.token_sets()
    Kn, qn = K[layer].float().cpu().numpy(), q.float().cpu().numpy()
    scale = 1 / np.sqrt(d)
    for b in range(B):
        pooled = orc.gqa_pool_queries(qn[b], G)
        for hg in range(H):
            if select == "blocks":
                nblk = min((val + 63) // 64, (L + 63) // 64)
                ref = orc.block_select(pooled[hg], Kn[b, hg], L, scale, 64, nblk)
                np.testing.assert_array_equal(sets[b][hg], ref)
                continue
            _, w = orc.dense_attention(pooled[hg], Kn[b, hg, :L], Kn[b, hg, :L], scale)
            k = val if kind == "topk" else 1
            ref = orc.select_tokens(kind, w, k=k, value=0.0 if kind == "topk" else val)
            scores = Kn[b, hg, :L].astype(np.float64) @ pooled[hg]
            if kind in ("topk", "ratio"):
                check_set(sets[b][hg], ref, scores, len(ref))
            else:
                check_policy_set(sets[b][hg], ref, w, kind, val)
