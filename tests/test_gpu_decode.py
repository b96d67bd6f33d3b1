"""GPU parity of the hybrid-head decode step (decode_engine.hpp:109-151)
against the oracle restatement of the same loop on identical inputs.

Index sets: the GPU ranks fp32 pooled scores (sum_j q_j.k over the packed GQA
rows, fused in the attention kernel); the oracle ranks f64 softmax weights of
the pooled query (decode_engine.hpp:129-132).  Softmax is monotone, so the
sets agree exactly except where fp rounding reorders scores that are equal to
within DELTA of the k-th score (the documented tie band); swaps are counted
and must lie inside that band.
"""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

FP32_TOL = 1e-5
BF16_TOL = 2e-2


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2602_04541_b200  # noqa: F401
    torch.cuda.set_device(0)


def rel_err(got, ref):
    got = np.asarray(got, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    return np.abs(got - ref).max() / max(np.abs(ref).max(), 1e-3)


def synth(seed, NL, B, H, G, d, seq, seq_cap, dtype):
    g = torch.Generator().manual_seed(seed)
    q = (torch.rand((NL, B, H * G, d), generator=g) * 2 - 1).to(dtype)
    K = (torch.rand((NL, B, H, seq_cap, d), generator=g) * 2 - 1).to(dtype)
    V = (torch.rand((NL, B, H, seq_cap, d), generator=g) * 2 - 1).to(dtype)
    return q, K, V


def roles_for(NL, H, retrieval_above_0, seed=0):
    r = np.ones((NL, H), dtype=np.uint8)
    r[0] = 0
    for (l, g) in retrieval_above_0:
        r[l, g] = 0
    return r


def pooled_scores(q_l, K_lg, group, g, seq):
    """f64 pooled-query scores (without scale) of head g at one layer."""
    qq = q_l[g * group:(g + 1) * group].astype(np.float64)
    pooled = qq.sum(0) / group
    return K_lg[:seq].astype(np.float64) @ pooled


def check_set(got, ref, scores, k, rel_band=2e-6):
    """Exact, or swaps confined to |s - s_(k)| <= band."""
    got, ref = set(got.tolist()), set(ref.tolist())
    assert len(got) == len(ref)
    if got == ref:
        return 0
    kth = np.sort(scores)[::-1][min(k, len(scores)) - 1]
    band = rel_band * np.abs(scores).max() * 4
    for t in got ^ ref:
        assert abs(scores[t] - kth) <= band, (t, scores[t], kth)
    return len(got - ref)


def run_case(orc, *, NL, B, H, G, d, seq, seq_cap, dtype, roles, policy, select="tokens",
             seed=0, layerwise=False):
    import paper_2602_04541_b200 as P
    q, K, V = synth(seed, NL, B, H, G, d, seq, seq_cap, dtype)
    dec = P.HybridDecoder(n_layers=NL, batch=B, n_kv_heads=H, group_size=G, d_head=d,
                          seq_cap=seq_cap, roles=roles, policy=policy, dtype=dtype, select=select)
    qd, Kd, Vd = q.cuda(), K.cuda(), V.cuda()
    traces = []
    if layerwise:
        out = torch.empty_like(qd)
        for l in range(NL):
            dec.layer(l, qd[l], Kd, Vd, seq, out[l])
            traces.append(dec.token_sets())
    else:
        out = dec.decode_step(qd, Kd, Vd, seq)
    torch.cuda.synchronize()
    return dec, q.float().numpy(), K.float().numpy(), V.float().numpy(), out.float().cpu().numpy(), traces


@pytest.mark.parametrize("seed", [0, 1])
def test_tiny_config_fp32_token_mode(orc, seed):
    """BASELINE configs[0]: 4 layers, 8 q / 2 KV heads, d 64, 4K context,
    top-k 256, fp32, batch 1 -- outputs, final sets and per-layer traces."""
    import paper_2602_04541_b200 as P
    NL, B, H, G, d, seq = 4, 1, 2, 4, 64, 4096
    roles = roles_for(NL, H, [(2, 1)])
    dec, q, K, V, out, traces = run_case(orc, NL=NL, B=B, H=H, G=G, d=d, seq=seq, seq_cap=seq,
                                         dtype=torch.float32, roles=roles,
                                         policy=P.SparsityPolicy.top_k(256), seed=seed,
                                         layerwise=True)
    r = orc.decode_step(q[:, 0], K[:, 0], V[:, 0], roles, seq=seq, scale=1 / np.sqrt(d),
                        kind="topk", k=256, trace=True)
    assert rel_err(out[:, 0], r["out"]) < FP32_TOL
    swaps = 0
    for l in range(NL):
        for g in range(H):
            src = max(ll for ll in range(l + 1) if roles[ll, g] == 0 or ll == 0)
            sc = pooled_scores(q[src, 0], K[src, 0, g], G, g, seq)
            swaps += check_set(traces[l][0][g], r["trace"][l][g], sc, 256)
    assert swaps == 0


def test_llama_like_bf16_token_mode(orc):
    """Llama-3-8B head shapes (32 q / 8 KV, d 128), bf16, shortened context."""
    import paper_2602_04541_b200 as P
    NL, B, H, G, d, seq = 3, 1, 8, 4, 128, 8192
    roles = roles_for(NL, H, [(1, 3), (2, 5)])
    dec, q, K, V, out, traces = run_case(orc, NL=NL, B=B, H=H, G=G, d=d, seq=seq, seq_cap=seq + 64,
                                         dtype=torch.bfloat16, roles=roles,
                                         policy=P.SparsityPolicy.top_k(512), seed=3,
                                         layerwise=True)
    Kc, Vc = K[:, 0], V[:, 0]
    r = orc.decode_step(q[:, 0], Kc, Vc, roles, seq=seq, scale=1 / np.sqrt(d), kind="topk", k=512,
                        trace=True)
    assert rel_err(out[:, 0], r["out"]) < BF16_TOL
    swaps = 0
    for l in range(NL):
        for g in range(H):
            src = max(ll for ll in range(l + 1) if roles[ll, g] == 0)
            sc = pooled_scores(q[src, 0], K[src, 0, g], G, g, seq)
            swaps += check_set(traces[l][0][g], r["trace"][l][g], sc, 512)
    print("tie-band swaps:", swaps)
    assert swaps == 0


def test_batch_and_ratio_policy(orc):
    """Batch > 1 (independent sequences) and the Ratio policy (policy.hpp:71-72)."""
    import paper_2602_04541_b200 as P
    NL, B, H, G, d, seq = 3, 3, 2, 2, 64, 1000
    roles = roles_for(NL, H, [(1, 0)])
    dec, q, K, V, out, _ = run_case(orc, NL=NL, B=B, H=H, G=G, d=d, seq=seq, seq_cap=1024,
                                    dtype=torch.float32, roles=roles,
                                    policy=P.SparsityPolicy.ratio(0.8), seed=5)
    sets = dec.token_sets()
    for b in range(B):
        r = orc.decode_step(q[:, b], K[:, b], V[:, b], roles, seq=seq, scale=1 / np.sqrt(d),
                            kind="ratio", value=0.8)
        assert rel_err(out[:, b], r["out"]) < FP32_TOL
        for g in range(H):
            assert len(sets[b][g]) == orc.fraction_budget(0.2, seq)
            assert np.array_equal(sets[b][g], r["sets"][g])


def test_full_budget_sparse_equals_dense(orc):
    """decode_engine_test.cpp:184-222: a budget >= seq makes sparse heads dense."""
    import paper_2602_04541_b200 as P
    NL, B, H, G, d, seq = 3, 1, 2, 4, 64, 700
    sparse = roles_for(NL, H, [])
    dense = np.zeros((NL, H), dtype=np.uint8)
    _, q, K, V, out_s, _ = run_case(orc, NL=NL, B=B, H=H, G=G, d=d, seq=seq, seq_cap=768,
                                    dtype=torch.float32, roles=sparse,
                                    policy=P.SparsityPolicy.top_k(100000), seed=9)
    _, _, _, _, out_d, _ = run_case(orc, NL=NL, B=B, H=H, G=G, d=d, seq=seq, seq_cap=768,
                                    dtype=torch.float32, roles=dense,
                                    policy=P.SparsityPolicy.top_k(4), seed=9)
    assert rel_err(out_s, out_d) < FP32_TOL


def test_block_mode_matches_composed_oracle(orc):
    """Block-sparse selection (the paper's kernel): block score = max pooled
    score over the block's rows; top ceil(k/64) blocks; kernel::run on them."""
    import paper_2602_04541_b200 as P
    NL, B, H, G, d, seq, k = 2, 1, 4, 4, 128, 4000, 640
    roles = roles_for(NL, H, [])
    dec, q, K, V, out, traces = run_case(orc, NL=NL, B=B, H=H, G=G, d=d, seq=seq, seq_cap=4096,
                                         dtype=torch.bfloat16, roles=roles,
                                         policy=P.SparsityPolicy.top_k(k), select="blocks",
                                         seed=11, layerwise=True)
    nblk = (k + 63) // 64
    # layer 0: dense retrieval for every head
    r0 = orc.kernel_run(K[0, 0, :, :seq], V[0, 0, :, :seq], q[0, 0], [list(range((seq + 63) // 64))] * H, batch=1,
                        group=G, seq_len=seq, scale=1 / np.sqrt(d), dtype=np.float64,
                        num_splits=4)
    assert rel_err(out[0, 0], r0) < BF16_TOL
    blocks = []
    for g in range(H):
        pq = q[0, 0, g * G:(g + 1) * G].astype(np.float64).mean(0)
        ref_blocks = orc.block_select(pq, K[0, 0, g], seq, 1 / np.sqrt(d), 64, nblk)
        got = traces[0][0][g]
        if not np.array_equal(got, ref_blocks):
            sc = orc.pooled_scores(pq, K[0, 0, g], seq, 1.0)
            bm = np.array([sc[i * 64:(i + 1) * 64].max() for i in range((seq + 63) // 64)])
            check_set(got, ref_blocks, bm, nblk)
        blocks.append(got.tolist())
    r1 = orc.kernel_run(K[1, 0, :, :seq], V[1, 0, :, :seq], q[1, 0], blocks, batch=1, group=G, seq_len=seq,
                        scale=1 / np.sqrt(d), dtype=np.float64, num_splits=3)
    assert rel_err(out[1, 0], r1) < BF16_TOL


def test_graph_replay_matches_eager_and_is_deterministic(orc):
    import paper_2602_04541_b200 as P
    NL, B, H, G, d, seq = 4, 1, 8, 4, 128, 5000
    roles = roles_for(NL, H, [(1, 2), (3, 7)])
    q, K, V = synth(21, NL, B, H, G, d, seq, 5120, torch.bfloat16)
    q, K, V = q.cuda(), K.cuda(), V.cuda()
    dec = P.HybridDecoder(n_layers=NL, batch=B, n_kv_heads=H, group_size=G, d_head=d, seq_cap=5120,
                          roles=roles, policy=P.SparsityPolicy.top_k(300))
    eager = dec.decode_step(q, K, V, seq)
    sets_eager = dec.token_sets()
    out = torch.empty_like(q)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        dec.capture(q, K, V, seq, out, stream=s)
        for _ in range(3):
            dec.replay(stream=s)
    s.synchronize()
    assert torch.equal(out, eager)
    sets = dec.token_sets()
    assert all(np.array_equal(a, b) for ra, rb in zip(sets, sets_eager) for a, b in zip(ra, rb))


def test_decoder_errors():
    import paper_2602_04541_b200 as P
    bad = np.ones((2, 2), dtype=np.uint8)  # layer 0 must be retrieval (rolemap.hpp:54-56)
    with pytest.raises(P.InvalidArgument):
        P.HybridDecoder(n_layers=2, batch=1, n_kv_heads=2, group_size=2, d_head=64, seq_cap=128,
                        roles=bad, policy=P.SparsityPolicy.top_k(4))
    with pytest.raises(P.InvalidArgument):
        P.SparsityPolicy.top_k(0)
    with pytest.raises(P.NotSupported):  # TopP selects tokens only
        P.HybridDecoder(n_layers=2, batch=1, n_kv_heads=2, group_size=2, d_head=64, seq_cap=128,
                        roles=np.zeros((2, 2)), policy=P.SparsityPolicy.top_p(0.9), select="blocks")
    dec = P.HybridDecoder(n_layers=2, batch=1, n_kv_heads=2, group_size=2, d_head=64, seq_cap=128,
                          roles=np.zeros((2, 2)), policy=P.SparsityPolicy.top_k(4))
    q = torch.zeros((2, 1, 4, 64), dtype=torch.bfloat16, device="cuda")
    kv = torch.zeros((2, 1, 2, 128, 64), dtype=torch.bfloat16, device="cuda")
    with pytest.raises(P.InvalidArgument):
        dec.decode_step(q, kv, kv, 129)  # beyond seq_cap
    with pytest.raises(P.LogicError):
        dec.replay()


@pytest.mark.parametrize("select", ["tokens", "blocks"])
def test_fused_step_matches_per_layer_kernels(orc, select):
    """The persistent whole-step kernel (one launch: attention, merge and the
    grid-wide radix selection of every layer) against the per-layer kernels
    (attention + merge + cluster top-k launches) on the same inputs: identical
    index sets, outputs equal up to merge-order rounding."""
    import paper_2602_04541_b200 as P
    NL, B, H, G, d, seq = 5, 2, 8, 4, 128, 6000
    roles = roles_for(NL, H, [(1, 3), (2, 5), (3, 0), (4, 3)])
    q, K, V = synth(17, NL, B, H, G, d, seq, 6016, torch.bfloat16)
    q, K, V = q.cuda(), K.cuda(), V.cuda()
    mk = lambda: P.HybridDecoder(n_layers=NL, batch=B, n_kv_heads=H, group_size=G, d_head=d,
                                 seq_cap=6016, roles=roles, policy=P.SparsityPolicy.top_k(700),
                                 select=select)
    fused = mk()
    assert fused.fused
    out_f = fused.decode_step(q, K, V, seq)
    per = mk()
    per.tune(P._lib.TUNE_PER_LAYER_KERNELS, 1)  # attention + merge + cluster top-k launches
    assert not per.fused
    out_p = torch.empty_like(q)
    for l in range(NL):
        per.layer(l, q[l], K, V, seq, out_p[l])
    torch.cuda.synchronize()
    sf, sp = fused.token_sets(), per.token_sets()
    assert all(np.array_equal(a, b) for ra, rb in zip(sf, sp) for a, b in zip(ra, rb))
    assert rel_err(out_f.float().cpu().numpy(), out_p.float().cpu().numpy()) < 1e-2


def test_fused_step_llama_like_vs_oracle(orc):
    """decode_step through the fused kernel vs the oracle decode loop."""
    import paper_2602_04541_b200 as P
    NL, B, H, G, d, seq = 4, 1, 8, 4, 128, 9000
    roles = roles_for(NL, H, [(1, 1), (2, 6), (3, 1)])
    dec, q, K, V, out, _ = run_case(orc, NL=NL, B=B, H=H, G=G, d=d, seq=seq, seq_cap=9024,
                                    dtype=torch.bfloat16, roles=roles,
                                    policy=P.SparsityPolicy.top_k(1000), seed=23)
    assert dec.fused
    r = orc.decode_step(q[:, 0], K[:, 0], V[:, 0], roles, seq=seq, scale=1 / np.sqrt(d), kind="topk",
                        k=1000)
    assert rel_err(out[:, 0], r["out"]) < BF16_TOL
    sets = dec.token_sets()[0]
    for g in range(H):
        src = max(l for l in range(NL) if roles[l, g] == 0)
        sc = pooled_scores(q[src, 0], K[src, 0, g], G, g, seq)
        check_set(sets[g], r["sets"][g], sc, 1000)


def test_fused_step_repeated_and_replanned(orc):
    """Step counters are monotonic across launches and reset on re-plan: the
    same step twice is bitwise identical; a different seq_len re-plans."""
    import paper_2602_04541_b200 as P
    NL, B, H, G, d = 3, 1, 4, 4, 64
    roles = roles_for(NL, H, [(2, 1)])
    q, K, V = synth(29, NL, B, H, G, d, 3000, 3072, torch.bfloat16)
    q, K, V = q.cuda(), K.cuda(), V.cuda()
    dec = P.HybridDecoder(n_layers=NL, batch=B, n_kv_heads=H, group_size=G, d_head=d, seq_cap=3072,
                          roles=roles, policy=P.SparsityPolicy.top_k(200))
    a = dec.decode_step(q, K, V, 3000).clone()
    sa = dec.token_sets()
    for _ in range(3):
        b = dec.decode_step(q, K, V, 3000)
    torch.cuda.synchronize()
    assert torch.equal(a, b)
    assert all(np.array_equal(x, y) for rx, ry in zip(sa, dec.token_sets()) for x, y in zip(rx, ry))
    c = dec.decode_step(q, K, V, 2999)
    r = orc.decode_step(q[:, 0].float().cpu().numpy(), K[:, 0].float().cpu().numpy(),
                        V[:, 0].float().cpu().numpy(), roles, seq=2999, scale=1 / np.sqrt(d),
                        kind="topk", k=200)
    assert rel_err(c[:, 0].float().cpu().numpy(), r["out"]) < BF16_TOL


@pytest.mark.parametrize("n_ties", [2000, 6000])
def test_fused_step_exact_ties_lowest_index(orc, n_ties):
    """Exact score ties at the top-k boundary (attention.hpp:117-118: ties go
    to the lower index).  Rows are built so the pooled scores take three values:
    800 rows at 2|qbar|^2, n_ties identical rows at |qbar|^2 straddling the
    boundary, the rest 0 -- the fused selection's tie path (and, with 6000 ties,
    its off-chip candidate path) must take exactly the lowest-index ties."""
    import paper_2602_04541_b200 as P
    NL, B, H, G, d, seq, k = 2, 1, 2, 4, 64, 20000, 1000
    roles = roles_for(NL, H, [])
    q, K, V = synth(11, NL, B, H, G, d, seq, seq, torch.float32)
    rng = np.random.default_rng(5)
    for l in range(NL):
        for g in range(H):
            qbar = q[l, 0, g * G:(g + 1) * G].double().mean(0)
            rows = rng.permutation(seq)
            Kl = torch.zeros(seq, d, dtype=torch.float64)
            Kl[rows[:800]] = 2 * qbar
            Kl[rows[800:800 + n_ties]] = qbar
            K[l, 0, g] = Kl.float()
    dec = P.HybridDecoder(n_layers=NL, batch=B, n_kv_heads=H, group_size=G, d_head=d, seq_cap=seq,
                          roles=roles, policy=P.SparsityPolicy.top_k(k), dtype=torch.float32)
    assert dec.fused
    out = dec.decode_step(q.cuda(), K.cuda(), V.cuda(), seq)
    torch.cuda.synchronize()
    sets = dec.token_sets()[0]
    r = orc.decode_step(q[:, 0].numpy(), K[:, 0].numpy(), V[:, 0].numpy(), roles, seq=seq,
                        scale=1 / np.sqrt(d), kind="topk", k=k)
    for g in range(H):
        np.testing.assert_array_equal(sets[g], r["sets"][g])
    assert rel_err(out[:, 0].cpu().numpy(), r["out"]) < FP32_TOL


def test_fused_step_batch4_many_items_per_cta(orc):
    """Batch 4 x 8 KV heads, 40K context: layer 0 has 32 selection rows x 5
    items = 160 items for 148 CTAs (several items per CTA, no role split);
    later layers use the split roles.  Every batch item against the oracle."""
    import paper_2602_04541_b200 as P
    NL, B, H, G, d, seq, k = 3, 4, 8, 4, 128, 40000, 2048
    roles = roles_for(NL, H, [(1, 2), (2, 5), (2, 7)])
    dec, q, K, V, out, _ = run_case(orc, NL=NL, B=B, H=H, G=G, d=d, seq=seq, seq_cap=seq,
                                    dtype=torch.bfloat16, roles=roles,
                                    policy=P.SparsityPolicy.top_k(k), seed=31)
    assert dec.fused
    sets = dec.token_sets()
    for b in range(B):
        r = orc.decode_step(q[:, b], K[:, b], V[:, b], roles, seq=seq, scale=1 / np.sqrt(d),
                            kind="topk", k=k)
        assert rel_err(out[:, b], r["out"]) < BF16_TOL
        for g in range(H):
            src = max(l for l in range(NL) if roles[l, g] == 0)
            sc = pooled_scores(q[src, b], K[src, b, g], G, g, seq)
            check_set(sets[b][g], r["sets"][g], sc, k)


def _policy_weights(q_l, K_lg, group, g, seq, scale):
    s = pooled_scores(q_l, K_lg, group, g, seq) * scale
    w = np.exp(s - s.max())
    return w / w.sum()


def check_policy_set(got, ref, w, kind, value, rel_band=1e-6):
    """TopP / Threshold sets: exact, or differences confined to weights within
    rel_band of the cut (tau, or the weight where the cumulative mass crosses p)."""
    got, ref = set(got.tolist()), set(ref.tolist())
    if got == ref:
        return 0
    if kind == "threshold":
        cut = value
    else:
        order = sorted(range(len(w)), key=lambda t: (-w[t], t))
        cut = w[order[len(ref) - 1]]
        assert abs(len(got) - len(ref)) <= 1
    for t in got ^ ref:
        assert abs(w[t] - cut) <= rel_band * cut, (kind, t, w[t], cut)
    return len(got ^ ref)


@pytest.mark.parametrize("kind,value", [("topp", 0.5), ("topp", 0.9), ("topp", 1.0),
                                        ("threshold", 1.3 / 4096), ("threshold", 0.5)])
def test_topp_threshold_policies_vs_oracle(orc, kind, value):
    """policy.hpp:73-101 on the device (csrc/policy.cu): TopP (cumulative mass,
    stable descending order) and Threshold (w > tau, argmax fallback) from the
    pooled-query weights; sparse heads consume the variable-size sets through
    their device counts.  Tiny fp32 config, per-layer sets vs the oracle."""
    import paper_2602_04541_b200 as P
    NL, B, H, G, d, seq = 4, 1, 2, 4, 64, 4096
    roles = roles_for(NL, H, [(2, 1)])
    policy = P.SparsityPolicy.top_p(value) if kind == "topp" else P.SparsityPolicy.threshold(value)
    dec, q, K, V, out, traces = run_case(orc, NL=NL, B=B, H=H, G=G, d=d, seq=seq, seq_cap=seq,
                                         dtype=torch.float32, roles=roles, policy=policy, seed=5,
                                         layerwise=True)
    scale = 1 / np.sqrt(d)
    r = orc.decode_step(q[:, 0], K[:, 0], V[:, 0], roles, seq=seq, scale=scale, kind=kind,
                        value=value, trace=True)
    diffs = 0
    for l in range(NL):
        for g in range(H):
            src = max(ll for ll in range(l + 1) if roles[ll, g] == 0 or ll == 0)
            w = _policy_weights(q[src, 0], K[src, 0, g], G, g, seq, scale)
            diffs += check_policy_set(traces[l][0][g], r["trace"][l][g], w, kind, value)
    if diffs == 0:
        assert rel_err(out[:, 0], r["out"]) < FP32_TOL
    if kind == "threshold" and value == 0.5:  # nothing clears the bar: the argmax alone
        assert all(len(traces[l][0][g]) == 1 for l in range(NL) for g in range(H))


def test_topp_bf16_llama_heads_graph_replay(orc):
    """TopP at Llama head shapes in bf16, through the eager step and a CUDA-graph
    replay (variable-size sets are device counts, so the graph is reusable)."""
    import paper_2602_04541_b200 as P
    NL, B, H, G, d, seq = 3, 1, 8, 4, 128, 8192
    roles = roles_for(NL, H, [(1, 3), (2, 5)])
    q, K, V = synth(7, NL, B, H, G, d, seq, seq, torch.bfloat16)
    dec = P.HybridDecoder(n_layers=NL, batch=B, n_kv_heads=H, group_size=G, d_head=d, seq_cap=seq,
                          roles=roles, policy=P.SparsityPolicy.top_p(0.3), dtype=torch.bfloat16)
    qd, Kd, Vd = q.cuda(), K.cuda(), V.cuda()
    out = dec.decode_step(qd, Kd, Vd, seq)
    sets = dec.token_sets()
    torch.cuda.synchronize()
    scale = 1 / np.sqrt(d)
    qf, Kf, Vf = q.float().numpy(), K.float().numpy(), V.float().numpy()
    r = orc.decode_step(qf[:, 0], Kf[:, 0], Vf[:, 0], roles, seq=seq, scale=scale, kind="topp",
                        value=0.3, trace=True)
    assert rel_err(out.float().cpu().numpy()[:, 0], r["out"]) < BF16_TOL
    for g in range(H):
        src = max(ll for ll in range(NL) if roles[ll, g] == 0)
        w = _policy_weights(qf[src, 0], Kf[src, 0, g], G, g, seq, scale)
        check_policy_set(sets[0][g], r["sets"][g], w, "topp", 0.3)
    out2 = torch.empty_like(out)
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        dec.capture(qd, Kd, Vd, seq, out2, stream=st)
        dec.replay(stream=st)
    st.synchronize()
    assert torch.equal(out2, out)
    assert all(np.array_equal(a, b) for a, b in zip(dec.token_sets()[0], sets[0]))


@pytest.mark.parametrize("num_splits", [1, 2])
def test_fused_step_single_unit_slots(orc, num_splits):
    """One or two splits per batch item (the default at batch >= 75): slots of
    a single unit write the output directly from the unit epilogue, with no
    merge -- against the oracle, every batch item."""
    import paper_2602_04541_b200 as P
    NL, B, H, G, d, seq, k = 2, 3, 2, 4, 128, 6000, 300
    roles = roles_for(NL, H, [(1, 1)])
    q, K, V = synth(41, NL, B, H, G, d, seq, seq, torch.bfloat16)
    dec = P.HybridDecoder(n_layers=NL, batch=B, n_kv_heads=H, group_size=G, d_head=d, seq_cap=seq,
                          roles=roles, policy=P.SparsityPolicy.top_k(k), dtype=torch.bfloat16,
                          num_splits=num_splits)
    out = dec.decode_step(q.cuda(), K.cuda(), V.cuda(), seq)
    torch.cuda.synchronize()
    assert dec.fused
    qf, Kf, Vf, of = q.float().numpy(), K.float().numpy(), V.float().numpy(), out.float().cpu().numpy()
    for b in range(B):
        r = orc.decode_step(qf[:, b], Kf[:, b], Vf[:, b], roles, seq=seq, scale=1 / np.sqrt(d),
                            kind="topk", k=k)
        assert rel_err(of[:, b], r["out"]) < BF16_TOL
