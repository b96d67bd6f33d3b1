"""KV-sequence sharding on ONE GPU: P ranks emulated with
their row slices of the same cache and one shared gathered buffer (the packed
all-gather layout of lyc_shard_merge).  Every rank must produce bitwise the
same outputs and global index sets; those must match the unsharded decoder
and the oracle's decode_step (decode_engine.hpp:109-151, oracle/hh_oracle.c)
within the north_star tolerances, index sets exactly."""
import numpy as np
import pytest
import torch

from tests.test_gpu_decode import BF16_TOL, FP32_TOL, rel_err, roles_for, synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.set_device(0)


def _run(P_, *, NL, B, H, G, d, seq, k, dtype, roles, seed=0):
    import paper_2602_04541_b200 as P
    from paper_2602_04541_b200.sharded import ShardedDecoder, emulate_step
    q, K, V = synth(seed, NL, B, H, G, d, seq, seq, dtype)
    qd, Kd, Vd = q.cuda(), K.cuda(), V.cuda()
    pol = P.SparsityPolicy.top_k(k)
    full = P.HybridDecoder(n_layers=NL, batch=B, n_kv_heads=H, group_size=G, d_head=d,
                           seq_cap=seq, roles=roles, policy=pol, dtype=dtype)
    ref_out = full.decode_step(qd, Kd, Vd, seq)
    ref_sets = full.token_sets()
    decs, recv = [], None
    for r in range(P_):
        sd = ShardedDecoder(n_layers=NL, batch=B, n_kv_heads=H, group_size=G, d_head=d,
                            seq_cap=seq, roles=roles, policy=pol, dtype=dtype, world=P_, rank=r,
                            recv=recv, exchange=False)
        recv = sd.recv
        decs.append(sd)
    kcap = decs[0].k_cap
    gsets = [torch.full((NL, B * H, kcap), -7, dtype=torch.int32, device="cuda") for _ in range(P_)]
    outs = emulate_step(decs, qd, Kd, Vd, seq, global_sets=gsets)
    torch.cuda.synchronize()
    return q, K, V, full, ref_out, ref_sets, decs, outs, gsets


def _last_retrieval(roles, g):
    return max(l for l in range(roles.shape[0]) if l == 0 or roles[l, g] == 0)


def _vs_oracle(orc, q, K, V, roles, seq, k, d, out, gsets, tol):
    """The rank-0 output and global sets against the oracle, per batch item."""
    NL, B, H = K.shape[0], K.shape[1], K.shape[2]
    g0 = gsets[0].cpu().numpy()
    for b in range(B):
        ref = orc.decode_step(q[:, b].float().numpy(), K[:, b].float().numpy(),
                              V[:, b].float().numpy(), roles, seq=seq, scale=1 / np.sqrt(d),
                              kind="topk", k=k)
        err = rel_err(out[:, b].float().cpu().numpy(), ref["out"])
        assert err < tol, (b, err)
        for g in range(H):
            l = _last_retrieval(roles, g)
            np.testing.assert_array_equal(g0[l, b * H + g, :k], ref["sets"][g])


@pytest.mark.parametrize("P_", [2, 3, 4, 8])
def test_sequence_shards_fp32_match_unsharded(orc, P_):
    NL, B, H, G, d, seq, k = 4, 1, 2, 4, 64, 4096, 256
    roles = roles_for(NL, H, [(2, 1)])
    q, K, V, full, ref_out, ref_sets, decs, outs, gsets = _run(
        P_, NL=NL, B=B, H=H, G=G, d=d, seq=seq, k=k, dtype=torch.float32, roles=roles)
    for p in range(1, P_):
        assert torch.equal(outs[p], outs[0]), f"rank {p} output differs from rank 0"
        assert torch.equal(gsets[p], gsets[0]), f"rank {p} global sets differ"
    err = rel_err(outs[0].cpu().numpy(), ref_out.cpu().numpy())
    assert err < FP32_TOL, err
    g0 = gsets[0].cpu().numpy()
    for g in range(H):
        l = _last_retrieval(roles, g)
        np.testing.assert_array_equal(g0[l, g, :k], ref_sets[0][g])
    _vs_oracle(orc, q, K, V, roles, seq, k, d, outs[0], gsets, FP32_TOL)


@pytest.mark.parametrize("P_", [2, 8])
def test_sequence_shards_bf16_llama_like(orc, P_):
    NL, B, H, G, d, seq, k = 3, 2, 8, 4, 128, 16384, 1024
    roles = roles_for(NL, H, [(1, 3), (2, 5), (2, 0)])
    q, K, V, full, ref_out, ref_sets, decs, outs, gsets = _run(
        P_, NL=NL, B=B, H=H, G=G, d=d, seq=seq, k=k, dtype=torch.bfloat16, roles=roles, seed=3)
    for p in range(1, P_):
        assert torch.equal(outs[p], outs[0])
    err = rel_err(outs[0].float().cpu().numpy(), ref_out.float().cpu().numpy())
    assert err < BF16_TOL, err
    g0 = gsets[0].cpu().numpy()
    for b in range(B):
        for g in range(H):
            l = _last_retrieval(roles, g)
            np.testing.assert_array_equal(g0[l, b * H + g, :k], ref_sets[b][g])
    _vs_oracle(orc, q, K, V, roles, seq, k, d, outs[0], gsets, BF16_TOL)


def test_sequence_shard_local_sets_partition_the_global_set():
    """Each rank's filtered index cache is its slice of the global set, made local."""
    NL, B, H, G, d, seq, k, P_ = 2, 1, 2, 4, 64, 3000, 200, 3
    roles = roles_for(NL, H, [])
    from paper_2602_04541_b200.sharded import shard_rows
    q, K, V, full, ref_out, ref_sets, decs, outs, gsets = _run(
        P_, NL=NL, B=B, H=H, G=G, d=d, seq=seq, k=k, dtype=torch.float32, roles=roles)
    for g in range(H):
        glob = ref_sets[0][g]
        pieces = []
        for p, sd in enumerate(decs):
            rb, nl = shard_rows(seq, P_, p)
            ids, cnt = sd.dec.index_cache()
            loc = ids[g, : int(cnt[g])].cpu().numpy()
            assert (loc >= 0).all() and (loc < nl).all()
            pieces.append(loc + rb)
        np.testing.assert_array_equal(np.concatenate(pieces), glob)
