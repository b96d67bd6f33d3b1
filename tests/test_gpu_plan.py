"""The device-planned step kernel: per-layer launches, token-after-token
decode without host synchronisation, device-resident lengths and graph
replay (include/lyc.h lyc_decoder_layer / lyc_decoder_step_dev /
lyc_decoder_capture_dev / lyc_kv_append_dev; decode_engine.hpp:97-151)."""
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


def _roles(NL, H, extra):
    r = np.ones((NL, H), np.uint8)
    r[0] = 0
    for (l, g) in extra:
        r[l, g] = 0
    return r


def _inputs(seed, NL, B, H, G, d, cap, dtype=torch.bfloat16):
    g = torch.Generator(device="cuda").manual_seed(seed)
    K = torch.empty((NL, B, H, cap, d), dtype=dtype, device="cuda").uniform_(-1, 1, generator=g)
    V = torch.empty_like(K).uniform_(-1, 1, generator=g)
    q = torch.empty((NL, B, H * G, d), dtype=dtype, device="cuda").uniform_(-1, 1, generator=g)
    return q, K, V


def _dec(NL, B, H, G, d, cap, roles, k, dtype=torch.bfloat16, policy=None, select="tokens"):
    import paper_2602_04541_b200 as P
    return P.HybridDecoder(n_layers=NL, batch=B, n_kv_heads=H, group_size=G, d_head=d,
                           seq_cap=cap, roles=roles, policy=policy or P.SparsityPolicy.top_k(k),
                           dtype=dtype, select=select)


def _sets_equal(a, b):
    return all(np.array_equal(x, y) for ra, rb in zip(a, b) for x, y in zip(ra, rb))


@pytest.mark.parametrize("B,select", [(1, "tokens"), (3, "tokens"), (2, "blocks")])
def test_layer_launches_equal_whole_step(B, select):
    """lyc_decoder_layer on the step kernel (one launch per layer) computes
    exactly what the whole-step launch computes: same plan, same units, same
    merge order -> bitwise equal outputs and index sets."""
    NL, H, G, d, cap, seq = 5, 8, 4, 128, 9000, 8700
    roles = _roles(NL, H, [(1, 3), (2, 5), (3, 0), (3, 4), (4, 3)])
    q, K, V = _inputs(5, NL, B, H, G, d, cap)
    a = _dec(NL, B, H, G, d, cap, roles, 900, select=select)
    b = _dec(NL, B, H, G, d, cap, roles, 900, select=select)
    assert a.fused and b.fused
    out_a = a.decode_step(q, K, V, seq)
    out_b = torch.empty_like(q)
    for l in range(NL):
        b.layer(l, q[l], K, V, seq, out_b[l])
    torch.cuda.synchronize()
    assert torch.equal(out_a, out_b)
    assert _sets_equal(a.token_sets(), b.token_sets())


def test_growing_seq_without_host_sync():
    """Token-after-token decode (decode_engine.hpp:97-99, seq = t + 1 grows):
    consecutive steps at seq, seq+1, ... issued back to back on a side stream
    (no synchronisation in between) equal steps of fresh decoders at each
    length, bitwise."""
    NL, B, H, G, d, cap = 4, 2, 8, 4, 128, 4200
    roles = _roles(NL, H, [(1, 2), (3, 6)])
    q, K, V = _inputs(7, NL, B, H, G, d, cap)
    lens = list(range(4090, 4100))  # crosses the 64-row block boundary at 4096
    dec = _dec(NL, B, H, G, d, cap, roles, 500)
    outs = [torch.empty_like(q) for _ in lens]
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        for L, o in zip(lens, outs):
            dec.decode_step(q, K, V, L, o, stream=st)
    st.synchronize()
    for L, o in zip(lens, outs):
        ref = _dec(NL, B, H, G, d, cap, roles, 500)
        r = ref.decode_step(q, K, V, L)
        torch.cuda.synchronize()
        assert torch.equal(o, r), L


def test_growing_seq_per_layer_kernels_stream_ordered():
    """The per-layer-kernel path (TopP) re-plans every new length on the host
    and uploads the plan stream-ordered: steps at growing lengths issued on a
    side stream without synchronisation match fresh decoders."""
    import paper_2602_04541_b200 as P
    NL, B, H, G, d, cap = 3, 1, 4, 4, 64, 3000
    roles = _roles(NL, H, [(2, 1)])
    q, K, V = _inputs(9, NL, B, H, G, d, cap)
    pol = P.SparsityPolicy.top_p(0.5)
    dec = _dec(NL, B, H, G, d, cap, roles, 0, policy=pol)
    assert not dec.fused
    lens = [2900, 2950, 2999, 3000]
    outs = [torch.empty_like(q) for _ in lens]
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        for L, o in zip(lens, outs):
            dec.decode_step(q, K, V, L, o, stream=st)
    st.synchronize()
    for L, o in zip(lens, outs):
        r = _dec(NL, B, H, G, d, cap, roles, 0, policy=pol).decode_step(q, K, V, L)
        torch.cuda.synchronize()
        assert torch.equal(o, r), L


@pytest.mark.parametrize("ragged", [False, True])
def test_device_lengths_graph_replay(ragged):
    """A graph captured with device-resident lengths (lyc_decoder_capture_dev)
    replays t, t+1, ...: the caller advances the lengths and appends the new
    token's K/V rows (lyc_kv_append_dev) inside the stream; every replay equals
    the eager host-length step at those lengths."""
    import ctypes as C
    import paper_2602_04541_b200 as P
    from paper_2602_04541_b200 import _lib as LL
    NL, B, H, G, d, cap = 3, 3, 8, 4, 128, 2100
    roles = _roles(NL, H, [(1, 5), (2, 2)])
    q, K, V = _inputs(13, NL, B, H, G, d, cap)
    K2, V2 = K.clone(), V.clone()
    start = [2000, 1500, 1990] if ragged else [2000] * B
    lens = torch.tensor(start, dtype=torch.int64, device="cuda")
    dec = _dec(NL, B, H, G, d, cap, roles, 300)
    ref = _dec(NL, B, H, G, d, cap, roles, 300)
    out = torch.empty_like(q)
    lay = LL.lyc_kv_layout(n_layers=NL, batch=B, n_kv_heads=H, d_head=d, dtype=LL.DTYPE_BF16,
                           pad=0, seq_cap=cap)
    g = torch.Generator(device="cuda").manual_seed(99)
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        dec.capture_dev(q, K, V, lens, out, stream=st)
    for t in range(6):
        rows_k = torch.empty((NL, B, H, d), dtype=torch.bfloat16, device="cuda").uniform_(-1, 1, generator=g)
        rows_v = torch.empty_like(rows_k).uniform_(-1, 1, generator=g)
        torch.cuda.synchronize()
        with torch.cuda.stream(st):
            lens.add_(1)
            LL.check(LL.lib().lyc_kv_append_dev(K.data_ptr(), V.data_ptr(), C.byref(lay), -1,
                                                lens.data_ptr(), rows_k.data_ptr(),
                                                rows_v.data_ptr(), st.cuda_stream))
            dec.replay(stream=st)
        st.synchronize()
        host = [s + t + 1 for s in start]
        for b in range(B):  # the same rows appended through the host-position write path
            K2[:, b, :, host[b] - 1] = rows_k[:, b]
            V2[:, b, :, host[b] - 1] = rows_v[:, b]
        assert torch.equal(K, K2) and torch.equal(V, V2)
        r = ref.decode_step(q, K2, V2, host if ragged else host[0])
        torch.cuda.synchronize()
        assert torch.equal(out, r), t
        assert _sets_equal(dec.token_sets(), ref.token_sets())
    dec.status()


def test_invalid_device_lengths_are_a_flagged_noop():
    import paper_2602_04541_b200 as P
    NL, B, H, G, d, cap = 2, 2, 2, 4, 64, 512
    roles = _roles(NL, H, [])
    q, K, V = _inputs(3, NL, B, H, G, d, cap)
    dec = _dec(NL, B, H, G, d, cap, roles, 32)
    out = torch.full_like(q, 7.0)
    bad = torch.tensor([100, 513], dtype=torch.int64, device="cuda")
    dec.decode_step_dev(q, K, V, bad, out)
    with pytest.raises(P.InvalidArgument):
        dec.status()
    assert torch.all(out == 7.0)
    good = torch.tensor([100, 512], dtype=torch.int64, device="cuda")
    dec.decode_step_dev(q, K, V, good, out)
    dec.status()
    r = _dec(NL, B, H, G, d, cap, roles, 32).decode_step(q, K, V, [100, 512])
    torch.cuda.synchronize()
    assert torch.equal(out, r)


def test_replay_after_replan_per_layer_kernels():
    """A graph captured on the per-layer kernels replays its captured length
    even after another length was planned (replay restores the plan)."""
    import paper_2602_04541_b200 as P
    NL, B, H, G, d, cap = 3, 1, 4, 4, 64, 2048
    roles = _roles(NL, H, [(1, 2)])
    q, K, V = _inputs(21, NL, B, H, G, d, cap)
    pol = P.SparsityPolicy.threshold(2.0 / 2000)
    dec = _dec(NL, B, H, G, d, cap, roles, 0, policy=pol)
    out = torch.empty_like(q)
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        dec.capture(q, K, V, 2000, out, stream=st)
        other = dec.decode_step(q, K, V, 1500, stream=st)
        dec.replay(stream=st)
    st.synchronize()
    r = _dec(NL, B, H, G, d, cap, roles, 0, policy=pol).decode_step(q, K, V, 2000)
    torch.cuda.synchronize()
    assert torch.equal(out, r)
    assert not torch.equal(other, r)


def test_step_is_bitwise_deterministic():
    """Repeated steps (fresh decoders and reused ones) of the 32K Llama config
    are bitwise identical.  Regression: a stage of the K/V ring was released
    before its final V ldmatrix had returned, so the producer's next copy
    could race it (columns 112..127 of the sparse head after a layer's single
    retrieval head, roughly one step in three)."""
    import bench
    import paper_2602_04541_b200 as P
    NL, B, H, G, d, L, k = 32, 1, 8, 4, 128, 32768, 2048
    roles = bench.make_roles(NL, H, 0.125, 2602)
    q, K, V = _inputs(11, NL, B, H, G, d, L)
    ref = None
    for trial in range(4):
        dec = _dec(NL, B, H, G, d, L, roles, k)
        for _ in range(4):
            out = dec.decode_step(q, K, V, L)
            torch.cuda.synchronize()
            if ref is None:
                ref = out.clone()
            assert torch.equal(out, ref)
        dec.close()
