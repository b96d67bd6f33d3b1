"""GPU parity of the CUDA path (through the C-ABI) against the oracle.

Tolerances (north_star; SURVEY.md 8(a) parity rules):
  fp32: max|o_gpu - o_ref| / max(max|o_ref|, 1e-3) <= 1e-5 relative
        (reference's own f32 gate is 1e-5 absolute, kernel_sim_test.cpp:230)
  bf16: <= 2e-2 relative, against the f64 oracle on the bf16-rounded inputs
  index sets: bit-exact except swaps inside the documented fp score tie band.
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
    import paper_2602_04541_b200  # noqa: F401  (fails loudly without liblyc.so)
    torch.cuda.set_device(0)


def rel_err(got, ref):
    got = np.asarray(got, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    return np.abs(got - ref).max() / max(np.abs(ref).max(), 1e-3)


def make_workload(rng, B, H, G, d, seq, bs, keep, n_retr, dtype):
    import paper_2602_04541_b200 as P
    nb = (seq + bs - 1) // bs
    K = rng.uniform(-1, 1, (B * H, seq, d)).astype(np.float32)
    V = rng.uniform(-1, 1, (B * H, seq, d)).astype(np.float32)
    Q = rng.uniform(-1, 1, (B * H * G, d)).astype(np.float32)
    tK, tV, tQ = (torch.from_numpy(x).to(dtype) for x in (K, V, Q))
    # the oracle sees exactly what the GPU sees (bf16-rounded, upcast)
    K, V, Q = (t.float().numpy() for t in (tK, tV, tQ))
    blocks = []
    for b in range(B):
        for g in range(H):
            if g < n_retr:
                blocks.append(list(range(nb)))
            else:
                c = max(1, int(np.ceil(keep * nb)))
                blocks.append(sorted(rng.choice(nb, c, replace=False).tolist()))
    w = P.Workload(batch=B, n_kv_heads=H, group_size=G, d_head=d, seq_len=seq, block_size=bs,
                   scale=float(1 / np.sqrt(d)), keys=tK, values=tV, queries=tQ,
                   blocks=P.BlockIndexSet(B, H, blocks))
    return w, K, V, Q, blocks


# ------------------------------------------------------------------ kernel::run
@pytest.mark.parametrize("seed", range(6))
def test_run_fp32_matches_reference_sweep(orc, seed):
    """kernel_sim_test.cpp:219-239 / acceptance criterion 3(c) on the GPU."""
    import paper_2602_04541_b200 as P
    rng = np.random.default_rng(100 + seed)
    B, H, G = int(rng.integers(1, 5)), int(rng.integers(1, 9)), int(rng.integers(1, 5))
    d = [16, 32, 64, 128][seed % 4]
    seq = int(rng.integers(64, 4097))
    S = int(rng.integers(1, 9))
    w, K, V, Q, blocks = make_workload(rng, B, H, G, d, seq, 64, 0.1, int(rng.integers(0, H + 1)),
                                       torch.float32)
    res = P.run(w, S)
    ref = orc.kernel_run(K, V, Q, blocks, batch=B, group=G, seq_len=seq, scale=w.scale,
                         num_splits=S, dtype=np.float64)
    assert rel_err(res.outputs.cpu().numpy(), ref) < FP32_TOL
    assert all(c == 1 for c in res.block_exec_counts)  # conservation (kernel_sim_test.cpp:241-248)


@pytest.mark.parametrize("d", [64, 128, 256])
@pytest.mark.parametrize("G", [1, 4, 8])
def test_run_bf16_matches_reference(orc, d, G):
    import paper_2602_04541_b200 as P
    rng = np.random.default_rng(d * 10 + G)
    B, H, seq = 2, 4, 1500
    w, K, V, Q, blocks = make_workload(rng, B, H, G, d, seq, 64, 0.2, 2, torch.bfloat16)
    for S in (1, 3, 37):
        res = P.run(w, S)
        ref = orc.kernel_run(K, V, Q, blocks, batch=B, group=G, seq_len=seq, scale=w.scale,
                             num_splits=S, dtype=np.float64)
        assert rel_err(res.outputs.float().cpu().numpy(), ref) < BF16_TOL


@pytest.mark.parametrize("bs", [16, 48, 64, 100, 200])
def test_run_block_sizes(orc, bs):
    """Workload::block_size is a free parameter (kernel_sim.hpp:127)."""
    import paper_2602_04541_b200 as P
    rng = np.random.default_rng(bs)
    w, K, V, Q, blocks = make_workload(rng, 1, 3, 2, 32, 777, bs, 0.3, 1, torch.float32)
    res = P.run(w, 5)
    ref = orc.kernel_run(K, V, Q, blocks, batch=1, group=2, seq_len=777, block_size=bs,
                         scale=w.scale, num_splits=5, dtype=np.float64)
    assert rel_err(res.outputs.cpu().numpy(), ref) < FP32_TOL


def test_run_golden_vectors(golden):
    """The reference's own kernel::run<float> outputs (tests/golden)."""
    import paper_2602_04541_b200 as P
    g = golden["kernel_run"]
    n = len([k for k in g if k.startswith("meta")])
    for i in range(n):
        B, H, G, d, seq, bs, S = g[f"meta{i}"].tolist()
        off, ids = g[f"off{i}"], g[f"ids{i}"]
        blocks = [ids[off[j]: off[j + 1]].tolist() for j in range(B * H)]
        w = P.Workload(batch=B, n_kv_heads=H, group_size=G, d_head=d, seq_len=seq, block_size=bs,
                       scale=0.25, keys=torch.from_numpy(g[f"K{i}"]),
                       values=torch.from_numpy(g[f"V{i}"]), queries=torch.from_numpy(g[f"Q{i}"]),
                       blocks=P.BlockIndexSet(B, H, blocks))
        res = P.run(w, S)
        assert np.abs(res.outputs.cpu().numpy() - g[f"out{i}"]).max() < 1e-5  # reference f32 gate
        assert res.block_exec_counts == [1] * len(ids)


def test_run_split_invariance_and_determinism(orc):
    """kernel_sim_test.cpp:201-209 and the bitwise worker-count test (250-264):
    for a fixed plan, outputs are bitwise reproducible run to run."""
    import paper_2602_04541_b200 as P
    rng = np.random.default_rng(43)
    w, K, V, Q, blocks = make_workload(rng, 2, 4, 2, 64, 777, 64, 0.25, 2, torch.float32)
    base = P.run(w, 1).outputs.cpu()
    for S in (2, 3, 5, 8, 150):
        a = P.run(w, S).outputs.cpu()
        b = P.run(w, S, n_workers=7).outputs.cpu()
        assert torch.equal(a, b)
        assert (a - base).abs().max().item() < 1e-5


def test_run_errors():
    """Reference exceptions map to InvalidArgument (kernel_sim.hpp:27-41, 64, 79, 211)."""
    import paper_2602_04541_b200 as P
    rng = np.random.default_rng(42)
    w, *_ = make_workload(rng, 1, 2, 1, 16, 128, 64, 0.5, 1, torch.float32)
    w.blocks.ids[1] = []
    with pytest.raises(P.InvalidArgument):
        P.run(w, 2)
    w.blocks.ids[1] = [1, 0]
    with pytest.raises(P.InvalidArgument):
        P.run(w, 2)
    w.blocks.ids[1] = [5]
    with pytest.raises(P.InvalidArgument):
        P.run(w, 2)
    w.blocks.ids[1] = [0]
    with pytest.raises(P.InvalidArgument):
        P.run(w, 0)


# ------------------------------------------------------------------ args_top_k
def test_args_top_k_known_cases():
    import paper_2602_04541_b200 as P
    w = torch.tensor([0.4, 0.1, 0.3, 0.2])
    assert P.args_top_k(w, 2).tolist() == [0, 2]
    assert P.args_top_k(torch.full((5,), 0.2), 3).tolist() == [0, 1, 2]
    assert P.args_top_k(w, 9).tolist() == [0, 1, 2, 3]
    with pytest.raises(P.InvalidArgument):
        P.args_top_k(w, 0)


@pytest.mark.parametrize("n,k", [(1, 1), (7, 3), (1000, 10), (4096, 256), (32768, 2048),
                                 (131072, 4096), (131073, 4096), (262144, 8192), (300000, 1)])
def test_args_top_k_bitexact(orc, n, k):
    """Exact set equality vs the reference rule on identical fp32 scores,
    including heavy ties and -0.0/+0.0 (compared equal by the reference)."""
    import paper_2602_04541_b200 as P
    rng = np.random.default_rng(n + k)
    for variant in range(3):
        s = rng.standard_normal(n).astype(np.float32)
        if variant == 1:
            s = np.round(s * 4) / 4  # massive ties at the threshold
        if variant == 2:
            s[:] = 0.0
            s[::3] = -0.0
        got = P.args_top_k(torch.from_numpy(s), k).cpu().numpy()
        ref = orc.args_top_k(s, k)
        assert np.array_equal(got, ref), (n, k, variant)


def test_args_top_k_golden(golden):
    import paper_2602_04541_b200 as P
    g = golden["args_top_k"]
    n = len([k for k in g if k.startswith("out")])
    for i in range(n):
        w = g[f"w{i}"]
        if w.dtype != np.float32:
            continue  # device scores are fp32
        got = P.args_top_k(torch.from_numpy(w), int(g[f"k{i}"])).cpu().numpy()
        assert np.array_equal(got, g[f"out{i}"]), i
