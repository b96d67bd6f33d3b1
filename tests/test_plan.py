"""The seq-parametric device planner of the fused step (csrc/plan.cuh), run
sequentially on the host, against the host-order planner of the same split
plan (capi.cu plan_step_launch: Algorithm 2's pooling, kernel_sim.hpp:63-110,
in the step kernel's three-pool order) -- slots, units, split offsets, merge
tasks, selection rows and budgets must agree exactly.  CPU only."""
import numpy as np
import pytest

import paper_2602_04541_b200 as P
from paper_2602_04541_b200.decode import plan_selftest


def _random_case(rng):
    B = int(rng.choice([1, 1, 2, 3, 4, 8, 16]))
    H = int(rng.integers(1, 9))
    G = int(rng.choice([1, 2, 4, 8]))
    NL = int(rng.integers(1, 7))
    n_sms = 148
    splits = int(rng.choice([0, 0, 1, 2, 3, 5])) if B * 5 <= n_sms else 0
    select = str(rng.choice(["tokens", "tokens", "blocks", "none"]))
    roles = np.ones((NL, H), np.uint8)
    roles[0] = 0
    if select == "none":
        roles[:] = 0
    else:
        roles[1:] = rng.random((NL - 1, H)) < rng.choice([0.1, 0.3, 0.7])
        roles[1:] = 1 - roles[1:]
    seq_cap = int(rng.choice([64, 1000, 8192, 40000, 131072]))
    if rng.random() < 0.5:
        pol = P.SparsityPolicy.top_k(int(rng.choice([1, 63, 64, 65, 256, 4096, 10 ** 6])))
    else:
        pol = P.SparsityPolicy.ratio(float(rng.choice([0.1, 0.5, 0.9, 0.99])))
    if rng.random() < 0.4 and B > 1:
        lens = [int(rng.integers(1, seq_cap + 1)) for _ in range(B)]
        return dict(n_layers=NL, batch=B, n_kv_heads=H, group_size=G, d_head=128,
                    seq_cap=seq_cap, roles=roles, policy=pol, select=select, seq_lens=lens,
                    n_sms=n_sms, num_splits=splits)
    seq = int(rng.choice([1, 63, 64, 65, seq_cap // 2 + 1, seq_cap]))
    return dict(n_layers=NL, batch=B, n_kv_heads=H, group_size=G, d_head=128, seq_cap=seq_cap,
                roles=roles, policy=pol, select=select, seq_len=max(1, min(seq, seq_cap)), n_sms=n_sms,
                num_splits=splits)


@pytest.mark.parametrize("seed", range(8))
def test_device_planner_equals_host_planner(seed):
    rng = np.random.default_rng(1000 + seed)
    for _ in range(40):
        case = _random_case(rng)
        plan_selftest(**case)


def test_bench_configs():
    import bench
    for name in ("qwen3-8b-128k", "llama3-8b-32k", "llama3-8b-64k-b16", "llama3-8b-256k-b4"):
        wl = bench.WORKLOADS[name]
        roles = bench.make_roles(wl["NL"], wl["H"], 0.125, 2602)
        for seq in (1, 4096, wl["L"] - 1, wl["L"]):
            plan_selftest(n_layers=wl["NL"], batch=wl["B"], n_kv_heads=wl["H"], group_size=wl["G"],
                          d_head=wl["d"], seq_cap=wl["L"], roles=roles,
                          policy=P.SparsityPolicy.top_k(wl["k"]), seq_len=seq)


def test_invalid_lengths_are_rejected():
    roles = np.zeros((2, 2), np.uint8)
    with pytest.raises(P.InvalidArgument):
        plan_selftest(n_layers=2, batch=2, n_kv_heads=2, group_size=2, d_head=64, seq_cap=100,
                      roles=roles, policy=P.SparsityPolicy.top_k(8), seq_lens=[5, 101])
