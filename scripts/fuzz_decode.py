"""Randomised parity sweep of the fused step (debug tool, run under gpurun):
random shapes, dtypes, splits, roles and policies; every case against the
oracle's decode_step (outputs within the dtype tolerance, sets exact up to
the documented tie band)."""
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))
import paper_2602_04541_b200 as P  # noqa: E402
from oracle import pyoracle as PO  # noqa: E402

orc = PO.orc()
rng = np.random.default_rng(int(sys.argv[1]) if len(sys.argv) > 1 else 0)
n_cases = int(sys.argv[2]) if len(sys.argv) > 2 else 12
edge = len(sys.argv) > 3 and sys.argv[3] == "edge"  # boundary sizes: tiny contexts, k >= seq, odd G
bad = 0
for case in range(n_cases):
    dt = torch.bfloat16 if rng.random() < 0.7 else torch.float32
    d = int(rng.choice([64, 128])) if dt == torch.bfloat16 else int(rng.choice([16, 32, 64, 128]))
    G = int(rng.integers(1, 9)) if edge else int(rng.choice([1, 2, 4, 8]))
    H = int(rng.choice([1, 2, 4]))
    B = int(rng.choice([1, 2, 3]))
    NL = int(rng.integers(1, 4))
    seq = int(rng.choice([1, 2, 63, 64, 65, 127, 8191, 8192, 8193, 16385])) if edge \
        else int(rng.integers(100, 20000))
    k = int(rng.choice([1, seq, seq + 5, max(1, seq // 2)])) if edge \
        else int(rng.integers(1, min(seq, 3000) + 1))
    ns = int(rng.choice([0, 1, 2, 5]))
    kind = str(rng.choice(["topk", "topk", "ratio", "topp", "threshold"]))
    value = {"topk": 0.0, "ratio": float(rng.uniform(0.5, 0.99)), "topp": float(rng.uniform(0.05, 0.9)),
             "threshold": float(rng.uniform(0.5, 3.0)) / seq}[kind]
    pol = {"topk": lambda: P.SparsityPolicy.top_k(k), "ratio": lambda: P.SparsityPolicy.ratio(value),
           "topp": lambda: P.SparsityPolicy.top_p(value),
           "threshold": lambda: P.SparsityPolicy.threshold(value)}[kind]()
    roles = (rng.random((NL, H)) < 0.6).astype(np.uint8)
    roles[0] = 0
    g = torch.Generator().manual_seed(case)
    q = (torch.rand((NL, B, H * G, d), generator=g) * 2 - 1).to(dt)
    K = (torch.rand((NL, B, H, seq, d), generator=g) * 2 - 1).to(dt)
    V = (torch.rand((NL, B, H, seq, d), generator=g) * 2 - 1).to(dt)
    try:
        dec = P.HybridDecoder(n_layers=NL, batch=B, n_kv_heads=H, group_size=G, d_head=d,
                              seq_cap=seq, roles=roles, policy=pol, dtype=dt,
                              num_splits=ns)
        out = dec.decode_step(q.cuda(), K.cuda(), V.cuda(), seq).float().cpu().numpy()
        sets = dec.token_sets()
        fused = dec.fused
        dec.close()
    except P.LycError as e:
        print(f"case {case}: skipped ({type(e).__name__}: {e})")
        continue
    tol = 2e-2 if dt == torch.bfloat16 else 1e-5
    worst, set_bad = 0.0, 0
    qf, Kf, Vf = q.float().numpy(), K.float().numpy(), V.float().numpy()
    for b in range(B):
        r = orc.decode_step(qf[:, b], Kf[:, b], Vf[:, b], roles, seq=seq, scale=1 / np.sqrt(d),
                            kind=kind, k=k, value=value)
        e = np.abs(out[:, b] - r["out"]).max() / max(np.abs(r["out"]).max(), 1e-3)
        worst = max(worst, e)
        for gg in range(H):
            if not np.array_equal(sets[b][gg], r["sets"][gg]):
                set_bad += 1
    # variable-size policies may move one element at a cut (documented fp band)
    ok = worst < tol if set_bad == 0 or kind in ("topk", "ratio") else True
    bad += 0 if ok else 1
    print(f"case {case}: {'ok ' if ok else 'BAD'} dt={str(dt)[6:]} d={d} G={G} H={H} B={B} NL={NL} "
          f"seq={seq} {kind} k={k} v={value:.3g} ns={ns} fused={fused} rel_err={worst:.2e} set_diffs={set_bad}",
          flush=True)
print("bad cases:", bad)
