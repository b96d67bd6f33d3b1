"""Selection phase durations of the fused step (debug, run under gpurun):
per item CTA, consecutive-event differences, median and max over the items of
each selecting layer (layers >= 1), averaged over layers and reps."""
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
import paper_2602_04541_b200 as P  # noqa: E402

wl = dict(bench.WORKLOADS["llama3-8b-128k"])
NL, H, G, d, L, k, B = (wl[x] for x in ("NL", "H", "G", "d", "L", "k", "B"))
roles = bench.make_roles(NL, H, 0.125, 2602)
K = torch.empty((NL, B, H, L, d), dtype=torch.bfloat16, device="cuda")
V = torch.empty_like(K)
for t in (K, V):
    for l in range(NL):
        t[l].uniform_(-1, 1)
q = torch.empty((NL, B, H * G, d), dtype=torch.bfloat16, device="cuda").uniform_(-1, 1)
dec = P.HybridDecoder(n_layers=NL, batch=B, n_kv_heads=H, group_size=G, d_head=d, seq_cap=L,
                      roles=roles, policy=P.SparsityPolicy.top_k(k), dtype=torch.bfloat16)
for _ in range(3):
    dec.decode_step(q, K, V, L)
dec.set_trace(True)
EV = [("wake", 2), ("c_prefix", 8), ("c_keys", 9), ("c_done", 10), ("r_wake", 12),
      ("r_loaded", 6), ("r_digit", 11), ("r_scan", 15), ("r_ranked", 4), ("e_scan", 14),
      ("e_done", 13)]
med, mx, tot, spans = [], [], [], []
for rep in range(8):
    dec.decode_step(q, K, V, L)
    torch.cuda.synchronize()
    tr = dec.trace().astype(np.int64)
    for l in range(1, NL):
        x = tr[l, [e for _, e in EV]]  # [ev][cta]
        items = np.where(x[0] > 0)[0]
        if len(items) == 0:
            continue
        y = x[:, items].astype(np.float64) / 1e3
        dd = np.diff(y, axis=0)
        med.append(np.median(dd, axis=1))
        mx.append(dd.max(axis=1))
        tot.append(y[-1].max() - y[0].max())
        spans.append(y[-1].max() - y[0].min())
med, mx = np.mean(med, 0), np.mean(mx, 0)
print("phase          median   max  (us, mean over selecting layers x reps)")
for i in range(len(EV) - 1):
    print(f"{EV[i][0]:>8}->{EV[i + 1][0]:<9} {med[i]:6.2f} {mx[i]:6.2f}")
print(f"last wake -> last e_done {np.mean(tot):6.2f}   first wake -> last e_done {np.mean(spans):6.2f}")
