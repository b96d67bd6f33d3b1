"""Which CTAs end each layer's consumer phase last (debug, run under gpurun)."""
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
acc = []
for rep in range(5):
    dec.decode_step(q, K, V, L)
    torch.cuda.synchronize()
    tr = dec.trace().astype(np.int64)
    t0 = tr[0, 0].min()
    acc.append((tr - t0) / 1e3)
rel = np.stack(acc)  # [rep][L][ev][cta]
n = rel.shape[-1]
for l in range(NL):
    nr = int((roles[l] == 0).sum()) if l else H
    pr = int((roles[l - 1] == 0).sum()) if l > 1 else (H if l == 1 else 0)
    b = rel[:, l, 0]
    e = rel[:, l, 1]
    span = (e - b).mean(0)
    end_rel = (e - b.max(1, keepdims=True)).mean(0)
    late = np.argsort(-end_rel)[:8]
    items_prev = 16 * pr
    tail = np.arange(n) >= n - items_prev if items_prev else np.zeros(n, bool)
    msg = ""
    if tail.any():
        msg = f" prev-item CTAs span {span[tail].mean():5.1f} others {span[~tail].mean():5.1f}"
    print(f"l{l:2d} R{nr} prevR{pr} span p50 {np.median(span):5.1f} max {span.max():5.1f} "
          f"end-rel p50 {np.median(end_rel):5.1f} max {end_rel.max():5.1f} late {list(late)}{msg}")
# consumer events of the latest CTA vs the median CTA (first rep)
names = ["q_staged", "first_tile", "unit1_done", "last_tile", "ue_enter", "ue_bar", "ue_stored", "u1_signalled"]
for l in (5, 6, 7, 12, 13, 17, 20):
    b = rel[:, l, 0]
    e = rel[:, l, 1]
    end_rel = (e - b.max(1, keepdims=True)).mean(0)
    order = np.argsort(end_rel)
    for tag, c in (("median", order[n // 2]), ("latest", order[-1])):
        ev = " ".join(f"{nm} {(rel[:, l, 16 + i, c] - rel[:, l, 0, c]).mean():5.1f}" for i, nm in enumerate(names))
        print(f"l{l:2d} {tag:6s} cta {c:3d} begin {(b[:, c] - b.min(1)).mean():4.1f} span {(e[:, c]-b[:, c]).mean():5.1f} | {ev}")
