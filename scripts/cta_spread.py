"""Per-CTA spread of the consumer spans of selected layers (debug, run under gpurun)."""
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
dec.decode_step(q, K, V, L)
torch.cuda.synchronize()
tr = dec.trace().astype(np.int64)
t0 = tr[0, 0].min()
rel = (tr - t0) / 1e3
for l in range(NL):
    nr = int((roles[l] == 0).sum()) if l else H
    b, e = rel[l, 0], rel[l, 1]
    span = e - b
    qs, t1, u1, tl = rel[l, 16] - b, rel[l, 17] - b, rel[l, 18] - b, rel[l, 19] - b
    print(f"l{l:2d} R{nr} begin max {b.max():7.1f} end p50/max {np.percentile(e,50):7.1f}/{e.max():7.1f}"
          f"  span p50 {np.percentile(span,50):5.1f} | q_staged p50 {np.percentile(qs,50):4.1f} "
          f"first_tile p50 {np.percentile(t1,50):4.1f} first_unit_done p50 {np.percentile(u1,50):5.1f} "
          f"last_tile p50 {np.percentile(tl,50):5.1f} | ue_enter {np.percentile(rel[l,20]-b,50):5.1f} "
          f"ue_bar {np.percentile(rel[l,21]-b,50):5.1f} ue_stored {np.percentile(rel[l,22]-b,50):5.1f}")
