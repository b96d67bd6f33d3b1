"""Per-CTA spread of the consumer phase of selected layers of one fused step
(debug, run under gpurun): python scripts/cta_spread.py [workload] [layers...]"""
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
import paper_2602_04541_b200 as P  # noqa: E402

wname = sys.argv[1] if len(sys.argv) > 1 else "qwen3-8b-128k"
wl = dict(bench.WORKLOADS[wname])
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
tr = dec.trace().astype(np.int64)  # [NL][events][ctas]
t0 = tr[0, 0].min()
rel = (tr - t0) / 1e3
layers = [int(x) for x in sys.argv[2:]] or list(range(1, 10))
for l in layers:
    nr = int((roles[l] == 0).sum())
    b = rel[l, 0]
    e = rel[l, 1]
    b0 = b.min()
    pe = np.percentile(e - b0, [10, 50, 90, 100])
    pb = np.percentile(b - b0, [50, 100])
    q16 = np.percentile(rel[l, 16] - b0, [50, 100])
    u18 = np.percentile(rel[l, 18] - b0, [10, 50, 90, 100])
    slow = np.argsort(-e)[:6]
    print(f"l{l:2d} R{nr} begin p50/max {pb[0]:4.1f}/{pb[1]:4.1f}  q_staged p50/max {q16[0]:4.1f}/{q16[1]:4.1f}  "
          f"first-unit-done p10/50/90/max {u18[0]:5.1f}/{u18[1]:5.1f}/{u18[2]:5.1f}/{u18[3]:5.1f}  "
          f"end p10/50/90/max {pe[0]:5.1f}/{pe[1]:5.1f}/{pe[2]:5.1f}/{pe[3]:5.1f}  slowest CTAs {slow.tolist()}")
