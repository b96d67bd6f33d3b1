"""Per-layer API timeline (lyc_decoder_layer, one step-kernel launch per layer):
per layer the first consumer start, the last consumer end, the last merge,
the last selection emission, and the gap to the next launch's first consumer
(debug, run under gpurun)."""
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
import paper_2602_04541_b200 as P  # noqa: E402

wl = dict(bench.WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "qwen3-8b-128k"])
NL, H, G, d, L, k, B = (wl[x] for x in ("NL", "H", "G", "d", "L", "k", "B"))
roles = bench.make_roles(NL, H, 0.125, 2602)
K = torch.empty((NL, B, H, L, d), dtype=torch.bfloat16, device="cuda")
V = torch.empty_like(K)
for t in (K, V):
    for l in range(NL):
        t[l].uniform_(-1, 1)
q = torch.empty((NL, B, H * G, d), dtype=torch.bfloat16, device="cuda").uniform_(-1, 1)
out = torch.empty_like(q)
dec = P.HybridDecoder(n_layers=NL, batch=B, n_kv_heads=H, group_size=G, d_head=d, seq_cap=L,
                      roles=roles, policy=P.SparsityPolicy.top_k(k), dtype=torch.bfloat16)
for _ in range(3):
    for l in range(NL):
        dec.layer(l, q[l], K, V, L, out[l])
dec.set_trace(True)
for l in range(NL):
    dec.layer(l, q[l], K, V, L, out[l])
torch.cuda.synchronize()
tr = dec.trace().astype(np.int64)
t0 = tr[0, 0].min()
r = (tr - t0) / 1e3
print(f"{'l':>3} {'R':>2} {'entry0':>8} {'pdl0':>8} {'bars':>8} {'prolog':>8} {'beg':>8} {'end':>8} {'merge':>8} "
      f"{'seldone':>8} {'exit':>8} {'next_beg':>8} {'gap':>6}")
for l in range(NL):
    nr = int((roles[l] == 0).sum()) if l else H
    beg, end, mrg = r[l, 0].min(), r[l, 1].max(), r[l, 3].max()
    sd = r[l, 13].max() if tr[l, 13].max() > t0 else float("nan")
    nb = r[l + 1, 0].min() if l + 1 < NL else float("nan")
    last = max(end, mrg, sd if sd == sd else 0)
    ent, pdl, pro, ex = r[l, 5].min(), r[l, 7].max(), r[l, 17].max(), r[l, 19].max()
    bars = r[l, 23].max()
    print(f"{l:3d} {nr:2d} {ent:8.1f} {pdl:8.1f} {bars:8.1f} {pro:8.1f} {beg:8.1f} {end:8.1f} {mrg:8.1f} {sd:8.1f} "
          f"{ex:8.1f} {nb:8.1f} {nb - last:6.1f}")
