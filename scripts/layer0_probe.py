"""One all-retrieval layer (layer 0 of the bench workload) for ncu source-level capture."""
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
import paper_2602_04541_b200 as P  # noqa: E402

wl = dict(bench.WORKLOADS["llama3-8b-128k"])
NL, H, G, d, L, k, B = 1, wl["H"], wl["G"], wl["d"], wl["L"], wl["k"], wl["B"]
roles = bench.make_roles(NL, H, 0.125, 2602)
K = torch.empty((NL, B, H, L, d), dtype=torch.bfloat16, device="cuda").uniform_(-1, 1)
V = torch.empty_like(K).uniform_(-1, 1)
q = torch.empty((NL, B, H * G, d), dtype=torch.bfloat16, device="cuda").uniform_(-1, 1)
pol = P.SparsityPolicy.top_k(k) if len(sys.argv) < 2 else None
dec = P.HybridDecoder(n_layers=NL, batch=B, n_kv_heads=H, group_size=G, d_head=d, seq_cap=L,
                      roles=roles, policy=P.SparsityPolicy.top_k(k), dtype=torch.bfloat16)
for _ in range(5):
    dec.decode_step(q, K, V, L)
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(20):
    dec.decode_step(q, K, V, L)
e.record()
torch.cuda.synchronize()
print("layer-0 step us", s.elapsed_time(e) / 20 * 1e3)
