"""Debug: bitwise determinism of the fused step across fresh decoders and
repeated steps (a race shows up as differing (layer, head) blocks)."""
import sys
from pathlib import Path
import numpy as np
import torch
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench
import paper_2602_04541_b200 as P
from tests.parity_util import make_inputs

wl = sys.argv[1] if len(sys.argv) > 1 else "llama3-8b-32k"
w = bench.WORKLOADS[wl]
NL, B, H, G, d, L, k = (w[x] for x in ("NL", "B", "H", "G", "d", "L", "k"))
roles = bench.make_roles(NL, H, 0.125, 2602)
q, K, V = make_inputs(NL, B, H, G, d, L, L, torch.bfloat16, 11)
ref = None
for trial in range(int(sys.argv[2]) if len(sys.argv) > 2 else 8):
    dec = P.HybridDecoder(n_layers=NL, batch=B, n_kv_heads=H, group_size=G, d_head=d, seq_cap=L,
                          roles=roles, policy=P.SparsityPolicy.top_k(k), dtype=torch.bfloat16)
    for step in range(3):
        out = dec.decode_step(q, K, V, L)
        torch.cuda.synchronize()
        o = out.float().cpu().numpy().reshape(NL, B, H, G, d)
        if ref is None:
            ref = o
            continue
        diff = np.argwhere(np.any(o != ref, axis=(3, 4)))
        det = []
        for (l, b, g) in diff.tolist()[:4]:
            dj = [float(np.abs(o[l, b, g, j] - ref[l, b, g, j]).max()) for j in range(G)]
            ncol = [np.nonzero(o[l, b, g, j] != ref[l, b, g, j])[0].tolist() for j in range(1)]
            det.append((l, g, [round(x, 4) for x in dj], ncol))
        print(f"trial {trial} step {step}: {'same' if len(diff) == 0 else det}", flush=True)
    dec.close()
