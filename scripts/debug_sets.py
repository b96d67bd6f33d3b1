"""Debug: compare fused-step vs per-layer index sets and both vs the oracle."""
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_2602_04541_b200 as P  # noqa: E402
from oracle import pyoracle  # noqa: E402
from tests.test_gpu_decode import roles_for, synth  # noqa: E402


def main(select="tokens", B=2):
    NL, H, G, d, seq = 5, 8, 4, 128, 6000
    roles = roles_for(NL, H, [(1, 3), (2, 5), (3, 0), (4, 3)])
    q, K, V = synth(17, NL, B, H, G, d, seq, 6016, torch.bfloat16)
    qd, Kd, Vd = q.cuda(), K.cuda(), V.cuda()
    mk = lambda: P.HybridDecoder(n_layers=NL, batch=B, n_kv_heads=H, group_size=G, d_head=d,
                                 seq_cap=6016, roles=roles, policy=P.SparsityPolicy.top_k(700),
                                 select=select)
    fused = mk()
    print("fused:", fused.fused)
    traces_f = []
    out_f = fused.decode_step(qd, Kd, Vd, seq)
    torch.cuda.synchronize()
    sf = fused.token_sets()
    per = mk()
    out_p = torch.empty_like(qd)
    traces_p = []
    for l in range(NL):
        per.layer(l, qd[l], Kd, Vd, seq, out_p[l])
        traces_p.append(per.token_sets())
    torch.cuda.synchronize()
    sp = per.token_sets()
    orc = pyoracle.orc()
    qn, Kn, Vn = q.float().numpy(), K.float().numpy(), V.float().numpy()
    for b in range(B):
        r = orc.decode_step(qn[:, b], Kn[:, b], Vn[:, b], roles, seq=seq, scale=1 / np.sqrt(d),
                            kind="topk", k=700, trace=True)
        for g in range(H):
            a, c, o = set(sf[b][g].tolist()), set(sp[b][g].tolist()), set(r["sets"][g].tolist())
            print(f"b{b} g{g} |f|={len(a)} |p|={len(c)} f^p={len(a ^ c)} f^o={len(a ^ o)} "
                  f"p^o={len(c ^ o)} sorted_f={bool(np.all(np.diff(sf[b][g]) > 0))}")
    print("out rel diff", (out_f.float() - out_p.float()).abs().max().item())


if __name__ == "__main__":
    main(*(sys.argv[1:2] or ["tokens"]))
