import sys
from pathlib import Path
import numpy as np
import torch
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_2602_04541_b200 as P
from tests.test_gpu_decode import synth, roles_for

NL, B, H, G, d, seq, k = 2, 1, 2, 4, 64, 20000, 1000
n_ties = int(sys.argv[1]) if len(sys.argv) > 1 else 2000
roles = roles_for(NL, H, [])
q, K, V = synth(11, NL, B, H, G, d, seq, seq, torch.float32)
rng = np.random.default_rng(5)
cls = {}
for l in range(NL):
    for g in range(H):
        qbar = q[l, 0, g * G:(g + 1) * G].double().mean(0)
        rows = rng.permutation(seq)
        Kl = torch.zeros(seq, d, dtype=torch.float64)
        Kl[rows[:800]] = 2 * qbar
        Kl[rows[800:800 + n_ties]] = qbar
        K[l, 0, g] = Kl.float()
        c = np.zeros(seq, np.int64); c[rows[:800]] = 2; c[rows[800:800 + n_ties]] = 1
        cls[(l, g)] = c
dec = P.HybridDecoder(n_layers=NL, batch=B, n_kv_heads=H, group_size=G, d_head=d, seq_cap=seq,
                      roles=roles, policy=P.SparsityPolicy.top_k(k), dtype=torch.float32)
out = dec.decode_step(q.cuda(), K.cuda(), V.cuda(), seq)
torch.cuda.synchronize()
sets = dec.token_sets()[0]
for g in range(H):
    c = cls[(0, g)]
    s = np.asarray(sets[g])
    ties = np.nonzero(c == 1)[0]
    want = np.sort(np.concatenate([np.nonzero(c == 2)[0], ties[:200]]))
    print("head", g, "len", len(s), "sorted", bool(np.all(np.diff(s) > 0)), "class counts",
          [(int((c[s] == v).sum())) for v in (2, 1, 0)], "max tie idx taken",
          int(s[c[s] == 1].max()) if (c[s] == 1).any() else None, "want max tie", int(ties[199]))
    print("   first diffs:", np.setdiff1d(want, s)[:10], np.setdiff1d(s, want)[:10])
    # per item
    for it in range(3):
        lo, hi = it * 8192, min(seq, (it + 1) * 8192)
        print("   item", it, "got", int(((s >= lo) & (s < hi)).sum()), "want", int(((want >= lo) & (want < hi)).sum()))
