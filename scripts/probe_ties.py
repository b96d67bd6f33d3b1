import sys, numpy as np, torch
sys.path.insert(0, "/root/repo")
import paper_2602_04541_b200 as P
from tests.test_gpu_decode import synth
rng = np.random.default_rng(5)
s = np.zeros(20000, np.float32); perm = rng.permutation(20000)
s[perm[:800]] = 2.0; s[perm[800:2800]] = 1.0
got = P.args_top_k(torch.tensor(s).cuda(), 1000).cpu().numpy()
want = np.sort(np.concatenate([perm[:800], np.sort(perm[800:2800])[:200]]))
print("args_top_k equal:", np.array_equal(np.sort(got), want), len(got))
q, K, V = synth(11, 2, 1, 2, 4, 64, 20000, 20000, torch.float32)
qb = q[0, 0, 0:4].double().mean(0)
Kl = torch.zeros(20000, 64, dtype=torch.float64); Kl[perm[:800]] = 2 * qb; Kl[perm[800:2800]] = qb
Kf = Kl.float()
sc = (Kf.double() @ q[0, 0, 0:4].double().T).sum(1)
print("pooled score classes:", np.unique(sc.numpy().round(4)))
# decode layer 0 only through the per-layer path and compare the set
from tests.test_gpu_decode import roles_for
NL, H, G, d, seq, k = 1, 1, 4, 64, 20000, 1000
q1 = q[:1, :, :4].contiguous()
K1 = torch.zeros(1, 1, 1, seq, d); K1[0, 0, 0] = Kf
V1 = V[:1, :, :1].contiguous()
for fused in (True, False):
    dec = P.HybridDecoder(n_layers=1, batch=1, n_kv_heads=1, group_size=4, d_head=64, seq_cap=seq,
                          roles=np.zeros((1, 1), np.uint8), policy=P.SparsityPolicy.top_k(k),
                          dtype=torch.float32)
    if fused:
        out = dec.decode_step(q1.cuda(), K1.cuda(), V1.cuda(), seq)
    else:
        out = dec.layer(0, q1[0].cuda(), K1.cuda(), V1.cuda(), seq)
    torch.cuda.synchronize()
    s0 = dec.token_sets()[0][0]
    print("fused" if fused else "layer", "fused-flag", dec.fused, "equal:", np.array_equal(s0, want),
          "n2", int(np.isin(s0, perm[:800]).sum()), "n1", int(np.isin(s0, perm[800:2800]).sum()))
