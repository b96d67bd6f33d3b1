import sys, numpy as np, torch
sys.path.insert(0, "/root/repo")
import paper_2602_04541_b200 as P
from tests.test_gpu_decode import synth
d = 64
for seq, k, n2, n1 in [(16384, 1000, 800, 2000), (20000, 1000, 800, 2000), (20000, 1000, 100, 150),
                       (20000, 1000, 800, 100), (8192, 1000, 800, 2000)]:
    q, K, V = synth(11, 1, 1, 1, 4, d, seq, seq, torch.float32)
    qb = q[0, 0, 0:4].double().mean(0)
    rng = np.random.default_rng(5); perm = rng.permutation(seq)
    Kl = torch.randn(seq, d) * 1e-3
    Kl[perm[:n2]] = (2 * qb).float(); Kl[perm[n2:n2 + n1]] = qb.float()
    scores = (Kl.double() @ q[0, 0, :4].double().T).sum(1).numpy()
    order = np.lexsort((np.arange(seq), -scores))
    want = np.sort(order[:k])
    dec = P.HybridDecoder(n_layers=1, batch=1, n_kv_heads=1, group_size=4, d_head=d, seq_cap=seq,
                          roles=np.zeros((1, 1), np.uint8), policy=P.SparsityPolicy.top_k(k), dtype=torch.float32)
    dec.decode_step(q.cuda(), Kl.reshape(1, 1, 1, seq, d).cuda(), V.cuda(), seq)
    torch.cuda.synchronize()
    s0 = dec.token_sets()[0][0]
    print(seq, k, n2, n1, "equal:", np.array_equal(s0, want), "n2", int(np.isin(s0, perm[:n2]).sum()),
          "n1", int(np.isin(s0, perm[n2:n2 + n1]).sum()), "len", len(s0))
