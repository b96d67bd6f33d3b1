import sys, numpy as np, torch
sys.path.insert(0, "/root/repo")
import paper_2602_04541_b200 as P
from tests.test_gpu_decode import synth
seq, k, d = 20000, 1000, 64
q, K, V = synth(11, 1, 1, 1, 4, d, seq, seq, torch.float32)
qb = q[0, 0, 0:4].double().mean(0)
def run(Kf, dtype, label):
    rng = np.random.default_rng(5); perm = rng.permutation(seq)
    Kl = Kf.clone()
    Kl[perm[:800]] = (2 * qb).float(); Kl[perm[800:2800]] = qb.float()
    want = np.sort(np.concatenate([perm[:800], np.sort(perm[800:2800])[:200]]))
    K1 = Kl.reshape(1, 1, 1, seq, d).to(dtype)
    dec = P.HybridDecoder(n_layers=1, batch=1, n_kv_heads=1, group_size=4, d_head=d, seq_cap=seq,
                          roles=np.zeros((1, 1), np.uint8), policy=P.SparsityPolicy.top_k(k), dtype=dtype)
    dec.decode_step(q.to(dtype).cuda(), K1.cuda(), V.to(dtype).cuda(), seq)
    torch.cuda.synchronize()
    s0 = dec.token_sets()[0][0]
    print(label, "equal:", np.array_equal(s0, want), "n2", int(np.isin(s0, perm[:800]).sum()),
          "n1", int(np.isin(s0, perm[800:2800]).sum()), "len", len(s0))
run(torch.zeros(seq, d), torch.float32, "zeros fp32")
run(torch.randn(seq, d) * 1e-3, torch.float32, "tiny-random fp32")
run(torch.zeros(seq, d), torch.bfloat16, "zeros bf16")
run(-torch.ones(seq, d) * qb.float() * 0.5, torch.float32, "negative fp32")
