"""Variable-length batches vs a uniform batch at Llama-3-8B shapes (32 layers,
32 q / 8 KV heads, d 128, bf16, 12.5 % retrieval heads, TopK).  Uniform lengths
and unequal lengths (lyc_decoder_step_varlen) both run the fused step kernel.
Prints us per step for: uniform (fused), uniform through the per-layer kernels
(lyc_decoder_layer loop), and a ragged batch (fused)."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2602_04541_b200 as P  # noqa: E402


def roles(NL, H, frac, seed=0):
    r = np.ones((NL, H), dtype=np.uint8)
    r[0] = 0
    rng = np.random.default_rng(seed)
    cells = [(l, g) for l in range(1, NL) for g in range(H)]
    n = int(round(frac * NL * H)) - H
    for i in rng.choice(len(cells), size=max(n, 0), replace=False):
        r[cells[i]] = 0
    return r


def timed(fn, n=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(n):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / n * 1e3


for B, cap, k in ((1, 131072, 4096), (16, 65536, 512)):
    NL, H, G, d = 32, 8, 4, 128
    rl = roles(NL, H, 0.125)
    K = torch.empty((NL, B, H, cap, d), dtype=torch.bfloat16, device="cuda").uniform_(-1, 1)
    V = torch.empty_like(K).uniform_(-1, 1)
    q = torch.empty((NL, B, H * G, d), dtype=torch.bfloat16, device="cuda").uniform_(-1, 1)
    out = torch.empty_like(q)
    mk = lambda: P.HybridDecoder(n_layers=NL, batch=B, n_kv_heads=H, group_size=G, d_head=d,  # noqa: E731
                                 seq_cap=cap, roles=rl, policy=P.SparsityPolicy.top_k(k),
                                 dtype=torch.bfloat16)
    dec = mk()
    t_fused = timed(lambda: dec.decode_step(q, K, V, cap, out))
    dec_l = mk()
    t_layer = timed(lambda: [dec_l.layer(l, q[l], K, V, cap, out[l]) for l in range(NL)])
    dec_v = mk()
    lens = [cap - (i * 997) % (cap // 2) for i in range(B)] if B > 1 else [cap - 1]
    t_var = timed(lambda: dec_v.decode_step(q, K, V, lens, out))
    tot = sum(lens)
    print(f"B={B} cap={cap} k={k}: uniform fused {t_fused:.1f} us, uniform per-layer "
          f"{t_layer:.1f} us, ragged fused {t_var:.1f} us "
          f"(ragged rows {tot / (B * cap):.2f} of uniform)")
    del K, V, dec, dec_l, dec_v
    torch.cuda.empty_cache()
