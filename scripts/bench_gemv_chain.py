"""The toy model's GEMV chain alone (qwen3-8b shapes: per layer W_qkv with
rotary + cache append, W_o + residual, W_1 + silu, W_2 + residual; then the
logits), distinct weights per layer as in the model, one CUDA graph per
token: us per token and weight GB/s (run under gpurun)."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2602_04541_b200 import _lib as LL  # noqa: E402
from paper_2602_04541_b200 import SparsityPolicy  # noqa: E402
from paper_2602_04541_b200.model import PRESETS, DecodeModel, ModelConfig, gemv  # noqa: E402
import numpy as np  # noqa: E402

L = 4096
cfg = ModelConfig(max_seq_len=L, **PRESETS["qwen3-8b"])
roles = np.zeros((cfg.n_layers, cfg.n_kv_heads), np.uint8)
m = DecodeModel(cfg, roles=roles, policy=SparsityPolicy.top_k(256), attention="full", seed=1)
NL, d, H, nq, cap = cfg.n_layers, cfg.d_head, cfg.n_kv_heads, cfg.n_q_heads, cfg.max_seq_len
pos = L - 1
st = torch.cuda.Stream()


PF = int(sys.argv[1]) if len(sys.argv) > 1 else 0  # 0: no prefetch, -1: whole next matrix, else bytes


def chain(which):
    seq = []
    for l in range(NL):
        for n in ("qkv", "o", "w1", "w2"):
            if n in which:
                seq.append((n, l))
    wt = {"qkv": m.wqkv, "o": m.wo, "w1": m.w1, "w2": m.w2}
    for i, (n, l) in enumerate(seq):
        pf = {"next_is_gemv": i + 1 < len(seq)}
        if PF and i + 1 < len(seq):
            nw = wt[seq[i + 1][0]][seq[i + 1][1]]
            pf.update(prefetch=nw, prefetch_bytes=0 if PF < 0 else min(PF, nw.numel() * 2))
        if n == "qkv":
            gemv(m.wqkv[l], x=m.x, gain=m.attn_norm[l], mode=LL.GEMV_QKV_ROPE, q_out=m.q[l],
                 k_cache=m.k[l, 0], v_cache=m.v[l, 0], slab_stride=cap * d, nq=nq, nkv=H, d=d,
                 pos=pos, stream=st, **pf)
        elif n == "o":
            gemv(m.wo[l], xb=m.o[l].view(-1), mode=LL.GEMV_RESIDUAL, y=m.x, stream=st, **pf)
        elif n == "w1":
            gemv(m.w1[l], x=m.x, gain=m.ffn_norm[l], mode=LL.GEMV_SILU_BF16, yb=m.mid, stream=st,
                 **pf)
        else:
            gemv(m.w2[l], xb=m.mid, mode=LL.GEMV_RESIDUAL, y=m.x, stream=st, **pf)


m.x.fill_(0.5)
m.o.fill_(0.1)
for which, wts in ((("qkv", "o", "w1", "w2"), None), (("qkv",), "wqkv"), (("o",), "wo"),
                   (("w1",), "w1"), (("w2",), "w2")):
    with torch.cuda.stream(st):
        chain(which)
    st.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st):
        chain(which)
    with torch.cuda.stream(st):
        for _ in range(3):
            g.replay()
    st.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(st):
        e0.record(st)
        for _ in range(10):
            g.replay()
        e1.record(st)
    e1.synchronize()
    us = e0.elapsed_time(e1) / 10 * 1e3
    names = [wts] if wts else ["wqkv", "wo", "w1", "w2"]
    nbytes = sum(t.numel() * 2 for n in names for t in getattr(m, n))
    print(f"pf={PF} {'+'.join(which):14s}: {us:8.1f} us/token, {us / NL / len(which):6.1f} us/launch, "
          f"{nbytes / us / 1e3:6.0f} GB/s")
