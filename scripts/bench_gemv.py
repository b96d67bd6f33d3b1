"""lyc_gemv (csrc/model.cu) at the toy model's Qwen3-8B / Llama-3-8B shapes:
us per launch and weight GB/s, back-to-back launches of ONE matrix (run under
gpurun).  Matrices below the 126 MB L2 are then served from L2: this measures
the kernel, not the model's HBM stream -- scripts/bench_gemv_chain.py times
the model's chain with distinct weights per layer."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2602_04541_b200 import _lib as LL  # noqa: E402
from paper_2602_04541_b200.model import gemv  # noqa: E402

SHAPES = [("qkv", 6144, 4096, LL.GEMV_STORE), ("o", 4096, 4096, LL.GEMV_RESIDUAL),
          ("w1", 12288, 4096, LL.GEMV_SILU_BF16), ("w2", 4096, 12288, LL.GEMV_RESIDUAL),
          ("lm", 151936, 4096, LL.GEMV_STORE)]
for name, M, K, mode in SHAPES:
    w = torch.randn((M, K), device="cuda").bfloat16()
    x = torch.randn(K, device="cuda")
    gain = torch.ones(K, device="cuda")
    y = torch.zeros(M, device="cuda")
    yb = torch.empty(M, dtype=torch.bfloat16, device="cuda")
    kw = dict(mode=mode, y=y, yb=yb)
    if mode == LL.GEMV_RESIDUAL:
        kw.update(xb=x.bfloat16())
    else:
        kw.update(x=x, gain=gain)
    for _ in range(3):
        gemv(w, **kw)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(20):
            gemv(w, **kw)
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / 100 * 1e3
    print(f"{name:4s} M={M:6d} K={K:5d}: {us:7.1f} us, {M * K * 2 / us / 1e3:6.0f} GB/s")
