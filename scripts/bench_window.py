"""Cache-correction attention (csrc/window.cu) at Llama-3-8B shapes: W window
positions x 32 q heads against a 128K bf16 cache, one layer.  Prints us per
layer and the algorithmic K/V GB/s (every K/V row of the 8 heads read once)."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2602_04541_b200 as P  # noqa: E402

for W in (32, 64):
    L, B, H, G, d, cap = 1, 1, 8, 4, 128, 131072
    start = cap - W
    k = torch.empty((L, B, H, cap, d), dtype=torch.bfloat16, device="cuda").uniform_(-1, 1)
    v = torch.empty_like(k).uniform_(-1, 1)
    q = torch.empty((B, W, H * G, d), dtype=torch.bfloat16, device="cuda").uniform_(-1, 1)
    for _ in range(3):
        P.correction_attention(k, v, 0, q, start)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 20
    s.record()
    for _ in range(n):
        P.correction_attention(k, v, 0, q, start)
    e.record()
    torch.cuda.synchronize()
    us = s.elapsed_time(e) / n * 1e3
    gbs = 2 * B * H * cap * d * 2 / (us * 1e-6) / 1e9
    print(f"window W={W}: {us:.1f} us per layer, {gbs:.0f} GB/s of K/V, "
          f"{2 * 2 * B * H * G * W * cap * d / (us * 1e-6) / 1e12:.1f} TFLOP/s")
