"""One decode token of the toy model at Qwen3-8B shapes (131072 context),
eager, for an ncu launch list (debug, run under gpurun):
  ncu --metrics gpu__time_duration.sum --clock-control none --csv \\
      --log-file gpurun_out/model_launches.csv python scripts/model_launches.py"""
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
from paper_2602_04541_b200 import SparsityPolicy  # noqa: E402
from paper_2602_04541_b200.model import PRESETS, DecodeModel, ModelConfig  # noqa: E402

L = int(sys.argv[1]) if len(sys.argv) > 1 else 131072
cfg = ModelConfig(max_seq_len=L, **PRESETS["qwen3-8b"])
roles = bench.make_roles(cfg.n_layers, cfg.n_kv_heads, 0.125, 2602)
m = DecodeModel(cfg, roles=roles, policy=SparsityPolicy.top_k(4096), attention="hybrid", seed=1)
m.k.uniform_(-1, 1)
m.v.uniform_(-1, 1)
for _ in range(2):
    m.decode_token(7, L - 1)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
m.decode_token(7, L - 1)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print("weights GB", m.weight_bytes() / 1e9)
