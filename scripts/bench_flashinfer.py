"""External full-attention bar: FlashInfer's single-request
decode attention over every layer's full cache (HND layout = ours), CUDA-graph
replayed, vs our same-GPU full attention.  Prints one JSON line (run under
gpurun; FlashInfer JIT-compiles its kernel on first use)."""
import json
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402

wl_name = sys.argv[1] if len(sys.argv) > 1 else "qwen3-8b-128k"
wl = dict(bench.WORKLOADS[wl_name])
NL, H, G, d, L = wl["NL"], wl["H"], wl["G"], wl["d"], wl["L"]
import flashinfer  # noqa: E402

K = torch.empty((NL, H, L, d), dtype=torch.bfloat16, device="cuda").uniform_(-1, 1)
V = torch.empty_like(K).uniform_(-1, 1)
q = torch.empty((NL, H * G, d), dtype=torch.bfloat16, device="cuda").uniform_(-1, 1)
out = torch.empty_like(q)
t0 = time.time()
for tc in (False, True):
    flashinfer.single_decode_with_kv_cache(q[0], K[0], V[0], kv_layout="HND", use_tensor_cores=tc)
torch.cuda.synchronize()
compile_s = time.time() - t0
res = {}
for tc in (False, True):
    def step():
        for l in range(NL):
            out[l] = flashinfer.single_decode_with_kv_cache(q[l], K[l], V[l], kv_layout="HND",
                                                            use_tensor_cores=tc)
    for _ in range(3):
        step()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        step()
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    res["tensor_cores" if tc else "cuda_cores"] = e0.elapsed_time(e1) / 20 * 1e3
bytes_ = 2 * NL * H * L * d * 2
best = min(res.values())
print(json.dumps({"workload": wl_name, "flashinfer": flashinfer.__version__,
                  "us_per_token": res, "best_us": best,
                  "hbm_gbs_best": bytes_ / best / 1e3, "jit_compile_s": compile_s}))
