"""Per-layer timeline of one fused decode step (debug tool, run under gpurun).

    python scripts/step_timeline.py [--workload llama3-8b-128k] [--select tokens]

Prints, per layer, the retrieval-head count and (relative to the step start,
in microseconds): first consumer start, last consumer end (all attention
units done), merge done, selection barriers and selection done -- each the
max (or min for starts) over the CTAs.
"""
import argparse
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
import paper_2602_04541_b200 as P  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="llama3-8b-128k")
    ap.add_argument("--select", default="tokens")
    ap.add_argument("--layers", type=int, default=0)
    ap.add_argument("--save", default="")
    ap.add_argument("--top-k", type=int, default=0)
    ap.add_argument("--r-per-layer", type=int, default=-1)
    a = ap.parse_args()
    wl = dict(bench.WORKLOADS[a.workload])
    if a.layers:
        wl["NL"] = a.layers
    NL, H, G, d, L, k, B = (wl[x] for x in ("NL", "H", "G", "d", "L", "k", "B"))
    if a.top_k:
        k = a.top_k
    roles = bench.make_roles(NL, H, 0.125, 2602)
    if a.r_per_layer >= 0:
        rng = np.random.default_rng(2602)
        roles[1:] = 1
        for l in range(1, NL):
            roles[l, rng.choice(H, size=min(a.r_per_layer, H), replace=False)] = 0
    dt = torch.bfloat16 if wl["dtype"] == "bf16" else torch.float32
    K = torch.empty((NL, B, H, L, d), dtype=dt, device="cuda")
    V = torch.empty_like(K)
    for t in (K, V):
        for l in range(NL):
            t[l].uniform_(-1, 1)
    q = torch.empty((NL, B, H * G, d), dtype=dt, device="cuda").uniform_(-1, 1)
    dec = P.HybridDecoder(n_layers=NL, batch=B, n_kv_heads=H, group_size=G, d_head=d, seq_cap=L,
                          roles=roles, policy=P.SparsityPolicy.top_k(k), dtype=dt, select=a.select)
    assert dec.fused, "timeline needs the fused step kernel"

    for _ in range(3):
        out = dec.decode_step(q, K, V, L)
    dec.set_trace(True)
    out = dec.decode_step(q, K, V, L)
    torch.cuda.synchronize()
    tr = dec.trace().astype(np.int64)
    if a.save:
        np.save(a.save, tr)
    t0 = tr[0, 0].min()
    rel = (tr - t0) / 1e3
    # selection events in chronological order (max over CTAs; NaN = no selection)
    ev = [("cons_beg", 0, "min"), ("cons_end", 1, "max"), ("epi_wake", 2, "max"),
          ("merge", 3, "max"), ("c_prefix", 8, "max"), ("c_keys", 9, "max"),
          ("c_done", 10, "max"), ("r_wake", 12, "max"), ("r_loaded", 6, "max"),
          ("r_digit", 11, "max"), ("r_scan", 15, "max"), ("r_ranked", 4, "max"),
          ("e_scan", 14, "max"), ("e_done", 13, "max")]
    print(f"{'l':>3} {'R':>2} " + " ".join(f"{n:>9}" for n, _, _ in ev))
    for l in range(NL):
        nr = int((roles[l] == 0).sum()) if l else H
        vals = []
        for _, e, how in ev:
            x = tr[l, e]
            if how == "min":
                vals.append(rel[l, e].min())
            else:
                vals.append(rel[l, e].max() if x.max() > t0 else float("nan"))
        print(f"{l:3d} {nr:2d} " + " ".join(f"{v:9.1f}" for v in vals))
    print("step span us:", (tr.max() - t0) / 1e3)


if __name__ == "__main__":
    main()
