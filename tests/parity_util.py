"""Shared harness of the BASELINE-size parity tests (TEST INFRASTRUCTURE).

A whole decode step runs through the fused step kernel on the GPU with set
tracing on (every layer's emitted index sets are recorded, the StepTrace of
decode_engine.hpp:26-32, 144-147).  The oracle then replays the same step
layer by layer (oracle/hh_oracle.c orc_decode_layer_f32in, the f64
restatement of decode_engine.hpp:109-151) on host f32 copies of one
(layer, batch item) slab at a time, carrying its own sets_ forward.

Checked per (layer, batch item):
  * outputs: ||o_gpu - o_ref||_inf / max(||o_ref||_inf, 1e-3) <= 2e-2 (bf16),
    1e-5 (fp32) -- the north_star tolerances;
  * index sets of the retrieval heads: equal to the oracle's, except swaps
    confined to the fp tie band |s - s_(k)| <= 8e-6 * max|s| (the GPU ranks
    fp32 sums of per-head scores, the oracle f64 pooled-query weights);
    the swap count is returned.
"""
from __future__ import annotations

import numpy as np
import torch

BF16_TOL = 2e-2
FP32_TOL = 1e-5
TIE_BAND = 8e-6  # x max|s|: 2e-6 relative fp32 rounding of a 4-term sum


def rel_err(got, ref):
    got = np.asarray(got, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    return float(np.abs(got - ref).max() / max(np.abs(ref).max(), 1e-3))


def set_swaps(got, ref, scores, k):
    """0 when equal; otherwise every differing id must sit in the tie band
    around the k-th score; returns the number of swapped ids."""
    got, ref = set(np.asarray(got).tolist()), set(np.asarray(ref).tolist())
    assert len(got) == len(ref), (len(got), len(ref))
    if got == ref:
        return 0
    kth = np.sort(scores)[::-1][min(k, len(scores)) - 1]
    band = TIE_BAND * np.abs(scores).max()
    for t in got ^ ref:
        assert abs(scores[t] - kth) <= band, ("swap outside the tie band", t, scores[t], kth)
    return len(got - ref)


def make_inputs(NL, B, H, G, d, L, seq_cap, dtype, seed, dev="cuda"):
    """Seeded U(-1, 1) q / K / V generated on the device, one layer at a time."""
    gen = torch.Generator(device=dev).manual_seed(seed)
    K = torch.empty((NL, B, H, seq_cap, d), dtype=dtype, device=dev)
    V = torch.empty_like(K)
    for t in (K, V):
        for l in range(NL):
            t[l].uniform_(-1, 1, generator=gen)
    q = torch.empty((NL, B, H * G, d), dtype=dtype, device=dev).uniform_(-1, 1, generator=gen)
    return q, K, V


def run_and_check(orc, *, NL, B, H, G, d, L, k, roles, dtype=torch.bfloat16, seed=0,
                  select="tokens", policy=None, seq_cap=None, threads=0):
    """Fused GPU step vs the layer-by-layer oracle.  Returns a report dict
    (max rel err, swaps, rows checked)."""
    import paper_2602_04541_b200 as P
    from oracle import pyoracle
    seq_cap = seq_cap or L
    policy = policy or P.SparsityPolicy.top_k(k)
    q, K, V = make_inputs(NL, B, H, G, d, L, seq_cap, dtype, seed)
    dec = P.HybridDecoder(n_layers=NL, batch=B, n_kv_heads=H, group_size=G, d_head=d,
                          seq_cap=seq_cap, roles=roles, policy=policy, dtype=dtype, select=select)
    assert dec.fused, "the BASELINE configs must run on the fused step kernel"
    import os
    if os.environ.get("LYC_TEST_NO_PDL"):
        dec.tune(P._lib.TUNE_PDL, 0)
    dec.set_trace_sets(True)
    out = dec.decode_step(q, K, V, L)
    torch.cuda.synchronize()
    ids, cnt = dec.traced_sets()
    final = dec.token_sets()
    out_h = out.float().cpu().numpy()
    tol = BF16_TOL if dtype == torch.bfloat16 else FP32_TOL
    scale = 1 / np.sqrt(d)
    kind, kk, val = policy.kind, policy.k, policy.value
    worst, swaps, rows = 0.0, 0, 0
    for b in range(B):
        st = pyoracle.LayerState(H, L)
        for l in range(NL):
            ql = q[l, b].float().cpu().numpy()
            Kl = K[l, b, :, :L].float().cpu().numpy()
            Vl = V[l, b, :, :L].float().cpu().numpy()
            ref, ps = orc.decode_layer(ql, Kl, Vl, roles[l], st, layer0=(l == 0), seq=L,
                                       scale=scale, kind=kind, k=kk, value=val,
                                       pooled_scores=True, threads=threads)
            e = rel_err(out_h[l, b], ref)
            worst = max(worst, e)
            if e > tol:  # diagnose: per-head errors, roles, the GPU set vs the oracle's
                G_ = H and out_h.shape[2] // H
                per = [round(rel_err(out_h[l, b, g * G_:(g + 1) * G_], ref[g * G_:(g + 1) * G_]), 4)
                       for g in range(H)]
                info = {"layer": l, "item": b, "err": e, "per_head": per,
                        "roles": roles[l].tolist(),
                        "set_sizes_gpu": [int(cnt[l, b * H + g]) for g in range(H)],
                        "set_sizes_ref": st.len.tolist()}
                raise AssertionError(f"rel err {e:.3e} > {tol}: {info}")
            for g in range(H):
                if l == 0 or roles[l, g] == 0:
                    r = b * H + g
                    n = int(cnt[l, r])
                    assert n == st.len[g], (l, b, g, n, st.len[g])
                    got = ids[l, r, :n]
                    assert np.all(np.diff(got) > 0), "set not strictly ascending"
                    swaps += set_swaps(got, st.set(g), ps[g], int(st.len[g]))
                    rows += 1
        for g in range(H):  # the final index cache (sets_ after the step)
            assert len(final[b][g]) == st.len[g]
    dec.close()
    return {"max_rel_err": worst, "swaps": swaps, "rows_checked": rows}


def roles_with(NL, H, retrieval):
    """Layer 0 all Retrieval; (l, g) pairs of `retrieval` above it."""
    r = np.ones((NL, H), dtype=np.uint8)
    r[0] = 0
    for (l, g) in retrieval:
        r[l, g] = 0
    return r
