"""Generate the golden fixtures of tests/golden/ from the REFERENCE itself.

Runs the unmodified reference headers (compiled in place into
oracle/_ref/libhh_ref.so by oracle/Makefile) on seeded inputs and stores
inputs + outputs as compressed npz.  The C restatement (oracle/liborc.so) and
the GPU path are checked against these files on machines without
/root/reference (the GPU box).

    python tests/golden/make_golden.py        # rewrites tests/golden/*.npz
"""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
from oracle import pyoracle  # noqa: E402

OUT = Path(__file__).resolve().parent


def main():
    pyoracle.build()
    ref = pyoracle.ref()
    if ref is None:
        raise SystemExit("oracle/_ref/libhh_ref.so missing: run make -C oracle with /root/reference present")
    rng = np.random.default_rng(20260214)

    # ---- args_top_k (attention.hpp:108-123), f64 and f32, with injected ties
    topk = {}
    for i in range(40):
        n = int(rng.integers(1, 3000))
        k = int(rng.integers(1, n + 5))
        w = rng.uniform(0, 1, n)
        if i % 3 == 0:
            w = np.round(w * 16) / 16  # heavy ties
        if i % 5 == 0 and n > 2:
            w[n // 2] = w[0]
        dt = np.float32 if i % 2 else np.float64
        w = w.astype(dt)
        topk[f"w{i}"] = w
        topk[f"k{i}"] = np.array(k)
        topk[f"out{i}"] = ref.args_top_k(w, k)
    np.savez_compressed(OUT / "args_top_k.npz", **topk)

    # ---- select_tokens (policy.hpp:64-104), all four kinds
    sel = {}
    for i in range(40):
        n = int(rng.integers(1, 500))
        w = rng.uniform(0, 1, n)
        w = w / w.sum()
        kind = ["topk", "topp", "threshold", "ratio"][i % 4]
        k = int(rng.integers(1, n + 3))
        value = {"topk": 0.0, "topp": float(rng.uniform(0.05, 1.0)),
                 "threshold": float(rng.uniform(0.1, 3.0)) / n, "ratio": float(rng.uniform(0.05, 0.95))}[kind]
        sel[f"w{i}"] = w
        sel[f"kind{i}"] = np.array(kind)
        sel[f"k{i}"] = np.array(k)
        sel[f"value{i}"] = np.array(value)
        sel[f"out{i}"] = ref.select_tokens(kind, w, k=k, value=value)
    np.savez_compressed(OUT / "select_tokens.npz", **sel)

    # ---- plan_splits + latency_model (kernel_sim.hpp:63-110, 284-316)
    plan = {}
    for i in range(30):
        B = int(rng.integers(1, 4))
        H = int(rng.integers(1, 9))
        hb = rng.integers(0, 40, size=(B, H))
        hb[:, 0] = np.maximum(hb[:, 0], 1)
        S = int(rng.integers(1, 12))
        units, sb, hsc = ref.plan_splits(hb, S)
        lm = ref.latency_model(hb, S, 4096)
        plan[f"hb{i}"] = hb
        plan[f"S{i}"] = np.array(S)
        plan[f"units{i}"] = units
        plan[f"sb{i}"] = sb
        plan[f"hsc{i}"] = hsc
        plan[f"lm_int{i}"] = np.array([lm[k] for k in ("total_blocks", "pooled_critical_blocks",
                                                        "naive_critical_blocks", "bytes_per_block",
                                                        "pooled_critical_bytes", "naive_critical_bytes")])
        plan[f"lm_f{i}"] = np.array([lm["mean_split_blocks"], lm["balance_ratio"]])
    np.savez_compressed(OUT / "plan_splits.npz", **plan)

    # ---- kernel::run<float> (kernel_sim.hpp:237-279), kernel_sim_test-style workloads
    run = {}
    for i in range(12):
        B = int(rng.integers(1, 3))
        H = int(rng.integers(1, 5))
        G = int(rng.integers(1, 5))
        d = 16
        seq = int(rng.integers(64, 700))
        bs = 64
        nb = (seq + bs - 1) // bs
        K = rng.uniform(-1, 1, (B * H, seq, d)).astype(np.float32)
        V = rng.uniform(-1, 1, (B * H, seq, d)).astype(np.float32)
        Q = rng.uniform(-1, 1, (B * H * G, d)).astype(np.float32)
        n_retr = int(rng.integers(0, H + 1))
        blocks = []
        for b in range(B):
            for g in range(H):
                if g < n_retr:
                    blocks.append(np.arange(nb))
                else:
                    keep = max(1, int(np.ceil(0.3 * nb)))
                    blocks.append(np.sort(rng.choice(nb, keep, replace=False)))
        S = int(rng.integers(1, 9))
        out, ec = ref.kernel_run(K, V, Q, blocks, batch=B, group=G, seq_len=seq, block_size=bs,
                                 scale=0.25, num_splits=S, dtype=np.float32, n_workers=2,
                                 exec_counts=True)
        off = np.zeros(len(blocks) + 1, dtype=np.int64)
        for j, bl in enumerate(blocks):
            off[j + 1] = off[j] + len(bl)
        run.update({f"K{i}": K, f"V{i}": V, f"Q{i}": Q, f"off{i}": off,
                    f"ids{i}": np.concatenate(blocks).astype(np.int64),
                    f"meta{i}": np.array([B, H, G, d, seq, bs, S]), f"out{i}": out, f"ec{i}": ec})
    np.savez_compressed(OUT / "kernel_run.npz", **run)

    # ---- decode_step attention loop (decode_engine.hpp:109-151), f64
    dec = {}
    for i in range(6):
        Lyr, H, G, d = 3, 2, 2, 8
        seq = int(rng.integers(10, 90))
        q = rng.uniform(-1, 1, (Lyr, H * G, d))
        K = rng.uniform(-1, 1, (Lyr, H, seq, d))
        V = rng.uniform(-1, 1, (Lyr, H, seq, d))
        roles = np.ones((Lyr, H), dtype=np.uint8)
        roles[0] = 0
        roles[int(rng.integers(1, Lyr)), int(rng.integers(0, H))] = 0
        kind = "topk" if i % 2 == 0 else "ratio"
        k = int(rng.integers(1, seq))
        value = 0.0 if kind == "topk" else float(rng.uniform(0.3, 0.9))
        r = ref.decode_step(q, K, V, roles, seq=seq, scale=1 / np.sqrt(d), kind=kind, k=k,
                            value=value, trace=True)
        dec.update({f"q{i}": q, f"K{i}": K, f"V{i}": V, f"roles{i}": roles,
                    f"kind{i}": np.array(kind), f"k{i}": np.array(k), f"value{i}": np.array(value),
                    f"seq{i}": np.array(seq), f"out{i}": r["out"]})
        for l in range(Lyr):
            for g in range(H):
                dec[f"trace{i}_{l}_{g}"] = r["trace"][l][g]
    np.savez_compressed(OUT / "decode_step.npz", **dec)
    print("wrote", sorted(p.name for p in OUT.glob("*.npz")))


if __name__ == "__main__":
    main()
