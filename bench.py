"""Benchmark of the B200 hybrid-head decode attention (one JSON line on rank 0).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload llama3-8b-128k|llama3-8b-32k|qwen3-8b-128k|llama3-8b-64k-b16|tiny]
                    [--select tokens|blocks]

A STEP is one decode step of hybrid-head attention over ALL layers
(decode_engine.hpp:109-151): per layer the retrieval heads' dense split-KV
attention with the fused pooled-query scoring, the sparse heads' attention over
the index sets of earlier layers, the split-KV merge and the top-k selection
into the per-head index cache -- one launch of the persistent step kernel,
CUDA-graph replayed.  Default workload: BASELINE's 128K single-GPU config
(Qwen3-8B shapes, 36 layers).  Inputs (q, K/V caches, 19 GiB at 128K) are
resident in HBM and far larger than the 126 MB L2, so no flush is needed.

value     : device time per decode step in us (= us/token at batch 1), max over
            ranks, CUDA events around exactly K replays.
e2e       : token after token through the public C-ABI call
            (HybridDecoder.decode_step, eager): every step uploads q of every
            layer + the new token's K/V rows from pinned host memory, appends
            the rows at the growing length (lyc_kv_write), runs the step at
            seq = t + 1 (device-side re-plan, no host sync) and copies the
            outputs back, all inside the timed region.
roofline  : dominant kernel = hybrid_step_kernel (the whole step); achieved =
            algorithmic bytes (K/V rows touched + q + out + index reads,
            SURVEY.md 8(d)) / its CUDA-event duration on the launching stream.
per_layer_api : the same step through lyc_decoder_layer (one launch per layer,
            the entry a model calls between its own projections).
selection_swaps : the step kernel's per-layer sets vs an exact f64 top-k.
cpu_baseline / --impl reference : the reference's own CPU path (oracle/_ref,
            the unmodified reference headers compiled here): hh::kernel::run<float>
            for every layer with std::thread workers on all host cores, plus the
            f64 selection pass of every retrieval head -- whole steps, timed.
Multi-GPU (torchrun): KV heads are sharded across ranks (index propagation is
per head index, so the attention needs no collective); the headline for N > 1
keeps the model's per-layer dependency -- one lyc_decoder_layer launch and one
all-gather of the layer's [B][Hq][d] outputs per layer, max over ranks.
--shard seq: KV-sequence sharding with one packed NCCL all-gather of
partials + top-k candidates per layer.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "decode attention us/token at 128K (1/2/4/8 B200); achieved HBM GB/s vs peak"

WORKLOADS = {
    # name: (layers, kv heads, group, d, context, top-k, batch, dtype)
    "llama3-8b-128k": dict(NL=32, H=8, G=4, d=128, L=131072, k=4096, B=1, dtype="bf16"),
    "llama3-8b-32k": dict(NL=32, H=8, G=4, d=128, L=32768, k=2048, B=1, dtype="bf16"),
    "qwen3-8b-128k": dict(NL=36, H=8, G=4, d=128, L=131072, k=4096, B=1, dtype="bf16"),
    "llama3-8b-64k-b16": dict(NL=32, H=8, G=4, d=128, L=65536, k=2048, B=16, dtype="bf16"),
    "llama3-8b-256k-b4": dict(NL=32, H=8, G=4, d=128, L=262144, k=2048, B=4, dtype="bf16"),
    "tiny": dict(NL=4, H=2, G=4, d=64, L=4096, k=256, B=1, dtype="f32"),
}


def make_roles(NL, H, frac, seed):
    """Layer 0 all retrieval (decode_engine.hpp:121); above it a seeded choice
    of retrieval heads so that frac of all (layer, head) slots are retrieval
    (12.5 % = 32/256 on Llama-3-8B)."""
    roles = np.ones((NL, H), dtype=np.uint8)
    roles[0] = 0
    n_extra = max(0, int(round(frac * NL * H)) - H)
    rng = np.random.default_rng(seed)
    slots = rng.choice((NL - 1) * H, size=min(n_extra, (NL - 1) * H), replace=False)
    for s in slots:
        roles[1 + s // H, s % H] = 0
    return roles


def shard_heads(roles, L, k, world, rank):
    """Assign KV heads to ranks, balancing per-token rows (LPT greedy)."""
    NL, H = roles.shape
    work = [sum(L if roles[l, g] == 0 else min(k, L) for l in range(NL)) for g in range(H)]
    load = [0] * world
    owner = [0] * H
    for g in sorted(range(H), key=lambda g: -work[g]):
        r = min(range(world), key=lambda r: load[r])
        owner[g] = r
        load[r] += work[g]
    return [g for g in range(H) if owner[g] == rank]


class ClockSampler:
    """NVML sampling of SM clock and throttle reasons during the timed region."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
        0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
        0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
        0x100: "display_clock_setting",
    }

    def __init__(self, index):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None
        self.t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit and bit != 0x1:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.02)

    def __enter__(self):
        if self.nv:
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.nv:
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["nvml unavailable"]}
        return {"sm_mhz": float(np.median(self.samples)), "sm_max_mhz": self.max_mhz,
                "samples": len(self.samples), "reasons": sorted(self.reasons)}


def ncu_traffic(workload):
    """dram read+write bytes per launch of the step kernel from the committed
    `ncu --set full` capture (profiles/ncu_traffic.json), or None."""
    try:
        t = json.loads((ROOT / "profiles" / "ncu_traffic.json").read_text())[workload]
        return float(t["dram_bytes_read"] + t["dram_bytes_write"])
    except Exception:
        return None


def peaks():
    try:
        return json.loads((ROOT / "MEASURED_PEAKS.json").read_text()), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}, "fallback (B200_PROFILING.md)"


# ----------------------------------------------------------------------- CPU
def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


class CpuStep:
    """The reference CPU path for one decode step of the workload, every layer
    executed (oracle/ref_shim.cpp ref_step_run over the unmodified reference
    headers): per layer hh::kernel::run<float> (kernel_sim.hpp:237-279) with
    the reference's own std::thread pool over the layer's block lists
    (retrieval heads: all ceil(L/64) blocks; sparse heads: a seeded
    ceil(k/64)-block subset, the same rows as their k-token sets), then the
    serial f64 selection pass of every retrieval head (gqa_pool_queries +
    dense_attention weights + select_tokens TopK, decode_engine.hpp:129-132).
    One layer's K/V (batch item 0) is built once and reused for every layer:
    the CPU time does not depend on the values.  Batch items are independent,
    so a batch-B step costs B batch-1 steps (us/token = the batch-1 step)."""

    def __init__(self, wl, roles, K=None, V=None, q=None, seed=7):
        from oracle import pyoracle
        self.o = pyoracle.ref()
        if self.o is None:
            raise RuntimeError("oracle/_ref (the reference compiled here) is missing")
        self.kind = "reference"
        NL, H, G, d, L, k = (wl[x] for x in ("NL", "H", "G", "d", "L", "k"))
        self.wl, self.roles = wl, roles
        rng = np.random.default_rng(seed)
        if K is None:
            K = rng.uniform(-1, 1, (H, L, d)).astype(np.float32)
            V = rng.uniform(-1, 1, (H, L, d)).astype(np.float32)
            q = rng.uniform(-1, 1, (H * G, d)).astype(np.float32)
        self.ctx = self.o.step_context(K, V, q, group=G, scale=1 / np.sqrt(d))
        nb = (L + 63) // 64
        self.nb, self.nblk = nb, min((k + 63) // 64, nb)
        self.blocks = [[np.arange(nb) if (l == 0 or roles[l, g] == 0)
                        else np.sort(rng.choice(nb, self.nblk, replace=False)) for g in range(H)]
                       for l in range(NL)]
        self.cores = os.cpu_count() or 1
        self.splits = 16 * H

    def step(self, workers=None):
        """-> (seconds, attention seconds, selection seconds) of one step."""
        return self.ctx.run(self.roles, self.blocks, num_splits=self.splits,
                            n_workers=workers or self.cores, top_k=min(self.wl["k"], self.wl["L"]))

    def thread_scaling(self):
        """kernel::run time of one hybrid layer (1 retrieval + H-1 sparse heads)
        at 1, 2, 4, ... workers (ms)."""
        H = self.wl["H"]
        r = np.ones((1, H), np.uint8)
        r[0, 0] = 0
        blk = [[np.arange(self.nb)] + [self.blocks[-1][g] if self.roles[-1, g] else
                                       np.arange(self.nblk) for g in range(1, H)]]
        out, w = {}, 1
        while True:
            _, ta, _ = self.ctx.run(r, blk, num_splits=self.splits, n_workers=w,
                                    top_k=min(self.wl["k"], self.wl["L"]))
            out[str(w)] = round(ta * 1e3, 2)
            if w >= self.cores:
                break
            w = min(2 * w, self.cores)
        return out

    def sample(self, nsteps, t_step, t_attn, t_sel):
        wl = self.wl
        nret = int(sum(1 for l in range(wl["NL"]) for g in range(wl["H"])
                       if l == 0 or self.roles[l, g] == 0))
        return (f"{nsteps} whole decode step(s) of the reference CPU path, all {wl['NL']} layers "
                f"executed: per layer hh::kernel::run<float> over H={wl['H']} heads "
                f"(retrieval {self.nb} blocks, sparse {self.nblk} blocks), {self.splits} splits, "
                f"{self.cores} std::thread workers ({t_attn * 1e3:.0f} ms/step); plus the serial f64 "
                f"selection pass of each of the {nret} retrieval (layer, head) slots "
                f"({t_sel * 1e3:.0f} ms/step); L={wl['L']}, d={wl['d']}, G={wl['G']}, batch 1 "
                f"(a batch-{wl['B']} step = {wl['B']} independent batch-1 steps)")

    def close(self):
        self.ctx.close()


def run_reference_arm(args, wl, roles, rank, world):
    if rank != 0:
        return
    cs = CpuStep(wl, roles)
    for _ in range(args.warmup):
        cs.step()
    vals, ta, tsel = [], [], []
    t0 = time.perf_counter()
    for _ in range(args.steps):
        sec, a, sl = cs.step()
        vals.append(sec)
        ta.append(a)
        tsel.append(sl)
    wall = time.perf_counter() - t0
    v = float(np.mean(vals)) * 1e6  # us per step of one batch item = us/token
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "us/token",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": v / 1e3 * wl["B"], "higher_is_better": False, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32 (selection f64)", "data": "synthetic U(-1,1)",
        "config": config_of(args, wl),
        "cpu_baseline": {"value": v, "unit": "us/token", "kind": cs.kind, "cores": cs.cores,
                         "cpu_model": cpu_model(),
                         "sample": cs.sample(args.steps, np.mean(vals), np.mean(ta), np.mean(tsel)),
                         "thread_scaling_layer_ms": cs.thread_scaling()},
        "e2e": {"value": v, "unit": "us/token", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "timed_s": float(np.sum(vals)), "wall_s": wall,
    }
    cs.close()
    print(json.dumps(line), flush=True)


def selection_swaps(dec, q, K, V, L, wl, roles, stream):
    """Per-layer index sets of one traced step vs the exact top-k of f64
    pooled-query scores (numpy; ties to the lower index).  Returns the swap
    count, and how many differing ids sit outside the fp tie band
    |s - s_(k)| <= 8e-6 max|s| (must be 0)."""
    import torch
    NL, H, G, k = wl["NL"], roles.shape[1], wl["G"], min(wl["k"], L)
    B = q.shape[1]
    dec.set_trace_sets(True)
    with torch.cuda.stream(stream):
        dec.decode_step(q, K, V, L, stream=stream)
    stream.synchronize()
    ids, cnt = dec.traced_sets()
    dec.set_trace_sets(False)
    swaps = out_band = rows = 0
    for l in range(NL):
        for g in range(H):
            if not (l == 0 or roles[l, g] == 0):
                continue
            for b in range(B):
                r = b * H + g
                got = ids[l, r, :cnt[l, r]]
                pq = q[l, b, g * G:(g + 1) * G].double().sum(0) / G
                s_ = (K[l, b, g, :L].double() @ pq).cpu().numpy()
                order = np.lexsort((np.arange(L), -s_))
                ref = np.sort(order[:k])
                rows += 1
                if got.shape[0] != k or not np.array_equal(got, ref):
                    diff = np.setxor1d(got, ref)
                    swaps += len(np.setdiff1d(got, ref))
                    kth = s_[order[k - 1]]
                    out_band += int(np.sum(np.abs(s_[diff] - kth) > 8e-6 * np.abs(s_).max()))
    return {"count": int(swaps), "outside_tie_band": int(out_band), "rows_checked": rows,
            "method": "sets emitted by the step kernel (set trace) vs numpy exact top-k of f64 "
                      "pooled scores, ties to the lower index"}


def config_of(args, wl):
    c = {"workload": args.workload, "layers": wl["NL"], "q_heads": wl["H"] * wl["G"],
         "kv_heads": wl["H"], "head_dim": wl["d"], "context": wl["L"], "top_k": wl["k"],
         "batch": wl["B"], "retrieval_fraction": args.retrieval_frac, "select": args.select,
         "parallelism": (f"{args.shard}-sharded x{args.gpus}" if args.gpus > 1 else "single GPU"),
         "l2": "inputs larger than L2 (KV caches >> 126 MB), no flush"}
    return c


# ----------------------------------------------------------------------- GPU
def run_seq_sharded(args, wl, roles, rank, world, local):
    """KV-sequence sharding: every rank holds L/N rows of every
    head; per layer one packed NCCL all-gather of [partials | top-k candidates]
    (paper_2602_04541_b200/sharded.py).  Total work fixed: strong scaling."""
    import torch
    import torch.distributed as dist
    import paper_2602_04541_b200 as P
    from paper_2602_04541_b200.sharded import ShardedDecoder, shard_rows
    NL, H, G, d, L, k, B = (wl[x] for x in ("NL", "H", "G", "d", "L", "k", "B"))
    dev = torch.device("cuda", local)
    dt = torch.bfloat16 if wl["dtype"] == "bf16" else torch.float32
    rb, nl = shard_rows(L, world, rank)
    gen = torch.Generator(device=dev).manual_seed(args.seed + 17 * rank)
    K = torch.empty((NL, B, H, nl, d), dtype=dt, device=dev)
    V = torch.empty_like(K)
    for t in (K, V):
        for l in range(NL):
            t[l].uniform_(-1, 1, generator=gen)
    qgen = torch.Generator(device=dev).manual_seed(args.seed)  # q identical on every rank
    q = torch.empty((NL, B, H * G, d), dtype=dt, device=dev).uniform_(-1, 1, generator=qgen)
    out = torch.empty_like(q)
    sd = ShardedDecoder(n_layers=NL, batch=B, n_kv_heads=H, group_size=G, d_head=d, seq_cap=nl,
                        roles=roles, policy=P.SparsityPolicy.top_k(k), dtype=dt, world=world,
                        rank=rank)
    for _ in range(args.warmup):
        sd.decode_step(q, K, V, nl, rb, L, out)
    torch.cuda.synchronize()
    dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        e0.record()
        for _ in range(args.steps):
            sd.decode_step(q, K, V, nl, rb, L, out)
        e1.record()
        e1.synchronize()
    torch.cuda.synchronize()
    dist.barrier()
    t = torch.tensor([e0.elapsed_time(e1) / args.steps], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    # algorithmic bytes of the whole job per step (all ranks): K/V rows touched + q/out
    e = 2 if dt == torch.bfloat16 else 4
    kb = min(k, L)
    rows = sum(L if (l == 0 or roles[l, g] == 0) else kb for l in range(NL) for g in range(H))
    job_bytes = B * rows * 2 * d * e + NL * B * H * G * d * e * 2
    if rank == 0:
        pk, pk_kind = peaks()
        achieved = job_bytes / (ms / 1e3) / 1e9 / world  # per GPU
        line = {
            "metric": METRIC, "value": ms * 1e3 / B, "unit": "us/token", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": False, "scaling": "strong", "vs_baseline": None,
            "dtype": wl["dtype"], "data": "synthetic U(-1,1) q/K/V, seeded roles",
            "config": config_of(args, wl), "tokens_per_s": B / (ms / 1e3),
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": float(pk["hbm_gbs"]),
                         "unit": "GB/s", "frac": achieved / float(pk["hbm_gbs"]),
                         "traffic": None, "peak_kind": pk_kind,
                         "kernel": "per-layer attention + merge + top-k + packed NCCL all-gather"},
            "cpu_baseline": None,
            "e2e": None,
            "gpu_launches": int(args.steps * NL * 6),
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    sd.close()
    dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="qwen3-8b-128k", choices=list(WORKLOADS))
    ap.add_argument("--select", default="tokens", choices=["tokens", "blocks"])
    ap.add_argument("--retrieval-frac", type=float, default=0.125)
    ap.add_argument("--r-per-layer", type=int, default=-1,
                    help="(diagnostic) exactly this many seeded retrieval heads in every layer "
                         "above 0, instead of --retrieval-frac")
    ap.add_argument("--top-k", type=int, default=0, help="override the workload's top-k budget")
    ap.add_argument("--seed", type=int, default=2602)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-full", action="store_true")
    ap.add_argument("--no-swaps", action="store_true")
    ap.add_argument("--no-sweep", action="store_true",
                    help="skip the 25 %% / 50 %% retrieval-fraction points (BASELINE config 3)")
    ap.add_argument("--no-flashinfer", action="store_true",
                    help="skip the external full-attention bar (FlashInfer decode)")
    ap.add_argument("--no-model", action="store_true",
                    help="skip the end-to-end toy-model TPOT (hybrid vs full attention)")
    ap.add_argument("--no-pdl", action="store_true",
                    help="plain stream serialisation of the planner / step launches")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="process-group backend for N > 1 (gloo: host-staged, for checking the "
                         "multi-rank code path with several ranks on one GPU)")
    ap.add_argument("--shard", default="heads", choices=["heads", "seq"],
                    help="multi-GPU split: KV heads (no collective) or KV sequence "
                         "(one packed NCCL all-gather of partials + top-k candidates per layer)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    wl = dict(WORKLOADS[args.workload])
    if args.top_k:
        wl["k"] = args.top_k
    roles = make_roles(wl["NL"], wl["H"], args.retrieval_frac, args.seed)
    if args.r_per_layer >= 0:
        rng = np.random.default_rng(args.seed)
        roles[1:] = 1
        for l in range(1, wl["NL"]):
            roles[l, rng.choice(wl["H"], size=min(args.r_per_layer, wl["H"]), replace=False)] = 0

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference_arm(args, wl, roles, rank, world)
        return

    import torch
    import torch.distributed as dist

    # one rank per GPU; ranks beyond the visible GPUs share them (a protocol
    # check of the multi-rank code path with --dist-backend gloo on one GPU)
    local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    if world > 1:
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group("gloo")
    import paper_2602_04541_b200 as P

    if world > 1 and args.shard == "seq":
        run_seq_sharded(args, wl, roles, rank, world, local)
        return
    NL, H, G, d, L, k, B = (wl[x] for x in ("NL", "H", "G", "d", "L", "k", "B"))
    my_heads = shard_heads(roles, L, k, world, rank) if world > 1 else list(range(H))
    Hr = len(my_heads)
    r_roles = np.ascontiguousarray(roles[:, my_heads])
    dt = torch.bfloat16 if wl["dtype"] == "bf16" else torch.float32
    esz = 2 if dt == torch.bfloat16 else 4
    seq_cap = L
    dev = torch.device("cuda", local)
    gen = torch.Generator(device=dev).manual_seed(args.seed + rank)
    K = torch.empty((NL, B, Hr, seq_cap, d), dtype=dt, device=dev)
    V = torch.empty_like(K)
    for t in (K, V):
        for l in range(NL):
            t[l].uniform_(-1, 1, generator=gen)
    q = torch.empty((NL, B, Hr * G, d), dtype=dt, device=dev).uniform_(-1, 1, generator=gen)
    out = torch.empty_like(q)
    stream = torch.cuda.Stream(device=dev)
    pol = P.SparsityPolicy.top_k(k)
    dec = P.HybridDecoder(n_layers=NL, batch=B, n_kv_heads=Hr, group_size=G, d_head=d,
                          seq_cap=seq_cap, roles=r_roles, policy=pol, dtype=dt, select=args.select)
    if args.no_pdl:
        dec.tune(P._lib.TUNE_PDL, 0)

    def barrier():
        if world > 1:
            dist.barrier()

    def allmax(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64,
                         device=dev if args.dist_backend == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def time_graph(dd, steps, warm):
        with torch.cuda.stream(stream):
            for _ in range(warm):
                dd.replay(stream=stream)
        stream.synchronize()
        barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            e0.record(stream)
            for _ in range(steps):
                dd.replay(stream=stream)
            e1.record(stream)
        e1.synchronize()
        torch.cuda.synchronize()
        barrier()
        return e0.elapsed_time(e1) / steps  # ms per step

    # ---- headline: graph-replayed decode steps
    with torch.cuda.stream(stream):
        dec.capture(q, K, V, L, out, stream=stream)
    launches_per_step = dec.launches_per_step(L)
    fused = dec.fused
    lc0 = P.lib().lyc_launch_count()
    with ClockSampler(local) as clk:
        ms = time_graph(dec, args.steps, args.warmup)
        # keep the GPU busy >= ~1 s so the sampler sees the loaded clock
        t_end = time.time() + max(0.0, 1.0 - ms * args.steps / 1e3)
        with torch.cuda.stream(stream):
            while time.time() < t_end:
                for _ in range(20):
                    dec.replay(stream=stream)
                stream.synchronize()
    launched = P.lib().lyc_launch_count() - lc0
    ms = allmax(ms)
    step_us = ms * 1e3
    step_bytes = dec.step_bytes(L)

    # ---- N > 1, head sharding with the model's per-layer dependency: the
    # o-projection of layer l needs every head's output, so each layer is one
    # lyc_decoder_layer launch followed by an all-gather of the [B][Hq][d]
    # outputs of all ranks (decode_engine.hpp:149-150); layer l+1 starts after
    # it.  The critical path is sum_l max_p work(l, p).  This is the headline
    # for N > 1; the independent whole-step time is reported beside it.
    layer_sync = None
    head_ms = ms  # the headline step time (N > 1: the layer-synchronous step)
    if world > 1:
        hmax = max(len(shard_heads(roles, L, k, world, r)) for r in range(world))
        send = torch.zeros((B, hmax * G, d), dtype=dt, device=dev)
        out_s = torch.empty_like(q)
        staged = args.dist_backend != "nccl"
        gath = torch.empty((world * B, hmax * G, d), dtype=dt,
                           device="cpu" if staged else dev)

        def sync_step():
            for l in range(NL):
                dec.layer(l, q[l], K, V, L, out_s[l], stream=stream)
                send[:, :Hr * G].copy_(out_s[l])
                if staged:
                    stream.synchronize()
                    dist.all_gather_into_tensor(gath, send.cpu())
                else:
                    dist.all_gather_into_tensor(gath, send)

        with torch.cuda.stream(stream):
            for _ in range(args.warmup):
                sync_step()
        torch.cuda.synchronize()
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            e0.record(stream)
            for _ in range(args.steps):
                sync_step()
            e1.record(stream)
        e1.synchronize()
        torch.cuda.synchronize()
        barrier()
        sync_ms = allmax(e0.elapsed_time(e1) / args.steps)
        layer_sync = {"us_per_token": sync_ms * 1e3 / B, "ms_per_step": sync_ms,
                      "fused_independent_us_per_token": step_us / B,
                      "collective": f"all_gather of [B][Hq][d] per layer ({args.dist_backend})",
                      "heads_per_rank": Hr, "launches_per_step": NL}
        head_ms = sync_ms

    # ---- roofline of the dominant kernel (attention), events inside the graph
    dec.set_timing(True)
    with torch.cuda.stream(stream):
        dec.capture(q, K, V, L, out, stream=stream)
        for _ in range(args.warmup):
            dec.replay(stream=stream)
    stream.synchronize()
    per_layer = np.zeros(NL)
    for _ in range(args.steps):
        with torch.cuda.stream(stream):
            dec.replay(stream=stream)
        per_layer += dec.attn_ms()
    per_layer /= args.steps
    attn_bytes = np.array([dec.layer_attn_bytes(l, L) for l in range(NL)], dtype=np.float64)
    attn_ms_total = float(per_layer.sum())
    achieved = attn_bytes.sum() / (attn_ms_total / 1e3) / 1e9
    dec.set_timing(False)
    pk, pk_kind = peaks()
    peak = float(pk["hbm_gbs"])

    # ---- same-GPU full-attention decode (every head dense, no selection)
    full = None
    if not args.no_full:
        fdec = P.HybridDecoder(n_layers=NL, batch=B, n_kv_heads=Hr, group_size=G, d_head=d,
                               seq_cap=seq_cap, roles=np.zeros((NL, Hr), np.uint8), policy=pol,
                               dtype=dt, select="none")
        fout = torch.empty_like(q)
        with torch.cuda.stream(stream):
            fdec.capture(q, K, V, L, fout, stream=stream)
        fms = allmax(time_graph(fdec, args.steps, args.warmup))
        fbytes = fdec.step_bytes(L)
        full = {"us_per_token": fms * 1e3, "hbm_gbs": fbytes / (fms / 1e3) / 1e9,
                "speedup_hybrid_vs_full": fms / ms}
        fdec.close()

    # ---- external full-attention bar: FlashInfer's decode
    # attention (library code, JIT-compiled on first use) over every layer's
    # full cache in our HND layout, CUDA-graph replayed
    flashinfer_full = None
    if world == 1 and not args.no_flashinfer and dt == torch.bfloat16 and B == 1:
        try:
            import flashinfer
            fo = torch.empty((NL, Hr * G, d), dtype=dt, device=dev)

            def fi_step():
                for l in range(NL):
                    fo[l] = flashinfer.single_decode_with_kv_cache(
                        q[l, 0], K[l, 0], V[l, 0], kv_layout="HND", use_tensor_cores=True)
            with torch.cuda.stream(stream):
                for _ in range(3):
                    fi_step()
                stream.synchronize()
                gfi = torch.cuda.CUDAGraph()
                with torch.cuda.graph(gfi, stream=stream):
                    fi_step()
                for _ in range(args.warmup):
                    gfi.replay()
            stream.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            with torch.cuda.stream(stream):
                e0.record(stream)
                for _ in range(args.steps):
                    gfi.replay()
                e1.record(stream)
            e1.synchronize()
            fi_us = e0.elapsed_time(e1) / args.steps * 1e3
            flashinfer_full = {"us_per_token": fi_us, "version": flashinfer.__version__,
                               "api": "flashinfer.single_decode_with_kv_cache (tensor cores), "
                                      "every layer, full cache",
                               "speedup_hybrid_vs_flashinfer_full": fi_us / step_us}
            if full:
                flashinfer_full["our_full_vs_flashinfer_full"] = fi_us / full["us_per_token"]
            del gfi
        except Exception as e:  # an external bar must not kill the bench line
            flashinfer_full = {"error": repr(e)[:200]}

    # ---- BASELINE config 3 is a retrieval-head fraction sweep at fixed top-k:
    # the same caches and queries with 25 % and 50 % retrieval heads (the
    # headline is the 12.5 % point), whole-step time, graph replayed
    sweep = None
    if world == 1 and fused and not args.no_sweep:
        sweep = []
        for fr in (0.25, 0.5):
            sroles = make_roles(NL, H, fr, args.seed)
            sdec = P.HybridDecoder(n_layers=NL, batch=B, n_kv_heads=H, group_size=G, d_head=d,
                                   seq_cap=seq_cap, roles=sroles, policy=pol, dtype=dt,
                                   select=args.select)
            sout = torch.empty_like(q)
            with torch.cuda.stream(stream):
                sdec.capture(q, K, V, L, sout, stream=stream)
            sms = time_graph(sdec, args.steps, args.warmup)
            sbytes = sdec.step_bytes(L)
            sweep.append({"retrieval_fraction": fr, "us_per_token": sms * 1e3 / B,
                          "bytes_per_step": sbytes,
                          "hbm_gbs": sbytes / (sms / 1e3) / 1e9,
                          "frac": sbytes / (sms / 1e3) / 1e9 / peak})
            sdec.close()

    # ---- the per-layer public API (lyc_decoder_layer, what a model calls
    # between its own projections): one step-kernel launch per layer (plus
    # the planner at layer 0), eager and CUDA-graph captured
    per_layer = None
    if fused:
        out_l = torch.empty_like(q)

        def layers_step():
            for l in range(NL):
                dec.layer(l, q[l], K, V, L, out_l[l], stream=stream)

        with torch.cuda.stream(stream):
            for _ in range(args.warmup):
                layers_step()
        stream.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            e0.record(stream)
            for _ in range(args.steps):
                layers_step()
            e1.record(stream)
        e1.synchronize()
        eager_ms = allmax(e0.elapsed_time(e1) / args.steps)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=stream):
            layers_step()
        with torch.cuda.stream(stream):
            for _ in range(args.warmup):
                g.replay()
        stream.synchronize()
        with torch.cuda.stream(stream):
            e0.record(stream)
            for _ in range(args.steps):
                g.replay()
            e1.record(stream)
        e1.synchronize()
        graph_ms = allmax(e0.elapsed_time(e1) / args.steps)
        same = bool(torch.equal(out_l, out))
        per_layer = {"api": "HybridDecoder.layer x n_layers (lyc_decoder_layer)",
                     "us_per_token_eager": eager_ms * 1e3 / B,
                     "us_per_token_graph": graph_ms * 1e3 / B,
                     "vs_whole_step_graph": graph_ms / ms,
                     "launches_per_step": NL + 1, "outputs_equal_whole_step": same}
        del g

    # ---- selection parity of the measured step (in-bench numpy check): the
    # per-layer sets the step kernel emitted (set tracing) against the exact
    # top-k of f64 pooled-query scores, ties to the lower index
    # (attention.hpp:108-123, decode_engine.hpp:129-132)
    swaps = None
    if rank == 0 and fused and args.select == "tokens" and not args.no_swaps:
        swaps = selection_swaps(dec, q, K, V, L, wl, r_roles, stream)

    # ---- e2e through the public API with host buffers, token after token:
    # every step uploads its inputs in one packed pinned copy (q of every layer
    # + the new token's K/V rows), appends the rows at the growing length
    # (lyc_kv_write, all layers in one launch), runs the step at seq = t + 1
    # through HybridDecoder.decode_step (the device planner re-plans the new
    # length in the stream: no host synchronisation) and reads the outputs
    # back.  The same loop at a fixed length is reported beside it.
    import ctypes as C
    from paper_2602_04541_b200 import _lib as LL
    nq, nkv = q.numel(), NL * B * Hr * d
    in_h = torch.empty(nq + 2 * nkv, dtype=dt, pin_memory=True)
    in_h[:nq].copy_(q.cpu().reshape(-1))
    in_h[nq:nq + nkv].copy_(K[:, :, :, L - 1].cpu().reshape(-1))
    in_h[nq + nkv:].copy_(V[:, :, :, L - 1].cpu().reshape(-1))
    in_d = torch.empty_like(in_h, device=dev)
    q_in = in_d[:nq].view(q.shape)
    k_new, v_new = in_d[nq:nq + nkv], in_d[nq + nkv:]
    lay = LL.lyc_kv_layout(n_layers=NL, batch=B, n_kv_heads=Hr, d_head=d,
                           dtype=LL.DTYPE_BF16 if dt == torch.bfloat16 else LL.DTYPE_F32, pad=0,
                           seq_cap=seq_cap)
    out_h = torch.empty(out.shape, dtype=dt, pin_memory=True)
    e2e_steps = max(3, args.steps)

    def e2e_step(seq):
        in_d.copy_(in_h, non_blocking=True)
        LL.check(LL.lib().lyc_kv_write(K.data_ptr(), V.data_ptr(), C.byref(lay), -1, seq - 1, 1,
                                       k_new.data_ptr(), v_new.data_ptr(), stream.cuda_stream))
        dec.decode_step(q_in, K, V, seq, out, stream=stream)
        out_h.copy_(out, non_blocking=True)

    def time_e2e(seqs):
        with torch.cuda.stream(stream):
            for s_ in seqs[:2]:
                e2e_step(s_)
        stream.synchronize()
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            e0.record(stream)
            for s_ in seqs:
                e2e_step(s_)
            e1.record(stream)
        e1.synchronize()
        barrier()
        return allmax(e0.elapsed_time(e1) / len(seqs))

    growing = list(range(L - e2e_steps + 1, L + 1))
    e2e_ms = time_e2e(growing)
    e2e_fixed_ms = time_e2e([L] * e2e_steps)
    h2d = in_h.numel() * esz
    d2h = out_h.numel() * esz

    # ---- end-to-end TPOT of the toy model's decode step:
    # per layer the Q/K/V GEMV (rmsnorm + rotary + cache append fused), the
    # attention through lyc_decoder_layer, the output projection and the FFN
    # GEMVs (lyc_gemv), then the logits -- hybrid vs full attention on the same
    # weights and cache, each token one CUDA graph replay
    model_tpot = None
    if world == 1 and not args.no_model and dt == torch.bfloat16 and B == 1:
        from paper_2602_04541_b200.model import PRESETS, DecodeModel, ModelConfig
        preset = "qwen3-8b" if NL == 36 else "llama3-8b"
        mcfg = ModelConfig(max_seq_len=seq_cap, **PRESETS[preset])
        if mcfg.n_layers == NL and mcfg.n_kv_heads == Hr and mcfg.d_head == d:
            dm = DecodeModel(mcfg, roles=r_roles, policy=pol, attention="hybrid", seed=args.seed,
                             k_cache=K, v_cache=V)
            res = {}
            for att in ("hybrid", "full"):
                dm.set_attention(att)
                with torch.cuda.stream(stream):
                    for _ in range(3):
                        dm.decode_token(7, L - 1, stream=stream)
                stream.synchronize()
                gph = torch.cuda.CUDAGraph()
                with torch.cuda.graph(gph, stream=stream):
                    dm.decode_token(7, L - 1, stream=stream)
                with torch.cuda.stream(stream):
                    for _ in range(args.warmup):
                        gph.replay()
                stream.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                n_rep = max(5, args.steps // 2)
                with torch.cuda.stream(stream):
                    e0.record(stream)
                    for _ in range(n_rep):
                        gph.replay()
                    e1.record(stream)
                e1.synchronize()
                res[att] = e0.elapsed_time(e1) / n_rep * 1e3
                del gph
            wb = dm.weight_bytes()
            model_tpot = {
                "model": f"{preset} shapes, toy_model.hpp structure (two-matrix FFN), random bf16 "
                         f"weights, batch 1, context {L}",
                "tpot_us_hybrid": res["hybrid"], "tpot_us_full": res["full"],
                "speedup_hybrid_vs_full": res["full"] / res["hybrid"],
                "weight_bytes": wb,
                "launches_per_token": 4 * NL + 1 + NL,
                "api": "DecodeModel.decode_token: lyc_gemv x (4 per layer + logits) + "
                       "lyc_decoder_layer per layer, CUDA-graph replayed"}
            dm.close()

    # ---- CPU baseline (rank 0, N == 1): the reference CPU path, whole steps
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            Kh = K[0, 0].float().cpu().numpy()
            Vh = V[0, 0].float().cpu().numpy()
            qh = q[0, 0].float().cpu().numpy()
            cs = CpuStep(wl, roles, Kh, Vh, qh)
            cs.step()  # warm-up
            n_cpu = 2
            res = [cs.step() for _ in range(n_cpu)]
            us = float(np.mean([r[0] for r in res])) * 1e6
            cpu = {"value": us, "unit": "us/token", "kind": cs.kind, "cores": cs.cores,
                   "cpu_model": cpu_model(),
                   "sample": cs.sample(n_cpu, *np.mean(np.array(res), axis=0))}
            cs.close()
        except Exception as e:  # the baseline must not kill the bench line
            cpu = {"value": None, "unit": "us/token", "error": repr(e)[:200]}

    if rank == 0:
        line = {
            "metric": METRIC, "value": head_ms * 1e3 / B,
            "unit": "us/token", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": head_ms, "higher_is_better": False,
            "scaling": "strong" if world > 1 else "weak", "vs_baseline": None,
            "dtype": wl["dtype"], "data": "synthetic U(-1,1) q/K/V, seeded roles",
            "config": config_of(args, wl),
            "tokens_per_s": B / (head_ms / 1e3),
            "step_hbm_gbs": step_bytes / (ms / 1e3) / 1e9 if world == 1 else None,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak,
                         "traffic": ncu_traffic(args.workload) if fused and world == 1 else None,
                         "traffic_unit": "bytes per launch (= step), ncu --set full",
                         "peak_kind": pk_kind,
                         "frac_of_8TBs": achieved / 8000.0,
                         "kernel": ("hybrid_step_kernel (whole step: attention + merge + "
                                    "selection of all layers, 1 launch)") if fused
                                   else "hybrid_attn_kernel (all layers)",
                         "attn_us_per_step": attn_ms_total * 1e3,
                         "layer0_gbs": None if fused
                                       else attn_bytes[0] / (per_layer[0] / 1e3) / 1e9,
                         "bytes_per_step": float(attn_bytes.sum())},
            "full_attention": full,
            "retrieval_fraction_sweep": sweep,
            "flashinfer_full_attention": flashinfer_full,
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_ms * 1e3 / B, "unit": "us/token", "h2d_bytes_per_step": int(h2d),
                    "d2h_bytes_per_step": int(d2h),
                    "api": "HybridDecoder.decode_step (eager C-ABI), token after token",
                    "seq_lens": f"{growing[0]}..{growing[-1]}",
                    "fixed_seq_us_per_token": e2e_fixed_ms * 1e3 / B,
                    "growing_vs_fixed": e2e_ms / e2e_fixed_ms},
            "per_layer_api": per_layer,
            "model_tpot": model_tpot,
            "head_shard_layer_sync": layer_sync,
            "selection_swaps": swaps,
            "gpu_launches": int((NL if layer_sync else launches_per_step) * args.steps),
            "launches_per_step": int(NL if layer_sync else launches_per_step),
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    dec.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
