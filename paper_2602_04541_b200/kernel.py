"""Mirror of ``hh::kernel`` (reference kernel_sim.hpp) over the C-ABI.

Same names, argument meaning and error behaviour as the reference operator
API: ``plan_splits`` (kernel_sim.hpp:63-110), ``Workload`` (120-146), ``run``
(237-279) and ``latency_model`` (284-316).  ``run`` executes on the B200
through ``lyc_workload_run``; host tensors are staged to the device (the
reference-facing end-to-end path), device tensors are used in place.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np
import torch

from . import _lib
from ._lib import InvalidArgument, check, lib


@dataclass
class BlockIndexSet:
    """kernel_sim.hpp:20-42: per (b, g) ascending block ids, slot b*H+g."""
    batch: int = 0
    n_kv_heads: int = 0
    ids: List[Sequence[int]] = field(default_factory=list)

    def slot(self, b: int, g: int) -> int:
        return b * self.n_kv_heads + g


@dataclass
class WorkUnit:
    """kernel_sim.hpp:45-50."""
    kv_head: int
    begin: int
    end: int
    head_local_split: int


@dataclass
class SplitSchedule:
    """kernel_sim.hpp:54-61."""
    batch: int
    num_splits: int
    units: list            # [b][split] -> [WorkUnit]
    split_blocks: list     # [b][split]
    head_blocks: list      # [b][kv head]
    head_split_count: list # [b][kv head]


def plan_splits(blocks: BlockIndexSet, num_splits: int) -> SplitSchedule:
    """kernel_sim.hpp:63-110 (host planner of the C-ABI, lyc_plan_splits)."""
    B, H = blocks.batch, blocks.n_kv_heads
    hb = np.array([[len(blocks.ids[b * H + g]) for g in range(H)] for b in range(B)],
                  dtype=np.int64).reshape(B, H)
    sb = np.zeros((B, max(num_splits, 1)), dtype=np.int64)
    hsc = np.zeros((B, H), dtype=np.int64)
    n = check(lib().lyc_plan_splits(B, H, hb.ctypes.data, num_splits, sb.ctypes.data,
                                     hsc.ctypes.data, None, 0))
    rec = np.zeros((max(n, 1), 6), dtype=np.int64)
    check(lib().lyc_plan_splits(B, H, hb.ctypes.data, num_splits, sb.ctypes.data,
                                hsc.ctypes.data, rec.ctypes.data, n))
    units = [[[] for _ in range(num_splits)] for _ in range(B)]
    for b, s, g, beg, end, hls in rec[:n].tolist():
        units[b][s].append(WorkUnit(g, beg, end, hls))
    return SplitSchedule(B, num_splits, units, sb.tolist(), hb.tolist(), hsc.tolist())


@dataclass
class Workload:
    """kernel_sim.hpp:120-146.

    keys/values: tensor [B*H][seq][d] (or [B*H][S_cap][d] with S_cap >= seq);
    queries: [B*Hq][d] with h = g*G + j; dtype float32 or bfloat16."""
    batch: int = 0
    n_kv_heads: int = 0
    group_size: int = 1
    d_head: int = 0
    seq_len: int = 0
    block_size: int = 64
    scale: float = 1.0
    keys: Optional[torch.Tensor] = None
    values: Optional[torch.Tensor] = None
    queries: Optional[torch.Tensor] = None
    blocks: BlockIndexSet = field(default_factory=BlockIndexSet)

    def n_q_heads(self) -> int:
        return self.n_kv_heads * self.group_size

    def n_blocks(self) -> int:
        return (self.seq_len + self.block_size - 1) // self.block_size


@dataclass
class RunResult:
    """kernel_sim.hpp:227-232."""
    outputs: torch.Tensor            # [B*Hq][d]
    schedule: SplitSchedule
    block_exec_counts: list


def _dtype_code(t: torch.Tensor) -> int:
    if t.dtype == torch.float32:
        return _lib.DTYPE_F32
    if t.dtype == torch.bfloat16:
        return _lib.DTYPE_BF16
    raise InvalidArgument(f"Workload: unsupported dtype {t.dtype}")


def run(w: Workload, num_splits: int, n_workers: int = 1, *, stream=None,
        exec_counts: bool = True) -> RunResult:
    """kernel_sim.hpp:237-279 on the GPU.  ``n_workers`` is accepted for API
    parity and ignored: outputs are bitwise independent of it by construction
    (one CTA per (b, split) cell, fixed merge order)."""
    if w.keys is None or w.values is None or w.queries is None:
        raise InvalidArgument("Workload: KV slot count mismatch")
    if w.keys.shape[0] != w.batch * w.n_kv_heads or w.values.shape != w.keys.shape:
        raise InvalidArgument("Workload: KV slot count mismatch")
    if w.queries.shape[0] != w.batch * w.n_q_heads():
        raise InvalidArgument("Workload: query slot count mismatch")
    if len(w.blocks.ids) != w.batch * w.n_kv_heads:
        raise InvalidArgument("BlockIndexSet: slot count mismatch")
    dev = torch.device("cuda", torch.cuda.current_device())
    k = w.keys.to(dev).contiguous()
    v = w.values.to(dev).contiguous()
    q = w.queries.to(dev).contiguous()
    dt = _dtype_code(k)
    if v.dtype != k.dtype or q.dtype != k.dtype:
        raise InvalidArgument("Workload: mixed dtypes")
    off = np.zeros(len(w.blocks.ids) + 1, dtype=np.int64)
    for i, ids in enumerate(w.blocks.ids):
        off[i + 1] = off[i] + len(ids)
    flat = np.zeros(max(int(off[-1]), 1), dtype=np.int64)
    if off[-1]:
        flat[: off[-1]] = np.concatenate([np.asarray(x, dtype=np.int64) for x in w.blocks.ids])
    cw = _lib.lyc_workload(
        batch=w.batch, n_kv_heads=w.n_kv_heads, group_size=w.group_size, d_head=w.d_head,
        seq_len=w.seq_len, block_size=w.block_size, kv_row_stride=k.shape[1], scale=w.scale,
        dtype=dt, k=k.data_ptr(), v=v.data_ptr(), q=q.data_ptr(), blk_off=off.ctypes.data,
        blk_ids=flat.ctypes.data)
    out = torch.empty((q.shape[0], w.d_head), dtype=k.dtype, device=dev)
    nb = w.n_blocks()
    counts = (torch.zeros((w.batch * w.n_kv_heads, nb), dtype=torch.int32, device=dev)
              if exec_counts else None)
    st = stream if stream is not None else torch.cuda.current_stream(dev)
    check(lib().lyc_workload_run(C.byref(cw), num_splits, out.data_ptr(),
                                 counts.data_ptr() if counts is not None else None,
                                 st.cuda_stream))
    sched = plan_splits(w.blocks, num_splits)
    flat_counts = []
    if counts is not None:
        c = counts.cpu().numpy()
        for s in range(w.batch * w.n_kv_heads):
            flat_counts.extend(c[s, : len(w.blocks.ids[s])].tolist())
    return RunResult(out, sched, flat_counts)


@dataclass
class CostReport:
    """kernel_sim.hpp:284-293."""
    total_blocks: int = 0
    pooled_critical_blocks: int = 0
    naive_critical_blocks: int = 0
    mean_split_blocks: float = 0.0
    balance_ratio: float = 0.0
    bytes_per_block: int = 0
    pooled_critical_bytes: int = 0
    naive_critical_bytes: int = 0


def latency_model(sched: SplitSchedule, bytes_per_block: int) -> CostReport:
    """kernel_sim.hpp:295-316 (recomputed by the C-ABI from the head sizes)."""
    hb = np.asarray(sched.head_blocks, dtype=np.int64)
    o = np.zeros(6, dtype=np.int64)
    d = np.zeros(2)
    check(lib().lyc_latency_model(sched.batch, hb.shape[1], hb.ctypes.data, sched.num_splits,
                                  bytes_per_block, o.ctypes.data, d.ctypes.data))
    return CostReport(int(o[0]), int(o[1]), int(o[2]), float(d[0]), float(d[1]), int(o[3]),
                      int(o[4]), int(o[5]))
