"""Mirror of the reference decode-step attention loop and its selection API.

* ``SparsityPolicy`` / ``fraction_budget`` -- policy.hpp:20-62 (all four kinds
  run on the device; TopP / Threshold through per-layer kernels, csrc/policy.cu).
* ``args_top_k``   -- attention.hpp:108-123 on a device score vector.
* ``HybridDecoder`` -- decode_engine.hpp:109-151: per layer, retrieval heads
  (layer 0, or role R in the RoleMap, rolemap.hpp:33-35) run dense split-KV
  attention and refresh the per-KV-head index cache (``sets_``,
  decode_engine.hpp:251) from the pooled-query scores; sparse heads attend to
  the set inherited from the nearest earlier retrieval layer of the same head
  index.  All of it runs in the in-tree ``liblyc.so``.

Device layouts (the C-ABI, include/lyc.h):
  q, out : [n_layers][B][Hq][d]          K, V : [n_layers][B][H][seq_cap][d]
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import List, Optional

import numpy as np
import torch

from . import _lib
from ._lib import InvalidArgument, NotSupported, check, lib


def fraction_budget(frac: float, n: int) -> int:
    """policy.hpp:57-62."""
    return int(lib().lyc_fraction_budget(float(frac), int(n)))


@dataclass
class SparsityPolicy:
    """policy.hpp:20-53."""
    kind: str = "topk"
    k: int = 1
    value: float = 0.0

    @staticmethod
    def top_k(k: int) -> "SparsityPolicy":
        if k < 1:
            raise InvalidArgument("top_k: k must be >= 1")
        return SparsityPolicy("topk", k, 0.0)

    @staticmethod
    def ratio(theta: float) -> "SparsityPolicy":
        if not (0.0 < theta < 1.0):
            raise InvalidArgument("ratio: theta must lie in (0,1)")
        return SparsityPolicy("ratio", 0, theta)

    @staticmethod
    def top_p(p: float) -> "SparsityPolicy":
        if not (0.0 < p <= 1.0):
            raise InvalidArgument("top_p: p must lie in (0,1]")
        return SparsityPolicy("topp", 0, p)

    @staticmethod
    def threshold(tau: float) -> "SparsityPolicy":
        if not (tau > 0.0):
            raise InvalidArgument("threshold: tau must be positive")
        return SparsityPolicy("threshold", 0, tau)

    def code(self) -> int:
        return {"topk": _lib.POLICY_TOPK, "topp": _lib.POLICY_TOPP,
                "threshold": _lib.POLICY_THRESHOLD, "ratio": _lib.POLICY_RATIO}[self.kind]

    def budget(self, n: int) -> int:
        if self.kind == "topk":
            return min(self.k, n)
        if self.kind == "ratio":
            return fraction_budget(1.0 - self.value, n)
        raise NotSupported(f"{self.kind}: data-dependent budget")


def args_top_k(scores: torch.Tensor, k: int, *, stream=None) -> torch.Tensor:
    """attention.hpp:108-123 on the GPU: indices of the min(k, n) largest
    fp32 scores, ties to the lower index, ascending (int32 device tensor)."""
    s = scores.to(torch.float32).contiguous()
    if not s.is_cuda:
        s = s.cuda()
    n = s.numel()
    out = torch.empty(max(min(k, n), 1), dtype=torch.int32, device=s.device)
    st = stream if stream is not None else torch.cuda.current_stream(s.device)
    cnt = check(lib().lyc_args_top_k(s.data_ptr(), n, k, out.data_ptr(), st.cuda_stream))
    return out[:cnt]


class HybridDecoder:
    """Device decode engine for the hybrid-head attention of one step.

    roles: [n_layers][n_kv_heads] with 0 = Retrieval, 1 = Sparse (RoleMap).
    select: 'tokens' (TokenSet, decode_engine.hpp:132) or 'blocks'
    (BlockIndexSet of ceil(k/64) blocks, the paper's block-sparse kernel)."""

    def __init__(self, *, n_layers: int, batch: int, n_kv_heads: int, group_size: int,
                 d_head: int, seq_cap: int, roles, policy: SparsityPolicy,
                 dtype: torch.dtype = torch.bfloat16, select: str = "tokens",
                 num_splits: int = 0, scale: float = 0.0):
        self.n_layers, self.batch, self.n_kv_heads = n_layers, batch, n_kv_heads
        self.group_size, self.d_head, self.seq_cap = group_size, d_head, seq_cap
        self.dtype = dtype
        self.policy = policy
        self.select = select
        r = np.ascontiguousarray(np.asarray(roles, dtype=np.uint8).reshape(n_layers, n_kv_heads))
        self.roles = r
        cfg = _lib.lyc_decode_config(
            n_layers=n_layers, batch=batch, n_kv_heads=n_kv_heads, group_size=group_size,
            d_head=d_head,
            dtype=_lib.DTYPE_BF16 if dtype == torch.bfloat16 else _lib.DTYPE_F32,
            seq_cap=seq_cap, policy_kind=policy.code(),
            select_mode={"tokens": _lib.SELECT_TOKENS, "blocks": _lib.SELECT_BLOCKS,
                         "none": _lib.SELECT_NONE}[select],
            top_k=policy.k, ratio=policy.value, block_size=64, num_splits=num_splits,
            scale=scale, roles=r.ctypes.data)
        h = C.c_void_p()
        check(lib().lyc_decoder_create(C.byref(cfg), C.byref(h)))
        self._h = h
        self.captured = None

    def close(self):
        if getattr(self, "_h", None):
            lib().lyc_decoder_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @staticmethod
    def _stream(stream):
        return (stream if stream is not None else torch.cuda.current_stream()).cuda_stream

    def decode_step(self, q, k_cache, v_cache, seq_len, out=None, *, stream=None):
        """All layers of one step (decode_engine.hpp:109-151).

        seq_len is an int (every batch item), or one length per batch item (a
        variable-length batch: B independent sequences, lyc_decoder_step_varlen).
        """
        if out is None:
            out = torch.empty_like(q)
        if isinstance(seq_len, (int, np.integer)):
            check(lib().lyc_decoder_step(self._h, q.data_ptr(), k_cache.data_ptr(),
                                         v_cache.data_ptr(), seq_len, out.data_ptr(),
                                         self._stream(stream)))
            return out
        lens = [int(x) for x in seq_len]
        if len(lens) != self.batch:
            raise ValueError("decode_step: one seq_len per batch item")
        arr = (C.c_int64 * len(lens))(*lens)
        check(lib().lyc_decoder_step_varlen(self._h, q.data_ptr(), k_cache.data_ptr(),
                                            v_cache.data_ptr(), arr, out.data_ptr(),
                                            self._stream(stream)))
        return out

    def decode_step_dev(self, q, k_cache, v_cache, seq_lens, out=None, *, stream=None):
        """A step whose lengths live on the device (int64 [B] tensor, current
        token included), read by the device planner when the step runs
        (lyc_decoder_step_dev).  No host synchronisation."""
        if out is None:
            out = torch.empty_like(q)
        _check_lens_tensor(seq_lens, self.batch)
        check(lib().lyc_decoder_step_dev(self._h, q.data_ptr(), k_cache.data_ptr(),
                                         v_cache.data_ptr(), seq_lens.data_ptr(), out.data_ptr(),
                                         self._stream(stream)))
        return out

    def capture_dev(self, q, k_cache, v_cache, seq_lens, out, *, stream=None):
        """Capture a step with device-resident lengths: every replay plans the
        lengths `seq_lens` holds when it runs (lyc_decoder_capture_dev)."""
        _check_lens_tensor(seq_lens, self.batch)
        check(lib().lyc_decoder_capture_dev(self._h, q.data_ptr(), k_cache.data_ptr(),
                                            v_cache.data_ptr(), seq_lens.data_ptr(),
                                            out.data_ptr(), self._stream(stream)))
        self.captured = (q, k_cache, v_cache, seq_lens, out)

    def status(self, *, stream=None):
        """Raise InvalidArgument if the last device-planned step rejected its
        lengths (synchronises the stream)."""
        check(lib().lyc_decoder_status(self._h, self._stream(stream)))

    def tune(self, what: int, value: int):
        """Experiment knobs (_lib.TUNE_RING_STAGES, _lib.TUNE_PER_LAYER_KERNELS)."""
        check(lib().lyc_decoder_tune(self._h, int(what), int(value)))

    def layer(self, l: int, q_l, k_cache, v_cache, seq_len: int, out_l=None, *, stream=None):
        """One layer (decode_engine.hpp:120-143); layers in order within a step."""
        if out_l is None:
            out_l = torch.empty_like(q_l)
        check(lib().lyc_decoder_layer(self._h, l, q_l.data_ptr(), k_cache.data_ptr(),
                                      v_cache.data_ptr(), seq_len, out_l.data_ptr(),
                                      self._stream(stream)))
        return out_l

    def refresh_sets(self, layer: int, q_last, k_cache, length: int, *, stream=None):
        """Cache-correction set refresh (decode_engine.hpp:190-197): re-select
        every KV head's index set from the pooled query of the last window
        position (q_last [B][Hq][d] at `layer`) over keys [0, length)."""
        check(lib().lyc_decoder_refresh_sets(self._h, layer, q_last.data_ptr(), k_cache.data_ptr(),
                                             int(length), self._stream(stream)))

    def capture(self, q, k_cache, v_cache, seq_len: int, out, *, stream=None):
        """Capture one step into a CUDA graph (fixed pointers and seq_len)."""
        if isinstance(seq_len, (int, np.integer)):
            check(lib().lyc_decoder_capture(self._h, q.data_ptr(), k_cache.data_ptr(),
                                            v_cache.data_ptr(), seq_len, out.data_ptr(),
                                            self._stream(stream)))
        else:
            lens = [int(x) for x in seq_len]
            if len(lens) != self.batch:
                raise ValueError("capture: one seq_len per batch item")
            arr = (C.c_int64 * len(lens))(*lens)
            check(lib().lyc_decoder_capture_varlen(self._h, q.data_ptr(), k_cache.data_ptr(),
                                                   v_cache.data_ptr(), arr, out.data_ptr(),
                                                   self._stream(stream)))
        self.captured = (q, k_cache, v_cache, seq_len, out)

    def replay(self, *, stream=None):
        check(lib().lyc_decoder_replay(self._h, self._stream(stream)))

    def sync_sets(self, *, stream=None):
        """Complete a selection deferred by the last per-layer call (in `stream`)."""
        check(lib().lyc_decoder_sync_sets(self._h, self._stream(stream)))

    def index_cache(self):
        """(ids [B*H][k_cap] int32 device view, counts [B*H]) -- the sets_."""
        self.sync_sets()
        ids, cnt, kcap = C.c_void_p(), C.c_void_p(), C.c_int64()
        check(lib().lyc_decoder_index_cache(self._h, C.byref(ids), C.byref(cnt), C.byref(kcap)))
        rows = self.batch * self.n_kv_heads
        dev = torch.device("cuda", torch.cuda.current_device())
        ids_t = _wrap_device(ids.value, rows * kcap.value, dev).view(rows, kcap.value)
        cnt_t = _wrap_device(cnt.value, rows, dev)
        return ids_t, cnt_t

    def token_sets(self) -> List[List[np.ndarray]]:
        """Host copy of the index cache as [b][g] ascending id arrays."""
        ids, cnt = self.index_cache()
        ids, cnt = ids.cpu().numpy(), cnt.cpu().numpy()
        H = self.n_kv_heads
        return [[ids[b * H + g, : cnt[b * H + g]].copy() for g in range(H)]
                for b in range(self.batch)]

    def launches_per_step(self, seq_len: int) -> int:
        return check(lib().lyc_decoder_launches_per_step(self._h, seq_len))

    def step_bytes(self, seq_len: int) -> int:
        return check(lib().lyc_decoder_step_bytes(self._h, seq_len))

    def layer_attn_bytes(self, layer: int, seq_len: int) -> int:
        return check(lib().lyc_decoder_layer_attn_bytes(self._h, layer, seq_len))

    @property
    def fused(self) -> bool:
        """True when decode_step runs the persistent whole-step kernel."""
        return bool(lib().lyc_decoder_is_fused(self._h))

    def set_trace(self, enable: bool = True):
        """Per-layer/per-CTA %globaltimer timeline of the fused step kernel."""
        check(lib().lyc_decoder_set_trace(self._h, int(bool(enable))))

    def trace(self) -> np.ndarray:
        """[n_layers][24 events][n_ctas] ns stamps of the last traced step."""
        n = check(lib().lyc_decoder_trace(self._h, None, 0))
        buf = np.zeros(n, dtype=np.uint64)
        check(lib().lyc_decoder_trace(self._h, buf.ctypes.data, n))
        return buf.reshape(self.n_layers, 24, -1)

    def set_trace_sets(self, enable: bool = True):
        """Record every layer's emitted index sets (fused step kernel)."""
        check(lib().lyc_decoder_set_trace_sets(self._h, int(bool(enable))))

    def traced_sets(self):
        """(ids [n_layers][B*H][k_cap] int32, counts [n_layers][B*H]; -1 = no
        set emitted at that layer) of the last traced step."""
        kcap = check(lib().lyc_decoder_traced_sets(self._h, None, None, 0))
        rows = self.n_layers * self.batch * self.n_kv_heads
        ids = np.zeros((rows, kcap), dtype=np.int32)
        cnt = np.zeros(rows, dtype=np.int32)
        check(lib().lyc_decoder_traced_sets(self._h, ids.ctypes.data, cnt.ctypes.data, ids.size))
        H = self.batch * self.n_kv_heads
        return ids.reshape(self.n_layers, H, kcap), cnt.reshape(self.n_layers, H)

    def set_timing(self, enable: bool = True):
        """CUDA events around every attention-kernel launch (graph-capturable)."""
        check(lib().lyc_decoder_set_timing(self._h, int(bool(enable))))

    def attn_ms(self) -> np.ndarray:
        """Per-layer attention-kernel durations (ms) of the last completed step."""
        ms = np.zeros(self.n_layers, dtype=np.float32)
        check(lib().lyc_decoder_attn_ms(self._h, ms.ctypes.data))
        return ms


def _check_lens_tensor(t, batch):
    if not (isinstance(t, torch.Tensor) and t.is_cuda and t.dtype == torch.int64 and
            t.numel() == batch and t.is_contiguous()):
        raise InvalidArgument("seq_lens: a contiguous int64 CUDA tensor with one length per batch item")


def plan_selftest(*, n_layers, batch, n_kv_heads, group_size, d_head, seq_cap, roles, policy,
                  select="tokens", seq_len=0, seq_lens=None, n_sms=148, num_splits=0) -> None:
    """The device planner (plan.cuh, run on the host) against the host-order
    planner; raises LogicError on the first difference.  No GPU needed."""
    r = np.ascontiguousarray(np.asarray(roles, dtype=np.uint8).reshape(n_layers, n_kv_heads))
    cfg = _lib.lyc_decode_config(
        n_layers=n_layers, batch=batch, n_kv_heads=n_kv_heads, group_size=group_size,
        d_head=d_head, dtype=_lib.DTYPE_BF16, seq_cap=seq_cap, policy_kind=policy.code(),
        select_mode={"tokens": _lib.SELECT_TOKENS, "blocks": _lib.SELECT_BLOCKS,
                     "none": _lib.SELECT_NONE}[select],
        top_k=policy.k, ratio=policy.value, block_size=64, num_splits=num_splits, scale=0.0,
        roles=r.ctypes.data)
    arr = None
    if seq_lens is not None:
        arr = (C.c_int64 * batch)(*[int(x) for x in seq_lens])
    check(lib().lyc_plan_selftest(C.byref(cfg), int(seq_len), arr, int(n_sms)))


def _wrap_device(ptr: int, n: int, dev) -> torch.Tensor:
    """Zero-copy int32 view of library-owned device memory (no ownership)."""
    class _Holder:
        __cuda_array_interface__ = {
            "shape": (n,), "typestr": "<i4", "data": (ptr, False), "version": 3, "strides": None}
    return torch.as_tensor(_Holder(), device=dev)
