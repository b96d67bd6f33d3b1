"""Device KV cache with the reference's write path (kv_cache.hpp:14-69).

The cache is the decoder's layout: K and V tensors [n_layers][B][H][seq_cap][d]
on the GPU.  ``append`` writes one row per (b, g) of a layer at the current
length (KvCache::append, 23-29), ``commit_row`` advances the shared length once
every layer appended (32), ``overwrite`` rewrites rows below the length
(34-42; a window of rows for cache correction).  Writes go through the C-ABI
``lyc_kv_write`` (include/lyc.h): one coalesced copy kernel, stream-ordered.
"""
from __future__ import annotations

import ctypes as C

import torch

from . import _lib
from ._lib import InvalidArgument, check, lib


class KvCache:
    def __init__(self, *, n_layers: int, batch: int, n_kv_heads: int, d_head: int, seq_cap: int,
                 dtype: torch.dtype = torch.bfloat16, device=None):
        if min(n_layers, batch, n_kv_heads, d_head, seq_cap) < 1:
            raise InvalidArgument("KvCache: all dimensions must be >= 1")
        dev = device or torch.device("cuda", torch.cuda.current_device())
        shape = (n_layers, batch, n_kv_heads, seq_cap, d_head)
        self.k = torch.zeros(shape, dtype=dtype, device=dev)
        self.v = torch.zeros(shape, dtype=dtype, device=dev)
        self.length = 0
        self._lay = _lib.lyc_kv_layout(
            n_layers=n_layers, batch=batch, n_kv_heads=n_kv_heads, d_head=d_head,
            dtype=_lib.DTYPE_BF16 if dtype == torch.bfloat16 else _lib.DTYPE_F32, pad=0,
            seq_cap=seq_cap)
        self.seq_cap = seq_cap

    def _write(self, layer: int, pos: int, k_rows: torch.Tensor, v_rows: torch.Tensor,
               stream=None):
        k_rows = k_rows.to(self.k.dtype).contiguous()
        v_rows = v_rows.to(self.v.dtype).contiguous()
        n_rows = k_rows.shape[-2] if k_rows.dim() == 4 else 1
        st = stream.cuda_stream if stream is not None else torch.cuda.current_stream().cuda_stream
        check(lib().lyc_kv_write(self.k.data_ptr(), self.v.data_ptr(), C.byref(self._lay), layer,
                                 pos, n_rows, k_rows.data_ptr(), v_rows.data_ptr(), st))

    def append(self, layer: int, k_rows: torch.Tensor, v_rows: torch.Tensor, *, stream=None):
        """Rows [B][H][d] of every head of `layer` at position `length`."""
        if self.length >= self.seq_cap:
            raise InvalidArgument("KvCache: cache is full")
        self._write(layer, self.length, k_rows, v_rows, stream)

    def commit_row(self):
        self.length += 1

    def overwrite(self, layer: int, pos: int, k_rows: torch.Tensor, v_rows: torch.Tensor, *,
                  stream=None):
        """Rows [B][H][d] (one position) or [B][H][n][d] (a window from pos)."""
        n = k_rows.shape[-2] if k_rows.dim() == 4 else 1
        if pos < 0 or pos + n > self.length:
            raise InvalidArgument("KvCache: overwrite beyond the committed length")
        self._write(layer, pos, k_rows, v_rows, stream)


def correction_attention(k_cache: torch.Tensor, v_cache: torch.Tensor, layer: int,
                         q_window: torch.Tensor, start: int, *, scale: float = 0.0,
                         stream=None) -> torch.Tensor:
    """Cache-correction attention (decode_engine.hpp:164-204): window position
    i (p = start + i) of q_window [B][W][Hq][d] attends keys [0, p] of `layer`
    of the cache [L][B][H][cap][d] (bf16 or fp32), after the window's K/V rows
    were rewritten (KvCache.overwrite).  Returns [B][W][Hq][d] in the cache dtype."""
    L, B, H, cap, d = k_cache.shape
    Bq, W, Hq, dq = q_window.shape
    if Bq != B or dq != d or Hq % H:
        raise InvalidArgument("correction_attention: shape mismatch")
    G = Hq // H
    lay = _lib.lyc_kv_layout(n_layers=L, batch=B, n_kv_heads=H, d_head=d,
                             dtype=_lib.DTYPE_BF16 if k_cache.dtype == torch.bfloat16 else _lib.DTYPE_F32,
                             pad=0, seq_cap=cap)
    need = check(lib().lyc_window_workspace(C.byref(lay), G, W))
    ws = torch.empty(need // 4 + 1, dtype=torch.float32, device=k_cache.device)
    q = q_window.contiguous()
    out = torch.empty_like(q)
    st = stream.cuda_stream if stream is not None else torch.cuda.current_stream().cuda_stream
    check(lib().lyc_window_attention(C.byref(lay), layer, k_cache.data_ptr(), v_cache.data_ptr(), G,
                                     scale, start, W, q.data_ptr(), out.data_ptr(), ws.data_ptr(),
                                     ws.numel() * 4, st))
    return out


__all__ = ["KvCache", "correction_attention"]
