"""KV-sequence sharded hybrid decode across GPUs.

The inter-GPU form of the reference's split pooling (kernel_sim.hpp:63-110)
and combine (205-225): rank p of P holds rows [row_begin, row_begin + n_local)
of EVERY head's cache.  Per layer (include/lyc.h, lyc_shard_layer /
lyc_shard_merge):

  1. local attention partials (fp32 o + base-2 LSE) and, for retrieval heads,
     the exact local top-k candidates (key, global token id);
  2. ONE packed all-gather of [o | lse | keys | ids] (NCCL over NVLink);
  3. on every rank identically: rank-ordered LSE merge -> the layer output,
     and the global top-k over the P candidate lists (ties to the lower
     global id, attention.hpp:117-118) -> the global index set, filtered to
     this rank's rows for the sparse heads of later layers.

Head sharding (no collective at all, index propagation is per head index,
decode_engine.hpp:132-134) is bench.py's default multi-GPU mode; this is the
mode for contexts where one head's history should not sit on one GPU
(BASELINE config 5: 256K, batch 4, 8 GPUs).
"""
from __future__ import annotations

from typing import Callable, Optional

import numpy as np
import torch

from ._lib import check, lib
from .decode import HybridDecoder, SparsityPolicy


def shard_rows(seq_total: int, world: int, rank: int):
    """Contiguous, near-equal row ranges (the first seq_total % world ranks get
    one more row): returns (row_begin, n_local)."""
    base, rem = divmod(seq_total, world)
    begin = rank * base + min(rank, rem)
    return begin, base + (1 if rank < rem else 0)


class ShardedDecoder:
    """One rank of a sequence-sharded decode step.

    ``exchange(send, recv)`` gathers every rank's packed block into ``recv``
    in rank order (default: ``torch.distributed.all_gather_into_tensor``).
    ``recv`` may be supplied so several ranks can share one gathered buffer
    (single-GPU emulation in the tests: rank p's send block IS recv[p])."""

    def __init__(self, *, n_layers: int, batch: int, n_kv_heads: int, group_size: int,
                 d_head: int, seq_cap: int, roles, policy: SparsityPolicy,
                 dtype: torch.dtype = torch.bfloat16, world: int = 1, rank: int = 0,
                 num_splits: int = 0, group=None, recv: Optional[torch.Tensor] = None,
                 exchange: Optional[Callable] = None):
        self.dec = HybridDecoder(n_layers=n_layers, batch=batch, n_kv_heads=n_kv_heads,
                                 group_size=group_size, d_head=d_head, seq_cap=seq_cap,
                                 roles=roles, policy=policy, dtype=dtype, select="tokens",
                                 num_splits=num_splits)
        self.world, self.rank, self.group = world, rank, group
        self.n_layers = n_layers
        ids, _ = self.dec.index_cache()
        self.k_cap = ids.shape[1]
        self.rows = batch * n_kv_heads * group_size
        self.bh = batch * n_kv_heads
        d = d_head
        # packed per-rank block, 4-byte words: o [rows*d] | lse [rows] | key [bh*k_cap] | id [bh*k_cap]
        self.off_lse = self.rows * d
        self.off_key = self.off_lse + self.rows
        self.off_idx = self.off_key + self.bh * self.k_cap
        words = self.off_idx + self.bh * self.k_cap
        self.block_words = (words + 3) // 4 * 4
        dev = torch.device("cuda", torch.cuda.current_device())
        if recv is None:
            recv = torch.empty(world * self.block_words, dtype=torch.float32, device=dev)
        self.recv = recv
        self.send = recv[rank * self.block_words:(rank + 1) * self.block_words] \
            if exchange is False else torch.empty(self.block_words, dtype=torch.float32, device=dev)
        self.exchange = exchange

    def _ptr(self, t: torch.Tensor, word: int) -> int:
        return t.data_ptr() + 4 * word

    def layer_local(self, l: int, q_l, k_cache, v_cache, n_local: int, row_begin: int, *,
                    stream=None):
        """Step 1: local partials + candidates into this rank's send block."""
        st = HybridDecoder._stream(stream)
        s = self.send
        check(lib().lyc_shard_layer(self.dec._h, l, q_l.data_ptr(), k_cache.data_ptr(),
                                    v_cache.data_ptr(), n_local, row_begin, self._ptr(s, 0),
                                    self._ptr(s, self.off_lse), self._ptr(s, self.off_key),
                                    self._ptr(s, self.off_idx), st))

    def gather(self):
        """Step 2: one packed all-gather (rank order)."""
        if self.exchange is False:  # send is a view into the shared recv
            return
        if self.exchange is not None:
            self.exchange(self.send, self.recv)
        else:
            import torch.distributed as dist
            dist.all_gather_into_tensor(self.recv, self.send, group=self.group)

    def layer_combine(self, l: int, out_l, n_local: int, row_begin: int, seq_total: int,
                      global_sets: Optional[torch.Tensor] = None, *, stream=None):
        """Step 3: identical on every rank -- merged output and global set."""
        st = HybridDecoder._stream(stream)
        r = self.recv
        check(lib().lyc_shard_merge(
            self.dec._h, l, self.world, self._ptr(r, 0), self._ptr(r, self.off_lse),
            self._ptr(r, self.off_key), self._ptr(r, self.off_idx), self.block_words, n_local,
            row_begin, seq_total, out_l.data_ptr(),
            global_sets.data_ptr() if global_sets is not None else None, st))

    def decode_step(self, q, k_cache, v_cache, n_local: int, row_begin: int, seq_total: int,
                    out=None, global_sets: Optional[torch.Tensor] = None, *, stream=None):
        """All layers: q/out [L][B][Hq][d]; k/v this rank's [L][B][H][seq_cap][d]
        (local row 0 = global row row_begin).  global_sets: optional
        [L][B*H][k_cap] int32 receiving each layer's global sets."""
        if out is None:
            out = torch.empty_like(q)
        for l in range(self.n_layers):
            self.layer_local(l, q[l], k_cache, v_cache, n_local, row_begin, stream=stream)
            self.gather()
            self.layer_combine(l, out[l], n_local, row_begin, seq_total,
                               global_sets[l] if global_sets is not None else None, stream=stream)
        return out

    def close(self):
        self.dec.close()


def emulate_step(decoders, q, k_full, v_full, seq_total: int, out=None, global_sets=None):
    """Run a P-rank sequence-sharded step on ONE GPU: rank p's cache is the row
    slice [row_begin, row_begin + n_local) of the full cache (same slab stride),
    all ranks share one gathered buffer.  Returns the outputs of every rank
    ([P][L][B][Hq][d]) -- identical by construction -- for checking."""
    P = len(decoders)
    outs = [torch.empty_like(q) for _ in range(P)]
    d = q.shape[-1]
    for l in range(decoders[0].n_layers):
        for p, sd in enumerate(decoders):
            rb, nl = shard_rows(seq_total, P, p)
            sd.layer_local(l, q[l], k_full[..., rb:, :], v_full[..., rb:, :], nl, rb)
        for p, sd in enumerate(decoders):
            rb, nl = shard_rows(seq_total, P, p)
            gs = global_sets[p][l] if global_sets is not None else None
            sd.layer_combine(l, outs[p][l], nl, rb, seq_total, gs)
    del d
    return outs


__all__ = ["ShardedDecoder", "emulate_step", "shard_rows"]
