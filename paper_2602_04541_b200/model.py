"""End-to-end decode step of the reference's toy model (toy_model.hpp:161-274,
decode_engine.hpp:95-151) on the device: per layer

    h = rmsnorm(x); q, k, v = W_qkv h; rotary(q, k); K/V rows -> cache   (compute_qkv)
    o = attention(q, cache)                                              (the hybrid decoder)
    x += W_o o                                                           (attn_project_residual)
    x += W_2 silu(W_1 rmsnorm(x))                                        (ffn_residual)

and logits = W_lm rmsnorm(x) (output_logits).  Every projection is one
lyc_gemv launch (csrc/model.cu: bf16 weights streamed once, the vector work
fused in), the attention one lyc_decoder_layer launch -- the per-layer call a
model makes between its own projections (end-to-end TPOT
with the surrounding GEMVs).  Weights are random bf16 with the reference
model's structure; `attention="full"` runs every head dense on the same
kernels (the full-attention baseline)."""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib as LL
from ._lib import check, lib
from .decode import HybridDecoder, SparsityPolicy


@dataclass(frozen=True)
class ModelConfig:
    """toy_model.hpp:21-46 ModelConfig (RoPE positions)."""
    n_layers: int
    n_q_heads: int
    n_kv_heads: int
    d_head: int
    d_ff: int
    vocab_size: int
    max_seq_len: int

    @property
    def d_model(self) -> int:
        return self.n_q_heads * self.d_head

    @property
    def kv_dim(self) -> int:
        return self.n_kv_heads * self.d_head

    @property
    def group_size(self) -> int:
        return self.n_q_heads // self.n_kv_heads


PRESETS = {
    # public model shapes with the toy model's two-matrix FFN (toy_model.hpp:259-267)
    "llama3-8b": dict(n_layers=32, n_q_heads=32, n_kv_heads=8, d_head=128, d_ff=14336,
                      vocab_size=128256),
    "qwen3-8b": dict(n_layers=36, n_q_heads=32, n_kv_heads=8, d_head=128, d_ff=12288,
                     vocab_size=151936),
    "tiny": dict(n_layers=4, n_q_heads=8, n_kv_heads=2, d_head=64, d_ff=256, vocab_size=512),
}


def gemv(w, x=None, xb=None, *, mode, y=None, yb=None, gain=None, eps=1e-6, q_out=None,
         k_cache=None, v_cache=None, slab_stride=0, nq=0, nkv=0, d=0, pos=0, stream=None,
         prefetch=None, prefetch_bytes=0, next_is_gemv=False):
    """One lyc_gemv launch (include/lyc.h): w bf16 [M][K]; `prefetch`: the
    next launch's weight tensor, whose first prefetch_bytes (default all) are
    pulled into L2 as this launch's warps finish; next_is_gemv: another
    lyc_gemv follows in the stream (LYC_GEMV_FLAG_NEXT_IS_GEMV)."""
    M, K = w.shape
    g = LL.lyc_gemv_desc(M=M, K=K, w=w.data_ptr(), x=x.data_ptr() if x is not None else None,
                         xb=xb.data_ptr() if xb is not None else None,
                         gain=gain.data_ptr() if gain is not None else None, eps=eps, mode=mode,
                         y=y.data_ptr() if y is not None else None,
                         yb=yb.data_ptr() if yb is not None else None,
                         q_out=q_out.data_ptr() if q_out is not None else None,
                         k_cache=k_cache.data_ptr() if k_cache is not None else None,
                         v_cache=v_cache.data_ptr() if v_cache is not None else None,
                         slab_stride=slab_stride, nq=nq, nkv=nkv, d=d,
                         flags=LL.GEMV_FLAG_NEXT_IS_GEMV if next_is_gemv else 0, pos=pos,
                         prefetch=prefetch.data_ptr() if prefetch is not None else None,
                         prefetch_bytes=(prefetch_bytes or prefetch.numel() * prefetch.element_size())
                         if prefetch is not None else 0)
    st = (stream if stream is not None else torch.cuda.current_stream()).cuda_stream
    check(lib().lyc_gemv(C.byref(g), st))


class DecodeModel:
    """A batch-1 decoder of the toy model's structure on the device (random
    bf16 weights, std 1/sqrt(fan_in)), its K/V cache, and the attention
    decoder (hybrid: the role map + policy; full: every head dense)."""

    def __init__(self, cfg: ModelConfig, *, roles=None, policy: SparsityPolicy | None = None,
                 attention: str = "hybrid", seed: int = 0, device="cuda", k_cache=None,
                 v_cache=None):
        self.cfg = cfg
        dev = torch.device(device)
        g = torch.Generator(device=dev).manual_seed(seed)
        bf = torch.bfloat16

        def w(out_dim, in_dim):
            t = torch.empty((out_dim, in_dim), dtype=bf, device=dev)
            return t.normal_(0.0, in_dim ** -0.5, generator=g)

        D, NL, H, d = cfg.d_model, cfg.n_layers, cfg.n_kv_heads, cfg.d_head
        qkv_rows = (cfg.n_q_heads + 2 * H) * d
        self.wqkv = [w(qkv_rows, D) for _ in range(NL)]
        self.wo = [w(D, D) for _ in range(NL)]
        self.w1 = [w(cfg.d_ff, D) for _ in range(NL)]
        self.w2 = [w(D, cfg.d_ff) for _ in range(NL)]
        self.attn_norm = [1 + 0.1 * torch.randn(D, generator=g, device=dev) for _ in range(NL)]
        self.ffn_norm = [1 + 0.1 * torch.randn(D, generator=g, device=dev) for _ in range(NL)]
        self.final_norm = 1 + 0.1 * torch.randn(D, generator=g, device=dev)
        self.lm_head = w(cfg.vocab_size, D)
        self.embedding = torch.empty((cfg.vocab_size, D), dtype=bf, device=dev).normal_(
            0.0, 1.0, generator=g)
        cap = cfg.max_seq_len
        if k_cache is not None:  # a caller-owned cache [NL][1][H][cap][d] bf16
            if tuple(k_cache.shape) != (NL, 1, H, cap, d) or k_cache.dtype != bf:
                raise ValueError("DecodeModel: cache must be bf16 [n_layers][1][H][max_seq_len][d]")
            self.k, self.v = k_cache, v_cache
        else:
            self.k = torch.zeros((NL, 1, H, cap, d), dtype=bf, device=dev)
            self.v = torch.zeros_like(self.k)
        self.roles, self.policy = roles, policy or SparsityPolicy.top_k(4096)
        # L2 prefetch of the next GEMV's first weight bytes (lyc_gemv_desc.prefetch);
        # 0 disables (scripts/bench_gemv_chain.py: 8 MB measured best)
        self.prefetch_bytes = 8 << 20
        # early scheduling of the next GEMV (LYC_GEMV_FLAG_NEXT_IS_GEMV): off --
        # it speeds a bare GEMV chain up by 3 % but slows this decode step
        # (interleaved with the attention step kernel) by 6 %
        # (profiles/r2_decode_gemv.md)
        self.early_next = False
        self.dec = None
        self.set_attention(attention)
        # per-token buffers
        self.x = torch.empty(D, dtype=torch.float32, device=dev)       # the residual stream
        self.q = torch.empty((NL, 1, cfg.n_q_heads, d), dtype=bf, device=dev)
        self.o = torch.empty_like(self.q)
        self.mid = torch.empty(cfg.d_ff, dtype=bf, device=dev)
        self.logits = torch.empty(cfg.vocab_size, dtype=torch.float32, device=dev)

    def set_attention(self, attention: str):
        """'hybrid' (the role map + policy) or 'full' (every head dense)."""
        cfg = self.cfg
        if attention == "full":
            roles = np.zeros((cfg.n_layers, cfg.n_kv_heads), np.uint8)
        elif self.roles is None:
            raise ValueError("hybrid attention needs a role map")
        else:
            roles = self.roles
        if self.dec is not None:
            self.dec.close()
        self.attention = attention
        self.dec = HybridDecoder(n_layers=cfg.n_layers, batch=1, n_kv_heads=cfg.n_kv_heads,
                                 group_size=cfg.group_size, d_head=cfg.d_head,
                                 seq_cap=cfg.max_seq_len, roles=roles, policy=self.policy,
                                 dtype=torch.bfloat16,
                                 select="none" if attention == "full" else "tokens")

    def fill_cache(self, length: int, seed: int = 1):
        """Synthetic history rows [0, length) (the prefill is out of scope)."""
        g = torch.Generator(device=self.k.device).manual_seed(seed)
        for t in (self.k, self.v):
            for l in range(self.cfg.n_layers):
                t[l, :, :, :length].uniform_(-1, 1, generator=g)

    def decode_token(self, token: int, pos: int, *, stream=None) -> torch.Tensor:
        """decode_engine.hpp:95-151 for one token at position pos (the cache
        holds rows [0, pos)); returns the logits (device fp32 [vocab])."""
        cfg, NL, d = self.cfg, self.cfg.n_layers, self.cfg.d_head
        H, nq = cfg.n_kv_heads, cfg.n_q_heads
        cap = cfg.max_seq_len

        def pf(w):  # the next GEMV's first weight bytes into L2 as this one finishes
            if not self.prefetch_bytes:
                return {}
            return dict(prefetch=w, prefetch_bytes=min(self.prefetch_bytes, w.numel() * 2))

        self.x.copy_(self.embedding[token].float())
        for l in range(NL):
            nxt = self.wqkv[l + 1] if l + 1 < NL else self.lm_head
            gemv(self.wqkv[l], x=self.x, gain=self.attn_norm[l], mode=LL.GEMV_QKV_ROPE,
                 q_out=self.q[l], k_cache=self.k[l, 0], v_cache=self.v[l, 0], slab_stride=cap * d,
                 nq=nq, nkv=H, d=d, pos=pos, stream=stream, **pf(self.wo[l]))
            self.dec.layer(l, self.q[l], self.k, self.v, pos + 1, self.o[l], stream=stream)
            gemv(self.wo[l], xb=self.o[l].view(-1), mode=LL.GEMV_RESIDUAL, y=self.x, stream=stream,
                 next_is_gemv=self.early_next, **pf(self.w1[l]))
            gemv(self.w1[l], x=self.x, gain=self.ffn_norm[l], mode=LL.GEMV_SILU_BF16, yb=self.mid,
                 stream=stream, next_is_gemv=self.early_next, **pf(self.w2[l]))
            gemv(self.w2[l], xb=self.mid, mode=LL.GEMV_RESIDUAL, y=self.x, stream=stream,
                 next_is_gemv=self.early_next, **pf(nxt))
        gemv(self.lm_head, x=self.x, gain=self.final_norm, mode=LL.GEMV_STORE, y=self.logits,
             stream=stream)
        return self.logits

    def weight_bytes(self) -> int:
        ts = self.wqkv + self.wo + self.w1 + self.w2 + [self.lm_head]
        return sum(t.numel() * t.element_size() for t in ts)

    def close(self):
        self.dec.close()


__all__ = ["DecodeModel", "ModelConfig", "PRESETS", "gemv"]
