// model.cu -- the decode-step operations that surround the attention in the
// reference's toy model (toy_model.hpp:161-274):
// rmsnorm, the Q/K/V projections with rotary embedding, the output projection
// with its residual, the FFN (W2 silu(W1 h)) with its residual and the logits.
// At batch 1 every one of them is a GEMV over a bf16 weight matrix -- bound by
// the HBM stream of the weights -- so each is ONE kernel with the small
// vector work fused into its prologue (rmsnorm of the residual stream, staged
// in shared memory per CTA) and epilogue (residual add, silu, rotary
// embedding + the new token's K/V rows written into the attention cache).
//
// Weights are stored [out][in] (row-major per output), the transpose of the
// reference's Matrix<float> [in][out] (matvec_f, toy_model.hpp:171-180):
// y_j = sum_i x_i W[i][j] -- the same sums, coalesced per output row.
//
// GEMV: 8 warps per CTA, each warp two adjacent output rows at a time (a
// rotary pair stays in one warp); lanes stream 16-B chunks of both rows with
// eight loads in flight per row, dot them with the fp32 input vector in
// shared memory, and reduce with shuffles.
#include <algorithm>

#include "lyc_common.cuh"
#include "lyc_plan.h"

namespace lyc {

constexpr int kGemvThreads = 256;
constexpr int kGemvUnroll = 8;  // 16-B chunks in flight per row per lane

enum { GEMV_STORE = 0, GEMV_RESIDUAL = 1, GEMV_SILU_BF16 = 2, GEMV_QKV_ROPE = 3 };  // = LYC_GEMV_*


__device__ __forceinline__ uint4 ld_stream(const void* p) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p));
  return v;
}

__device__ __forceinline__ float dot8(const uint4& w, const float* x) {
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&w);
  const float4 x0 = *reinterpret_cast<const float4*>(x);
  const float4 x1 = *reinterpret_cast<const float4*>(x + 4);
  const float2 a = __bfloat1622float2(h[0]), b = __bfloat1622float2(h[1]);
  const float2 c = __bfloat1622float2(h[2]), e = __bfloat1622float2(h[3]);
  float s = a.x * x0.x;
  s = fmaf(a.y, x0.y, s);
  s = fmaf(b.x, x0.z, s);
  s = fmaf(b.y, x0.w, s);
  s = fmaf(c.x, x1.x, s);
  s = fmaf(c.y, x1.y, s);
  s = fmaf(e.x, x1.z, s);
  return fmaf(e.y, x1.w, s);
}

// The epilogue of one row pair (lane 0 of its warp).
__device__ __forceinline__ void gemv_epilogue(const LycGemvParams& p, int64_t r0, bool two,
                                              float s0, float s1) {
  {  // (one block: the modes are exclusive)
    if (p.mode == GEMV_STORE) {
      p.y[r0] = s0;
      if (two) p.y[r0 + 1] = s1;
    } else if (p.mode == GEMV_RESIDUAL) {
      p.y[r0] += s0;
      if (two) p.y[r0 + 1] += s1;
    } else if (p.mode == GEMV_SILU_BF16) {
      __nv_bfloat16* yb = static_cast<__nv_bfloat16*>(p.yb);
      yb[r0] = __float2bfloat16_rn(s0 / (1.f + __expf(-s0)));
      if (two) yb[r0 + 1] = __float2bfloat16_rn(s1 / (1.f + __expf(-s1)));
    } else {  // GEMV_QKV_ROPE (d even: a rotary pair never straddles heads)
      const int d = p.d;
      const int64_t qk_rows = (int64_t)(p.nq + p.nkv) * d;
      float y0 = s0, y1 = s1;
      if (r0 < qk_rows) {  // toy_model.hpp:184-194: pair (i, i+1), freq 10000^(-i/d)
        const int i = (int)(r0 % d);
        const double freq = pow(10000.0, -(double)i / (double)d);
        double sn, cs;
        sincos((double)p.pos * freq, &sn, &cs);
        y0 = (float)((double)s0 * cs - (double)s1 * sn);
        y1 = (float)((double)s0 * sn + (double)s1 * cs);
      }
      const int64_t qrows = (int64_t)p.nq * d;
      if (r0 < qrows) {
        __nv_bfloat16* q = static_cast<__nv_bfloat16*>(p.q_out);
        q[r0] = __float2bfloat16_rn(y0);
        q[r0 + 1] = __float2bfloat16_rn(y1);
      } else {
        const bool is_k = r0 < qk_rows;
        const int64_t rr = r0 - (is_k ? qrows : qk_rows);
        const int g = (int)(rr / d), i = (int)(rr % d);
        __nv_bfloat16* dst = static_cast<__nv_bfloat16*>(is_k ? p.k_cache : p.v_cache) +
                             g * p.slab_stride + p.pos * d + i;
        dst[0] = __float2bfloat16_rn(y0);
        dst[1] = __float2bfloat16_rn(y1);
      }
    }
  }
}

// This warp's share of the next launch's weights into L2 (bulk prefetches
// through the TMA engine; fire and forget), after its own rows.
__device__ __forceinline__ void gemv_prefetch_next(const LycGemvParams& p, int warp, int lane) {
  if (p.pf && lane == 0) {
    const int64_t warps = (int64_t)gridDim.x * (kGemvThreads / 32);
    const int64_t wid = (int64_t)blockIdx.x * (kGemvThreads / 32) + warp;
    const int64_t share = ((p.pf_bytes / 16 + warps - 1) / warps) * 16;
    const int64_t b0 = wid * share, b1 = b0 + share < p.pf_bytes ? b0 + share : p.pf_bytes;
    for (int64_t b = b0; b < b1; b += 65536) {
      const uint32_t n = (uint32_t)(b1 - b < 65536 ? b1 - b : 65536);
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(static_cast<const char*>(p.pf) + b),
                   "r"(n)
                   : "memory");
    }
  }
}

// The input vector into shared memory, rmsnorm'ed when a gain is given
// (toy_model.hpp:161-169: x * inv_rms * gain, eps 1e-6); all threads of the
// CTA, ends with a barrier.
__device__ __forceinline__ void gemv_stage_x(const LycGemvParams& p, float* xs, float* red, int tid,
                                             int warp, int lane) {
  const int K = (int)p.K;
  // 16-B vectors, kPro of them in flight per thread before any is used: one
  // L2 round trip per kPro * 256 vectors (K = 4096: one) -- an element loop
  // would wait for every load in turn.
  constexpr int kPro = 4;
  float ss = 0.f;
  if (p.x) {
    const float4* x4 = reinterpret_cast<const float4*>(p.x);
    for (int c0 = tid; c0 < K / 4; c0 += kGemvThreads * kPro) {
      float4 v[kPro];
#pragma unroll
      for (int u = 0; u < kPro; ++u)
        if (c0 + u * kGemvThreads < K / 4) v[u] = __ldcg(x4 + c0 + u * kGemvThreads);
#pragma unroll
      for (int u = 0; u < kPro; ++u) {
        const int c = c0 + u * kGemvThreads;
        if (c < K / 4) {
          reinterpret_cast<float4*>(xs)[c] = v[u];
          ss = fmaf(v[u].x, v[u].x, fmaf(v[u].y, v[u].y, fmaf(v[u].z, v[u].z, fmaf(v[u].w, v[u].w, ss))));
        }
      }
    }
  } else {
    const uint4* x8 = static_cast<const uint4*>(p.xb);
    for (int c0 = tid; c0 < K / 8; c0 += kGemvThreads * kPro) {
      uint4 v[kPro];
#pragma unroll
      for (int u = 0; u < kPro; ++u)
        if (c0 + u * kGemvThreads < K / 8) v[u] = __ldcg(x8 + c0 + u * kGemvThreads);
#pragma unroll
      for (int u = 0; u < kPro; ++u) {
        const int c = c0 + u * kGemvThreads;
        if (c < K / 8) {
          const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&v[u]);
          float f[8];
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const float2 t = __bfloat1622float2(h[e]);
            f[2 * e] = t.x;
            f[2 * e + 1] = t.y;
          }
          reinterpret_cast<float4*>(xs)[2 * c] = make_float4(f[0], f[1], f[2], f[3]);
          reinterpret_cast<float4*>(xs)[2 * c + 1] = make_float4(f[4], f[5], f[6], f[7]);
#pragma unroll
          for (int e = 0; e < 8; ++e) ss = fmaf(f[e], f[e], ss);
        }
      }
    }
  }
  if (p.gain) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, off);
    if (lane == 0) red[warp] = ss;
    __syncthreads();
    float tot = 0.f;
#pragma unroll
    for (int w = 0; w < kGemvThreads / 32; ++w) tot += red[w];
    const float inv = rsqrtf(tot / (float)K + p.eps);
    const float4* g4 = reinterpret_cast<const float4*>(p.gain);
    for (int c0 = tid; c0 < K / 4; c0 += kGemvThreads * kPro) {
      float4 g[kPro];
#pragma unroll
      for (int u = 0; u < kPro; ++u)
        if (c0 + u * kGemvThreads < K / 4) g[u] = __ldg(g4 + c0 + u * kGemvThreads);
#pragma unroll
      for (int u = 0; u < kPro; ++u) {
        const int c = c0 + u * kGemvThreads;
        if (c < K / 4) {
          float4 v = reinterpret_cast<float4*>(xs)[c];
          v.x = v.x * inv * g[u].x;
          v.y = v.y * inv * g[u].y;
          v.z = v.z * inv * g[u].z;
          v.w = v.w * inv * g[u].w;
          reinterpret_cast<float4*>(xs)[c] = v;
        }
      }
    }
  }
  __syncthreads();
}

__global__ void __launch_bounds__(kGemvThreads) gemv_kernel(const __grid_constant__ LycGemvParams p) {
  extern __shared__ float xs[];  // [K] the (normalised) input vector
  __shared__ float red[kGemvThreads / 32];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int K = (int)p.K;
  const int64_t pairs = (p.M + 1) / 2;
  const int chunks = K / 8;
  // ---- the first weight chunks of this warp's first row pair are loaded
  // before waiting for the previous kernel (programmatic dependent launch):
  // weights do not depend on it, so their HBM stream overlaps its tail
  int64_t pr = (int64_t)blockIdx.x * (kGemvThreads / 32) + warp;
  uint4 a[kGemvUnroll], b[kGemvUnroll];
  auto load_batch = [&](int64_t r0, int c0) {
    const bool two = r0 + 1 < p.M;
    const __nv_bfloat16* w0 = static_cast<const __nv_bfloat16*>(p.w) + r0 * p.K;
    const __nv_bfloat16* w1 = two ? w0 + p.K : w0;
#pragma unroll
    for (int u = 0; u < kGemvUnroll; ++u) {
      const int c = c0 + u * 32;
      if (c < chunks) {
        a[u] = ld_stream(w0 + (int64_t)c * 8);
        b[u] = ld_stream(w1 + (int64_t)c * 8);
      }
    }
  };
  if (pr < pairs) load_batch(2 * pr, lane);
  pdl_wait();
  gemv_stage_x(p, xs, red, tid, warp, lane);
  // ---- two adjacent rows per warp
  bool first = true;
  for (; pr < pairs; pr += (int64_t)gridDim.x * (kGemvThreads / 32)) {
    const int64_t r0 = 2 * pr;
    const bool two = r0 + 1 < p.M;
    float s0 = 0.f, s1 = 0.f;
    for (int c0 = lane; c0 < chunks; c0 += 32 * kGemvUnroll) {
      if (!first) load_batch(r0, c0);  // (the first batch was loaded before the wait)
      first = false;
#pragma unroll
      for (int u = 0; u < kGemvUnroll; ++u) {
        const int c = c0 + u * 32;
        if (c < chunks) {
          s0 += dot8(a[u], xs + c * 8);
          s1 += dot8(b[u], xs + c * 8);
        }
      }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      s0 += __shfl_xor_sync(0xffffffffu, s0, off);
      s1 += __shfl_xor_sync(0xffffffffu, s1, off);
    }
    if (lane != 0) continue;
    gemv_epilogue(p, r0, two, s0, s1);
  }
  // this CTA's rows are done: when another GEMV follows, its CTAs may be
  // scheduled as the SM frees up (they still wait for this grid's completion
  // before reading its outputs).  A trigger at the start was slower (its CTAs
  // competed with this grid's streaming); this one saves ~3 % of the GEMV
  // chain (the toy model's step, whose GEMV chains alternate with the
  // attention step, does not set the flag: 6 % slower with it).
  if (p.flags & 1) pdl_trigger();
  gemv_prefetch_next(p, warp, lane);
}

cudaError_t launch_gemv(const LycGemvParams& p, int n_sms, cudaStream_t st) {
  const size_t smem = (size_t)p.K * 4;
  static bool configured_[64] = {};
  bool& configured = device_flag(configured_);
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(gemv_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         200 * 1024);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  const int64_t pairs = (p.M + 1) / 2;
  const int64_t need = (pairs + kGemvThreads / 32 - 1) / (kGemvThreads / 32);
  // one wave of resident CTAs (registers and the input vector's shared
  // memory bound them) with a grid-stride loop: a second wave would compete
  // with the next kernel's early (programmatic-dependent) CTAs for the slots
  int per_sm = 1;
  cudaError_t oe = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, gemv_kernel, kGemvThreads, smem);
  if (oe != cudaSuccess) return oe;
  per_sm = std::max(1, per_sm);
  const int grid = (int)std::min<int64_t>(need, (int64_t)n_sms * per_sm);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kGemvThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, gemv_kernel, p);
}

}  // namespace lyc
