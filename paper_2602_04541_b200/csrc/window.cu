// window.cu -- causal window attention for cache correction
// (decode_engine.hpp:164-204): the last W decoded
// positions are re-run densely after their K/V rows were rewritten
// (kv_cache.hpp:34-42, lyc_kv_write): position p = start + i attends keys
// [0, p] (the rewritten rows of earlier window positions included).
//
// Per (b, KV head g) the W x G query rows form one M = W*G block (<= 128 rows
// per CTA, 8 warps x 16 rows), so every K/V tile is read from HBM once for all
// of them -- a prefill-style flash-attention pass over the cache with a causal
// edge, not W decode passes.  The key range is split across CTAs
// (flash-decoding); a second kernel merges the splits (base-2 LSE) and writes
// the rows back in the caller's [B][W][Hq][d] layout.
//   * tiles of 64 keys, cp.async double buffer, 16-B chunks XOR-swizzled by
//     row (conflict-free ldmatrix);
//   * S = Q K^T and O += P V with mma.sync m16n8k16 (bf16 -> fp32), P kept in
//     registers (C fragment -> A fragment);
//   * online softmax in the exp2 domain, two rows per thread.
#include <algorithm>

#include "lyc_common.cuh"
#include "lyc_plan.h"

namespace lyc {

constexpr int kWinRows = 128;  // query rows per CTA (8 warps x 16)
constexpr int kWinThreads = 256;
constexpr int kWinTile = 64;   // keys per tile

template <int D>
struct WinSmem {
  __nv_bfloat16 q[kWinRows * D];
  __nv_bfloat16 k[2][kWinTile * D];
  __nv_bfloat16 v[2][kWinTile * D];
};

// byte offset of 16-B chunk c of row r in a [rows][D] bf16 tile, swizzled
template <int D>
__device__ __forceinline__ uint32_t win_off(int r, int c) {
  return (uint32_t)(r * (D * 2) + ((c ^ (r & 7)) << 4));
}

struct WinParams {
  const __nv_bfloat16* q;   // [B][W][Hq][D]
  const __nv_bfloat16* k;   // cache [L][B][H][cap][D]
  const __nv_bfloat16* v;
  float* part_o;            // [B*H][rb][n_split][128][D]
  float* part_lse;          // [B*H][rb][n_split][128]
  int64_t slab0;            // element offset of (layer, b=0, g=0) row 0
  int64_t cap;
  int32_t B, H, G, W, rows, rb, n_split;
  int64_t start;            // first window position
  int64_t keys;             // start + W
  int64_t split_keys;       // keys per split (multiple of kWinTile)
  float scale_log2;
};

template <int D>
__global__ void __launch_bounds__(kWinThreads, 1) window_attn_kernel(const __grid_constant__ WinParams p) {
  extern __shared__ uint8_t win_raw[];
  WinSmem<D>& sm = *reinterpret_cast<WinSmem<D>*>(win_raw);
  constexpr int CH = D / 8;  // 16-B chunks per row
  constexpr int KS = D / 16;
  const int split = blockIdx.x, bh = blockIdx.y, rblk = blockIdx.z;
  const int b = bh / p.H, g = bh - b * p.H;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int row0 = rblk * kWinRows;
  const int nrows = min(kWinRows, p.rows - row0);
  const int64_t k_lo = (int64_t)split * p.split_keys;
  const int64_t k_hi = min(p.keys, k_lo + p.split_keys);
  const int64_t slab = p.slab0 + ((int64_t)b * p.H + g) * p.cap * D;

  // stage Q rows r = i*G + j -> q[b][i][g*G + j]
  for (int x = tid; x < kWinRows * CH; x += kWinThreads) {
    const int r = x / CH, c = x - r * CH;
    const int rr = row0 + r;
    const void* src = p.q;
    uint32_t bytes = 0;
    if (r < nrows) {
      const int i = rr / p.G, j = rr - i * p.G;
      src = p.q + (((int64_t)b * p.W + i) * (p.H * p.G) + g * p.G + j) * D + c * 8;
      bytes = 16;
    }
    cp_async_16(reinterpret_cast<uint8_t*>(sm.q) + win_off<D>(r, c), src, bytes);
  }
  auto load_tile = [&](int buf, int64_t t0) {
    for (int x = tid; x < kWinTile * CH; x += kWinThreads) {
      const int r = x / CH, c = x - r * CH;
      const int64_t key = t0 + r;
      const bool ok = key < k_hi;
      const int64_t off = slab + (ok ? key : 0) * D + c * 8;
      cp_async_16(reinterpret_cast<uint8_t*>(sm.k[buf]) + win_off<D>(r, c), p.k + off, ok ? 16u : 0u);
      cp_async_16(reinterpret_cast<uint8_t*>(sm.v[buf]) + win_off<D>(r, c), p.v + off, ok ? 16u : 0u);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  const int ntiles = k_hi > k_lo ? (int)((k_hi - k_lo + kWinTile - 1) / kWinTile) : 0;
  if (ntiles > 0) load_tile(0, k_lo);
  else asm volatile("cp.async.commit_group;" ::: "memory");

  // this thread's two rows (g, g + 8 of the warp's 16) and their causal limits
  const int qg = lane >> 2, qt = lane & 3;
  const int ra = row0 + warp * 16 + qg, rb2 = ra + 8;
  const int64_t lim_a = ra < p.rows ? p.start + ra / p.G : -1;
  const int64_t lim_b = rb2 < p.rows ? p.start + rb2 / p.G : -1;

  float m_a = -INFINITY, m_b = -INFINITY, l_a = 0.f, l_b = 0.f;
  float o[D / 8][4];
#pragma unroll
  for (int n = 0; n < D / 8; ++n) o[n][0] = o[n][1] = o[n][2] = o[n][3] = 0.f;
  uint32_t qa[KS][4];
  bool q_loaded = false;

  for (int ti = 0; ti < ntiles; ++ti) {
    const int buf = ti & 1;
    const int64_t t0 = k_lo + (int64_t)ti * kWinTile;
    if (ti + 1 < ntiles) {
      load_tile(buf ^ 1, t0 + kWinTile);
      asm volatile("cp.async.wait_group 1;" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;" ::: "memory");
    }
    __syncthreads();
    if (!q_loaded) {  // A fragments of the warp's 16 rows, once
      const uint8_t* qs = reinterpret_cast<const uint8_t*>(sm.q);
      const int r = warp * 16 + (lane & 7) + ((lane >> 3) & 1) * 8;
#pragma unroll
      for (int kk = 0; kk < KS; ++kk)
        ldsm_x4(qa[kk][0], qa[kk][1], qa[kk][2], qa[kk][3], qs + win_off<D>(r, kk * 2 + (lane >> 4)));
      q_loaded = true;
    }
    const uint8_t* ks = reinterpret_cast<const uint8_t*>(sm.k[buf]);
    const uint8_t* vs = reinterpret_cast<const uint8_t*>(sm.v[buf]);
    // ---- S = Q K^T: 8 n-tiles of 8 keys
    float s[8][4];
#pragma unroll
    for (int n = 0; n < 8; ++n) s[n][0] = s[n][1] = s[n][2] = s[n][3] = 0.f;
#pragma unroll
    for (int kk = 0; kk < KS; ++kk) {
#pragma unroll
      for (int n2 = 0; n2 < 4; ++n2) {  // two n-tiles per ldmatrix.x4
        uint32_t b0, b1, b2, b3;
        const int key = n2 * 16 + (lane & 7) + (lane >> 4) * 8;
        ldsm_x4(b0, b1, b2, b3, ks + win_off<D>(key, kk * 2 + ((lane >> 3) & 1)));
        mma_bf16(s[2 * n2], qa[kk][0], qa[kk][1], qa[kk][2], qa[kk][3], b0, b1);
        mma_bf16(s[2 * n2 + 1], qa[kk][0], qa[kk][1], qa[kk][2], qa[kk][3], b2, b3);
      }
    }
    // ---- mask (split end, causal limit) and online softmax, rows a and b
    float mx_a = -INFINITY, mx_b = -INFINITY;
#pragma unroll
    for (int n = 0; n < 8; ++n) {
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        const int64_t key = t0 + n * 8 + 2 * qt + c;
        const bool in = key < k_hi;
        s[n][c] = (in && key <= lim_a) ? s[n][c] * p.scale_log2 : -INFINITY;
        s[n][2 + c] = (in && key <= lim_b) ? s[n][2 + c] * p.scale_log2 : -INFINITY;
        mx_a = fmaxf(mx_a, s[n][c]);
        mx_b = fmaxf(mx_b, s[n][2 + c]);
      }
    }
    mx_a = fmaxf(mx_a, __shfl_xor_sync(0xffffffffu, mx_a, 1));
    mx_a = fmaxf(mx_a, __shfl_xor_sync(0xffffffffu, mx_a, 2));
    mx_b = fmaxf(mx_b, __shfl_xor_sync(0xffffffffu, mx_b, 1));
    mx_b = fmaxf(mx_b, __shfl_xor_sync(0xffffffffu, mx_b, 2));
    const float mn_a = fmaxf(m_a, mx_a), mn_b = fmaxf(m_b, mx_b);
    const float rs_a = m_a == -INFINITY ? 0.f : fast_exp2(m_a - mn_a);
    const float rs_b = m_b == -INFINITY ? 0.f : fast_exp2(m_b - mn_b);
    const float mu_a = mn_a == -INFINITY ? 0.f : mn_a, mu_b = mn_b == -INFINITY ? 0.f : mn_b;
    float sum_a = 0.f, sum_b = 0.f;
#pragma unroll
    for (int n = 0; n < 8; ++n) {
      s[n][0] = fast_exp2(s[n][0] - mu_a);
      s[n][1] = fast_exp2(s[n][1] - mu_a);
      s[n][2] = fast_exp2(s[n][2] - mu_b);
      s[n][3] = fast_exp2(s[n][3] - mu_b);
      sum_a += s[n][0] + s[n][1];
      sum_b += s[n][2] + s[n][3];
    }
    l_a = l_a * rs_a + sum_a;
    l_b = l_b * rs_b + sum_b;
    m_a = mn_a;
    m_b = mn_b;
#pragma unroll
    for (int n = 0; n < D / 8; ++n) {
      o[n][0] *= rs_a;
      o[n][1] *= rs_a;
      o[n][2] *= rs_b;
      o[n][3] *= rs_b;
    }
    // ---- O += P V: 4 k-steps of 16 keys, P from registers
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const uint32_t a0 = pack_bf16(s[2 * j][0], s[2 * j][1]);
      const uint32_t a1 = pack_bf16(s[2 * j][2], s[2 * j][3]);
      const uint32_t a2 = pack_bf16(s[2 * j + 1][0], s[2 * j + 1][1]);
      const uint32_t a3 = pack_bf16(s[2 * j + 1][2], s[2 * j + 1][3]);
#pragma unroll
      for (int n2 = 0; n2 < D / 16; ++n2) {  // two n-tiles of 8 dims per ldmatrix.x4.trans
        uint32_t b0, b1, b2, b3;
        const int key = j * 16 + (lane & 7) + ((lane >> 3) & 1) * 8;
        ldsm_x4_t(b0, b1, b2, b3, vs + win_off<D>(key, n2 * 2 + (lane >> 4)));
        mma_bf16(o[2 * n2], a0, a1, a2, a3, b0, b1);
        mma_bf16(o[2 * n2 + 1], a0, a1, a2, a3, b2, b3);
      }
    }
    __syncthreads();  // the buffer is refilled next iteration
  }
  // ---- partials: normalized o and base-2 LSE per row
  l_a += __shfl_xor_sync(0xffffffffu, l_a, 1);
  l_a += __shfl_xor_sync(0xffffffffu, l_a, 2);
  l_b += __shfl_xor_sync(0xffffffffu, l_b, 1);
  l_b += __shfl_xor_sync(0xffffffffu, l_b, 2);
  const int64_t unit = ((int64_t)bh * p.rb + rblk) * p.n_split + split;
  float* po = p.part_o + unit * kWinRows * D;
  float* pl = p.part_lse + unit * kWinRows;
  const int la = warp * 16 + qg, lb = la + 8;
  const float ia = l_a > 0.f ? 1.f / l_a : 0.f, ib = l_b > 0.f ? 1.f / l_b : 0.f;
#pragma unroll
  for (int n = 0; n < D / 8; ++n) {
    const int c = n * 8 + 2 * qt;
    *reinterpret_cast<float2*>(po + (int64_t)la * D + c) = make_float2(o[n][0] * ia, o[n][1] * ia);
    *reinterpret_cast<float2*>(po + (int64_t)lb * D + c) = make_float2(o[n][2] * ib, o[n][3] * ib);
  }
  if (qt == 0) {
    pl[la] = l_a > 0.f ? log2f(l_a) + m_a : -INFINITY;
    pl[lb] = l_b > 0.f ? log2f(l_b) + m_b : -INFINITY;
  }
}

// Merge the splits of every row (one warp per row, lanes over d) and write
// the row to out[b][i][g*G + j].
__global__ void window_merge_kernel(const __grid_constant__ WinParams p, int d,
                                    __nv_bfloat16* __restrict__ out) {
  const int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int64_t total = (int64_t)p.B * p.H * p.rows;
  if (w >= total) return;
  const int bh = (int)(w / p.rows), r = (int)(w - (int64_t)bh * p.rows);
  const int rblk = r / kWinRows, rr = r - rblk * kWinRows;
  const int64_t u0 = ((int64_t)bh * p.rb + rblk) * p.n_split;
  float M = -INFINITY;
  for (int s = 0; s < p.n_split; ++s) M = fmaxf(M, p.part_lse[(u0 + s) * kWinRows + rr]);
  const float Mz = M == -INFINITY ? 0.f : M;
  float den = 0.f;
  float acc[4] = {0.f, 0.f, 0.f, 0.f};
  for (int s = 0; s < p.n_split; ++s) {
    const float ls = p.part_lse[(u0 + s) * kWinRows + rr];
    const float wgt = ls == -INFINITY ? 0.f : exp2f(ls - Mz);
    den += wgt;
    const float* po = p.part_o + ((u0 + s) * kWinRows + rr) * d;
#pragma unroll
    for (int c = 0; c < 4; ++c)
      if (c * 32 + lane < d) acc[c] = fmaf(wgt, po[c * 32 + lane], acc[c]);
  }
  const int b = bh / p.H, g = bh - b * p.H;
  const int i = r / p.G, j = r - i * p.G;
  __nv_bfloat16* dst = out + (((int64_t)b * p.W + i) * (p.H * p.G) + g * p.G + j) * d;
#pragma unroll
  for (int c = 0; c < 4; ++c)
    if (c * 32 + lane < d) dst[c * 32 + lane] = __float2bfloat16_rn(den > 0.f ? acc[c] / den : 0.f);
}

int64_t window_workspace_bytes(int B, int H, int G, int W, int n_split) {
  const int rows = W * G, rb = (rows + kWinRows - 1) / kWinRows;
  const int64_t units = (int64_t)B * H * rb * n_split;
  return units * kWinRows * (128 + 1) * 4;  // d <= 128
}

template <int D>
static cudaError_t launch_window_t(const WinParams& p, void* out, cudaStream_t st) {
  static bool configured_[64] = {};
  bool& configured = device_flag(configured_);
  const int smem = (int)sizeof(WinSmem<D>);
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(window_attn_kernel<D>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  window_attn_kernel<D><<<dim3(p.n_split, p.B * p.H, p.rb), kWinThreads, smem, st>>>(p);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  const int64_t warps = (int64_t)p.B * p.H * p.rows;
  window_merge_kernel<<<(unsigned)((warps + 7) / 8), 256, 0, st>>>(p, D,
                                                                     static_cast<__nv_bfloat16*>(out));
  return cudaGetLastError();
}

// fp32 caches (small configs): one warp per window row, keys in chunks of 32
// (a lane per key for the scores, lanes over d for P V), online softmax.
__global__ void window_attn_f32_kernel(const float* __restrict__ q, const float* __restrict__ k,
                                       const float* __restrict__ v, int64_t slab0, int64_t cap,
                                       int B, int H, int G, int W, int d, int64_t start,
                                       float scale, float* __restrict__ out) {
  extern __shared__ float qs_all[];
  const int wib = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t row = (int64_t)blockIdx.x * (blockDim.x >> 5) + wib;  // (b, i, hq)
  const int Hq = H * G;
  if (row >= (int64_t)B * W * Hq) return;
  const int hq = (int)(row % Hq), i = (int)((row / Hq) % W), b = (int)(row / ((int64_t)Hq * W));
  const int g = hq / G;
  float* qs = qs_all + wib * d;
  const float* qr = q + row * d;
  for (int c = lane; c < d; c += 32) qs[c] = qr[c];
  __syncwarp();
  const float* ks = k + slab0 + ((int64_t)b * H + g) * cap * d;
  const float* vs = v + slab0 + ((int64_t)b * H + g) * cap * d;
  const int64_t n = start + i + 1;  // keys [0, start + i]
  float m = -INFINITY, l = 0.f, o[4] = {0.f, 0.f, 0.f, 0.f};
  for (int64_t t0 = 0; t0 < n; t0 += 32) {
    const int64_t t = t0 + lane;
    float sc = -INFINITY;
    if (t < n) {
      float acc = 0.f;
      for (int c = 0; c < d; ++c) acc = fmaf(qs[c], ks[t * d + c], acc);
      sc = acc * scale;
    }
    float mx = sc;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, off));
    const float mn = fmaxf(m, mx);
    const float rs = m == -INFINITY ? 0.f : expf(m - mn);
    const float w = t < n ? expf(sc - mn) : 0.f;
    float ws = w;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) ws += __shfl_xor_sync(0xffffffffu, ws, off);
    l = l * rs + ws;
    m = mn;
#pragma unroll
    for (int c = 0; c < 4; ++c) o[c] *= rs;
    const int cnt = (int)(n - t0 < 32 ? n - t0 : 32);
    for (int j = 0; j < cnt; ++j) {
      const float wj = __shfl_sync(0xffffffffu, w, j);
      const float* vr = vs + (t0 + j) * d;
#pragma unroll
      for (int c = 0; c < 4; ++c)
        if (c * 32 + lane < d) o[c] = fmaf(wj, vr[c * 32 + lane], o[c]);
    }
  }
  float* dst = out + row * d;
#pragma unroll
  for (int c = 0; c < 4; ++c)
    if (c * 32 + lane < d) dst[c * 32 + lane] = l > 0.f ? o[c] / l : 0.f;
}

cudaError_t launch_window_f32(const void* q, const void* k, const void* v, int layer, int B, int H,
                              int G, int d, int64_t cap, int64_t start, int W, float scale,
                              void* out, cudaStream_t st) {
  const int64_t rows = (int64_t)B * W * H * G;
  const int wpb = 8;
  window_attn_f32_kernel<<<(unsigned)((rows + wpb - 1) / wpb), wpb * 32, wpb * d * 4, st>>>(
      static_cast<const float*>(q), static_cast<const float*>(k), static_cast<const float*>(v),
      (int64_t)layer * B * H * cap * d, cap, B, H, G, W, d, start, scale, static_cast<float*>(out));
  return cudaGetLastError();
}

// q, out: [B][W][Hq][d] bf16; k, v: cache [L][B][H][cap][d] bf16.
cudaError_t launch_window(const void* q, const void* k, const void* v, int L, int layer, int B,
                          int H, int G, int d, int64_t cap, int64_t start, int W, float scale,
                          float* workspace, int n_split, void* out, cudaStream_t st) {
  WinParams p;
  p.q = static_cast<const __nv_bfloat16*>(q);
  p.k = static_cast<const __nv_bfloat16*>(k);
  p.v = static_cast<const __nv_bfloat16*>(v);
  p.B = B;
  p.H = H;
  p.G = G;
  p.W = W;
  p.rows = W * G;
  p.rb = (p.rows + kWinRows - 1) / kWinRows;
  p.cap = cap;
  p.slab0 = (int64_t)layer * B * H * cap * d;
  p.start = start;
  p.keys = start + W;
  const int64_t tiles = (p.keys + kWinTile - 1) / kWinTile;
  p.n_split = (int)std::max<int64_t>(1, std::min<int64_t>(n_split, tiles));
  p.split_keys = ((tiles + p.n_split - 1) / p.n_split) * kWinTile;
  p.n_split = (int)((p.keys + p.split_keys - 1) / p.split_keys);
  const int64_t units = (int64_t)B * H * p.rb * p.n_split;
  p.part_o = workspace;
  p.part_lse = workspace + units * kWinRows * 128;
  p.scale_log2 = scale * 1.4426950408889634f;
  (void)L;
  switch (d) {
    case 64: return launch_window_t<64>(p, out, st);
    case 128: return launch_window_t<128>(p, out, st);
  }
  return cudaErrorInvalidValue;
}

}  // namespace lyc
