// window.cu -- the split merge of the cache-correction window attention
// (window_tc.cu computes the splits on the tensor cores) and the fp32-cache
// path for small configs (decode_engine.hpp:164-204).
#include <algorithm>

#include "lyc_common.cuh"
#include "lyc_plan.h"

namespace lyc {

constexpr int kWinRows = 128;  // rows per split partial block (= window_tc.cu kTcRows)

// Merge the splits of every row (one warp per row, lanes over d) and write
// the row to out[b][i][g*G + j].
struct WinMergeParams {
  const float* part_o;      // [B*H][rb][n_split][128][d]
  const float* part_lse;    // [B*H][rb][n_split][128]
  int32_t B, H, G, W, rows, rb, n_split;
};

__global__ void window_merge_kernel(const __grid_constant__ WinMergeParams p, int d,
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

cudaError_t launch_window_merge(const float* part_o, const float* part_lse, int B, int H, int G,
                                int W, int rows, int rb, int n_split, int d, void* out,
                                cudaStream_t st) {
  WinMergeParams p;
  p.part_o = part_o;
  p.part_lse = part_lse;
  p.B = B;
  p.H = H;
  p.G = G;
  p.W = W;
  p.rows = rows;
  p.rb = rb;
  p.n_split = n_split;
  const int64_t warps = (int64_t)B * H * rows;
  window_merge_kernel<<<(unsigned)((warps + 7) / 8), 256, 0, st>>>(p, d,
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

}  // namespace lyc
