// refresh.cu -- the index-set refresh of cache correction
// (decode_engine.hpp:190-197, refresh_sets_on_correction): after the window
// pass, every KV head's set is re-selected from the pooled query of the last
// window position (gqa_pool_queries, attention.hpp:127-146) against keys
// [0, len) of the layer -- selection weights of dense_attention
// (attention.hpp:50-75), which select_tokens ranks like the raw pooled scores
// (softmax is monotone).  This kernel writes the scores as order-preserving
// keys (token mode) or the max key of every 64-row block (block mode); the
// decoder's cluster top-k / policy kernels then write the index cache.
//
// HBM-bound GEMV over the K slabs: grid (row chunks, B*H), 16-B loads, one
// row per LPR lanes (a row's bytes in one coalesced request), a shuffle
// reduction over those lanes.
#include <algorithm>

#include "lyc_common.cuh"

namespace lyc {

constexpr int kRefreshThreads = 256;
constexpr int kRefreshRowsPerBlock = 1024;

template <typename T>
__device__ __forceinline__ float dot_chunk(const uint4& v, const float* q) {
  if constexpr (sizeof(T) == 2) {
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&v);
    float acc = 0.f;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float2 f = __bfloat1622float2(h[i]);
      acc = fmaf(f.x, q[2 * i], acc);
      acc = fmaf(f.y, q[2 * i + 1], acc);
    }
    return acc;
  } else {
    const float* f = reinterpret_cast<const float*>(&v);
    float acc = 0.f;
#pragma unroll
    for (int i = 0; i < 4; ++i) acc = fmaf(f[i], q[i], acc);
    return acc;
  }
}

// q: [B][Hq][d] of the last window position; k: this layer's [B][H][cap][d].
// keys [B*H][key_stride]: token mode -> key of row t; block mode -> atomicMax
// into key of block t / 64 (zeroed by the caller).
template <typename T, int D>
__global__ void __launch_bounds__(kRefreshThreads) refresh_scores_kernel(
    const T* __restrict__ q, const T* __restrict__ k, int64_t cap, int H, int G, int64_t len,
    uint32_t* __restrict__ keys, int64_t key_stride, int blocks) {
  constexpr int EPC = 16 / (int)sizeof(T);  // elements per 16-B chunk
  constexpr int CPR = D / EPC;              // chunks per row
  static_assert(CPR <= 32 && 32 % CPR == 0, "row must fit one warp");
  constexpr int RPW = 32 / CPR;             // rows per warp per step
  __shared__ float pooled[D];
  const int bh = blockIdx.y, b = bh / H, g = bh - b * H;
  const int Hq = H * G;
  // gqa_pool_queries: acc += q_j over the group, then / G (attention.hpp:138-143)
  for (int c = threadIdx.x; c < D; c += blockDim.x) {
    float acc = 0.f;
    for (int j = 0; j < G; ++j) acc += (float)q[((int64_t)b * Hq + g * G + j) * D + c];
    pooled[c] = acc / (float)G;
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int sub = lane / CPR, ch = lane - sub * CPR;
  float qc[EPC];
#pragma unroll
  for (int i = 0; i < EPC; ++i) qc[i] = pooled[ch * EPC + i];
  const T* slab = k + (int64_t)bh * cap * D;
  uint32_t* krow = keys + (int64_t)bh * key_stride;
  const int64_t r0 = (int64_t)blockIdx.x * kRefreshRowsPerBlock;
  const int64_t r1 = min(len, r0 + kRefreshRowsPerBlock);
  for (int64_t base = r0 + (int64_t)warp * RPW; base < r1; base += (int64_t)RPW * (kRefreshThreads / 32)) {
    const int64_t t = base + sub;
    float s = 0.f;
    if (t < r1) {
      const uint4 v = __ldcs(reinterpret_cast<const uint4*>(slab + t * D) + ch);
      s = dot_chunk<T>(v, qc);
    }
#pragma unroll
    for (int off = CPR / 2; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
    if (ch == 0 && t < r1) {
      const uint32_t key = float_key(s);
      if (blocks) atomicMax(krow + t / 64, key);
      else krow[t] = key;
    }
  }
}

template <typename T, int D>
static cudaError_t launch_refresh_t(const void* q, const void* k, int64_t cap, int B, int H, int G,
                                    int64_t len, uint32_t* keys, int64_t key_stride, int blocks,
                                    cudaStream_t st) {
  const dim3 grid((unsigned)((len + kRefreshRowsPerBlock - 1) / kRefreshRowsPerBlock), (unsigned)(B * H));
  refresh_scores_kernel<T, D><<<grid, kRefreshThreads, 0, st>>>(
      static_cast<const T*>(q), static_cast<const T*>(k), cap, H, G, len, keys, key_stride, blocks);
  return cudaGetLastError();
}

cudaError_t launch_refresh_scores(const void* q, const void* k_layer, int64_t cap, int B, int H,
                                  int G, int d, int dtype, int64_t len, uint32_t* keys,
                                  int64_t key_stride, int blocks, cudaStream_t st) {
  if (dtype == 1) {
    switch (d) {
      case 64: return launch_refresh_t<__nv_bfloat16, 64>(q, k_layer, cap, B, H, G, len, keys, key_stride, blocks, st);
      case 128: return launch_refresh_t<__nv_bfloat16, 128>(q, k_layer, cap, B, H, G, len, keys, key_stride, blocks, st);
      case 256: return launch_refresh_t<__nv_bfloat16, 256>(q, k_layer, cap, B, H, G, len, keys, key_stride, blocks, st);
    }
  } else {
    switch (d) {
      case 16: return launch_refresh_t<float, 16>(q, k_layer, cap, B, H, G, len, keys, key_stride, blocks, st);
      case 32: return launch_refresh_t<float, 32>(q, k_layer, cap, B, H, G, len, keys, key_stride, blocks, st);
      case 64: return launch_refresh_t<float, 64>(q, k_layer, cap, B, H, G, len, keys, key_stride, blocks, st);
      case 128: return launch_refresh_t<float, 128>(q, k_layer, cap, B, H, G, len, keys, key_stride, blocks, st);
    }
  }
  return cudaErrorInvalidValue;
}

}  // namespace lyc
