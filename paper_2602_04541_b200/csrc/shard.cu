// shard.cu -- KV-sequence sharding across GPUs: the small
// kernels around the all-gather of one layer.
//
// Rank p holds rows [row_begin, row_begin + n_local) of every head.  Locally
// it runs the ordinary per-layer attention (partials exported as fp32 o +
// base-2 LSE) and the exact top-k of its own pooled scores.  After one packed
// all-gather every rank runs the SAME deterministic combine:
//   * LSE merge of the P partials in rank order (kernel_sim.hpp:205-225 applied
//     across ranks);
//   * global top-k over the P local candidate lists.  The union of the local
//     top-k's contains the global top-k; concatenated in rank order the
//     candidates are in ascending global index, so the radix select's
//     lower-position tie-break IS attention.hpp:117-118's lower-index rule;
//   * the global set is filtered to this rank's rows (local numbering) for
//     the sparse heads of later layers.
#include "lyc_common.cuh"
#include "lyc_plan.h"

namespace lyc {

// Local candidates: the local top-k ids of selection row r (ascending, local
// numbering, `cnt[row]` of them) -> (key, global id) at cache row `row`,
// padded to k_cap with key 0 / id -1.
__global__ void shard_candidates_kernel(const uint32_t* __restrict__ keys, int64_t key_stride,
                                        const int32_t* __restrict__ local_ids,
                                        const int32_t* __restrict__ cnt,
                                        const int32_t* __restrict__ sel_rows, int64_t k_cap,
                                        int64_t row_begin, uint32_t* __restrict__ cand_key,
                                        int32_t* __restrict__ cand_idx) {
  const int r = blockIdx.x;
  const int row = sel_rows[r];
  const int n = cnt[row];
  const uint32_t* kr = keys + (int64_t)r * key_stride;
  for (int64_t i = threadIdx.x; i < k_cap; i += blockDim.x) {
    const int64_t o = (int64_t)row * k_cap + i;
    if (i < n) {
      const int32_t id = local_ids[o];
      cand_key[o] = kr[id];
      cand_idx[o] = (int32_t)(id + row_begin);
    } else {
      cand_key[o] = 0u;
      cand_idx[o] = -1;
    }
  }
}

// Rank-ordered LSE merge: one warp per (output row, 32-column chunk).
template <typename T>
__global__ void shard_merge_kernel(const float* __restrict__ all_o,
                                   const float* __restrict__ all_lse, int64_t stride_o,
                                   int64_t stride_lse, int world, int rows, int d,
                                   T* __restrict__ out) {
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int chunks = (d + 31) / 32;
  const int row = gw / chunks, chunk = gw - row * chunks;
  if (row >= rows) return;
  float M = -INFINITY;
  for (int p = 0; p < world; ++p) M = fmaxf(M, all_lse[p * stride_lse + row]);
  const float Mz = M == -INFINITY ? 0.f : M;
  const int c = chunk * 32 + lane;
  float den = 0.f, acc = 0.f;
  for (int p = 0; p < world; ++p) {  // fixed rank order: bitwise identical on every rank
    const float w = exp2f(all_lse[p * stride_lse + row] - Mz);
    den += w;
    if (c < d) acc = fmaf(w, all_o[p * stride_o + (int64_t)row * d + c], acc);
  }
  if (c < d) {
    const float v = den > 0.f ? acc / den : 0.f;
    if constexpr (sizeof(T) == 2)
      out[(int64_t)row * d + c] = __float2bfloat16_rn(v);
    else
      out[(int64_t)row * d + c] = v;
  }
}

// Concatenate the ranks' candidate segments of each selection row.
__global__ void shard_gather_candidates_kernel(const uint32_t* __restrict__ all_key,
                                               const int32_t* __restrict__ all_idx,
                                               int64_t stride, int world, int64_t k_cap,
                                               const int32_t* __restrict__ sel_rows,
                                               uint32_t* __restrict__ keys,
                                               int32_t* __restrict__ ids) {
  const int r = blockIdx.x;
  const int row = sel_rows[r];
  const int64_t n = (int64_t)world * k_cap;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    const int64_t p = i / k_cap, j = i - p * k_cap;
    const int64_t src = p * stride + (int64_t)row * k_cap + j;
    keys[(int64_t)r * n + i] = all_key[src];
    ids[(int64_t)r * n + i] = all_idx[src];
  }
}

// Positions of the global top-k (ascending) -> global ids (ascending) -> the
// global set (optional) and this rank's filtered local index-cache row.
__global__ void shard_finalize_kernel(const int32_t* __restrict__ pos, int64_t pos_stride,
                                      const int32_t* __restrict__ ids, int64_t id_stride, int k,
                                      const int32_t* __restrict__ sel_rows, int64_t row_begin,
                                      int64_t n_local, int32_t* __restrict__ global_sets,
                                      int64_t global_stride, int32_t* __restrict__ cache,
                                      int64_t cache_stride, int32_t* __restrict__ cache_count) {
  __shared__ int s_lt, s_in;
  const int r = blockIdx.x;
  const int row = sel_rows[r];
  if (threadIdx.x == 0) {
    s_lt = 0;
    s_in = 0;
  }
  __syncthreads();
  int lt = 0, in = 0;
  for (int i = threadIdx.x; i < k; i += blockDim.x) {
    const int32_t g = ids[(int64_t)r * id_stride + pos[(int64_t)r * pos_stride + i]];
    if (global_sets) global_sets[(int64_t)row * global_stride + i] = g;
    lt += g < row_begin;
    in += g >= row_begin && g < row_begin + n_local;
  }
  atomicAdd(&s_lt, lt);
  atomicAdd(&s_in, in);
  __syncthreads();
  // ascending ids: the ones in this shard are the contiguous run [s_lt, s_lt + s_in)
  for (int i = threadIdx.x; i < s_in; i += blockDim.x) {
    const int32_t g = ids[(int64_t)r * id_stride + pos[(int64_t)r * pos_stride + s_lt + i]];
    cache[(int64_t)row * cache_stride + i] = (int32_t)(g - row_begin);
  }
  if (threadIdx.x == 0) cache_count[row] = s_in;
}

cudaError_t launch_shard_candidates(const uint32_t* keys, int64_t key_stride,
                                    const int32_t* local_ids, const int32_t* cnt,
                                    const int32_t* sel_rows, int n_sel, int64_t k_cap,
                                    int64_t row_begin, uint32_t* cand_key, int32_t* cand_idx,
                                    cudaStream_t st) {
  if (n_sel == 0) return cudaSuccess;
  shard_candidates_kernel<<<n_sel, 256, 0, st>>>(keys, key_stride, local_ids, cnt, sel_rows, k_cap,
                                                 row_begin, cand_key, cand_idx);
  return cudaGetLastError();
}

cudaError_t launch_shard_merge(const float* all_o, const float* all_lse, int64_t stride_o,
                               int64_t stride_lse, int world, int rows, int d, void* out,
                               int dtype, cudaStream_t st) {
  const int warps = rows * ((d + 31) / 32);
  const int blocks = (warps + 3) / 4;
  if (dtype == 1)
    shard_merge_kernel<__nv_bfloat16><<<blocks, 128, 0, st>>>(
        all_o, all_lse, stride_o, stride_lse, world, rows, d, static_cast<__nv_bfloat16*>(out));
  else
    shard_merge_kernel<float><<<blocks, 128, 0, st>>>(all_o, all_lse, stride_o, stride_lse, world,
                                                      rows, d, static_cast<float*>(out));
  return cudaGetLastError();
}

cudaError_t launch_shard_gather(const uint32_t* all_key, const int32_t* all_idx, int64_t stride,
                                int world, int64_t k_cap, const int32_t* sel_rows, int n_sel,
                                uint32_t* keys, int32_t* ids, cudaStream_t st) {
  if (n_sel == 0) return cudaSuccess;
  shard_gather_candidates_kernel<<<n_sel, 256, 0, st>>>(all_key, all_idx, stride, world, k_cap,
                                                        sel_rows, keys, ids);
  return cudaGetLastError();
}

cudaError_t launch_shard_finalize(const int32_t* pos, int64_t pos_stride, const int32_t* ids,
                                  int64_t id_stride, int k, const int32_t* sel_rows, int n_sel,
                                  int64_t row_begin, int64_t n_local, int32_t* global_sets,
                                  int64_t global_stride, int32_t* cache, int64_t cache_stride,
                                  int32_t* cache_count, cudaStream_t st) {
  if (n_sel == 0) return cudaSuccess;
  shard_finalize_kernel<<<n_sel, 256, 0, st>>>(pos, pos_stride, ids, id_stride, k, sel_rows,
                                               row_begin, n_local, global_sets, global_stride,
                                               cache, cache_stride, cache_count);
  return cudaGetLastError();
}

}  // namespace lyc
