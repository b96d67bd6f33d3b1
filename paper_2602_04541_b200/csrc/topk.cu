// topk.cu -- exact top-k selection into the per-head index cache
// (reference: args_top_k attention.hpp:108-123 via select_tokens
// policy.hpp:64-72, called at decode_engine.hpp:132).
//
// Semantics reproduced exactly: the min(k, n) largest scores, ties broken by
// the LOWER index, emitted in ascending index order.  Scores arrive as
// order-preserving uint32 keys (lyc_common.cuh float_key), written by the
// attention kernel's fused selection epilogue.
//
// One thread-block CLUSTER per selection row (b, retrieval head):
//   * each CTA loads its contiguous slice of the row's keys into smem once
//     (L2-resident: the attention kernel wrote them microseconds earlier);
//   * 3 radix passes (11 + 11 + 10 bits, MSB first) find the k-th largest key
//     T exactly; per pass every CTA builds a smem histogram of the candidates
//     that still match the prefix, one cluster barrier publishes them, and every
//     CTA sums the C histograms through DSMEM (double-buffered so one barrier
//     per pass suffices);
//   * emission: keys > T are all taken, keys == T are taken in index order
//     until k are emitted (the tie rule).  Slices are contiguous and in rank
//     order, so a cluster-wide exclusive scan of (count > T, count == T) gives
//     every CTA its output offset, and an in-CTA ordered scan compacts its
//     slice -> ascending indices with no sort.
#include <cooperative_groups.h>

#include <algorithm>

#include "lyc_common.cuh"
#include "lyc_plan.h"

namespace cg = cooperative_groups;

namespace lyc {

constexpr int kTopkThreads = 1024;
constexpr int kBins = 2048;

struct TopkShared {
  uint32_t hist[2][kBins];
  uint32_t ghist[kBins];
  uint32_t warp_tot[32];
  uint32_t counts[2];   // this CTA's (count > T, count == T)
  uint32_t digit, above;
};

// Inclusive scan of one value per thread across the block (1024 threads).
__device__ __forceinline__ uint32_t block_inclusive_scan(uint32_t v, uint32_t* warp_tot,
                                                         uint32_t& total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const uint32_t n = __shfl_up_sync(0xffffffffu, v, off);
    if (lane >= off) v += n;
  }
  if (lane == 31) warp_tot[warp] = v;
  __syncthreads();
  if (warp == 0) {
    uint32_t w = warp_tot[lane];
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const uint32_t n = __shfl_up_sync(0xffffffffu, w, off);
      if (lane >= off) w += n;
    }
    warp_tot[lane] = w;  // inclusive prefix over warps
  }
  __syncthreads();
  const uint32_t before = warp == 0 ? 0u : warp_tot[warp - 1];
  total = warp_tot[31];
  __syncthreads();
  return v + before;
}

__global__ void __launch_bounds__(kTopkThreads, 1) topk_cluster_kernel(const __grid_constant__ LycTopkParams p) {
  cg::cluster_group cluster = cg::this_cluster();
  const int C = (int)cluster.num_blocks();
  const int rank = (int)cluster.block_rank();
  const int row = blockIdx.x / C;
  const int tid = threadIdx.x;

  extern __shared__ __align__(16) uint8_t smem_raw[];
  TopkShared& sh = *reinterpret_cast<TopkShared*>(smem_raw);
  uint32_t* keys = reinterpret_cast<uint32_t*>(smem_raw + sizeof(TopkShared));

  uint32_t* gkeys = p.keys + (int64_t)row * p.key_stride;
  const int n_row = p.row_n ? p.row_n[row] : p.n;  // variable-length batch: this row's keys
  const int k_row = p.row_k ? p.row_k[row] : p.k;
  const int lo = rank * p.slice;
  const int cnt = max(0, min(p.slice, n_row - lo));
  for (int i = tid; i < cnt; i += kTopkThreads) {
    keys[i] = gkeys[lo + i];
    if (p.clear_keys) gkeys[lo + i] = 0u;
  }

  uint32_t prefix = 0, pmask = 0;
  uint32_t krem = (uint32_t)k_row;  // still to take among keys matching the prefix
  constexpr int kShift[3] = {21, 10, 0};
  constexpr uint32_t kMask[3] = {0x7ffu, 0x7ffu, 0x3ffu};
#pragma unroll
  for (int pass = 0; pass < 3; ++pass) {
    uint32_t* h = sh.hist[pass & 1];
    for (int b = tid; b < kBins; b += kTopkThreads) h[b] = 0u;
    __syncthreads();
    const int sft = kShift[pass];
    const uint32_t msk = kMask[pass];
    for (int i = tid; i < cnt; i += kTopkThreads) {
      const uint32_t key = keys[i];
      if ((key & pmask) == prefix) atomicAdd(&h[(key >> sft) & msk], 1u);
    }
    cluster.sync();
    const int nb = (int)msk + 1;
    for (int b = tid; b < nb; b += kTopkThreads) {
      uint32_t s = 0;
      for (int c = 0; c < C; ++c) s += cluster.map_shared_rank(h, c)[b];
      sh.ghist[b] = s;
    }
    __syncthreads();
    // Suffix scan from the top bin down: thread t owns bins nb-1-2t, nb-2-2t.
    const int b_hi = nb - 1 - 2 * tid, b_lo = b_hi - 1;
    const uint32_t c_hi = b_hi >= 0 ? sh.ghist[b_hi] : 0u;
    const uint32_t c_lo = b_lo >= 0 ? sh.ghist[b_lo] : 0u;
    uint32_t total;
    const uint32_t incl = block_inclusive_scan(c_hi + c_lo, sh.warp_tot, total);
    const uint32_t excl = incl - c_hi - c_lo;  // count in bins above b_hi
    if (excl < krem && krem <= incl) {
      if (krem <= excl + c_hi) {
        sh.digit = (uint32_t)b_hi;
        sh.above = excl;
      } else {
        sh.digit = (uint32_t)b_lo;
        sh.above = excl + c_hi;
      }
    }
    __syncthreads();
    prefix |= sh.digit << sft;
    pmask |= msk << sft;
    krem -= sh.above;
    __syncthreads();
  }
  const uint32_t T = prefix;  // exact k-th largest key; krem ties of T to take

  // ---- emission
  uint32_t gt = 0, eq = 0;
  for (int i = tid; i < cnt; i += kTopkThreads) {
    const uint32_t key = keys[i];
    gt += key > T;
    eq += key == T;
  }
  uint32_t tot_gt, tot_eq;
  block_inclusive_scan(gt, sh.warp_tot, tot_gt);
  block_inclusive_scan(eq, sh.warp_tot, tot_eq);
  if (tid == 0) {
    sh.counts[0] = tot_gt;
    sh.counts[1] = tot_eq;
  }
  cluster.sync();
  uint32_t out_base = 0, eq_before = 0;
  for (int c = 0; c < rank; ++c) {
    const uint32_t* rc = cluster.map_shared_rank(sh.counts, c);
    const uint32_t cg_ = rc[0], ce = rc[1];
    const uint32_t take = krem > eq_before ? min(ce, krem - eq_before) : 0u;
    out_base += cg_ + take;
    eq_before += ce;
  }
  const uint32_t take_eq = krem > eq_before ? min(sh.counts[1], krem - eq_before) : 0u;

  int32_t* out = p.out + (int64_t)p.out_row[row] * p.out_stride;
  uint32_t run_gt = 0, run_eq = 0;  // counts before the current chunk
  constexpr int kPer = 4;
  for (int base = 0; base < cnt; base += kTopkThreads * kPer) {
    const int i0 = base + tid * kPer;
    uint32_t kv[kPer];
    uint32_t g = 0, e = 0;
#pragma unroll
    for (int q = 0; q < kPer; ++q) {
      kv[q] = i0 + q < cnt ? keys[i0 + q] : 0u;
      const bool ok = i0 + q < cnt;
      g += ok && kv[q] > T;
      e += ok && kv[q] == T;
    }
    uint32_t tot;
    const uint32_t incl = block_inclusive_scan((e << 16) | g, sh.warp_tot, tot);
    uint32_t gb = run_gt + ((incl - ((e << 16) | g)) & 0xffffu);
    uint32_t eb = run_eq + ((incl - ((e << 16) | g)) >> 16);
#pragma unroll
    for (int q = 0; q < kPer; ++q) {
      if (i0 + q >= cnt) break;
      const bool is_gt = kv[q] > T, is_eq = kv[q] == T;
      if (is_gt || (is_eq && eb < take_eq)) {
        const uint32_t pos = out_base + gb + min(eb, take_eq);
        out[pos] = lo + i0 + q;
      }
      gb += is_gt;
      eb += is_eq;
    }
    run_gt += tot & 0xffffu;
    run_eq += tot >> 16;
  }
  if (rank == 0 && tid == 0 && p.out_count) p.out_count[p.out_row[row]] = k_row;
  cluster.sync();  // keep smem alive until every CTA has read our counts
}

size_t topk_smem_bytes(int slice) { return sizeof(TopkShared) + (size_t)slice * 4; }

// Cluster size: smallest power of two C <= 16 with ceil(n / C) <= max_slice.
int topk_cluster_size(int n, int max_slice) {
  int c = 1;
  while (c < 16 && (n + c - 1) / c > max_slice) c <<= 1;
  return c;
}

cudaError_t launch_topk(const LycTopkParams& p, int rows, int cluster, cudaStream_t st) {
  if (rows == 0) return cudaSuccess;
  const size_t smem = topk_smem_bytes(p.slice);
  static size_t configured_[64] = {};  // per device: attributes are per-device state
  int dev = 0;
  cudaGetDevice(&dev);
  size_t& configured = configured_[dev & 63];
  if (configured < smem) {
    cudaError_t e = cudaFuncSetAttribute(topk_cluster_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(topk_cluster_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
    configured = smem;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(rows * cluster);
  cfg.blockDim = dim3(kTopkThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = cluster;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, topk_cluster_kernel, p);
}

}  // namespace lyc

namespace lyc {

__global__ void float_keys_kernel(const float* __restrict__ s, uint32_t* __restrict__ keys, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    keys[i] = float_key(s[i]);
}

cudaError_t launch_float_keys(const float* s, uint32_t* keys, int64_t n, cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  const int blocks = (int)std::min<int64_t>((n + 255) / 256, 148 * 8);
  float_keys_kernel<<<blocks, 256, 0, st>>>(s, keys, n);
  return cudaGetLastError();
}

}  // namespace lyc
