// policy.cu -- the TopP and Threshold token-selection policies on device
// (reference: select_tokens policy.hpp:73-101, fed by the pooled-query
// weights of dense_attention, attention.hpp:51-75, at decode_engine.hpp:128-132).
//
// Inputs are the order-preserving keys the attention consumers wrote while
// scoring (lyc_common.cuh float_key of sum_j q_j.k = G * pooled_q.k for bf16,
// of pooled_q.k for fp32).  One CTA per selection row:
//   * weights: w_t = exp(x_t - x_max) / Z, x_t = key_float(key_t) * score_scale,
//     Z accumulated in f64 (the reference's dense_attention runs in f64);
//   * Threshold(tau): every t with w_t > tau, ascending; if none clears the
//     bar, the first index of the maximum weight (policy.hpp:89-101);
//   * TopP(p): the smallest prefix of the weights sorted descending (ties in
//     index order: stable_sort) whose cumulative mass reaches p
//     (policy.hpp:73-88).  The sort is replaced by a radix select on the keys
//     weighted by mass (12 + 10 + 10 bits): the boundary key K*, the mass
//     strictly above it, and how many of the keys equal to K* (in index
//     order) the prefix needs.  Output ascending, count in out_count.
// Weights are monotone in the keys, so the sets equal the reference's except
// where f64-vs-f32 score rounding reorders weights within the documented tie
// band or moves the cumulative crossing of p.
#include "lyc_common.cuh"
#include "lyc_plan.h"

namespace lyc {

constexpr int kPolThreads = 1024;

template <typename T, typename Op>
__device__ __forceinline__ T block_reduce(T v, T* red, Op op) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) v = op(v, __shfl_xor_sync(0xffffffffu, v, off));
  __syncthreads();
  if (lane == 0) red[w] = v;
  __syncthreads();
  v = red[0];
  for (int i = 1; i < kPolThreads / 32; ++i) v = op(v, red[i]);
  return v;
}

// Block-wide exclusive scan of one value per thread (thread order).
template <typename T>
__device__ __forceinline__ T block_excl_scan(T v, T* red, T& total) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  T x = v;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const T y = __shfl_up_sync(0xffffffffu, x, off);
    if (lane >= off) x += y;
  }
  __syncthreads();
  if (lane == 31) red[w] = x;
  __syncthreads();
  T before = 0;
  total = 0;
  for (int i = 0; i < kPolThreads / 32; ++i) {
    if (i < w) before += red[i];
    total += red[i];
  }
  return before + x - v;
}

struct PolSmem {
  double mass[4096];
  double dred[32];
  uint32_t ured[32];
  uint32_t pick;      // chosen bin
  double above;       // mass strictly above the chosen bin (running)
};

__device__ __forceinline__ double weight_of(uint32_t key, float xmax, double scale, double inv_z) {
  return exp(((double)key_float(key) - (double)xmax) * scale) * inv_z;
}

// Descending cumulative search over nb bins of s.mass: the bin where the mass
// above (starting from `above0`) first reaches `target`.  Sets s.pick and
// s.above (mass strictly above the picked bin); s.pick = 0xffffffff if the
// bins' total never reaches the target.
__device__ void pick_bin(PolSmem& s, int nb, double above0, double target) {
  const int per = nb / kPolThreads > 0 ? nb / kPolThreads : 1;
  const int t = threadIdx.x;
  // thread t owns bins [nb - (t+1)*per, nb - t*per) (highest first)
  double sum = 0.0;
  const int hi = nb - t * per;
  if (hi > 0)
    for (int i = 0; i < per; ++i) sum += s.mass[hi - 1 - i];
  double tot;
  const double ex = block_excl_scan<double>(sum, s.dred, tot);
  if (threadIdx.x == 0) s.pick = 0xffffffffu;
  __syncthreads();
  if (hi > 0 && above0 + ex < target && target <= above0 + ex + sum) {
    double run = above0 + ex;
    for (int i = 0; i < per; ++i) {
      const double m = s.mass[hi - 1 - i];
      if (target <= run + m) {
        s.pick = (uint32_t)(hi - 1 - i);
        s.above = run;
        break;
      }
      run += m;
    }
  }
  __syncthreads();
}

__global__ void __launch_bounds__(kPolThreads, 1) policy_select_kernel(const __grid_constant__ LycPolicyParams p) {
  __shared__ PolSmem s;
  const int r = blockIdx.x;
  const uint32_t* kr = p.keys + (int64_t)r * p.key_stride;
  const int n = p.row_n ? p.row_n[r] : p.n;  // variable-length batch: this row's tokens
  const int C = (n + kPolThreads - 1) / kPolThreads;  // contiguous keys per thread
  const int b0 = threadIdx.x * C, b1 = min(n, b0 + C);
  const int orow = p.out_row[r];
  int32_t* out = p.out + (int64_t)orow * p.out_stride;
  const double scale = (double)p.score_scale;

  // max key (the maximum weight) and its first index
  uint32_t kmax = 0u;
  for (int i = b0; i < b1; ++i) kmax = max(kmax, kr[i]);
  kmax = block_reduce<uint32_t>(kmax, s.ured, [](uint32_t a, uint32_t b) { return max(a, b); });
  const float xmax = key_float(kmax);
  double zsum = 0.0;
  for (int i = b0; i < b1; ++i) zsum += exp(((double)key_float(kr[i]) - (double)xmax) * scale);
  const double Z = block_reduce<double>(zsum, s.dred, [](double a, double b) { return a + b; });
  const double inv_z = 1.0 / Z;

  if (p.kind == LYC_POLICY_KIND_THRESHOLD) {
    uint32_t c = 0;
    for (int i = b0; i < b1; ++i) c += weight_of(kr[i], xmax, scale, inv_z) > p.value ? 1u : 0u;
    uint32_t total;
    uint32_t pos = block_excl_scan<uint32_t>(c, s.ured, total);
    if (total > 0) {
      for (int i = b0; i < b1; ++i)
        if (weight_of(kr[i], xmax, scale, inv_z) > p.value) out[pos++] = i;
    } else {
      // nothing cleared the bar: the first index of the maximum
      uint32_t first = 0xffffffffu;
      for (int i = b0; i < b1 && first == 0xffffffffu; ++i)
        if (kr[i] == kmax) first = (uint32_t)i;
      first = block_reduce<uint32_t>(first, s.ured, [](uint32_t a, uint32_t b) { return min(a, b); });
      if (threadIdx.x == 0) out[0] = (int32_t)first;
      total = 1;
    }
    if (threadIdx.x == 0 && p.out_count) p.out_count[orow] = (int32_t)total;
    return;
  }

  // ---- TopP: radix select by mass, 12 + 10 + 10 bits from the top
  const double target = p.value;
  uint32_t prefix = 0;
  int pbits = 0;
  double above = 0.0;
  bool all = false;
  const int widths[3] = {12, 10, 10};
  for (int pass = 0; pass < 3; ++pass) {
    const int wb = widths[pass];
    const int nb = 1 << wb;
    const int sh = 32 - pbits - wb;
    for (int b = threadIdx.x; b < nb; b += kPolThreads) s.mass[b] = 0.0;
    __syncthreads();
    for (int i = b0; i < b1; ++i) {
      const uint32_t k = kr[i];
      if (pbits == 0 || (k >> (32 - pbits)) == prefix)
        atomicAdd(&s.mass[(k >> sh) & (uint32_t)(nb - 1)], weight_of(k, xmax, scale, inv_z));
    }
    __syncthreads();
    pick_bin(s, nb, above, target);
    if (s.pick == 0xffffffffu) {  // rounding: the total mass never reaches p -> everything
      all = true;
      break;
    }
    prefix = (prefix << wb) | s.pick;
    pbits += wb;
    above = s.above;
    __syncthreads();
  }
  uint32_t kstar = prefix;      // the boundary key (all 32 bits)
  uint32_t take_tied = 0;       // keys == kstar taken, in index order
  if (!all) {
    const double wstar = weight_of(kstar, xmax, scale, inv_z);
    uint32_t ct = 0;
    for (int i = b0; i < b1; ++i) ct += kr[i] == kstar ? 1u : 0u;
    const uint32_t tied = block_reduce<uint32_t>(ct, s.ured, [](uint32_t a, uint32_t b) { return a + b; });
    // the smallest j >= 1 with above + j * w* >= p (sequential in the reference)
    double cum = above;
    uint32_t j = 0;
    while (j < tied) {
      cum += wstar;
      ++j;
      if (cum >= target) break;
    }
    take_tied = j;
  } else {
    kstar = 0u;
    take_tied = 0xffffffffu;  // every key (>= 0)
  }
  // emission in index order: keys > K*, and the first take_tied keys == K*
  uint32_t ca = 0, ct = 0;
  for (int i = b0; i < b1; ++i) {
    ca += kr[i] > kstar ? 1u : 0u;
    ct += kr[i] == kstar ? 1u : 0u;
  }
  uint32_t ttot;
  const uint32_t trank = block_excl_scan<uint32_t>(ct, s.ured, ttot);
  const uint32_t mine_t = trank >= take_tied ? 0u : min(ct, take_tied - trank);
  uint32_t total;
  uint32_t pos = block_excl_scan<uint32_t>(ca + mine_t, s.ured, total);
  uint32_t tr = trank;
  for (int i = b0; i < b1; ++i) {
    const uint32_t k = kr[i];
    if (k > kstar) {
      out[pos++] = i;
    } else if (k == kstar) {
      if (tr < take_tied) out[pos++] = i;
      ++tr;
    }
  }
  if (threadIdx.x == 0 && p.out_count) p.out_count[orow] = (int32_t)total;
}

cudaError_t launch_policy(const LycPolicyParams& p, int rows, cudaStream_t st) {
  if (rows == 0) return cudaSuccess;
  policy_select_kernel<<<rows, kPolThreads, 0, st>>>(p);
  return cudaGetLastError();
}

}  // namespace lyc
