// attn.cu -- the pooled hybrid-head split-KV decode attention kernel
// (Algorithm 2; CPU reference kernel_sim.hpp:169-201
// run_split and attention.hpp:50-104 dense/sparse attention).
//
// One CTA executes one split of the pooled plan: a sequence of UNITS, each a
// contiguous item range of one slot (b, KV head).  Retrieval (ITEM_DENSE),
// block-sparse (ITEM_BLOCKS) and token-sparse (ITEM_TOKENS) slots share the
// same pipeline; only the row addresses differ:
//
//   warp 4 (producer): for every 64-row tile, one lane per row issues a
//     cp.async.bulk (TMA engine) of the K row and the V row into a padded
//     smem ring (row stride d*e+16 B -> conflict-free ldmatrix), completion
//     counted in bytes on the stage's mbarrier.  Gathered and contiguous
//     tiles are the same instruction stream.
//   warps 0-3 (consumers): each owns 16 rows of every tile; all G query heads
//     of the GQA group are packed as the 16-row A operand of mma.sync
//     m16n8k16 (bf16 -> fp32), so K and V are read from smem exactly once per
//     tile for the whole group.  Online softmax (attention.hpp:161-181) in the
//     exp2 domain with warp-shuffle row max/sum.
//   Fused selection (retrieval slots with sel >= 0): the pooled-query score
//   of every row, sum_j q_j.k (= G * pooled_q.k, attention.hpp:127-146 and
//   decode_engine.hpp:129-132), is reduced across the packed rows with three
//   shuffles and written as an order-preserving uint32 key (token mode) or
//   atomically max-folded per block (block mode).
//   End of unit: the 4 warps' (m, l, o) states are merged through smem and
//   written as a normalized partial + base-2 LSE (kernel_sim.hpp:195-198), or
//   directly as the final output when the slot has a single unit.
#include "lyc_common.cuh"
#include "lyc_plan.h"

namespace lyc {

constexpr int kConsumerWarps = 4;
constexpr int kThreads = (kConsumerWarps + 1) * 32;

template <typename T>
struct ElemBytes;
template <>
struct ElemBytes<__nv_bfloat16> {
  static constexpr int v = 2;
};
template <>
struct ElemBytes<float> {
  static constexpr int v = 4;
};

template <typename T, int D>
struct AttnCfg {
  static constexpr int kRowBytes = D * ElemBytes<T>::v;
  static constexpr int kRowStride = kRowBytes + 16;  // +16 B: rows rotate 4 banks
  static constexpr int kTileBytes = LYC_TILE * kRowStride;
  static constexpr int kStageBytes = 2 * kTileBytes;  // K tile then V tile
  static constexpr int kMaxG = 16;
  static constexpr int kMergeBytes = kConsumerWarps * kMaxG * (D + 2) * 4;
  static constexpr int kQBytes = (ElemBytes<T>::v == 4) ? (kMaxG + 1) * D * 4 : 0;
  static constexpr int kBudget = 200 * 1024;
  static constexpr int kStagesRaw = (kBudget - kMergeBytes - kQBytes) / kStageBytes;
  static constexpr int kStages = kStagesRaw > 8 ? 8 : kStagesRaw;
  static constexpr int kSmem = kStages * kStageBytes + kMergeBytes + kQBytes + 2 * kStages * 8 + 16;
  static_assert(kStages >= 2, "not enough shared memory for a 2-stage ring");
};

struct Tile {
  int32_t lo;            // first row (contiguous tiles)
  int32_t nvalid;        // valid rows in this tile
  const int32_t* ids;    // token ids (gathered tiles) or nullptr
};

__device__ __forceinline__ int tiles_per_item(const LycSlot& s, int bs) {
  return s.kind == ITEM_TOKENS ? 1 : (bs + LYC_TILE - 1) / LYC_TILE;
}

__device__ __forceinline__ Tile tile_of(const LycSlot& s, int item, int sub, int seq, int bs) {
  Tile t;
  if (s.kind == ITEM_TOKENS) {
    t.ids = s.list + (int64_t)item * LYC_TILE;
    t.lo = 0;
    t.nvalid = min(LYC_TILE, s.list_len - item * LYC_TILE);
  } else {
    const int blk = s.kind == ITEM_DENSE ? item : __ldg(s.list + item);
    const int b0 = blk * bs;
    const int hi = min(b0 + bs, seq);
    t.ids = nullptr;
    t.lo = b0 + sub * LYC_TILE;
    t.nvalid = max(0, min(LYC_TILE, hi - t.lo));
  }
  return t;
}

__device__ __forceinline__ int tile_row(const Tile& t, int r) {
  const int rr = r < t.nvalid ? r : 0;  // invalid rows re-load row 0 (finite data, masked)
  return t.ids ? __ldg(t.ids + rr) : t.lo + rr;
}

// ---------------------------------------------------------------- producer
template <typename T, int D>
__device__ __forceinline__ void produce(const LycAttnParams& p, uint8_t* ring, uint64_t* full,
                                        uint64_t* empty, int ub, int ue, int lane) {
  using C = AttnCfg<T, D>;
  const uint64_t pol = policy_evict_first();
  const char* kbase = static_cast<const char*>(p.k);
  const char* vbase = static_cast<const char*>(p.v);
  int stage = 0;
  uint32_t phase = 0;
  for (int u = ub; u < ue; ++u) {
    const LycUnit un = p.units[u];
    const LycSlot s = p.slots[un.slot];
    const int tpi = tiles_per_item(s, p.block_size);
    const int64_t slab = s.kv_off * ElemBytes<T>::v;
    for (int it = un.begin; it < un.end; ++it) {
      if (p.exec_counts && lane == 0)
        atomicAdd(p.exec_counts + (int64_t)un.slot * p.counts_stride + it, 1u);
      for (int sub = 0; sub < tpi; ++sub) {
        const Tile t = tile_of(s, it, sub, p.seq_len, p.block_size);
        const int r0 = tile_row(t, lane), r1 = tile_row(t, lane + 32);
        mbar_wait(&empty[stage], phase ^ 1);
        if (lane == 0) mbar_arrive_expect_tx(&full[stage], 2 * LYC_TILE * C::kRowBytes);
        __syncwarp();
        uint8_t* kd = ring + stage * C::kStageBytes;
        uint8_t* vd = kd + C::kTileBytes;
        bulk_g2s_stream(kd + lane * C::kRowStride, kbase + slab + (int64_t)r0 * C::kRowBytes,
                        C::kRowBytes, &full[stage], pol);
        bulk_g2s_stream(vd + lane * C::kRowStride, vbase + slab + (int64_t)r0 * C::kRowBytes,
                        C::kRowBytes, &full[stage], pol);
        bulk_g2s_stream(kd + (lane + 32) * C::kRowStride,
                        kbase + slab + (int64_t)r1 * C::kRowBytes, C::kRowBytes, &full[stage],
                        pol);
        bulk_g2s_stream(vd + (lane + 32) * C::kRowStride,
                        vbase + slab + (int64_t)r1 * C::kRowBytes, C::kRowBytes, &full[stage],
                        pol);
        if (++stage == C::kStages) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  }
}

__device__ __forceinline__ void consumer_bar() {
  asm volatile("bar.sync 1, %0;" ::"n"(kConsumerWarps * 32) : "memory");
}

__device__ __forceinline__ float warp_max4(float v) {  // max over the 4 lanes of a quad
  v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, 1));
  return fmaxf(v, __shfl_xor_sync(0xffffffffu, v, 2));
}

template <typename T>
__device__ __forceinline__ void store_out(T* dst, float v);
template <>
__device__ __forceinline__ void store_out<float>(float* dst, float v) {
  *dst = v;
}
template <>
__device__ __forceinline__ void store_out<__nv_bfloat16>(__nv_bfloat16* dst, float v) {
  *dst = __float2bfloat16_rn(v);
}

// Merge the consumer warps' (m, l, o) for one unit and emit partial / output.
// merge smem layout: o[w][j][D] then ml[w][j][2].
template <typename T, int D>
__device__ __forceinline__ void unit_epilogue(const LycAttnParams& p, const LycSlot& s, int u,
                                              float* mo, float* ml, int tid) {
  using C = AttnCfg<T, D>;
  const int G = p.group;
  consumer_bar();
  const bool direct = s.n_units == 1;
  for (int idx = tid; idx < G * D; idx += kConsumerWarps * 32) {
    const int j = idx / D, d = idx - j * D;
    float M = -INFINITY;
#pragma unroll
    for (int w = 0; w < kConsumerWarps; ++w) M = fmaxf(M, ml[(w * C::kMaxG + j) * 2]);
    float L = 0.f, O = 0.f;
#pragma unroll
    for (int w = 0; w < kConsumerWarps; ++w) {
      const float mw = ml[(w * C::kMaxG + j) * 2];
      const float f = mw == -INFINITY ? 0.f : exp2f(mw - M);
      L += ml[(w * C::kMaxG + j) * 2 + 1] * f;
      O += mo[(w * C::kMaxG + j) * D + d] * f;
    }
    const float o = O / L;
    if (direct) {
      store_out<T>(static_cast<T*>(p.out) + (int64_t)(s.q_row + j) * D + d, o);
    } else {
      p.part_o[((int64_t)u * G + j) * D + d] = o;
      if (d == 0) p.part_lse[(int64_t)u * G + j] = log2f(L) + M;
    }
  }
  consumer_bar();
}

// ---------------------------------------------------------------- bf16 path
// Consumer warp w handles rows [16w, 16w+16) of each 64-row tile.
template <int D>
__device__ __forceinline__ void consume_bf16(const LycAttnParams& p, uint8_t* ring,
                                             uint64_t* full, uint64_t* empty, float* mo,
                                             float* ml, int ub, int ue, int warp, int lane) {
  using C = AttnCfg<__nv_bfloat16, D>;
  constexpr int KS = D / 16;  // k-steps over d for QK^T
  constexpr int NT = D / 8;   // n-tiles over d for PV
  const int G = p.group;
  const int qr = lane >> 2;   // A/C row of this lane (and qr + 8)
  const int qc = (lane & 3) * 2;
  const int t0 = warp * 16;
  int stage = 0;
  uint32_t phase = 0;
  const __nv_bfloat16* Q = static_cast<const __nv_bfloat16*>(p.q);

  for (int u = ub; u < ue; ++u) {
    const LycUnit un = p.units[u];
    const LycSlot s = p.slots[un.slot];
    const int tpi = tiles_per_item(s, p.block_size);
    // ---- Q fragments: rows j < G of the group, zero elsewhere.
    uint32_t qa[KS][4];
#pragma unroll
    for (int kk = 0; kk < KS; ++kk) {
#pragma unroll
      for (int h = 0; h < 4; ++h) {
        const int row = qr + (h & 1) * 8;
        const int col = kk * 16 + qc + (h >> 1) * 8;
        qa[kk][h] = row < G ? __ldg(reinterpret_cast<const uint32_t*>(
                                  Q + (int64_t)(s.q_row + row) * D + col))
                            : 0u;
      }
    }
    float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;
    float o[NT][4];
#pragma unroll
    for (int n = 0; n < NT; ++n) o[n][0] = o[n][1] = o[n][2] = o[n][3] = 0.f;
    const bool want_sel = s.sel >= 0 && p.sel_mode != SEL_NONE;

    for (int it = un.begin; it < un.end; ++it) {
      for (int sub = 0; sub < tpi; ++sub) {
        const Tile t = tile_of(s, it, sub, p.seq_len, p.block_size);
        mbar_wait(&full[stage], phase);
        const uint8_t* ks = ring + stage * C::kStageBytes;
        const uint8_t* vs = ks + C::kTileBytes;
        // ---- S = Q K^T for this warp's 16 rows (two n-tiles of 8)
        float sc[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
        {
          const uint8_t* kp = ks + (t0 + (lane >> 4) * 8 + (lane & 7)) * C::kRowStride +
                              ((lane >> 3) & 1) * 16;
#pragma unroll
          for (int kk = 0; kk < KS; ++kk) {
            uint32_t b0, b1, b2, b3;
            ldsm_x4(b0, b1, b2, b3, kp + kk * 32);
            mma_bf16(sc[0], qa[kk][0], qa[kk][1], qa[kk][2], qa[kk][3], b0, b1);
            mma_bf16(sc[1], qa[kk][0], qa[kk][1], qa[kk][2], qa[kk][3], b2, b3);
          }
        }
        // ---- fused selection score: sum over packed rows (rows >= G are 0)
        if (want_sel) {
          float ps[2][2];
#pragma unroll
          for (int n = 0; n < 2; ++n)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              float v = sc[n][e] + sc[n][e + 2];
              v += __shfl_xor_sync(0xffffffffu, v, 4);
              v += __shfl_xor_sync(0xffffffffu, v, 8);
              v += __shfl_xor_sync(0xffffffffu, v, 16);
              ps[n][e] = v;
            }
          if (p.sel_mode == SEL_TOKEN_KEYS) {
            if (lane < 4) {
#pragma unroll
              for (int n = 0; n < 2; ++n) {
                const int r = t0 + n * 8 + qc;
                uint32_t* dst = p.sel_keys + (int64_t)s.sel * p.sel_stride + t.lo + r;
                if (r < t.nvalid) dst[0] = float_key(ps[n][0]);
                if (r + 1 < t.nvalid) dst[1] = float_key(ps[n][1]);
              }
            }
          } else {  // SEL_BLOCK_KEYS: max over valid rows of this block
            uint32_t km = 0u;
#pragma unroll
            for (int n = 0; n < 2; ++n)
#pragma unroll
              for (int e = 0; e < 2; ++e)
                if (t0 + n * 8 + qc + e < t.nvalid) km = max(km, float_key(ps[n][e]));
            km = max(km, __shfl_xor_sync(0xffffffffu, km, 1));
            km = max(km, __shfl_xor_sync(0xffffffffu, km, 2));
            if (lane == 0 && km != 0u)
              atomicMax(p.sel_keys + (int64_t)s.sel * p.sel_stride + it, km);
          }
        }
        // ---- online softmax (exp2 domain), rows qr (e=0,1) and qr+8 (e=2,3)
        float x[2][4];
#pragma unroll
        for (int n = 0; n < 2; ++n)
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int r = t0 + n * 8 + qc + (e & 1);
            x[n][e] = r < t.nvalid ? sc[n][e] * p.scale_log2 : -INFINITY;
          }
        const float mx0 = warp_max4(fmaxf(fmaxf(x[0][0], x[0][1]), fmaxf(x[1][0], x[1][1])));
        const float mx1 = warp_max4(fmaxf(fmaxf(x[0][2], x[0][3]), fmaxf(x[1][2], x[1][3])));
        const float mn0 = fmaxf(m0, mx0), mn1 = fmaxf(m1, mx1);
        const float r0 = m0 == -INFINITY ? 0.f : fast_exp2(m0 - mn0);
        const float r1 = m1 == -INFINITY ? 0.f : fast_exp2(m1 - mn1);
        const float u0 = mn0 == -INFINITY ? 0.f : mn0;
        const float u1 = mn1 == -INFINITY ? 0.f : mn1;
        float pr[2][4];
#pragma unroll
        for (int n = 0; n < 2; ++n) {
          pr[n][0] = fast_exp2(x[n][0] - u0);
          pr[n][1] = fast_exp2(x[n][1] - u0);
          pr[n][2] = fast_exp2(x[n][2] - u1);
          pr[n][3] = fast_exp2(x[n][3] - u1);
        }
        l0 = l0 * r0 + pr[0][0] + pr[0][1] + pr[1][0] + pr[1][1];
        l1 = l1 * r1 + pr[0][2] + pr[0][3] + pr[1][2] + pr[1][3];
        m0 = mn0;
        m1 = mn1;
#pragma unroll
        for (int n = 0; n < NT; ++n) {
          o[n][0] *= r0;
          o[n][1] *= r0;
          o[n][2] *= r1;
          o[n][3] *= r1;
        }
        // ---- O += P V ; P (C layout) -> A fragment without a smem round trip
        const uint32_t pa0 = pack_bf16(pr[0][0], pr[0][1]);
        const uint32_t pa1 = pack_bf16(pr[0][2], pr[0][3]);
        const uint32_t pa2 = pack_bf16(pr[1][0], pr[1][1]);
        const uint32_t pa3 = pack_bf16(pr[1][2], pr[1][3]);
        {
          const uint8_t* vp = vs + (t0 + (lane & 7) + ((lane >> 3) & 1) * 8) * C::kRowStride +
                              (lane >> 4) * 16;
#pragma unroll
          for (int n2 = 0; n2 < D / 16; ++n2) {
            uint32_t b0, b1, b2, b3;
            ldsm_x4_t(b0, b1, b2, b3, vp + n2 * 32);
            mma_bf16(o[2 * n2], pa0, pa1, pa2, pa3, b0, b1);
            mma_bf16(o[2 * n2 + 1], pa0, pa1, pa2, pa3, b2, b3);
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[stage]);
        if (++stage == C::kStages) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
    // ---- per-warp state -> smem, then cross-warp merge
    l0 += __shfl_xor_sync(0xffffffffu, l0, 1);
    l0 += __shfl_xor_sync(0xffffffffu, l0, 2);
    l1 += __shfl_xor_sync(0xffffffffu, l1, 1);
    l1 += __shfl_xor_sync(0xffffffffu, l1, 2);
    if ((lane & 3) == 0) {
      if (qr < G) {
        ml[(warp * C::kMaxG + qr) * 2] = m0;
        ml[(warp * C::kMaxG + qr) * 2 + 1] = l0;
      }
      if (qr + 8 < G) {
        ml[(warp * C::kMaxG + qr + 8) * 2] = m1;
        ml[(warp * C::kMaxG + qr + 8) * 2 + 1] = l1;
      }
    }
#pragma unroll
    for (int n = 0; n < NT; ++n) {
      const int d = n * 8 + qc;
      if (qr < G) {
        mo[(warp * C::kMaxG + qr) * D + d] = o[n][0];
        mo[(warp * C::kMaxG + qr) * D + d + 1] = o[n][1];
      }
      if (qr + 8 < G) {
        mo[(warp * C::kMaxG + qr + 8) * D + d] = o[n][2];
        mo[(warp * C::kMaxG + qr + 8) * D + d + 1] = o[n][3];
      }
    }
    unit_epilogue<__nv_bfloat16, D>(p, s, u, mo, ml, warp * 32 + lane);
  }
}

// ---------------------------------------------------------------- fp32 path
// CUDA-core FP32 (exact fp32 products, serial-order-free accumulation); used
// for the fp32 parity configs.  Lane l of warp w owns row t0 + (l & 15) for the
// scores (half h = l >> 4 of the d range), and d columns l, l+32, ... for PV.
template <int D>
__device__ __forceinline__ void consume_f32(const LycAttnParams& p, uint8_t* ring,
                                            uint64_t* full, uint64_t* empty, float* mo,
                                            float* ml, float* qs, int ub, int ue, int warp,
                                            int lane) {
  using C = AttnCfg<float, D>;
  constexpr int MAXG = 8;
  constexpr int DH = D / 2;
  constexpr int DC = (D + 31) / 32;
  const int G = p.group;
  const int t0 = warp * 16;
  const int tr = lane & 15, half = lane >> 4;
  int stage = 0;
  uint32_t phase = 0;
  const float* Q = static_cast<const float*>(p.q);

  for (int u = ub; u < ue; ++u) {
    const LycUnit un = p.units[u];
    const LycSlot s = p.slots[un.slot];
    const int tpi = tiles_per_item(s, p.block_size);
    const bool want_sel = s.sel >= 0 && p.sel_mode != SEL_NONE;
    float m[MAXG], l[MAXG], o[MAXG][DC];
#pragma unroll
    for (int j = 0; j < MAXG; ++j) {
      m[j] = -INFINITY;
      l[j] = 0.f;
#pragma unroll
      for (int c = 0; c < DC; ++c) o[j][c] = 0.f;
    }
    // stage the group's queries (rows 0..G-1) and the pooled query (row G,
    // gqa_pool_queries order: acc += q_j for j = 0..G-1, then acc /= G)
    const int tid = warp * 32 + lane;
    for (int d = tid; d < D; d += kConsumerWarps * 32) {
      float acc = 0.f;
      for (int j = 0; j < G; ++j) {
        const float v = __ldg(Q + (int64_t)(s.q_row + j) * D + d);
        qs[j * D + d] = v;
        acc += v;
      }
      qs[G * D + d] = acc / (float)G;
    }
    consumer_bar();
    for (int it = un.begin; it < un.end; ++it) {
      for (int sub = 0; sub < tpi; ++sub) {
        const Tile t = tile_of(s, it, sub, p.seq_len, p.block_size);
        mbar_wait(&full[stage], phase);
        const float* krow =
            reinterpret_cast<const float*>(ring + stage * C::kStageBytes + (t0 + tr) * C::kRowStride);
        const float* vs = reinterpret_cast<const float*>(ring + stage * C::kStageBytes + C::kTileBytes);
        float sc[MAXG], pooled = 0.f;
#pragma unroll
        for (int j = 0; j < MAXG; ++j) sc[j] = 0.f;
        for (int dd = 0; dd < DH; ++dd) {
          const int d = half * DH + dd;
          const float kv = krow[d];
#pragma unroll
          for (int j = 0; j < MAXG; ++j)
            if (j < G) sc[j] = fmaf(qs[j * D + d], kv, sc[j]);
          if (want_sel) pooled = fmaf(qs[G * D + d], kv, pooled);
        }
#pragma unroll
        for (int j = 0; j < MAXG; ++j) sc[j] += __shfl_xor_sync(0xffffffffu, sc[j], 16);
        const bool valid = t0 + tr < t.nvalid;
        if (want_sel) {
          pooled += __shfl_xor_sync(0xffffffffu, pooled, 16);
          if (p.sel_mode == SEL_TOKEN_KEYS) {
            if (half == 0 && valid)
              p.sel_keys[(int64_t)s.sel * p.sel_stride + t.lo + t0 + tr] = float_key(pooled);
          } else {
            uint32_t km = (half == 0 && valid) ? float_key(pooled) : 0u;
#pragma unroll
            for (int off = 1; off < 16; off <<= 1) km = max(km, __shfl_xor_sync(0xffffffffu, km, off));
            if (lane == 0 && km != 0u) atomicMax(p.sel_keys + (int64_t)s.sel * p.sel_stride + it, km);
          }
        }
        float pr[MAXG];
#pragma unroll
        for (int j = 0; j < MAXG; ++j) {
          if (j >= G) break;
          const float x = valid ? sc[j] * p.scale_log2 : -INFINITY;
          float mx = x;
#pragma unroll
          for (int off = 1; off < 16; off <<= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, off));
          const float mn = fmaxf(m[j], mx);
          const float r = m[j] == -INFINITY ? 0.f : exp2f(m[j] - mn);
          const float uu = mn == -INFINITY ? 0.f : mn;
          pr[j] = exp2f(x - uu);
          float ps = half == 0 ? pr[j] : 0.f;
#pragma unroll
          for (int off = 1; off < 32; off <<= 1) ps += __shfl_xor_sync(0xffffffffu, ps, off);
          l[j] = l[j] * r + ps;
          m[j] = mn;
#pragma unroll
          for (int c = 0; c < DC; ++c) o[j][c] *= r;
        }
        for (int rr = 0; rr < 16; ++rr) {
          const float* vrow = reinterpret_cast<const float*>(
              reinterpret_cast<const uint8_t*>(vs) + (t0 + rr) * C::kRowStride);
#pragma unroll
          for (int j = 0; j < MAXG; ++j) {
            if (j >= G) break;
            const float pj = __shfl_sync(0xffffffffu, pr[j], rr);
#pragma unroll
            for (int c = 0; c < DC; ++c)
              if (c * 32 + lane < D) o[j][c] = fmaf(pj, vrow[c * 32 + lane], o[j][c]);
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[stage]);
        if (++stage == C::kStages) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
#pragma unroll
    for (int j = 0; j < MAXG; ++j) {
      if (j >= G) break;
      if (lane == 0) {
        ml[(warp * C::kMaxG + j) * 2] = m[j];
        ml[(warp * C::kMaxG + j) * 2 + 1] = l[j];
      }
#pragma unroll
      for (int c = 0; c < DC; ++c)
        if (c * 32 + lane < D) mo[(warp * C::kMaxG + j) * D + c * 32 + lane] = o[j][c];
    }
    unit_epilogue<float, D>(p, s, u, mo, ml, warp * 32 + lane);
  }
}

template <typename T, int D>
__global__ void __launch_bounds__(kThreads, 1) hybrid_attn_kernel(const __grid_constant__ LycAttnParams p) {
  using C = AttnCfg<T, D>;
  extern __shared__ __align__(128) uint8_t smem[];
  uint8_t* ring = smem;
  float* mo = reinterpret_cast<float*>(smem + C::kStages * C::kStageBytes);
  float* ml = mo + kConsumerWarps * C::kMaxG * D;
  float* qs = ml + kConsumerWarps * C::kMaxG * 2;
  uint64_t* full = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(qs) + C::kQBytes);
  uint64_t* empty = full + C::kStages;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int cell = blockIdx.y * p.n_splits + blockIdx.x;
  const int ub = p.split_off[cell], ue = p.split_off[cell + 1];

  if (threadIdx.x == 0) {
    for (int s = 0; s < C::kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kConsumerWarps);
    }
    fence_mbar_init();
  }
  __syncthreads();
  if (warp == kConsumerWarps) {
    produce<T, D>(p, ring, full, empty, ub, ue, lane);
  } else if constexpr (sizeof(T) == 2) {
    consume_bf16<D>(p, ring, full, empty, mo, ml, ub, ue, warp, lane);
  } else {
    consume_f32<D>(p, ring, full, empty, mo, ml, qs, ub, ue, warp, lane);
  }
}

// ---------------------------------------------------------------- merge
// kernel_sim.hpp:205-225 combine, for slots with > 1 unit.  One warp per
// (task = (slot, j), 32-column chunk); lanes stride over the slot's partials
// in head-local split order, then a fixed-shape butterfly reduces across
// lanes -> bitwise deterministic for a given plan.
template <typename T>
__global__ void __launch_bounds__(128) split_merge_kernel(const __grid_constant__ LycMergeParams p) {
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int task = gw / p.chunks, chunk = gw - task * p.chunks;
  if (task >= p.n_tasks) return;
  const LycMergeTask tk = p.tasks[task];
  const LycSlot s = p.slots[tk.slot];
  const int D = p.d;
  const int G = p.group;
  float M = -INFINITY;
  for (int i = lane; i < s.n_units; i += 32)
    M = fmaxf(M, __ldcg(p.part_lse + (int64_t)(s.first_unit + i) * G + tk.j));
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, off));
  float den = 0.f;
  float acc[32];
#pragma unroll
  for (int c = 0; c < 32; ++c) acc[c] = 0.f;
  for (int i = lane; i < s.n_units; i += 32) {
    const int64_t u = s.first_unit + i;
    const float w = exp2f(__ldcg(p.part_lse + u * G + tk.j) - M);
    den += w;
    const float4* src = reinterpret_cast<const float4*>(p.part_o + (u * G + tk.j) * D + chunk * 32);
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      if (chunk * 32 + 4 * c >= D) break;
      const float4 v = __ldcg(src + c);
      acc[4 * c] = fmaf(w, v.x, acc[4 * c]);
      acc[4 * c + 1] = fmaf(w, v.y, acc[4 * c + 1]);
      acc[4 * c + 2] = fmaf(w, v.z, acc[4 * c + 2]);
      acc[4 * c + 3] = fmaf(w, v.w, acc[4 * c + 3]);
    }
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) den += __shfl_xor_sync(0xffffffffu, den, off);
  // reduce-scatter butterfly: after 5 rounds lane l holds column l's sum.
#pragma unroll
  for (int r = 0; r < 5; ++r) {
    const int half = 16 >> r;
    const bool upper = (lane & half) != 0;
#pragma unroll
    for (int c = 0; c < half; ++c) {
      const float send = upper ? acc[c] : acc[c + half];
      const float keep = upper ? acc[c + half] : acc[c];
      acc[c] = keep + __shfl_xor_sync(0xffffffffu, send, half);
    }
  }
  // lane's column: bits of lane select the kept half at each round
  const int col = lane;  // round r keeps the half selected by lane bit (16 >> r)
  if (chunk * 32 + col < D)
    store_out<T>(static_cast<T*>(p.out) + (int64_t)(s.q_row + tk.j) * D + chunk * 32 + col,
               acc[0] / den);
}

// ---------------------------------------------------------------- launchers
template <typename T, int D>
static cudaError_t launch_attn_t(const LycAttnParams& p, int batch, cudaStream_t st) {
  using C = AttnCfg<T, D>;
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(hybrid_attn_kernel<T, D>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmem);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  dim3 grid(p.n_splits, batch);
  hybrid_attn_kernel<T, D><<<grid, kThreads, C::kSmem, st>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_attn(const LycAttnParams& p, int dtype, int d, int batch, cudaStream_t st) {
  if (dtype == 1) {
    switch (d) {
      case 64: return launch_attn_t<__nv_bfloat16, 64>(p, batch, st);
      case 128: return launch_attn_t<__nv_bfloat16, 128>(p, batch, st);
      case 256: return launch_attn_t<__nv_bfloat16, 256>(p, batch, st);
    }
  } else {
    switch (d) {
      case 16: return launch_attn_t<float, 16>(p, batch, st);
      case 32: return launch_attn_t<float, 32>(p, batch, st);
      case 64: return launch_attn_t<float, 64>(p, batch, st);
      case 128: return launch_attn_t<float, 128>(p, batch, st);
    }
  }
  return cudaErrorInvalidValue;
}

int attn_stages(int dtype, int d) {
  if (dtype == 1) {
    switch (d) {
      case 64: return AttnCfg<__nv_bfloat16, 64>::kStages;
      case 128: return AttnCfg<__nv_bfloat16, 128>::kStages;
      case 256: return AttnCfg<__nv_bfloat16, 256>::kStages;
    }
  } else {
    switch (d) {
      case 16: return AttnCfg<float, 16>::kStages;
      case 32: return AttnCfg<float, 32>::kStages;
      case 64: return AttnCfg<float, 64>::kStages;
      case 128: return AttnCfg<float, 128>::kStages;
    }
  }
  return 0;
}

cudaError_t launch_merge(const LycMergeParams& p, int dtype, cudaStream_t st) {
  const int warps = p.n_tasks * p.chunks;
  if (warps == 0) return cudaSuccess;
  const int blocks = (warps + 3) / 4;
  if (dtype == 1)
    split_merge_kernel<__nv_bfloat16><<<blocks, 128, 0, st>>>(p);
  else
    split_merge_kernel<float><<<blocks, 128, 0, st>>>(p);
  return cudaGetLastError();
}

}  // namespace lyc
