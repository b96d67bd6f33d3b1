// attn_core.cuh -- device building blocks of the hybrid-head decode attention
// (reference: kernel_sim.hpp:169-201 run_split, 205-225 combine;
// attention.hpp:50-104 dense/sparse attention, 161-181 online_update).
// Shared by the per-layer kernels (attn.cu) and the persistent step kernel
// (step.cu).
//
// A CTA streams the 64-row K/V tiles of its split through a smem ring:
//   producers (2 warps):
//     * full contiguous tiles (retrieval heads, selected blocks): one thread
//       issues 2D tensor-map TMA boxes (64 rows x one 128-B panel, 128B
//       swizzle for bf16) -- 4 instructions per 32 KB stage, completion
//       counted in bytes on the stage's mbarrier;
//     * gathered tiles (token-sparse heads, ragged tails): all 64 producer
//       threads issue coalesced 16-B cp.async (LDGSTS) of the indexed rows into
//       the same swizzled layout, zero-filling masked rows, and arrive on the
//       mbarrier when their copies land.
//   consumers (4 warps): each owns 16 rows of every tile; the G <= 8 query
//     heads of the GQA group are packed as the A operand of mma.sync m16n8k16
//     (bf16 -> fp32), so every K/V byte is read from smem once for the whole
//     group.  Online softmax in the exp2 domain with quad-shuffle row max/sum;
//     P goes C-fragment -> A-fragment in registers.
//   fused selection (retrieval slots with sel >= 0): the pooled-query score
//     sum_j q_j.k of every row (= G * pooled_q.k, attention.hpp:127-146,
//     decode_engine.hpp:129-132) is reduced across the packed rows with three
//     shuffles and written as an order-preserving uint32 key (token mode,
//     plus the first radix-pass histogram when hist1 is given) or max-folded
//     per block (block mode).
//   end of unit: the 4 warps' (m, l, o) are merged through smem and written as
//     a normalized partial + base-2 LSE (kernel_sim.hpp:195-198), or as the
//     final output when the slot has a single unit.
#pragma once
#include <type_traits>

#include "lyc_common.cuh"
#include "lyc_plan.h"

namespace lyc {

constexpr int kConsumerWarps = 4;
constexpr int kProducerWarps = 2;
constexpr int kProducerThreads = kProducerWarps * 32;
constexpr int kMaxG = 8;

template <typename T, int D>
struct AttnCfg {
  static constexpr int kE = (int)sizeof(T);
  static constexpr bool kSwizzle = kE == 2;        // bf16 tiles: 128-B swizzled panels
  static constexpr int kRowBytes = D * kE;
  static constexpr int kPanelBytes = LYC_TILE * 128;
  static constexpr int kTileBytes = LYC_TILE * kRowBytes;
  static constexpr int kStageBytes = 2 * kTileBytes;  // K tile then V tile
  static constexpr int kChunksPerRow = kRowBytes / 16;
  static constexpr int kMergeBytes = kConsumerWarps * kMaxG * (D + 3) * 4;  // mo, ml, coef
  static constexpr int kQBytes = kE == 4 ? (kMaxG + 1) * D * 4 : 0;
  static constexpr int kMaxSmem = 232448 - 1024;   // 227 KB opt-in minus alignment slack
  // the step kernel's epilogue warps (selection); the step kernel is built for d <= 128 only
  static constexpr int kExtraBytes = D <= 128 ? 43008 : 0;  // >= sizeof(EpiSmem), step.cu
  // layer-start staging of up to kQUnits unit descriptors + their queries (bf16)
  static constexpr int kQUnits = 8;
  static constexpr int kURecBytes = 80;  // LycUnit + LycSlot, padded
  static constexpr int kUStageBytes = kE == 2 ? 2 * kQUnits * kURecBytes : 0;  // double-buffered
  static constexpr int kQStageBytes = kE == 2 ? kQUnits * kMaxG * D * 2 : 0;
  static constexpr int kHistBytes = LYC_H1_BINS * 4;  // per-CTA first-pass selection histogram
  static constexpr int kFixed = kMergeBytes + kQBytes + 512 + kExtraBytes + kHistBytes +
                                kUStageBytes + kQStageBytes;  // 512: barriers + 128-B alignment
  static constexpr int kStagesRaw = (kMaxSmem - kFixed) / kStageBytes;
  static constexpr int kStages = kStagesRaw > 8 ? 8 : kStagesRaw;
  static constexpr int kSmem = kStages * kStageBytes + kFixed + 1024;
  static_assert(kStages >= 2, "not enough shared memory for a 2-stage ring");
  static_assert(kRowBytes % 16 == 0 && (!kSwizzle || kRowBytes % 128 == 0), "row layout");

  // byte offset of 16-B chunk c of tile row r
  __device__ __forceinline__ static uint32_t off(int r, int c) {
    if constexpr (kSwizzle)
      return (uint32_t)((c >> 3) * kPanelBytes + r * 128 + (((c & 7) ^ (r & 7)) << 4));
    else
      return (uint32_t)(r * kRowBytes + c * 16);
  }
};

// Carved shared memory of one attention CTA.
template <typename T, int D>
struct AttnSmem {
  uint8_t* ring;
  float* mo;       // [warps][kMaxG][D] per-warp unnormalised outputs
  float* ml;       // [warps][kMaxG][2] per-warp (m, l)
  float* qs;       // fp32 path: staged queries [kMaxG + 1][D]
  uint64_t* full;
  uint64_t* empty;
  int2* tinfo;     // [kStages] (first row, valid rows) of the tile in each stage, from the producer
  uint32_t* clayer;  // step kernel: 1 + the layer the consumers have started (they passed its wait)
  uint8_t* extra;  // kExtraBytes scratch for other warp roles
  uint32_t* hist;  // [LYC_H1_BINS] first radix pass of the unit's selection keys (zero between units)
  uint8_t* ustage; // [kQUnits] unit records staged at layer start (bf16 consumers)
  uint8_t* qstage; // [kQUnits][kMaxG][D] bf16 queries of those units

  // Offsets are applied to the __shared__ array itself (no integer round trip),
  // so the compiler keeps the shared address space and emits LDS/STS/ATOMS --
  // generic accesses would queue behind the thread's outstanding global stores.
  static constexpr int kMoOff = 0;
  static constexpr int kMlOff = kMoOff + kConsumerWarps * kMaxG * D * 4;
  static constexpr int kQsOff = kMlOff + kConsumerWarps * kMaxG * 3 * 4;  // ml + coef
  static constexpr int kBarOff = kQsOff + AttnCfg<T, D>::kQBytes;
  static constexpr int kTinfoOff = kBarOff + 2 * AttnCfg<T, D>::kStages * 8;
  static constexpr int kCLayerOff = kTinfoOff + AttnCfg<T, D>::kStages * 8;
  static constexpr int kExtraOff = (kCLayerOff + 16 + 127) & ~127;
  static constexpr int kHistOff = kExtraOff + AttnCfg<T, D>::kExtraBytes;
  static constexpr int kUStageOff = kHistOff + AttnCfg<T, D>::kHistBytes;
  static constexpr int kQStageOff = kUStageOff + AttnCfg<T, D>::kUStageBytes;

  static_assert(kQStageOff + AttnCfg<T, D>::kQStageBytes + 1024 <= AttnCfg<T, D>::kSmem -
                    AttnCfg<T, D>::kStages * AttnCfg<T, D>::kStageBytes,
                "shared-memory carve exceeds the allocation");
  __device__ __forceinline__ static AttnSmem carve(uint8_t* raw) {
    using C = AttnCfg<T, D>;
    AttnSmem s;
    uint8_t* base = raw + ((1024u - (smem_u32(raw) & 1023u)) & 1023u);
    s.ring = base;
    uint8_t* fx = base + C::kStages * C::kStageBytes;
    s.mo = reinterpret_cast<float*>(fx + kMoOff);
    s.ml = reinterpret_cast<float*>(fx + kMlOff);
    s.qs = reinterpret_cast<float*>(fx + kQsOff);
    s.full = reinterpret_cast<uint64_t*>(fx + kBarOff);
    s.empty = s.full + C::kStages;
    s.tinfo = reinterpret_cast<int2*>(fx + kTinfoOff);
    s.clayer = reinterpret_cast<uint32_t*>(fx + kCLayerOff);
    s.extra = fx + kExtraOff;
    s.hist = reinterpret_cast<uint32_t*>(fx + kHistOff);
    s.ustage = fx + kUStageOff;
    s.qstage = fx + kQStageOff;
    return s;
  }
};

// Ring depth in use: fewer stages than the smem capacity keep fewer bytes in
// flight per SM -- enough to saturate HBM without inflating the memory
// system's queueing latency for the latency-bound work (merge, selection).
template <typename C>
__device__ __forceinline__ int ring_stages(const LycView& p) {
  return (p.stages > 0 && p.stages < C::kStages) ? p.stages : C::kStages;
}

struct Tile {
  int32_t lo;            // first row (contiguous tiles)
  int32_t nvalid;        // valid rows in this tile
  const int32_t* ids;    // token ids (gathered tiles) or nullptr
  int32_t cap;           // gathered tiles: ids readable (list capacity) from ids
};

__device__ __forceinline__ int tiles_per_item(const LycSlot& s, int bs) {
  return s.kind == ITEM_TOKENS ? 1 : (bs + LYC_TILE - 1) / LYC_TILE;
}

__device__ __forceinline__ Tile tile_of(const LycSlot& s, int item, int sub, int bs) {
  Tile t;
  if (s.kind == ITEM_TOKENS) {
    t.ids = s.list + (int64_t)item * LYC_TILE;
    t.lo = 0;
    t.cap = s.list_len - item * LYC_TILE;
    const int len = s.count ? min(s.list_len, __ldcg(s.count)) : s.list_len;
    t.nvalid = min(LYC_TILE, len - item * LYC_TILE);
  } else {
    const int blk = s.kind == ITEM_DENSE ? item : __ldcg(s.list + item);
    const int b0 = blk * bs;
    const int hi = min(b0 + bs, s.seq);  // ragged last block of this slot's sequence
    t.ids = nullptr;
    t.cap = 0;
    t.lo = b0 + sub * LYC_TILE;
    t.nvalid = max(0, min(LYC_TILE, hi - t.lo));
  }
  return t;
}

struct NoWaits {
  __device__ __forceinline__ void unit(const LycSlot&) const {}
  __device__ __forceinline__ bool needed() const { return false; }
  __device__ __forceinline__ bool any(bool) const { return false; }
  __device__ __forceinline__ void last_tile() const {}
};

// ---------------------------------------------------------------- producer
// Streams the tiles of units [ub, ue) of one layer.  `stage`/`phase` persist
// across calls (the persistent kernel keeps one ring across layers).
template <typename T, int D, typename Waits, bool kEarlyExit = false>
__device__ __forceinline__ void produce_units(const LycView& p, const CUtensorMap* tmk,
                                              const CUtensorMap* tmv, uint8_t* ring,
                                              uint64_t* full, uint64_t* empty, int2* tinfo,
                                              int ub, int ue,
                                              int pt, int& stage, uint32_t& phase,
                                              const Waits& waits) {
  using C = AttnCfg<T, D>;
  constexpr int CPR = C::kChunksPerRow;
  constexpr int kRowsPerRound = kProducerThreads / CPR > 0 ? kProducerThreads / CPR : 1;
  constexpr int kRounds = LYC_TILE / kRowsPerRound;
  static_assert(kProducerThreads % CPR == 0 || CPR % kProducerThreads == 0, "producer mapping");
  const uint64_t pol = policy_evict_first();
  const char* kbase = static_cast<const char*>(p.k);
  const char* vbase = static_cast<const char*>(p.v);
  const int my_c = pt % CPR;
  const int my_r0 = pt / CPR;
  // Row indices (gathered tiles) and block ids (block lists) of the NEXT tile
  // are loaded while the current tile is issued: one L2 round trip per unit
  // instead of one per tile.
  // (token lists: the id loads are predicated on the list capacity only, so
  // they overlap the device count's load; rows past the count are masked after)
  auto load_rows = [&](const Tile& t, int* rows) {
    if (t.ids == nullptr && t.nvalid == LYC_TILE) return;
#pragma unroll
    for (int i = 0; i < kRounds; ++i) {
      const int r = my_r0 + i * kRowsPerRound;
      rows[i] = t.ids ? (r < t.cap ? __ldcg(t.ids + r) : -1) : t.lo + r;
    }
#pragma unroll
    for (int i = 0; i < kRounds; ++i)
      if (my_r0 + i * kRowsPerRound >= t.nvalid) rows[i] = -1;
  };
  // unit records are prefetched one unit ahead (two dependent loads that
  // would otherwise stall the ring at every unit start)
  LycUnit un_next;
  LycSlot s_next;
  if (ub < ue) {
    un_next = p.units[ub];
    s_next = p.slots[un_next.slot];
  }
  for (int u = ub; u < ue; ++u) {
    const LycUnit un = un_next;
    LycSlot s = s_next;
    // the step kernel's live length of this slot's batch item (its plan is
    // reused while the length stays in the same 64-row block)
    if (p.seq_of) s.seq = p.seq_of[s.item];
    if (u + 1 < ue) {
      un_next = p.units[u + 1];
      s_next = p.slots[un_next.slot];
    }
    waits.unit(s);
    const int tpi = tiles_per_item(s, p.block_size);
    const int row0 = (int)(s.kv_off / D);  // tensor-map row of the slab's row 0
    const int nt = (un.end - un.begin) * tpi;
    Tile t = tile_of(s, un.begin, 0, p.block_size);
    int rows[kRounds];
    load_rows(t, rows);
    for (int f = 0; f < nt; ++f) {
      const int it = un.begin + f / tpi, sub = f % tpi;
      if (p.exec_counts && pt == 0 && sub == 0)
        atomicAdd(p.exec_counts + (int64_t)un.slot * p.counts_stride + it, 1u);
      Tile tn = t;
      int rows_n[kRounds];
      if (f + 1 < nt) {
        tn = tile_of(s, un.begin + (f + 1) / tpi, (f + 1) % tpi, p.block_size);
        load_rows(tn, rows_n);
      }
      {
        // the current token's K/V row is produced after the previous layer:
        // only a tile that holds it waits (dense: the last tile always; a
        // selected set: iff its largest id is the current token)
        // (from the tile's own rows -- no extra loads: contiguous tiles by
        // their range, gathered tiles by the ids already loaded)
        if (it == s.n_items - 1 && waits.needed()) {
          bool mine = false;
          if (t.ids) {
#pragma unroll
            for (int i = 0; i < kRounds; ++i) mine |= rows[i] == s.seq - 1;
          } else {
            mine = t.nvalid > 0 && t.lo + t.nvalid == s.seq;
          }
          if (waits.any(mine)) waits.last_tile();
        }
        uint8_t* kd = ring + stage * C::kStageBytes;
        uint8_t* vd = kd + C::kTileBytes;
        if (kEarlyExit && t.nvalid <= 0) {
          // past the end of a variable-size set (device count): an empty tile,
          // no copies; the consumers skip it
          mbar_wait(&empty[stage], phase ^ 1);
          if (pt == 0) {
            tinfo[stage] = make_int2(t.lo, 0);
            mbar_arrive(&full[stage]);
          }
          mbar_arrive(&full[stage]);
        } else if (t.ids == nullptr && t.nvalid == LYC_TILE) {
          mbar_wait(&empty[stage], phase ^ 1);
          if (pt == 0) {
            // the tile's rows for the consumers (no global loads on their side);
            // released by this thread's extra arrival
            tinfo[stage] = make_int2(t.lo, t.nvalid);
            mbar_arrive(&full[stage]);
            mbar_arrive_expect_tx(&full[stage], C::kStageBytes);
            if constexpr (C::kSwizzle) {
#pragma unroll
              for (int h = 0; h < C::kRowBytes / 128; ++h) {
                tma_load_2d(kd + h * C::kPanelBytes, tmk, h * (128 / C::kE), row0 + t.lo,
                            &full[stage], pol);
                tma_load_2d(vd + h * C::kPanelBytes, tmv, h * (128 / C::kE), row0 + t.lo,
                            &full[stage], pol);
              }
            } else {
              tma_load_2d(kd, tmk, 0, row0 + t.lo, &full[stage], pol);
              tma_load_2d(vd, tmv, 0, row0 + t.lo, &full[stage], pol);
            }
          } else {
            mbar_arrive(&full[stage]);
          }
        } else {
          // gathered / ragged tile: coalesced 16-B cp.async, masked rows zero-filled
          mbar_wait(&empty[stage], phase ^ 1);
          if (pt == 0) {
            tinfo[stage] = make_int2(t.lo, t.nvalid);
            mbar_arrive(&full[stage]);
          }
#pragma unroll
          for (int i = 0; i < kRounds; ++i) {
            const int r = my_r0 + i * kRowsPerRound;
            const int64_t src = (int64_t)(rows[i] < 0 ? 0 : rows[i]) * C::kRowBytes + my_c * 16 +
                                s.kv_off * C::kE;
            const uint32_t nbytes = rows[i] < 0 ? 0u : 16u;
            cp_async_16(kd + C::off(r, my_c), kbase + src, nbytes);
            cp_async_16(vd + C::off(r, my_c), vbase + src, nbytes);
          }
          cp_async_mbar_arrive(&full[stage]);
        }
        if (++stage == ring_stages<C>(p)) {
          stage = 0;
          phase ^= 1;
        }
      }
      t = tn;
#pragma unroll
      for (int i = 0; i < kRounds; ++i) rows[i] = rows_n[i];
    }
  }
}

// A data dependency for a stage release: false for every value an MMA / FMA
// chain produces (hardware NaNs are canonical 0x7fffffff), but the compiler
// cannot know that, so the caller's branch waits for `v` -- and with it for
// the shared-memory loads that fed it.
__device__ __forceinline__ bool stage_reads_done_never(float v) {
  return __float_as_uint(v) == 0x7fc00001u;
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

// Consumer-side timeline stamps (events 16..23 of the step timeline).
__device__ __forceinline__ void cstamp(const LycView& p, int ev, int tid) {
  if (p.trace_l && tid == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    p.trace_l[(size_t)ev * p.trace_ctas + blockIdx.x] = t;
  }
}

// Merge the consumer warps' (m, l, o) for one unit and emit partial / output.
template <typename T, int D>
__device__ __forceinline__ void unit_epilogue(const LycView& p, const LycSlot& s, int u,
                                              float* mo, float* ml, int tid, uint32_t* hist_s,
                                              uint32_t* hist_g) {
  const int G = p.group;
  cstamp(p, 20, tid);
  consumer_bar();
  cstamp(p, 21, tid);
  const bool direct = s.n_units == 1;
  // per query head j (one thread each): the warps' rescale coefficients
  // f_w / L and the unit's LSE -- computed once, not once per column
  float* coef = ml + kConsumerWarps * kMaxG * 2;  // [kMaxG][kConsumerWarps]
  if (tid < G) {
    const int j = tid;
    float M = -INFINITY;
#pragma unroll
    for (int w = 0; w < kConsumerWarps; ++w) M = fmaxf(M, ml[(w * kMaxG + j) * 2]);
    float f[kConsumerWarps], L = 0.f;
#pragma unroll
    for (int w = 0; w < kConsumerWarps; ++w) {
      const float mw = ml[(w * kMaxG + j) * 2];
      f[w] = mw == -INFINITY ? 0.f : exp2f(mw - M);
      L += ml[(w * kMaxG + j) * 2 + 1] * f[w];
    }
    // L == 0: the unit saw no valid row (a shard holding none of a sparse
    // head's indices) -- an empty partial (o = 0, lse = -inf)
    const float inv = L > 0.f ? 1.f / L : 0.f;
#pragma unroll
    for (int w = 0; w < kConsumerWarps; ++w) coef[j * kConsumerWarps + w] = f[w] * inv;
    const float lse = L > 0.f ? log2f(L) + M : -INFINITY;
    if (direct && p.out_f32)
      p.out_lse[s.q_row + j] = lse;
    else if (!direct)
      p.part_lse[(int64_t)u * G + j] = lse;
  }
  consumer_bar();
#pragma unroll 4
  for (int idx = tid; idx < G * D; idx += kConsumerWarps * 32) {
    const int j = idx / D, d = idx - j * D;
    float o = 0.f;
#pragma unroll
    for (int w = 0; w < kConsumerWarps; ++w)
      o = fmaf(mo[(w * kMaxG + j) * D + d], coef[j * kConsumerWarps + w], o);
    if (direct && p.out_f32)
      p.out_f32[(int64_t)(s.q_row + j) * D + d] = o;
    else if (direct)
      store_out<T>(static_cast<T*>(p.out) + (int64_t)(s.q_row + j) * D + d, o);
    else
      p.part_o[((int64_t)u * G + j) * D + d] = o;
  }
  cstamp(p, 22, tid);
  static_assert(kConsumerWarps * 32 * 32 == LYC_H1_BINS && LYC_H1_COARSE * 64 == LYC_H1_BINS,
                "histogram flush mapping");
  if (hist_g) {
    // flush the unit's first-pass histogram and re-zero it: thread t owns 32
    // consecutive bins, read and re-zeroed as eight 16-B vectors in a rotated
    // order (conflict-free), then one predicated global atomic per non-empty
    // bin; the 64-bin coarse summary (top 6 bits) after the fine bins gets one
    // atomic per non-empty coarse bin (thread pairs share one)
    uint4* hv = reinterpret_cast<uint4*>(hist_s + tid * 32);
    uint4 v[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] = hv[(j + tid) & 7];
#pragma unroll
    for (int j = 0; j < 8; ++j) hv[(j + tid) & 7] = make_uint4(0u, 0u, 0u, 0u);
    uint32_t sum = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      uint32_t* g = hist_g + tid * 32 + ((j + tid) & 7) * 4;
      if (v[j].x) atomicAdd(g, v[j].x);
      if (v[j].y) atomicAdd(g + 1, v[j].y);
      if (v[j].z) atomicAdd(g + 2, v[j].z);
      if (v[j].w) atomicAdd(g + 3, v[j].w);
      sum += v[j].x + v[j].y + v[j].z + v[j].w;
    }
    sum += __shfl_xor_sync(0xffffffffu, sum, 1);
    if ((tid & 1) == 0 && sum) atomicAdd(hist_g + LYC_H1_BINS + (tid >> 1), sum);
  }
  consumer_bar();
}

// Warp-aggregated increment of hist[bin] by the lanes in `mask` (all lanes of
// `mask` must call it; ok = false lanes contribute nothing).
__device__ __forceinline__ void hist_add(uint32_t* hist, uint32_t bin, bool ok, unsigned mask,
                                         int lane) {
  const uint32_t b = ok ? bin : (0x80000000u | (uint32_t)lane);
  const unsigned grp = __match_any_sync(mask, b);
  if (ok && lane == __ffs(grp) - 1) atomicAdd(hist + bin, (uint32_t)__popc(grp));
}

// ---------------------------------------------------------------- bf16 path
// Consumer warp w handles rows [16w, 16w+16) of each 64-row tile.  Query rows
// j < G <= 8 sit in A-fragment rows 0..7; rows 8..15 are zero, so only the
// c0/c1 halves of the score / output fragments carry data.
struct UnitRec {
  LycUnit u;
  LycSlot s;
};

// Unit records [ub, ub + n) (n <= cap) of one layer into shared memory, by the
// first n threads of the caller's group.
__device__ __forceinline__ void stage_unit_records(const LycView& p, UnitRec* rec, int ub, int ue,
                                                   int tid, int cap) {
  if (tid < min(ue - ub, cap)) {
    UnitRec r;
    r.u = p.units[ub + tid];
    r.s = p.unit_slots ? p.unit_slots[ub + tid] : p.slots[r.u.slot];
    rec[tid] = r;
  }
}

template <int D, bool kEarlyExit = false>
__device__ __forceinline__ void consume_units_bf16(const LycView& p, const AttnSmem<__nv_bfloat16, D>& sm,
                                                   int ub, int ue, int warp, int lane, int& stage,
                                                   uint32_t& phase, int rec_buf = -1) {
  using C = AttnCfg<__nv_bfloat16, D>;
  constexpr int KS = D / 16;  // k-steps over d for QK^T
  constexpr int NT = D / 8;   // n-tiles over d for PV
  const int G = p.group;
  const int qr = lane >> 2;   // A/C row of this lane
  const int qc = (lane & 3) * 2;
  const int t0 = warp * 16;
  const int sw = lane & 7;    // every ldmatrix row address below has (row & 7) == lane & 7
  // K (non-trans): row t0 + (lane>>4)*8 + (lane&7), chunk 2kk + ((lane>>3)&1)
  const uint32_t k_row = (uint32_t)(t0 + (lane >> 4) * 8 + (lane & 7)) * 128;
  const int k_x = (lane >> 3) & 1;
  // V (trans): row t0 + (lane&7) + ((lane>>3)&1)*8, chunk 2*n2 + (lane>>4)
  const uint32_t v_row = (uint32_t)(t0 + (lane & 7) + ((lane >> 3) & 1) * 8) * 128;
  const int v_x = lane >> 4;
  const __nv_bfloat16* Q = static_cast<const __nv_bfloat16*>(p.q);

  // ---- layer start: the first kQUnits unit records and their queries are
  // staged on chip (records possibly pre-staged by the caller while it waited
  // for the previous layer -- rec_buf >= 0), instead of three dependent L2
  // round trips (unit -> slot -> q) at every unit boundary
  constexpr int kQU = C::kQUnits;
  using URec = UnitRec;
  static_assert(sizeof(URec) <= C::kURecBytes, "unit record");
  const int tid = warp * 32 + lane;
  const int nst = min(ue - ub, kQU);
  URec* rec = reinterpret_cast<URec*>(sm.ustage) + (rec_buf > 0 ? kQU : 0);
  if (rec_buf < 0) {
    stage_unit_records(p, rec, ub, ue, tid, kQU);
    consumer_bar();
  }
  {
    const int cpu = G * D / 8;  // 16-B chunks of one unit's G query rows
    for (int c = tid; c < nst * cpu; c += kConsumerWarps * 32) {
      const int uu = c / cpu, r = c - uu * cpu;
      const uint4 v = __ldcg(reinterpret_cast<const uint4*>(Q + (int64_t)rec[uu].s.q_row * D) + r);
      reinterpret_cast<uint4*>(sm.qstage + uu * kMaxG * D * 2)[r] = v;
    }
  }
  consumer_bar();
  cstamp(p, 16, tid);

  for (int u = ub; u < ue; ++u) {
    const bool staged = u - ub < kQU;
    const LycUnit un = staged ? rec[u - ub].u : p.units[u];
    const LycSlot s = staged ? rec[u - ub].s : p.slots[un.slot];
    const int tpi = tiles_per_item(s, p.block_size);
    uint32_t qa0[KS], qa2[KS];
    const __nv_bfloat16* qst =
        reinterpret_cast<const __nv_bfloat16*>(sm.qstage + (u - ub) * kMaxG * D * 2);
#pragma unroll
    for (int kk = 0; kk < KS; ++kk) {
      if (staged) {
        const __nv_bfloat16* qrow = qst + qr * D + kk * 16 + qc;
        qa0[kk] = qr < G ? *reinterpret_cast<const unsigned int*>(qrow) : 0u;
        qa2[kk] = qr < G ? *reinterpret_cast<const unsigned int*>(qrow + 8) : 0u;
      } else {
        const __nv_bfloat16* qrow = Q + (int64_t)(s.q_row + qr) * D + kk * 16 + qc;
        qa0[kk] = qr < G ? __ldcg(reinterpret_cast<const unsigned int*>(qrow)) : 0u;
        qa2[kk] = qr < G ? __ldcg(reinterpret_cast<const unsigned int*>(qrow + 8)) : 0u;
      }
    }
    float m0 = -INFINITY, l0 = 0.f;
    // full m16n8 C fragments, accumulated in place: entries [2], [3] (rows
    // 8..15 of the A operand, which are zero) stay 0 and are never read
    float o[NT][4];
#pragma unroll
    for (int n = 0; n < NT; ++n) o[n][0] = o[n][1] = o[n][2] = o[n][3] = 0.f;
    const bool want_sel = s.sel >= 0 && p.sel_mode != SEL_NONE;
    uint32_t* hist = (want_sel && p.hist1) ? p.hist1 + (int64_t)s.sel * LYC_H1_STRIDE +
                                                 (blockIdx.x % LYC_H1_COPIES) * LYC_H1_ROW
                                           : nullptr;

    // the tile loop in two copies: with the fused selection scoring
    // (retrieval units) and without it -- no per-tile branch on it
    auto tiles = [&](auto sel_c) {
      constexpr int kSel = decltype(sel_c)::value;  // 0 none, 1 token keys, 2 block keys
      // one flat loop over the unit's tiles (item it, sub-tile sub)
      const int nt = (un.end - un.begin) * tpi;
      int it = un.begin, sub = 0;
      for (int f = 0; f < nt; ++f) {
        {
          mbar_wait(&sm.full[stage], phase);
          const int2 t = sm.tinfo[stage];  // (first row, valid rows)
          if (kEarlyExit && t.y <= 0) {  // past the end of a variable-size set: skip
            __syncwarp();
            if (lane == 0) mbar_arrive(&sm.empty[stage]);
            if (++stage == ring_stages<C>(p)) {
              stage = 0;
              phase ^= 1;
            }
            if (++sub == tpi) {
              sub = 0;
              ++it;
            }
            continue;
          }
          const uint8_t* ks = sm.ring + stage * C::kStageBytes;
          const uint8_t* vs = ks + C::kTileBytes;
          // ---- S = Q K^T for this warp's 16 rows (two n-tiles of 8)
          // two independent accumulator chains (even / odd k-steps) halve the
          // dependent-MMA latency of a tile; summed once at the end
          float sc[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
          float sd[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
  #pragma unroll
          for (int kk = 0; kk < KS; ++kk) {
            uint32_t b0, b1, b2, b3;
            const int c = 2 * (kk & 3) + k_x;
            ldsm_x4(b0, b1, b2, b3, ks + (kk >> 2) * C::kPanelBytes + k_row + ((c ^ sw) << 4));
            float (&acc)[2][4] = (kk & 1) ? sd : sc;
            mma_bf16(acc[0], qa0[kk], 0u, qa2[kk], 0u, b0, b1);
            mma_bf16(acc[1], qa0[kk], 0u, qa2[kk], 0u, b2, b3);
          }
  #pragma unroll
          for (int n = 0; n < 2; ++n)
  #pragma unroll
            for (int e = 0; e < 4; ++e) sc[n][e] += sd[n][e];
          // ---- fused selection score: sum over packed rows (rows >= G are 0)
          if constexpr (kSel != 0) {
            float ps[2][2];
  #pragma unroll
            for (int n = 0; n < 2; ++n)
  #pragma unroll
              for (int e = 0; e < 2; ++e) {
                float v = sc[n][e];
                v += __shfl_xor_sync(0xffffffffu, v, 4);
                v += __shfl_xor_sync(0xffffffffu, v, 8);
                v += __shfl_xor_sync(0xffffffffu, v, 16);
                ps[n][e] = v;
              }
            if constexpr (kSel == 1) {
              // lane r < 16 gathers row t0 + r's score (held by lane (r & 7) >> 1
              // as ps[r >> 3][r & 1]) so the warp's 16 keys go out in one
              // coalesced 64-B store and one shared-memory atomic
              const int r = lane & 15, src = (r & 7) >> 1;
              const float v00 = __shfl_sync(0xffffffffu, ps[0][0], src);
              const float v01 = __shfl_sync(0xffffffffu, ps[0][1], src);
              const float v10 = __shfl_sync(0xffffffffu, ps[1][0], src);
              const float v11 = __shfl_sync(0xffffffffu, ps[1][1], src);
              const float mine = (r >> 3) ? ((r & 1) ? v11 : v10) : ((r & 1) ? v01 : v00);
              if (lane < 16 && t0 + r < t.y) {
                const uint32_t key = float_key(mine);
                p.sel_keys[(int64_t)s.sel * p.sel_stride + t.x + t0 + r] = key;
                if (hist) atomicAdd(sm.hist + (key >> (32 - LYC_H1_BITS)), 1u);
              }
            } else {  // SEL_BLOCK_KEYS: max over valid rows of this block
              uint32_t km = 0u;
  #pragma unroll
              for (int n = 0; n < 2; ++n)
  #pragma unroll
                for (int e = 0; e < 2; ++e)
                  if (t0 + n * 8 + qc + e < t.y) km = max(km, float_key(ps[n][e]));
              km = max(km, __shfl_xor_sync(0xffffffffu, km, 1));
              km = max(km, __shfl_xor_sync(0xffffffffu, km, 2));
              if (lane == 0 && km != 0u)
                atomicMax(p.sel_keys + (int64_t)s.sel * p.sel_stride + it, km);
            }
          }
          // ---- online softmax (exp2 domain) for row qr
          float x[2][2];
  #pragma unroll
          for (int n = 0; n < 2; ++n)
  #pragma unroll
            for (int e = 0; e < 2; ++e)
              x[n][e] = t0 + n * 8 + qc + e < t.y ? sc[n][e] * p.scale_log2 : -INFINITY;
          const float mx = warp_max4(fmaxf(fmaxf(x[0][0], x[0][1]), fmaxf(x[1][0], x[1][1])));
          const float mn = fmaxf(m0, mx);
          const float rs = m0 == -INFINITY ? 0.f : fast_exp2(m0 - mn);
          const float mu = mn == -INFINITY ? 0.f : mn;
          const float p00 = fast_exp2(x[0][0] - mu), p01 = fast_exp2(x[0][1] - mu);
          const float p10 = fast_exp2(x[1][0] - mu), p11 = fast_exp2(x[1][1] - mu);
          l0 = l0 * rs + p00 + p01 + p10 + p11;
          m0 = mn;
  #pragma unroll
          for (int n = 0; n < NT; ++n) {
            o[n][0] *= rs;
            o[n][1] *= rs;
          }
          // ---- O += P V ; P (C layout) -> A fragment without a smem round trip
          const uint32_t pa0 = pack_bf16(p00, p01);
          const uint32_t pa2 = pack_bf16(p10, p11);
  #pragma unroll
          for (int n2 = 0; n2 < D / 16; ++n2) {
            uint32_t b0, b1, b2, b3;
            const int c = 2 * (n2 & 3) + v_x;
            ldsm_x4_t(b0, b1, b2, b3, vs + (n2 >> 2) * C::kPanelBytes + v_row + ((c ^ sw) << 4));
            mma_bf16(o[2 * n2], pa0, 0u, pa2, 0u, b0, b1);
            mma_bf16(o[2 * n2 + 1], pa0, 0u, pa2, 0u, b2, b3);
          }
          // release the stage only after its last ldmatrix has returned: an
          // mbarrier arrive does not wait for in-flight shared-memory loads
          // (measured: the producer's next copy into this stage raced the
          // final V ldmatrix -- columns 112..127 of a head's output), so the
          // arrive is made data-dependent on the MMA that consumes it
          // (every accumulator -- the compiler reorders the n2 loop freely --
          // combined in a shallow xor tree)
          uint32_t dep[NT];
#pragma unroll
          for (int n = 0; n < NT; ++n) dep[n] = __float_as_uint(o[n][0]);
#pragma unroll
          for (int w = 1; w < NT; w *= 2)
#pragma unroll
            for (int n = 0; n + w < NT; n += 2 * w) dep[n] ^= dep[n + w];
          __syncwarp();
          if (lane == 0 && !stage_reads_done_never(__uint_as_float(dep[0])))
            mbar_arrive(&sm.empty[stage]);
          if (++stage == ring_stages<C>(p)) {
            stage = 0;
            phase ^= 1;
          }
        }
        if (++sub == tpi) {
          sub = 0;
          ++it;
        }
      }
    };
    if (!want_sel)
      tiles(std::integral_constant<int, 0>{});
    else if (p.sel_mode == SEL_TOKEN_KEYS)
      tiles(std::integral_constant<int, 1>{});
    else
      tiles(std::integral_constant<int, 2>{});
    // ---- per-warp state -> smem, then cross-warp merge
    l0 += __shfl_xor_sync(0xffffffffu, l0, 1);
    l0 += __shfl_xor_sync(0xffffffffu, l0, 2);
    if ((lane & 3) == 0 && qr < G) {
      sm.ml[(warp * kMaxG + qr) * 2] = m0;
      sm.ml[(warp * kMaxG + qr) * 2 + 1] = l0;
    }
    if (qr < G) {
#pragma unroll
      for (int n = 0; n < NT; ++n)
        *reinterpret_cast<float2*>(&sm.mo[(warp * kMaxG + qr) * D + n * 8 + qc]) =
            make_float2(o[n][0], o[n][1]);
    }
    unit_epilogue<__nv_bfloat16, D>(p, s, s.first_unit + un.hls, sm.mo, sm.ml, warp * 32 + lane,
                                    sm.hist, hist);
    if (u == ub) cstamp(p, 18, tid);
    // one more finished unit of a slot that is merged or selected: its
    // partial, keys and histogram counts are published (unit_epilogue ended
    // with a consumer barrier)
    if ((want_sel || s.n_units > 1) && p.slot_ctr && tid == 0)
      asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(p.slot_ctr + (int64_t)un.slot * 16 + 12)
                   : "memory");
  }
}

// ---------------------------------------------------------------- fp32 path
// CUDA-core FP32 (exact fp32 products); used for the fp32 parity configs.
// Lane l of warp w owns row t0 + (l & 15) for the scores (half h = l >> 4 of
// the d range), and d columns l, l+32, ... for PV.  Tiles are unswizzled.
template <int D, bool kEarlyExit = false>
__device__ __forceinline__ void consume_units_f32(const LycView& p, const AttnSmem<float, D>& sm,
                                                  int ub, int ue, int warp, int lane, int& stage,
                                                  uint32_t& phase) {
  using C = AttnCfg<float, D>;
  constexpr int DH = D / 2;
  constexpr int DC = (D + 31) / 32;
  const int G = p.group;
  const int t0 = warp * 16;
  const int tr = lane & 15, half = lane >> 4;
  const float* Q = static_cast<const float*>(p.q);
  float* qs = sm.qs;

  for (int u = ub; u < ue; ++u) {
    const LycUnit un = p.units[u];
    const LycSlot s = p.slots[un.slot];
    const int tpi = tiles_per_item(s, p.block_size);
    const bool want_sel = s.sel >= 0 && p.sel_mode != SEL_NONE;
    uint32_t* hist = (want_sel && p.hist1) ? p.hist1 + (int64_t)s.sel * LYC_H1_STRIDE +
                                                 (blockIdx.x % LYC_H1_COPIES) * LYC_H1_ROW
                                           : nullptr;
    float m[kMaxG], l[kMaxG], o[kMaxG][DC];
#pragma unroll
    for (int j = 0; j < kMaxG; ++j) {
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
        const float v = __ldcg(Q + (int64_t)(s.q_row + j) * D + d);
        qs[j * D + d] = v;
        acc += v;
      }
      qs[G * D + d] = acc / (float)G;
    }
    consumer_bar();
    for (int it = un.begin; it < un.end; ++it) {
      for (int sub = 0; sub < tpi; ++sub) {
        mbar_wait(&sm.full[stage], phase);
        const int2 t = sm.tinfo[stage];  // (first row, valid rows)
        if (kEarlyExit && t.y <= 0) {  // past the end of a variable-size set: skip
          __syncwarp();
          if (lane == 0) mbar_arrive(&sm.empty[stage]);
          if (++stage == ring_stages<C>(p)) {
            stage = 0;
            phase ^= 1;
          }
          continue;
        }
        const uint8_t* ks = sm.ring + stage * C::kStageBytes;
        const float* krow = reinterpret_cast<const float*>(ks + (t0 + tr) * C::kRowBytes);
        const uint8_t* vs = ks + C::kTileBytes;
        float sc[kMaxG], pooled = 0.f;
#pragma unroll
        for (int j = 0; j < kMaxG; ++j) sc[j] = 0.f;
        for (int dd = 0; dd < DH; ++dd) {
          const int d = half * DH + dd;
          const float kv = krow[d];
#pragma unroll
          for (int j = 0; j < kMaxG; ++j)
            if (j < G) sc[j] = fmaf(qs[j * D + d], kv, sc[j]);
          if (want_sel) pooled = fmaf(qs[G * D + d], kv, pooled);
        }
#pragma unroll
        for (int j = 0; j < kMaxG; ++j) sc[j] += __shfl_xor_sync(0xffffffffu, sc[j], 16);
        const bool valid = t0 + tr < t.y;
        if (want_sel) {
          pooled += __shfl_xor_sync(0xffffffffu, pooled, 16);
          if (p.sel_mode == SEL_TOKEN_KEYS) {
            if (half == 0) {
              const uint32_t key = float_key(pooled);
              if (valid) {
                p.sel_keys[(int64_t)s.sel * p.sel_stride + t.x + t0 + tr] = key;
                if (hist) atomicAdd(sm.hist + (key >> (32 - LYC_H1_BITS)), 1u);
              }
            }
          } else {
            uint32_t km = (half == 0 && valid) ? float_key(pooled) : 0u;
#pragma unroll
            for (int off = 1; off < 16; off <<= 1)
              km = max(km, __shfl_xor_sync(0xffffffffu, km, off));
            if (lane == 0 && km != 0u)
              atomicMax(p.sel_keys + (int64_t)s.sel * p.sel_stride + it, km);
          }
        }
        float pr[kMaxG];
#pragma unroll
        for (int j = 0; j < kMaxG; ++j) {
          if (j >= G) break;
          const float x = valid ? sc[j] * p.scale_log2 : -INFINITY;
          float mx = x;
#pragma unroll
          for (int off = 1; off < 16; off <<= 1)
            mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, off));
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
          const float* vrow = reinterpret_cast<const float*>(vs + (t0 + rr) * C::kRowBytes);
#pragma unroll
          for (int j = 0; j < kMaxG; ++j) {
            if (j >= G) break;
            const float pj = __shfl_sync(0xffffffffu, pr[j], rr);
#pragma unroll
            for (int c = 0; c < DC; ++c)
              if (c * 32 + lane < D) o[j][c] = fmaf(pj, vrow[c * 32 + lane], o[j][c]);
          }
        }
        // the stage's last loads must have returned before its release (see
        // the bf16 path): the arrive depends on the accumulators they feed
        float last = 0.f;
#pragma unroll
        for (int c = 0; c < DC; ++c) last += o[0][c];
        __syncwarp();
        if (lane == 0 && !stage_reads_done_never(last)) mbar_arrive(&sm.empty[stage]);
        if (++stage == ring_stages<C>(p)) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
#pragma unroll
    for (int j = 0; j < kMaxG; ++j) {
      if (j >= G) break;
      if (lane == 0) {
        sm.ml[(warp * kMaxG + j) * 2] = m[j];
        sm.ml[(warp * kMaxG + j) * 2 + 1] = l[j];
      }
#pragma unroll
      for (int c = 0; c < DC; ++c)
        if (c * 32 + lane < D) sm.mo[(warp * kMaxG + j) * D + c * 32 + lane] = o[j][c];
    }
    unit_epilogue<float, D>(p, s, s.first_unit + un.hls, sm.mo, sm.ml, warp * 32 + lane, sm.hist,
                            hist);
    if ((want_sel || s.n_units > 1) && p.slot_ctr && warp * 32 + lane == 0)
      asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(p.slot_ctr + (int64_t)un.slot * 16 + 12)
                   : "memory");
  }
}

// kEarlyExit: units may end early (variable-size sets with device counts:
// TopP / Threshold, sequence shards); compiled out of the step kernel, whose
// tile loop is sensitive to the extra exit path.
template <typename T, int D, bool kEarlyExit = false>
__device__ __forceinline__ void consume_units(const LycView& p, const AttnSmem<T, D>& sm, int ub,
                                              int ue, int warp, int lane, int& stage,
                                              uint32_t& phase, int rec_buf = -1) {
  if constexpr (sizeof(T) == 2)
    consume_units_bf16<D, kEarlyExit>(p, sm, ub, ue, warp, lane, stage, phase, rec_buf);
  else
    consume_units_f32<D, kEarlyExit>(p, sm, ub, ue, warp, lane, stage, phase);
}

// ---------------------------------------------------------------- merge
// kernel_sim.hpp:205-225 combine for one (slot, j, 32-column chunk) by one
// warp: lanes stride over the slot's partials in head-local split order, a
// fixed-shape butterfly reduces across lanes -> bitwise deterministic.
template <typename T>
__device__ __forceinline__ void merge_task(const float* part_o, const float* part_lse,
                                           const LycMergeTask& s, int chunk, int G, int D,
                                           void* out, int lane, float* out_f32 = nullptr,
                                           float* out_lse = nullptr) {
  const int j = s.j;
  // one pass (online rescaling) in batches of kB partials per lane: all of a
  // batch's LSE and output loads are issued before any is used -- a slot with
  // <= 32 * kB partials merges in ONE L2 round trip
  constexpr int kB = 4;
  float m = -INFINITY, den = 0.f;
  float acc[32];
#pragma unroll
  for (int c = 0; c < 32; ++c) acc[c] = 0.f;
  for (int base = 0; base < s.n_units; base += 32 * kB) {
    float lse[kB];
    float4 v[kB][8];
#pragma unroll
    for (int b = 0; b < kB; ++b) {
      const int i = base + b * 32 + lane;
      const bool ok = i < s.n_units;
      const int64_t u = s.first_unit + (ok ? i : 0);
      lse[b] = ok ? __ldcg(part_lse + u * G + j) : -INFINITY;
      const float4* src = reinterpret_cast<const float4*>(part_o + (u * G + j) * D + chunk * 32);
#pragma unroll
      for (int c = 0; c < 8; ++c)
        v[b][c] = (ok && chunk * 32 + 4 * c < D) ? __ldcg(src + c) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int b = 0; b < kB; ++b) {
      if (lse[b] == -INFINITY) continue;  // empty or absent partial
      if (lse[b] > m) {
        const float f = m == -INFINITY ? 0.f : exp2f(m - lse[b]);
        den *= f;
#pragma unroll
        for (int c = 0; c < 32; ++c) acc[c] *= f;
        m = lse[b];
      }
      const float w = exp2f(lse[b] - m);
      den += w;
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        acc[4 * c] = fmaf(w, v[b][c].x, acc[4 * c]);
        acc[4 * c + 1] = fmaf(w, v[b][c].y, acc[4 * c + 1]);
        acc[4 * c + 2] = fmaf(w, v[b][c].z, acc[4 * c + 2]);
        acc[4 * c + 3] = fmaf(w, v[b][c].w, acc[4 * c + 3]);
      }
    }
  }
  // rescale every lane to the warp maximum, then the fixed-shape reductions
  float M = m;
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, off));
  const float Mz = M == -INFINITY ? 0.f : M;  // all partials empty: output 0
  {
    const float f = m == -INFINITY ? 0.f : exp2f(m - Mz);
    den *= f;
#pragma unroll
    for (int c = 0; c < 32; ++c) acc[c] *= f;
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) den += __shfl_xor_sync(0xffffffffu, den, off);
  // reduce-scatter butterfly: after 5 rounds lane l holds column l's sum
  // (round r keeps the half selected by lane bit 16 >> r).
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
  const float o = den > 0.f ? acc[0] / den : 0.f;
  if (out_f32) {
    if (chunk * 32 + lane < D) out_f32[(int64_t)(s.q_row + j) * D + chunk * 32 + lane] = o;
    if (chunk == 0 && lane == 0) out_lse[s.q_row + j] = den > 0.f ? log2f(den) + Mz : -INFINITY;
  } else if (chunk * 32 + lane < D) {
    store_out<T>(static_cast<T*>(out) + (int64_t)(s.q_row + j) * D + chunk * 32 + lane, o);
  }
}

}  // namespace lyc
