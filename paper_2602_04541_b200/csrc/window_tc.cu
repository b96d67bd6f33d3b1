// window_tc.cu -- cache-correction window attention on the 5th-generation
// tensor cores (decode_engine.hpp:164-204): after the K/V
// rows of the last W positions were rewritten (kv_cache.hpp:34-42), window
// position p = start + i re-attends keys [0, p].  Per (b, KV head g) the W x G
// query rows are ONE M = 128 UMMA tile, so every K/V byte crosses HBM once for
// all of them (a prefill-style pass over the cache, not W decode passes).
//
// One CTA per (key split, b*H + g, 128-row block), 1 CTA per SM:
//   warps 0, 2    TMA producers: 64-key K and V tiles (128B-swizzled panels,
//                 3-D tensor maps whose row extent is the live length, so rows
//                 past it arrive as zeros) into separate rings -- K freed when
//                 its QK completes, V when its PV completes;
//   warps 1, 3    MMA issuers (one lane each; warp 1 also owns TMEM):
//                   S_t = Q K_t^T    tcgen05.mma kind::f16, M 128, N 64, K = d
//                   O_t = P_t V_t    M 128, N = d, K 64 (V is the MN-major operand)
//                 S double-buffered (2 x 64 TMEM columns); two O accumulators
//                 in TMEM (even / odd tiles, d columns each); completion via
//                 tcgen05.commit -> mbarrier;
//   warps 4-7, 8-11  two softmax warpgroups, even and odd tiles, each with its
//                 own S buffer, P buffer, O accumulator and (m, l) per row --
//                 two independent pipelines, merged per row at the end.
//                 Thread r of a group owns query row r (TMEM lane r): tcgen05.ld
//                 of its S row, causal / split mask, online softmax in the exp2
//                 domain, P_t (bf16) into shared memory in the UMMA K-major
//                 SW128 layout.  Lazy rescaling: P is taken against a reference
//                 max m_ref that moves only when the row max exceeds it by more
//                 than kRescale (P <= 2^kRescale), and only then is the row's O
//                 rescaled in TMEM (ld, scale, st) -- exact, just a different
//                 reference point, and rare after the first tiles.
// The key range is split across CTAs (flash-decoding); each split writes a
// normalized partial + base-2 LSE per row, merged by window_merge_kernel
// (window.cu) in split order.
#include <algorithm>

#include "lyc_common.cuh"
#include "lyc_plan.h"

namespace lyc {

constexpr int kTcRows = 128;   // UMMA M: query rows per CTA
constexpr int kTcKeys = 64;    // keys per tile (UMMA N of S, K of P V)
constexpr int kKStages = 4;   // K tiles in flight (released when their QK completes)
constexpr int kVStages = 4;   // V tiles in flight (released when their PV completes)
constexpr int kPBufs = 4;     // P tiles in shared memory (two per softmax group)
constexpr int kSBufs = 4;     // score tiles in TMEM (QK runs this far ahead of PV)
constexpr uint32_t kOCol = kSBufs * kTcKeys;  // TMEM column of the two O accumulators
constexpr int kTcThreads = 384;  // TMA warp, MMA warp, 2 idle, two softmax warpgroups

struct WinTcParams {
  CUtensorMap tmap_k;       // 3-D: {d, live rows, L*B*H slabs}, box {64, 64, 1}, SW128
  CUtensorMap tmap_v;
  const __nv_bfloat16* q;   // [B][W][Hq][d]
  float* part_o;            // [B*H][rb][n_split][128][d]
  float* part_lse;          // [B*H][rb][n_split][128]
  int32_t B, H, G, W, rows, rb, n_split, layer;
  int64_t start;            // first window position
  int64_t keys;             // start + W
  int64_t split_keys;       // keys per split (multiple of kTcKeys)
  float scale_log2;
};

template <int D>
struct WinTcSmem {
  static constexpr int kPanels = D / 64;
  static constexpr int kQBytes = kTcRows * D * 2;          // [panel][128 rows][128 B]
  static constexpr int kTileBytes = 2 * kTcKeys * D * 2;   // K + V of one tile
  static constexpr int kPBytes = kTcRows * kTcKeys * 2;    // one panel [128 rows][128 B] each
  static constexpr int kQOff = 0;
  static constexpr int kKOff = kQOff + kQBytes;
  static constexpr int kTileHalf = kTileBytes / 2;        // one of K or V: [panel][64 rows][128 B]
  static constexpr int kVOff = kKOff + kKStages * kTileHalf;
  static constexpr int kPOff = kVOff + kVStages * kTileHalf;
  static constexpr int kBarOff = kPOff + kPBufs * kPBytes;
  // barriers: k_full[KS], k_empty[KS], v_full[VS], v_empty[VS], s_full[4], s_empty[4],
  // pv_done[4], p_full[4]
  static constexpr int kNumBars = 2 * kKStages + 2 * kVStages + 2 * kSBufs + 2 * kPBufs;
  static constexpr int kMlOff = kBarOff + kNumBars * 8;     // [128] (m, l) of softmax group 1
  static constexpr int kTmemOff = kMlOff + kTcRows * 8;
  static constexpr int kBytes = kTmemOff + 16;
  static constexpr int kAlloc = kBytes + 1024;             // + alignment slack
};

// ---------------------------------------------------------------- tcgen05 PTX
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
// UMMA shared-memory descriptor (sm_100): start, leading / stride byte offsets
// (>> 4), version 1, 128B swizzle.  Atoms are 8 rows x 128 B, 1024-B aligned.
__device__ __forceinline__ uint64_t umma_desc_sw128(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  const uint64_t lo = (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16);
  const uint64_t hi = (uint64_t)((sbo >> 4) & 0x3FFFu) | (1ull << 14) | (2ull << 29);
  return lo | (hi << 32);
}
// kind::f16 instruction descriptor: bf16 A/B, fp32 D, M 128, N n; b_mn: B is MN-major.
__host__ __device__ constexpr uint32_t umma_idesc_bf16(int n, bool b_mn) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((b_mn ? 1u : 0u) << 16) | ((uint32_t)(n >> 3) << 17) |
         ((uint32_t)(kTcRows >> 4) << 24);
}
__device__ __forceinline__ void umma_bf16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                          uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}
// 32 consecutive TMEM columns of this thread's lane (warp w reads lanes 32*(w%4)..+31)
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float (&v)[32]) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
      "%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]),
        "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]),
        "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr)
      : "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
      "%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
      "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]),
      "r"(r[16]), "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]),
      "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
      : "memory");
}
__device__ __forceinline__ void tmem_st_wait() {
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_ld_wait() {
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* tmap, int c0, int c1,
                                            int c2, uint64_t* bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      ".L2::cache_hint [%0], [%1, {%2, %3, %4}], [%5], %6;" ::"r"(smem_u32(dst)),
      "l"(tmap), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}

// byte offset of 16-B chunk c (8 bf16) of row r in a [panel][rows][128 B] SW128 block
__device__ __forceinline__ uint32_t sw128_off(int r, int c, int panel_bytes) {
  return (uint32_t)((c >> 3) * panel_bytes + r * 128 + (((c & 7) ^ (r & 7)) << 4));
}

template <int D>
__global__ void __launch_bounds__(kTcThreads, 1) window_tc_kernel(const __grid_constant__ WinTcParams p) {
  using S = WinTcSmem<D>;
  extern __shared__ uint8_t tc_raw[];
  uint8_t* sm = tc_raw + ((1024u - (smem_u32(tc_raw) & 1023u)) & 1023u);
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + S::kBarOff);
  uint64_t* k_full = bars;
  uint64_t* k_empty = k_full + kKStages;
  uint64_t* v_full = k_empty + kKStages;
  uint64_t* v_empty = v_full + kVStages;
  uint64_t* s_full = v_empty + kVStages;
  uint64_t* s_empty = s_full + kSBufs;
  uint64_t* pv_done = s_full + 2 * kSBufs;  // [kPBufs]: PV_t commits to pv_done[t % kPBufs]
  uint64_t* p_full = pv_done + kPBufs;      // [kPBufs]: P_t (P buffer t % kPBufs) written
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(sm + S::kTmemOff);

  const int split = blockIdx.x, bh = blockIdx.y, rblk = blockIdx.z;
  const int b = bh / p.H, g = bh - b * p.H;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int row0 = rblk * kTcRows;
  const int64_t k_lo = (int64_t)split * p.split_keys;
  const int64_t k_hi = min(p.keys, k_lo + p.split_keys);
  const int nt = k_hi > k_lo ? (int)((k_hi - k_lo + kTcKeys - 1) / kTcKeys) : 0;
  const int slab = (p.layer * p.B + b) * p.H + g;

  if (tid == 0) {
    for (int s = 0; s < kKStages; ++s) {
      mbar_init(&k_full[s], 1);
      mbar_init(&k_empty[s], 1);
    }
    for (int s = 0; s < kVStages; ++s) {
      mbar_init(&v_full[s], 1);
      mbar_init(&v_empty[s], 1);
    }
    for (int i = 0; i < kSBufs; ++i) {
      mbar_init(&s_full[i], 1);
      mbar_init(&s_empty[i], 4);
    }
    for (int i = 0; i < kPBufs; ++i) {
      mbar_init(&pv_done[i], 1);
      mbar_init(&p_full[i], 4);
    }
    fence_mbar_init();
  }
  if (warp == 1) {  // TMEM: S [4][64 cols] at 0, O [2][D cols] at 256
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                     smem_u32(tmem_slot))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  // Q rows r = i*G + j of (b, g) -> q[b][i][g*G + j], zero past the window
  constexpr int CH = D / 8;
  for (int x = tid; x < kTcRows * CH; x += kTcThreads) {
    const int r = x / CH, c = x - r * CH;
    const int rr = row0 + r;
    const void* src = p.q;
    uint32_t bytes = 0;
    if (rr < p.rows) {
      const int i = rr / p.G, j = rr - i * p.G;
      src = p.q + (((int64_t)b * p.W + i) * (p.H * p.G) + g * p.G + j) * D + c * 8;
      bytes = 16;
    }
    cp_async_16(sm + S::kQOff + sw128_off(r, c, kTcRows * 128), src, bytes);
  }
  asm volatile("cp.async.wait_all;" ::: "memory");
  fence_proxy_async();  // generic-proxy Q writes -> the tensor cores' reads
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ---------------- TMA producer of the K tiles
    if (lane == 0 && nt > 0) {
      prefetch_tensormap(&p.tmap_k);
      const uint64_t pol = policy_evict_first();
      for (int t = 0; t < nt; ++t) {
        const int s = t % kKStages;
        mbar_wait(&k_empty[s], ((t / kKStages) & 1) ^ 1);
        mbar_arrive_expect_tx(&k_full[s], (uint32_t)S::kTileHalf);
        uint8_t* kd = sm + S::kKOff + s * S::kTileHalf;
#pragma unroll
        for (int h = 0; h < S::kPanels; ++h)
          tma_load_3d(kd + h * kTcKeys * 128, &p.tmap_k, h * 64, (int)(k_lo + (int64_t)t * kTcKeys),
                      slab, &k_full[s], pol);
      }
    }
  } else if (warp == 2) {
    // ---------------- TMA producer of the V tiles
    if (lane == 0 && nt > 0) {
      prefetch_tensormap(&p.tmap_v);
      const uint64_t pol = policy_evict_first();
      for (int t = 0; t < nt; ++t) {
        const int s = t % kVStages;
        mbar_wait(&v_empty[s], ((t / kVStages) & 1) ^ 1);
        mbar_arrive_expect_tx(&v_full[s], (uint32_t)S::kTileHalf);
        uint8_t* vd = sm + S::kVOff + s * S::kTileHalf;
#pragma unroll
        for (int h = 0; h < S::kPanels; ++h)
          tma_load_3d(vd + h * kTcKeys * 128, &p.tmap_v, h * 64, (int)(k_lo + (int64_t)t * kTcKeys),
                      slab, &v_full[s], pol);
      }
    }
  } else if (warp == 1 || warp == 3) {
    // ---------------- MMA issuers: warp 1 the scores (S = Q K^T), warp 3 the
    // P V products -- two threads, so neither waits behind the other's inputs
    // (each tcgen05.commit tracks its own thread's MMAs)
    if (lane == 0 && nt > 0) {
      constexpr uint32_t idesc_s = umma_idesc_bf16(kTcKeys, false);
      constexpr uint32_t idesc_o = umma_idesc_bf16(D, true);
      const uint32_t q_base = smem_u32(sm + S::kQOff);
      const uint32_t p_base = smem_u32(sm + S::kPOff);
      auto qk = [&](int t) {
        const int s = t % kKStages, sb = t % kSBufs;
        mbar_wait(&k_full[s], (t / kKStages) & 1);
        mbar_wait(&s_empty[sb], ((t / kSBufs) & 1) ^ 1);
        tc_fence_after();
        const uint32_t k_base = smem_u32(sm + S::kKOff + s * S::kTileHalf);
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint32_t koff = (uint32_t)(kk & 3) * 32u;  // 16 columns inside the 128-B row
          const uint64_t ad = umma_desc_sw128(q_base + (kk >> 2) * kTcRows * 128 + koff, 0, 1024);
          const uint64_t bd = umma_desc_sw128(k_base + (kk >> 2) * kTcKeys * 128 + koff, 0, 1024);
          umma_bf16(tmem + (uint32_t)(sb * kTcKeys), ad, bd, idesc_s, kk > 0 ? 1u : 0u);
        }
        umma_commit(&s_full[sb]);
        umma_commit(&k_empty[s]);
      };
      auto pv = [&](int t) {
        const int s = t % kVStages;
        mbar_wait(&v_full[s], (t / kVStages) & 1);
        mbar_wait(&p_full[t % kPBufs], (t / kPBufs) & 1);  // P_t written (O rescaled if it had to be)
        tc_fence_after();
        const uint32_t v_base = smem_u32(sm + S::kVOff + s * S::kTileHalf);
        const uint32_t pt_base = p_base + (uint32_t)((t % kPBufs) * S::kPBytes);
#pragma unroll
        for (int kk = 0; kk < kTcKeys / 16; ++kk) {
          const uint64_t ad = umma_desc_sw128(pt_base + (uint32_t)kk * 32u, 0, 1024);
          // V [keys][d]: d contiguous (MN-major); 8-key atoms 1024 B apart,
          // 64-column panels kTcKeys * 128 B apart
          const uint64_t bd = umma_desc_sw128(v_base + (uint32_t)kk * 16u * 128u, kTcKeys * 128, 1024);
          umma_bf16(tmem + kOCol + (uint32_t)((t & 1) * D), ad, bd, idesc_o,
                    (t > 1 || kk > 0) ? 1u : 0u);
        }
        umma_commit(&pv_done[t % kPBufs]);
        umma_commit(&v_empty[s]);
      };
      if (warp == 1)
        for (int t = 0; t < nt; ++t) qk(t);
      else
        for (int t = 0; t < nt; ++t) pv(t);
    }
  } else if (warp >= 4) {
    // ---------------- softmax group grp (tiles t = grp, grp + 2, ...): thread r owns row r
    const int grp = (warp - 4) >> 2;
    const int r = (warp & 3) * 32 + lane;    // = TMEM lane
    const int rr = row0 + r;
    const int64_t lim = rr < p.rows ? p.start + rr / p.G : -1;  // last key this row sees
    const int full_rows = row0 + kTcRows <= p.rows ? 1 : 0;     // every row of the block is live
    const uint32_t lane_base = (uint32_t)((warp & 3) * 32) << 16;
    constexpr float kRescale = 8.f;  // P <= 2^8 against the reference max
    float m = -INFINITY, l = 0.f;  // m: the reference max (exp2 domain)
    auto o_addr = [&](int g) { return tmem + lane_base + kOCol + (uint32_t)(g * D); };
    for (int t = grp; t < nt; t += 2) {
      const uint32_t sb = (uint32_t)(t % kSBufs);
      mbar_wait(&s_full[sb], (t / kSBufs) & 1);
      tc_fence_after();
      float sv[kTcKeys];
#pragma unroll
      for (int c0 = 0; c0 < kTcKeys; c0 += 32) {
        float v[32];
        tmem_ld32(tmem + lane_base + sb * kTcKeys + (uint32_t)c0, v);
        tmem_ld_wait();
#pragma unroll
        for (int i = 0; i < 32; ++i) sv[c0 + i] = v[i];
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&s_empty[sb]);
      // causal limit of this row and the split end: only edge tiles mask
      // (uniform over the block: interior tiles are below every row's limit)
      const int64_t key0 = k_lo + (int64_t)t * kTcKeys;
      if (key0 + kTcKeys > min(p.start + 1, k_hi) || full_rows == 0) {
        const int64_t hi = min(lim + 1, k_hi) - key0;  // keys [0, hi) of the tile are visible
#pragma unroll
        for (int c = 0; c < kTcKeys; ++c) sv[c] = c < hi ? sv[c] : -INFINITY;
      }
      float mx0 = -INFINITY, mx1 = -INFINITY;
#pragma unroll
      for (int c = 0; c < kTcKeys; c += 2) {
        mx0 = fmaxf(mx0, sv[c]);
        mx1 = fmaxf(mx1, sv[c + 1]);
      }
      const float mx = fmaxf(mx0, mx1) * p.scale_log2;  // scale > 0 keeps the order
      // move the reference only when the row max outgrows it by kRescale
      const bool move = mx > m + kRescale || (m == -INFINITY && mx > -INFINITY);
      const float mn = move ? mx : m;
      const float f = (move && m != -INFINITY) ? fast_exp2(m - mn) : 1.f;
      const float nmu = mn == -INFINITY ? 0.f : -mn;
      float sum0 = 0.f, sum1 = 0.f;
      uint32_t pk[kTcKeys / 2];
#pragma unroll
      for (int c = 0; c < kTcKeys; c += 2) {
        const float p0 = fast_exp2(fmaf(sv[c], p.scale_log2, nmu));
        const float p1 = fast_exp2(fmaf(sv[c + 1], p.scale_log2, nmu));
        sum0 += p0;
        sum1 += p1;
        pk[c / 2] = pack_bf16(p0, p1);
      }
      l = l * f + (sum0 + sum1);
      m = mn;
      // rescale the warp's O rows in TMEM when one of them moved its
      // reference: O is quiescent once PV_{t-2} (this group's last) completed
      if (t >= 2 && __any_sync(0xffffffffu, f != 1.f)) {
        mbar_wait(&pv_done[(t - 2) % kPBufs], ((t - 2) / kPBufs) & 1);
        tc_fence_after();
#pragma unroll
        for (int c0 = 0; c0 < D; c0 += 32) {
          float v[32];
          tmem_ld32(o_addr(grp) + (uint32_t)c0, v);
          tmem_ld_wait();
          uint32_t w[32];
#pragma unroll
          for (int i = 0; i < 32; ++i) w[i] = __float_as_uint(v[i] * f);
          tmem_st32(o_addr(grp) + (uint32_t)c0, w);
        }
        tmem_st_wait();
      }
      // P buffer t % kPBufs is free once PV_{t - kPBufs} completed
      const int pb = t % kPBufs;
      mbar_wait(&pv_done[pb], ((t / kPBufs) & 1) ^ 1);
      uint8_t* pt = sm + S::kPOff + pb * S::kPBytes;
#pragma unroll
      for (int c = 0; c < kTcKeys / 8; ++c)
        *reinterpret_cast<uint4*>(pt + sw128_off(r, c, kTcRows * 128)) =
            make_uint4(pk[4 * c], pk[4 * c + 1], pk[4 * c + 2], pk[4 * c + 3]);
      fence_proxy_async();  // generic-proxy P writes -> the PV MMA
      tc_fence_before();    // TMEM stores -> the PV MMA
      __syncwarp();
      if (lane == 0) mbar_arrive(&p_full[pb]);
    }
    // this group's last PV
    const int n_mine = nt > grp ? (nt - grp + 1) / 2 : 0;
    if (n_mine > 0) {
      const int t_last = grp + 2 * (n_mine - 1);
      mbar_wait(&pv_done[t_last % kPBufs], (t_last / kPBufs) & 1);
    }
    float2* ml = reinterpret_cast<float2*>(sm + S::kMlOff);
    if (grp == 1) ml[r] = make_float2(m, l);
    tc_fence_before();
    asm volatile("bar.sync 1, 256;" ::: "memory");  // the two softmax groups
    if (grp == 0) {
      tc_fence_after();
      // merge the groups' (m, l, O) of this row; normalized partial + base-2 LSE
      const float2 o1 = ml[r];
      const float M = fmaxf(m, o1.x);
      const float Mz = M == -INFINITY ? 0.f : M;
      const float f0 = m == -INFINITY ? 0.f : fast_exp2(m - Mz);
      const float f1 = o1.x == -INFINITY ? 0.f : fast_exp2(o1.x - Mz);
      const float L = l * f0 + o1.y * f1;
      const float inv = L > 0.f ? 1.f / L : 0.f;
      const float c0f = f0 * inv, c1f = f1 * inv;
      const int64_t unit = ((int64_t)bh * p.rb + rblk) * p.n_split + split;
      float* po = p.part_o + (unit * kTcRows + r) * D;
#pragma unroll
      for (int c0 = 0; c0 < D; c0 += 32) {
        float v0[32], v1[32];
        if (nt > 0) {
          tmem_ld32(o_addr(0) + (uint32_t)c0, v0);
        } else {
#pragma unroll
          for (int i = 0; i < 32; ++i) v0[i] = 0.f;
        }
        if (nt > 1) {
          tmem_ld32(o_addr(1) + (uint32_t)c0, v1);
        } else {
#pragma unroll
          for (int i = 0; i < 32; ++i) v1[i] = 0.f;
        }
        tmem_ld_wait();
#pragma unroll
        for (int c = 0; c < 32; c += 4)
          *reinterpret_cast<float4*>(po + c0 + c) =
              make_float4(v0[c] * c0f + v1[c] * c1f, v0[c + 1] * c0f + v1[c + 1] * c1f,
                          v0[c + 2] * c0f + v1[c + 2] * c1f, v0[c + 3] * c0f + v1[c + 3] * c1f);
      }
      p.part_lse[unit * kTcRows + r] = L > 0.f ? log2f(L) + M : -INFINITY;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
  }
}

template <int D>
static cudaError_t launch_window_tc_t(const WinTcParams& p, cudaStream_t st) {
  static bool configured_[64] = {};
  bool& configured = device_flag(configured_);
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(window_tc_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         WinTcSmem<D>::kAlloc);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  window_tc_kernel<D><<<dim3(p.n_split, p.B * p.H, p.rb), kTcThreads, WinTcSmem<D>::kAlloc, st>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_window_merge(const float* part_o, const float* part_lse, int B, int H, int G,
                                int W, int rows, int rb, int n_split, int d, void* out,
                                cudaStream_t st);

// Splits per (b, g, row block): about one CTA per SM.
int window_tc_splits(int B, int H, int G, int W, int n_sms, int64_t keys) {
  const int rows = W * G, rb = (rows + kTcRows - 1) / kTcRows;
  const int ctas = B * H * rb;
  const int64_t tiles = (keys + kTcKeys - 1) / kTcKeys;
  return (int)std::max<int64_t>(1, std::min<int64_t>(std::max(1, n_sms / ctas), tiles));
}

cudaError_t launch_window_tc(const CUtensorMap& tmap_k, const CUtensorMap& tmap_v, const void* q,
                             int layer, int B, int H, int G, int d, int64_t start, int W,
                             float scale, float* workspace, int n_split, void* out,
                             cudaStream_t st) {
  WinTcParams p;
  p.tmap_k = tmap_k;
  p.tmap_v = tmap_v;
  p.q = static_cast<const __nv_bfloat16*>(q);
  p.B = B;
  p.H = H;
  p.G = G;
  p.W = W;
  p.rows = W * G;
  p.rb = (p.rows + kTcRows - 1) / kTcRows;
  p.layer = layer;
  p.start = start;
  p.keys = start + W;
  const int64_t tiles = (p.keys + kTcKeys - 1) / kTcKeys;
  int ns = (int)std::max<int64_t>(1, std::min<int64_t>(n_split, tiles));
  p.split_keys = ((tiles + ns - 1) / ns) * kTcKeys;
  p.n_split = (int)((p.keys + p.split_keys - 1) / p.split_keys);
  const int64_t units = (int64_t)B * H * p.rb * p.n_split;
  p.part_o = workspace;
  p.part_lse = workspace + units * kTcRows * 128;
  p.scale_log2 = scale * 1.4426950408889634f;
  cudaError_t e = d == 64 ? launch_window_tc_t<64>(p, st)
                  : d == 128 ? launch_window_tc_t<128>(p, st)
                             : cudaErrorInvalidValue;
  if (e != cudaSuccess) return e;
  return launch_window_merge(p.part_o, p.part_lse, B, H, G, W, p.rows, p.rb, p.n_split, d, out, st);
}

}  // namespace lyc
