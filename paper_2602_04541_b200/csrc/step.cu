// step.cu -- the persistent decode-step kernel: every layer of one decode step
// (decode_engine.hpp:109-151) in ONE launch, one CTA per SM.
//
// The first n_ctas CTAs of the 1-D grid are ATTENTION CTAs (256 threads):
//   warps 0-3 consumers  attention of this CTA's split of layer l
//                        (attn_core.cuh); layer l+1 starts only after layer
//                        l's outputs are final (device counter) -- the model's
//                        layer dependency;
//   warps 4-5 producers  stream the K/V tiles of layer l, l+1, ... continuously
//                        through the smem ring: the next layer's history rows
//                        are in flight while layer l is being merged.  Tiles
//                        whose index list comes from a selection wait for it;
//                        the tile holding the current token waits for the
//                        previous layer (its K/V row is produced after it);
//   warps 6-7 epilogue   the split-KV LSE merge of layer l (kernel_sim.hpp:
//                        205-225), spread over every attention CTA.
// The last n_sel_ctas CTAs form SELECTION TEAMS of 4 (Algorithm 2's pooling
// applied to the selection): after layer l's attention, a team computes for
// each of its retrieval heads args_top_k over the pooled-query keys
// (attention.hpp:108-123: the k largest, ties to the lower index, ascending)
// as an exact radix select.  The consumers already produced the first 11-bit
// histogram while scoring; each team CTA holds a quarter of the keys in
// shared memory; two more passes exchange 2048-bin histograms through global
// memory behind per-row team barriers; an ordered compaction writes the
// index cache.  Selection runs concurrently with the next layer's attention.
// Grid-wide coordination uses monotonic counters in global memory (each step
// adds the number of participating CTAs); the launch is cooperative, so every
// CTA is co-resident.
#include "attn_core.cuh"

namespace lyc {

constexpr int kEpiWarps = 2;
constexpr int kEpiThreads = kEpiWarps * 32;
constexpr int kStepThreads = (kConsumerWarps + kProducerWarps + kEpiWarps) * 32;
constexpr int kTeam = 4;  // CTAs per selection team

__device__ __forceinline__ uint32_t ld_acquire(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Grid-level wait on a monotonic counter; traps after ~20 s (a lost signal is
// a bug -- fail the launch instead of hanging the GPU).
__device__ __forceinline__ void spin_until(const uint32_t* ctr, uint32_t target) {
  if ((int)(ld_acquire(ctr) - target) >= 0) return;
  const long long t0 = clock64();
  while ((int)(ld_acquire(ctr) - target) < 0) {
    __nanosleep(128);
    if (clock64() - t0 > 40000000000LL) __trap();
  }
}

__device__ __forceinline__ void group_bar(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

// One thread of a warp group signals after the group's global writes.
__device__ __forceinline__ void signal(uint32_t* ctr) {
  __threadfence();
  atomicAdd(ctr, 1u);
}

// Debug timeline: %globaltimer (ns) of event ev of layer l on slot `who`.
enum { EV_CONS_BEGIN = 0, EV_CONS_END, EV_EPI_ATTN, EV_MERGE, EV_SEL0, EV_SEL1, EV_SEL2, EV_SELDONE };
__device__ __forceinline__ void stamp(const LycStepParams& p, int l, int ev, int who) {
  if (p.trace) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    p.trace[((size_t)l * 8 + ev) * p.n_ctas + who] = t;
  }
}

struct StepWaits {
  const uint32_t* ctr;
  uint32_t t_attn, t_sel;
  int layer;
  int pt;
  __device__ __forceinline__ void wait(const uint32_t* c, uint32_t target) const {
    if (pt == 0) spin_until(c, target);
    group_bar(3, kProducerThreads);
  }
  __device__ __forceinline__ void unit(const LycSlot& s) const {
    if (s.dep >= 0) wait(LYC_CTR(ctr, s.dep, CTR_SELDONE), t_sel);
  }
  __device__ __forceinline__ void last_tile() const {
    if (layer > 0) wait(LYC_CTR(ctr, layer - 1, CTR_MERGE), t_attn);
  }
};

__device__ __forceinline__ LycView layer_view(const LycStepParams& p, const LycLayerDesc& L,
                                              int l, int esz) {
  LycView v;
  v.k = p.k;
  v.v = p.v;
  v.q = static_cast<const uint8_t*>(p.q) + (int64_t)l * p.q_layer_stride * esz;
  v.out = static_cast<uint8_t*>(p.out) + (int64_t)l * p.q_layer_stride * esz;
  v.slots = L.slots;
  v.units = L.units;
  v.split_off = L.split_off;
  v.part_o = p.part_o;
  v.part_lse = p.part_lse;
  v.sel_keys = p.sel_keys + (int64_t)(l & 1) * p.max_sel * p.sel_stride;
  v.hist1 = p.sel_mode == SEL_TOKEN_KEYS ? p.hist + (int64_t)(l & 1) * p.max_sel * LYC_BINS
                                         : nullptr;
  v.exec_counts = nullptr;
  v.sel_stride = p.sel_stride;
  v.counts_stride = 0;
  v.n_splits = p.n_splits;
  v.seq_len = p.seq_len;
  v.block_size = p.block_size;
  v.group = p.group;
  v.sel_mode = p.sel_mode;
  v.scale = p.scale;
  v.scale_log2 = p.scale_log2;
  return v;
}

// ---------------------------------------------------------------- selection
// Warp-level search of a histogram (from the top bin down) for the bin that
// holds the krem-th largest candidate.  Returns (digit, count above it).
__device__ __forceinline__ void find_digit(const uint32_t* h, int nbins, uint32_t krem,
                                           uint32_t& digit, uint32_t& above, int lane) {
  const int per = nbins / 32;  // 64 (11-bit) or 32 (10-bit) bins per lane
  const int hi = nbins - 1 - lane * per;  // lane owns bins hi, hi-1, ..., hi-per+1
  uint32_t cnt[64];
  uint32_t sum = 0;
  const uint4* src = reinterpret_cast<const uint4*>(h + hi - per + 1);
#pragma unroll
  for (int q = 0; q < 16; ++q) {
    if (q * 4 >= per) break;
    const uint4 v = src[q];
    cnt[4 * q] = v.x;
    cnt[4 * q + 1] = v.y;
    cnt[4 * q + 2] = v.z;
    cnt[4 * q + 3] = v.w;
    sum += v.x + v.y + v.z + v.w;
  }
  uint32_t incl = sum;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const uint32_t n = __shfl_up_sync(0xffffffffu, incl, off);
    if (lane >= off) incl += n;
  }
  const uint32_t excl = incl - sum;
  uint32_t d = 0, a = 0;
  const bool mine = excl < krem && krem <= incl;
  if (mine) {
    uint32_t run = excl;
    for (int i = per - 1; i >= 0; --i) {  // cnt[i] is bin hi - per + 1 + i
      if (krem <= run + cnt[i]) {
        d = (uint32_t)(hi - per + 1 + i);
        a = run;
        break;
      }
      run += cnt[i];
    }
  }
  const unsigned who = __ballot_sync(0xffffffffu, mine);
  const int src_lane = __ffs(who) - 1;
  digit = __shfl_sync(0xffffffffu, d, src_lane);
  above = __shfl_sync(0xffffffffu, a, src_lane);
}

// Shared memory of a selection CTA (carved from the same dynamic allocation).
struct SelSmem {
  uint32_t hist[LYC_BINS];   // this CTA's pass histogram
  uint32_t ghist[LYC_BINS];  // team-summed histogram
  uint32_t warp_tot[32];
  uint32_t digit, above;
  uint64_t bar;              // completion of the slice's bulk copy
  uint32_t keys[1];          // this CTA's slice of the row's keys (capacity sel_cap), 16-B aligned
};

// Block-wide inclusive scan (256 threads).
__device__ __forceinline__ uint32_t block_scan(uint32_t v, uint32_t* warp_tot, uint32_t& total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  constexpr int kWarps = kStepThreads / 32;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const uint32_t n = __shfl_up_sync(0xffffffffu, v, off);
    if (lane >= off) v += n;
  }
  if (lane == 31) warp_tot[warp] = v;
  __syncthreads();
  uint32_t before = 0;
  total = 0;
#pragma unroll
  for (int w = 0; w < kWarps; ++w) {
    const uint32_t t = warp_tot[w];
    before += w < warp ? t : 0u;
    total += t;
  }
  __syncthreads();
  return v + before;
}

struct Team {
  uint32_t* bar;        // this row's barrier counters (kTeam arrivals each per step)
  uint32_t* xch;        // [2][kTeam][LYC_BINS] histogram exchange buffers of this team
  uint32_t* cnt;        // [kTeam][2] count exchange
  uint32_t target;      // epoch1 * kTeam
  int rank;

  __device__ __forceinline__ void barrier(int b) const {
    __syncthreads();
    if (threadIdx.x == 0) {
      signal(bar + b * 16);
      spin_until(bar + b * 16, target);
    }
    __syncthreads();
  }
  // Publish the local histogram, barrier b, sum the team's histograms into ghist.
  __device__ __forceinline__ void exchange(SelSmem& sh, int buf, int nbins, int b) const {
    uint32_t* mine = xch + ((size_t)buf * kTeam + rank) * LYC_BINS;
    __syncthreads();  // the local histogram's shared-memory atomics are complete
    for (int i = threadIdx.x; i < nbins; i += kStepThreads) mine[i] = sh.hist[i];
    barrier(b);
    // thread t sums bins [4t, 4t+4) (+1024) of every member: all loads in flight
    const int nv = nbins / 4;
    for (int v0 = 0; v0 < nv; v0 += kStepThreads) {
      const int v = v0 + threadIdx.x;
      uint4 part[kTeam];
#pragma unroll
      for (int c = 0; c < kTeam; ++c)
        part[c] = __ldcg(reinterpret_cast<const uint4*>(xch + ((size_t)buf * kTeam + c) * LYC_BINS) + v);
      uint4 s = make_uint4(0, 0, 0, 0);
#pragma unroll
      for (int c = 0; c < kTeam; ++c) {
        s.x += part[c].x;
        s.y += part[c].y;
        s.z += part[c].z;
        s.w += part[c].w;
      }
      reinterpret_cast<uint4*>(sh.ghist)[v] = s;
    }
    __syncthreads();
  }
};

__device__ __forceinline__ void digit_of(SelSmem& sh, const uint32_t* h, int nbins, uint32_t krem) {
  if (threadIdx.x < 32) {
    uint32_t d, a;
    find_digit(h, nbins, krem, d, a, threadIdx.x);
    if (threadIdx.x == 0) {
      sh.digit = d;
      sh.above = a;
    }
  }
  __syncthreads();
}

// One row: the k largest of n keys (ties to the lower index), ascending,
// into out[0..k).  h1 (token mode) holds the grid-wide first-pass histogram.
__device__ void select_row(SelSmem& sh, const Team& tm, const LycStepParams& p, uint32_t* keys_g,
                           uint32_t* h1, int32_t* out, uint32_t& bar_phase, int l, int sid) {
  const int tid = threadIdx.x;
  const int n = p.n_keys;
  const int slice = ((n + kTeam - 1) / kTeam + 3) & ~3;
  const int lo = min(n, tm.rank * slice);
  const int cnt = max(0, min(slice, n - lo));
  // this CTA's slice (lo and slice are multiples of 4): the 16-B aligned body
  // by TMA bulk copies on one mbarrier, the < 4-key tail by plain loads
  {
    const int nv = cnt >> 2;
    if (tid == 0 && nv > 0) {
      fence_proxy_async();  // prior generic reads of keys[] before the async-proxy overwrite
      mbar_arrive_expect_tx(&sh.bar, (uint32_t)nv * 16u);
      constexpr int kChunk = 2048;  // 16-B vectors per bulk copy (32 KB)
      for (int v = 0; v < nv; v += kChunk)
        bulk_g2s(sh.keys + 4 * v, keys_g + lo + 4 * v, (uint32_t)min(kChunk, nv - v) * 16u,
                 &sh.bar);
    }
    for (int i = (nv << 2) + tid; i < cnt; i += kStepThreads) sh.keys[i] = __ldcg(keys_g + lo + i);
    if (nv > 0) {
      mbar_wait(&sh.bar, bar_phase);
      bar_phase ^= 1u;
      if (tid == 0) stamp(p, l, EV_SEL0, sid);
    }
    __syncthreads();
    if (p.sel_mode == SEL_BLOCK_KEYS) {
      __syncthreads();
      for (int i = tid; i < cnt; i += kStepThreads) keys_g[lo + i] = 0u;
    }
  }
  uint32_t krem = (uint32_t)p.k_sel;
  // ---- pass 1 (bits 31..21)
  if (h1) {
    const uint4* h = reinterpret_cast<const uint4*>(h1);
    uint4* g = reinterpret_cast<uint4*>(sh.ghist);
    uint4 buf[2];
#pragma unroll
    for (int q = 0; q < 2; ++q) buf[q] = __ldcg(h + q * kStepThreads + tid);
#pragma unroll
    for (int q = 0; q < 2; ++q) g[q * kStepThreads + tid] = buf[q];
    __syncthreads();
  } else {
    for (int b = tid; b < LYC_BINS; b += kStepThreads) sh.hist[b] = 0u;
    __syncthreads();
    for (int i = tid; i < cnt; i += kStepThreads) atomicAdd(&sh.hist[sh.keys[i] >> 21], 1u);
    tm.exchange(sh, 1, LYC_BINS, 0);
  }
  digit_of(sh, sh.ghist, LYC_BINS, krem);
  const uint32_t d1 = sh.digit;
  krem -= sh.above;
  // ---- pass 2 (bits 20..10) among keys whose top bits are d1
  for (int b = tid; b < LYC_BINS; b += kStepThreads) sh.hist[b] = 0u;
  __syncthreads();
  for (int i = tid; i < cnt; i += kStepThreads) {
    const uint32_t key = sh.keys[i];
    if ((key >> 21) == d1) atomicAdd(&sh.hist[(key >> 10) & 0x7ffu], 1u);
  }
  tm.exchange(sh, 0, LYC_BINS, 1);  // also orders every member's read of h1 before its reset
  if (tid == 0) stamp(p, l, EV_SEL1, sid);
  digit_of(sh, sh.ghist, LYC_BINS, krem);
  const uint32_t d2 = sh.digit;
  krem -= sh.above;
  if (h1 && tm.rank == 0)  // reset the fused histogram for its next use
    for (int b = tid; b < LYC_BINS; b += kStepThreads) h1[b] = 0u;
  // ---- pass 3 (bits 9..0)
  const uint32_t pre22 = (d1 << 11) | d2;
  for (int b = tid; b < 1024; b += kStepThreads) sh.hist[b] = 0u;
  __syncthreads();
  for (int i = tid; i < cnt; i += kStepThreads) {
    const uint32_t key = sh.keys[i];
    if ((key >> 10) == pre22) atomicAdd(&sh.hist[key & 0x3ffu], 1u);
  }
  tm.exchange(sh, 1, 1024, 2);
  if (tid == 0) stamp(p, l, EV_SEL2, sid);
  digit_of(sh, sh.ghist, 1024, krem);
  const uint32_t T = (pre22 << 10) | sh.digit;
  krem -= sh.above;  // ties of T to take, team-wide
  // ---- emission: team scan of (count > T, count == T) over ranks
  uint32_t gt = 0, eq = 0;
  for (int i = tid; i < cnt; i += kStepThreads) {
    const uint32_t key = sh.keys[i];
    gt += key > T;
    eq += key == T;
  }
  uint32_t tgt, teq;
  block_scan(gt, sh.warp_tot, tgt);
  block_scan(eq, sh.warp_tot, teq);
  if (tid == 0) {
    tm.cnt[tm.rank * 2] = tgt;
    tm.cnt[tm.rank * 2 + 1] = teq;
  }
  tm.barrier(3);
  uint32_t base = 0, eqb = 0;
  for (int c = 0; c < tm.rank; ++c) {
    const uint32_t cg_ = __ldcg(tm.cnt + 2 * c), ce = __ldcg(tm.cnt + 2 * c + 1);
    base += cg_ + (krem > eqb ? min(ce, krem - eqb) : 0u);
    eqb += ce;
  }
  const uint32_t take_eq = krem > eqb ? min(teq, krem - eqb) : 0u;
  uint32_t run_gt = 0, run_eq = 0;
  constexpr int kPer = 8;
  for (int b0 = 0; b0 < cnt; b0 += kStepThreads * kPer) {
    const int i0 = b0 + tid * kPer;
    uint32_t kv[kPer];
    uint32_t g = 0, e = 0;
#pragma unroll
    for (int q = 0; q < kPer; ++q) {
      const bool ok = i0 + q < cnt;
      kv[q] = ok ? sh.keys[i0 + q] : 0u;
      g += ok && kv[q] > T;
      e += ok && kv[q] == T;
    }
    uint32_t tot;
    const uint32_t mine = (e << 16) | g;
    const uint32_t incl = block_scan(mine, sh.warp_tot, tot);
    uint32_t gb = run_gt + ((incl - mine) & 0xffffu);
    uint32_t eb = run_eq + ((incl - mine) >> 16);
#pragma unroll
    for (int q = 0; q < kPer; ++q) {
      if (i0 + q >= cnt) break;
      const bool is_gt = kv[q] > T, is_eq = kv[q] == T;
      if (is_gt || (is_eq && eb < take_eq)) out[base + gb + min(eb, take_eq)] = lo + i0 + q;
      gb += is_gt;
      eb += is_eq;
    }
    run_gt += tot & 0xffffu;
    run_eq += tot >> 16;
  }
  __syncthreads();
}

// ---------------------------------------------------------------- kernel
template <typename T, int D>
__global__ void __launch_bounds__(kStepThreads, 1) hybrid_step_kernel(const __grid_constant__ LycStepParams p) {
  using C = AttnCfg<T, D>;
  extern __shared__ uint8_t smem_raw[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int cta = blockIdx.x;
  const int n_total = p.n_ctas + p.n_sel_ctas;
  uint32_t* ctrl = LYC_CTR(p.ctr, p.n_layers, 0);  // completed steps; exits at + stride
  __shared__ uint32_t s_epoch;
  if (threadIdx.x == 0) s_epoch = ld_acquire(ctrl);
  __syncthreads();
  const uint32_t epoch1 = s_epoch + 1u;
  const uint32_t t_attn = epoch1 * (uint32_t)p.n_ctas;
  const uint32_t t_sel = epoch1 * (uint32_t)p.n_sel_ctas;
  constexpr int esz = (int)sizeof(T);

  if (cta >= p.n_ctas) {
    // ======================== selection team ========================
    SelSmem& sh = *reinterpret_cast<SelSmem*>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
    const int sid = cta - p.n_ctas;
    const int team = sid / kTeam;
    const int n_teams = p.n_sel_ctas / kTeam;
    Team tm;
    tm.rank = sid % kTeam;
    tm.target = epoch1 * (uint32_t)kTeam;
    tm.xch = p.sel_xch + (size_t)team * (2 * kTeam * LYC_BINS + 64);
    tm.cnt = tm.xch + 2 * kTeam * LYC_BINS;
    if (threadIdx.x == 0) {
      mbar_init(&sh.bar, 1);
      fence_mbar_init();
    }
    __syncthreads();
    uint32_t bar_phase = 0;
    for (int l = 0; l < p.n_layers; ++l) {
      const LycLayerDesc L = p.layers[l];
      if (L.n_sel == 0 || p.sel_mode == SEL_NONE) continue;
      if (threadIdx.x == 0) {
        spin_until(LYC_CTR(p.ctr, l, CTR_ATTN), t_attn);
        __threadfence();
      }
      __syncthreads();
      for (int r = team; r < L.n_sel; r += n_teams) {
        uint32_t* kg = p.sel_keys + ((int64_t)(l & 1) * p.max_sel + r) * p.sel_stride;
        uint32_t* h1 = p.sel_mode == SEL_TOKEN_KEYS
                           ? p.hist + ((int64_t)(l & 1) * p.max_sel + r) * LYC_BINS
                           : nullptr;
        const int row = __ldg(L.sel_rows + r);
        tm.bar = p.sel_bar + ((size_t)l * p.max_sel + r) * 64;
        select_row(sh, tm, p, kg, h1, p.idx + (int64_t)row * p.idx_stride, bar_phase, l, sid);
        if (threadIdx.x == 0 && tm.rank == 0 && p.idx_count) p.idx_count[row] = p.k_sel;
      }
      __syncthreads();
      if (threadIdx.x == 0) {
        stamp(p, l, EV_SELDONE, sid);
        signal(LYC_CTR(p.ctr, l, CTR_SELDONE));
      }
    }
  } else {
    // ======================== attention CTA ========================
    const AttnSmem<T, D> sm = AttnSmem<T, D>::carve(smem_raw);
    if (threadIdx.x == 0) {
      for (int s = 0; s < C::kStages; ++s) {
        mbar_init(&sm.full[s], kProducerThreads);
        mbar_init(&sm.empty[s], kConsumerWarps);
      }
      fence_mbar_init();
    }
    for (int b = threadIdx.x; b < LYC_BINS; b += kStepThreads) sm.hist[b] = 0u;
    __syncthreads();
    const int cell = cta;  // = b * n_splits + split
    if (warp < kConsumerWarps) {
      const int tid = threadIdx.x;
      int stage = 0;
      uint32_t phase = 0;
      for (int l = 0; l < p.n_layers; ++l) {
        if (l > 0) {
          if (tid == 0) {
            spin_until(LYC_CTR(p.ctr, l - 1, CTR_MERGE), t_attn);
            // key / histogram buffers of this parity are free once layer l-2's
            // selection (if any) finished
            if (l >= 2 && p.layers[l - 2].n_sel > 0 && p.sel_mode != SEL_NONE)
              spin_until(LYC_CTR(p.ctr, l - 2, CTR_SELDONE), t_sel);
            __threadfence();
          }
          consumer_bar();
        }
        if (tid == 0) stamp(p, l, EV_CONS_BEGIN, cta);
        const LycLayerDesc L = p.layers[l];
        const LycView v = layer_view(p, L, l, esz);
        consume_units<T, D>(v, sm, L.split_off[cell], L.split_off[cell + 1], warp, lane, stage,
                            phase);
        consumer_bar();
        if (tid == 0) {
          stamp(p, l, EV_CONS_END, cta);
          signal(LYC_CTR(p.ctr, l, CTR_ATTN));
        }
      }
    } else if (warp < kConsumerWarps + kProducerWarps) {
      const int pt = threadIdx.x - kConsumerWarps * 32;
      if (pt == 0) {
        prefetch_tensormap(&p.tmap_k);
        prefetch_tensormap(&p.tmap_v);
      }
      int stage = 0;
      uint32_t phase = 0;
      for (int l = 0; l < p.n_layers; ++l) {
        const LycLayerDesc L = p.layers[l];
        const LycView v = layer_view(p, L, l, esz);
        StepWaits waits{p.ctr, t_attn, t_sel, l, pt};
        produce_units<T, D>(v, &p.tmap_k, &p.tmap_v, sm.ring, sm.full, sm.empty,
                            L.split_off[cell], L.split_off[cell + 1], pt, stage, phase, waits);
      }
    } else {
      const int et = threadIdx.x - (kConsumerWarps + kProducerWarps) * 32;
      const int ew = et >> 5;
      const int chunks = (D + 31) / 32;
      for (int l = 0; l < p.n_layers; ++l) {
        const LycLayerDesc L = p.layers[l];
        if (et == 0) {
          spin_until(LYC_CTR(p.ctr, l, CTR_ATTN), t_attn);
          __threadfence();
          stamp(p, l, EV_EPI_ATTN, cta);
        }
        group_bar(2, kEpiThreads);
        // split-KV merge, spread over all attention CTAs' epilogue warps
        const int total = L.n_merges * chunks;
        uint8_t* outl = static_cast<uint8_t*>(p.out) + (int64_t)l * p.q_layer_stride * esz;
        for (int t = cta * kEpiWarps + ew; t < total; t += p.n_ctas * kEpiWarps) {
          const LycMergeTask tk = L.merges[t / chunks];
          const LycSlot s = L.slots[tk.slot];
          merge_task<T>(p.part_o, p.part_lse, s, tk.j, t % chunks, p.group, D, outl, lane);
        }
        group_bar(2, kEpiThreads);
        if (et == 0) {
          stamp(p, l, EV_MERGE, cta);
          signal(LYC_CTR(p.ctr, l, CTR_MERGE));
        }
      }
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const uint32_t done = atomicAdd(ctrl + LYC_CTR_STRIDE, 1u);
    if (done == epoch1 * (uint32_t)n_total - 1u) atomicAdd(ctrl, 1u);  // last CTA out
  }
}

template <typename T, int D>
int step_sel_capacity() {  // keys a selection CTA keeps in shared memory
  using C = AttnCfg<T, D>;
  return (int)((C::kSmem - 1024 - (int)sizeof(SelSmem)) / 4);
}

template <typename T, int D>
static cudaError_t launch_step_t(const LycStepParams& p, cudaStream_t st) {
  using C = AttnCfg<T, D>;
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(hybrid_step_kernel<T, D>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmem);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(p.n_ctas + p.n_sel_ctas);
  cfg.blockDim = dim3(kStepThreads);
  cfg.dynamicSmemBytes = C::kSmem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, hybrid_step_kernel<T, D>, p);
}

cudaError_t launch_step(const LycStepParams& p, int dtype, int d, cudaStream_t st) {
  if (dtype == 1) {
    switch (d) {
      case 64: return launch_step_t<__nv_bfloat16, 64>(p, st);
      case 128: return launch_step_t<__nv_bfloat16, 128>(p, st);
    }
  } else {
    switch (d) {
      case 16: return launch_step_t<float, 16>(p, st);
      case 32: return launch_step_t<float, 32>(p, st);
      case 64: return launch_step_t<float, 64>(p, st);
      case 128: return launch_step_t<float, 128>(p, st);
    }
  }
  return cudaErrorInvalidValue;
}

int step_select_capacity(int dtype, int d) {
  if (dtype == 1) return d == 64 ? step_sel_capacity<__nv_bfloat16, 64>()
                                 : step_sel_capacity<__nv_bfloat16, 128>();
  switch (d) {
    case 16: return step_sel_capacity<float, 16>();
    case 32: return step_sel_capacity<float, 32>();
    case 64: return step_sel_capacity<float, 64>();
    default: return step_sel_capacity<float, 128>();
  }
}

// Global scratch of the selection teams (words): per team, 2 x kTeam
// histogram exchange buffers plus the count exchange; per (layer, row), the
// team-barrier counters (4 used, 64 words apart).
size_t step_sel_xch_words(int n_sel_ctas) {
  return (size_t)(n_sel_ctas / kTeam) * (2 * kTeam * LYC_BINS + 64);
}
size_t step_sel_bar_words(int n_layers, int max_sel) { return (size_t)n_layers * max_sel * 64; }

bool step_supported(int dtype, int d) {
  return dtype == 1 ? (d == 64 || d == 128) : (d == 16 || d == 32 || d == 64 || d == 128);
}

}  // namespace lyc
