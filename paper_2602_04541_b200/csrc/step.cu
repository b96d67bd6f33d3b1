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
// The last n_sel_ctas CTAs are SELECTION CTAs (Algorithm 2's pooling applied
// to the selection): after layer l's attention, each computes for its share of
// the layer's retrieval heads args_top_k over the pooled-query keys
// (attention.hpp:108-123: the k largest, ties to the lower index, ascending)
// as an exact radix select that needs no inter-CTA synchronisation: the
// consumers already produced the first 11-bit histogram while scoring, one
// TMA-pipelined pass over the keys builds an "above the boundary bin" bitmap
// plus the boundary-bin candidates, and the rest runs in shared memory.
// Selection runs concurrently with the next layer's attention.
// Grid-wide coordination uses monotonic counters in global memory (each step
// adds the number of participating CTAs); the launch is cooperative, so every
// CTA is co-resident.
#include "attn_core.cuh"

namespace lyc {

constexpr int kEpiWarps = 2;
constexpr int kEpiThreads = kEpiWarps * 32;
constexpr int kStepThreads = (kConsumerWarps + kProducerWarps + kEpiWarps) * 32;

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

// ---- selection CTA: one row at a time, entirely on-chip after one key stream
constexpr int kChunkKeys = 8192;  // keys per streamed chunk (32 KB, one TMA bulk copy)
constexpr int kRing = 3;          // chunks in flight

struct SelHdr {
  uint32_t hist[LYC_BINS];
  uint32_t warp_tot[32];
  uint64_t bars[kRing];
  uint32_t digit, above;
};

// Dynamic layout: ring | header | bitmap[nwords] | cand keys[cap] | cand idx[cap]
struct SelSmem {
  uint32_t (*ring)[kChunkKeys];
  SelHdr* h;
  uint32_t* bitmap;  // bit i: key i selected
  uint32_t* ckey;    // boundary-bin candidates, index order
  uint32_t* cidx;
  int cap;

  __device__ static SelSmem carve(uint8_t* raw, int total_bytes, int nwords) {
    SelSmem s;
    uint8_t* base = reinterpret_cast<uint8_t*>(
        (reinterpret_cast<uintptr_t>(raw) + 1023) & ~static_cast<uintptr_t>(1023));
    const int avail = total_bytes - (int)(base - raw);
    s.ring = reinterpret_cast<uint32_t(*)[kChunkKeys]>(base);
    s.h = reinterpret_cast<SelHdr*>(base + kRing * kChunkKeys * 4);
    s.bitmap = reinterpret_cast<uint32_t*>(s.h + 1);
    uint32_t* c = s.bitmap + ((nwords + 3) & ~3);
    const int used = (int)(reinterpret_cast<uint8_t*>(c) - base);
    s.cap = max(0, (avail - used) / 8);
    s.ckey = c;
    s.cidx = c + s.cap;
    return s;
  }
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

__device__ __forceinline__ void digit_of(SelHdr* h, int nbins, uint32_t krem) {
  if (threadIdx.x < 32) {
    uint32_t d, a;
    find_digit(h->hist, nbins, krem, d, a, threadIdx.x);
    if (threadIdx.x == 0) {
      h->digit = d;
      h->above = a;
    }
  }
  __syncthreads();
}

// Streams keys[0, n) through the TMA ring; f(base, chunk, cnt) runs on every
// thread for each chunk in order and must not read the chunk after returning.
// `phases` holds the per-slot mbarrier parities (persistent across calls).
template <typename F>
__device__ __forceinline__ void stream_keys(const SelSmem& sh, const uint32_t* keys, int n,
                                            uint32_t& phases, F&& f) {
  const int nck = (n + kChunkKeys - 1) / kChunkKeys;
  auto issue = [&](int c) {
    const int cnt = min(kChunkKeys, n - c * kChunkKeys);
    const uint32_t bytes = (uint32_t)((cnt + 3) & ~3) * 4u;  // key rows are padded to 4
    uint64_t* bar = &sh.h->bars[c % kRing];
    mbar_arrive_expect_tx(bar, bytes);
    bulk_g2s(sh.ring[c % kRing], keys + (size_t)c * kChunkKeys, bytes, bar);
  };
  __syncthreads();
  if (threadIdx.x == 0) {
    fence_proxy_async();  // earlier generic reads of the ring precede its async overwrite
    for (int c = 0; c < min(kRing, nck); ++c) issue(c);
  }
  for (int c = 0; c < nck; ++c) {
    const int slot = c % kRing;
    mbar_wait(&sh.h->bars[slot], (phases >> slot) & 1u);
    phases ^= 1u << slot;
    f(c * kChunkKeys, sh.ring[slot], min(kChunkKeys, n - c * kChunkKeys));
    __syncthreads();
    if (threadIdx.x == 0 && c + kRing < nck) {
      fence_proxy_async();
      issue(c + kRing);
    }
  }
}

// One row: the k largest of n keys (ties to the lower index), ascending,
// into out[0..k).  h1 (token mode) is the grid-wide first-pass histogram
// (bits 31..21) built by the attention consumers; otherwise it is computed
// here.  The radix descends until the boundary bin fits the candidate store
// (normally right after pass 1); ONE streaming pass then classifies every key:
// above the boundary prefix -> bitmap bit, inside it -> candidate (key, index)
// in index order.  The remaining radix passes run on the candidates in shared
// memory, the selected candidates join the bitmap, and a popcount scan of the
// bitmap emits the indices in ascending order.
__device__ void select_row(uint8_t* smem_raw, int smem_bytes, const LycStepParams& p,
                           uint32_t* keys_g, uint32_t* h1, int32_t* out, uint32_t& phases, int l,
                           int sid) {
  const int tid = threadIdx.x;
  const int n = p.n_keys;
  const int nwords = (n + 31) / 32;
  const SelSmem sh = SelSmem::carve(smem_raw, smem_bytes, nwords);
  SelHdr* H = sh.h;
  uint32_t krem = (uint32_t)p.k_sel;
  // ---- pass 1 (bits 31..21)
  if (h1) {
    const uint4* src = reinterpret_cast<const uint4*>(h1);
    uint4 buf[2];
#pragma unroll
    for (int q = 0; q < 2; ++q) buf[q] = __ldcg(src + q * kStepThreads + tid);
#pragma unroll
    for (int q = 0; q < 2; ++q) reinterpret_cast<uint4*>(H->hist)[q * kStepThreads + tid] = buf[q];
    __syncthreads();
  } else {
    for (int b = tid; b < LYC_BINS; b += kStepThreads) H->hist[b] = 0u;
    stream_keys(sh, keys_g, n, phases, [&](int, const uint32_t* ck, int cnt) {
      for (int i = tid; i < cnt; i += kStepThreads) atomicAdd(&H->hist[ck[i] >> 21], 1u);
    });
  }
  digit_of(H, LYC_BINS, krem);
  uint32_t P = H->digit;  // boundary prefix
  int shift = 21;         // key >> shift is the prefix
  krem -= H->above;
  uint32_t n_eq = H->hist[P];
  if (n_eq > (uint32_t)sh.cap) {  // rare: boundary bin too big -> descend on the stream
    for (int b = tid; b < LYC_BINS; b += kStepThreads) H->hist[b] = 0u;
    stream_keys(sh, keys_g, n, phases, [&](int, const uint32_t* ck, int cnt) {
      for (int i = tid; i < cnt; i += kStepThreads)
        if ((ck[i] >> 21) == P) atomicAdd(&H->hist[(ck[i] >> 10) & 0x7ffu], 1u);
    });
    digit_of(H, LYC_BINS, krem);
    P = (P << 11) | H->digit;
    shift = 10;
    krem -= H->above;
    n_eq = H->hist[H->digit];
    if (n_eq > (uint32_t)sh.cap) {
      for (int b = tid; b < 1024; b += kStepThreads) H->hist[b] = 0u;
      stream_keys(sh, keys_g, n, phases, [&](int, const uint32_t* ck, int cnt) {
        for (int i = tid; i < cnt; i += kStepThreads)
          if ((ck[i] >> 10) == P) atomicAdd(&H->hist[ck[i] & 0x3ffu], 1u);
      });
      digit_of(H, 1024, krem);
      P = (P << 10) | H->digit;  // the k-th key T itself; krem of its ties are taken
      shift = 0;
      krem -= H->above;
    }
  }
  if (tid == 0) stamp(p, l, EV_SEL0, sid);
  // ---- classify every key against the prefix P
  uint32_t run = 0;  // candidates (or ties of T) so far, index order
  stream_keys(sh, keys_g, n, phases, [&](int base, const uint32_t* ck, int cnt) {
    // thread t owns 32 consecutive keys = one bitmap word, read as 8 rotated
    // 16-B vectors (conflict-free)
    uint32_t word = 0, eqm = 0;
    const int k0 = tid * 32;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int qq = (q + tid) & 7;
      const uint4 v = reinterpret_cast<const uint4*>(ck + k0)[qq];
      const uint32_t kv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int j = qq * 4 + e;
        const bool ok = k0 + j < cnt;
        const uint32_t pre = shift ? kv[e] >> shift : kv[e];
        word |= (ok && pre > P) ? (1u << j) : 0u;
        eqm |= (ok && pre == P) ? (1u << j) : 0u;
      }
    }
    uint32_t tot;
    const uint32_t c = __popc(eqm);
    const uint32_t incl = block_scan(c, H->warp_tot, tot);
    uint32_t pos = run + incl - c;
    if (shift == 0) {  // ties of T: take the first krem by index
      while (eqm) {
        const int j = __ffs(eqm) - 1;
        eqm &= eqm - 1;
        if (pos < krem) word |= 1u << j;
        ++pos;
      }
    } else {
      while (eqm) {
        const int j = __ffs(eqm) - 1;
        eqm &= eqm - 1;
        sh.ckey[pos] = ck[k0 + j];
        sh.cidx[pos] = (uint32_t)(base + k0 + j);
        ++pos;
      }
    }
    if (k0 < cnt) sh.bitmap[base / 32 + tid] = word;
    run += tot;
  });
  // ---- finish the radix on the candidates
  if (shift > 0) {
    const int nc = (int)run;
    if (shift == 21) {
      for (int b = tid; b < LYC_BINS; b += kStepThreads) H->hist[b] = 0u;
      __syncthreads();
      for (int i = tid; i < nc; i += kStepThreads)
        atomicAdd(&H->hist[(sh.ckey[i] >> 10) & 0x7ffu], 1u);
      __syncthreads();
      digit_of(H, LYC_BINS, krem);
      P = (P << 11) | H->digit;
      krem -= H->above;
    }
    for (int b = tid; b < 1024; b += kStepThreads) H->hist[b] = 0u;
    __syncthreads();
    for (int i = tid; i < nc; i += kStepThreads)
      if ((sh.ckey[i] >> 10) == P) atomicAdd(&H->hist[sh.ckey[i] & 0x3ffu], 1u);
    __syncthreads();
    digit_of(H, 1024, krem);
    const uint32_t T = (P << 10) | H->digit;
    krem -= H->above;  // ties of T to take (lowest indices first)
    // selected candidates join the bitmap: key > T, or the first krem ties
    uint32_t tie_run = 0;
    for (int b0 = 0; b0 < nc; b0 += kStepThreads) {
      const int i = b0 + tid;
      const uint32_t key = i < nc ? sh.ckey[i] : 0u;
      const bool is_eq = i < nc && key == T;
      uint32_t tot;
      const uint32_t incl = block_scan(is_eq ? 1u : 0u, H->warp_tot, tot);
      const uint32_t rank = tie_run + incl - (is_eq ? 1u : 0u);
      if (i < nc && (key > T || (is_eq && rank < krem)))
        atomicOr(&sh.bitmap[sh.cidx[i] >> 5], 1u << (sh.cidx[i] & 31));
      tie_run += tot;
    }
    __syncthreads();
  }
  if (tid == 0) stamp(p, l, EV_SEL1, sid);
  // ---- emit the set bits in ascending order
  const int per = (nwords + kStepThreads - 1) / kStepThreads;
  const int w0 = min(nwords, tid * per), w1 = min(nwords, w0 + per);
  uint32_t cnt = 0;
  for (int w = w0; w < w1; ++w) cnt += __popc(sh.bitmap[w]);
  uint32_t tot;
  uint32_t pos = block_scan(cnt, H->warp_tot, tot) - cnt;
  for (int w = w0; w < w1; ++w) {
    uint32_t m = sh.bitmap[w];
    while (m) {
      const int j = __ffs(m) - 1;
      m &= m - 1;
      out[pos++] = w * 32 + j;
    }
  }
  if (h1)  // reset the fused histogram for its next use
    for (int b = tid; b < LYC_BINS; b += kStepThreads) h1[b] = 0u;
  if (p.sel_mode == SEL_BLOCK_KEYS)  // block keys are max-folded: reset the row
    for (int i = tid; i < n; i += kStepThreads) keys_g[i] = 0u;
  if (tid == 0) stamp(p, l, EV_SEL2, sid);
  __syncthreads();
}

// ---------------------------------------------------------------- kernel
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

    // ======================== selection CTA ========================
    const int sid = cta - p.n_ctas;
    if (threadIdx.x == 0) {
      SelHdr* H = SelSmem::carve(smem_raw, C::kSmem, 0).h;
      for (int s = 0; s < kRing; ++s) mbar_init(&H->bars[s], 1);
      fence_mbar_init();
    }
    __syncthreads();
    uint32_t phases = 0;
    for (int l = 0; l < p.n_layers; ++l) {
      const LycLayerDesc L = p.layers[l];
      if (L.n_sel == 0 || p.sel_mode == SEL_NONE) continue;
      if (threadIdx.x == 0) {
        spin_until(LYC_CTR(p.ctr, l, CTR_ATTN), t_attn);
        __threadfence();
      }
      __syncthreads();
      for (int r = sid; r < L.n_sel; r += p.n_sel_ctas) {
        uint32_t* kg = p.sel_keys + ((int64_t)(l & 1) * p.max_sel + r) * p.sel_stride;
        uint32_t* h1 = p.sel_mode == SEL_TOKEN_KEYS
                           ? p.hist + ((int64_t)(l & 1) * p.max_sel + r) * LYC_BINS
                           : nullptr;
        const int row = __ldg(L.sel_rows + r);
        select_row(smem_raw, C::kSmem, p, kg, h1, p.idx + (int64_t)row * p.idx_stride, phases, l,
                   sid);
        if (threadIdx.x == 0 && p.idx_count) p.idx_count[row] = p.k_sel;
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

int step_select_capacity(int, int) { return 1 << 16; }  // keys per row / 4 (bitmap bound)

bool step_supported(int dtype, int d) {
  return dtype == 1 ? (d == 64 || d == 128) : (d == 16 || d == 32 || d == 64 || d == 128);
}

}  // namespace lyc
