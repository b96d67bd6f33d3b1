// step.cu -- the persistent decode-step kernel: every layer of one decode step
// (decode_engine.hpp:109-151) in ONE launch, one CTA per SM, all SMs.
//
// Warp roles of every CTA (256 threads):
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
//   warps 6-7 epilogue   after the whole grid finished layer l's attention:
//                        (a) the split-KV LSE merge (kernel_sim.hpp:205-225);
//                        (b) the selection of the layer's retrieval heads --
//                            args_top_k over the pooled-query keys
//                            (attention.hpp:108-123: the k largest, ties to the
//                            lower index, ascending) as an exact radix select.
//                        Both are pooled over ALL CTAs (Algorithm 2's workload
//                        pooling applied to the epilogue): merge tasks and
//                        32 KB key "items" are dealt round-robin.
// Selection per retrieval head: the consumers built the first 11-bit
// histogram while scoring; every item classifies its 8192 keys against the
// boundary bin (bitmap word per 32 keys, boundary-bin candidates in index
// order); the CTA that completes a head's LAST item finishes the radix on the
// candidates, adds the selected ones to the bitmap and emits the set bits in
// ascending order into the index cache.  No grid barrier: a per-head counter.
// Grid-wide coordination uses monotonic counters in global memory (each step
// adds a fixed amount); the launch is cooperative, so every CTA is co-resident.
#include <climits>

#include "attn_core.cuh"
#include "plan.cuh"

namespace lyc {

constexpr int kEpiWarps = 2;
constexpr int kEpiThreads = kEpiWarps * 32;
constexpr int kStepThreads = (kConsumerWarps + kProducerWarps + kEpiWarps) * 32;
constexpr int kItemKeys = 8192;  // keys per selection item (32 KB, one TMA bulk copy)
constexpr int kSpec = 2048;     // candidates a resolver loads before it knows the count
constexpr int kRankMax = 256;    // boundary-bin candidates resolved by direct ranking (per warp list)

__device__ __forceinline__ uint32_t ld_acquire(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ uint32_t ld_relaxed(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Grid-level wait on a monotonic counter (acquire loads).  Traps after ~20 s
// (a lost signal is a bug -- fail the launch instead of hanging the GPU).
__device__ __forceinline__ void spin_until(const uint32_t* ctr, uint32_t target) {
  // acquire polls: no trailing fence (a fence would also wait for this
  // thread's own outstanding stores and copies)
  if ((int)(ld_acquire(ctr) - target) < 0) {
    const long long t0 = clock64();
    while ((int)(ld_acquire(ctr) - target) < 0) {
      __nanosleep(64);
      if (clock64() - t0 > 40000000000LL) __trap();
    }
  }
}

// spin_until on two counters at once (c2 may be null): both loads in flight
// per poll, so an already-reached second target costs no extra round trip.
__device__ __forceinline__ void spin_until2(const uint32_t* c1, uint32_t t1, const uint32_t* c2,
                                            uint32_t t2) {
  auto done = [&]() {
    const uint32_t a = ld_acquire(c1);
    const uint32_t b = c2 ? ld_acquire(c2) : t2;
    return (int)(a - t1) >= 0 && (int)(b - t2) >= 0;
  };
  if (!done()) {
    const long long t0 = clock64();
    while (!done()) {
      __nanosleep(64);
      if (clock64() - t0 > 40000000000LL) __trap();
    }
  }
}

__device__ __forceinline__ void group_bar(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

// One thread of a warp group signals after the group's global writes (the
// group synchronised with bar.sync first; the release is cumulative).
__device__ __forceinline__ void signal(uint32_t* ctr) {
  asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(ctr) : "memory");
}

__device__ __forceinline__ uint32_t atom_add_acq_rel(uint32_t* ctr, uint32_t v) {
  uint32_t old;
  asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], %2;" : "=r"(old) : "l"(ctr), "r"(v) : "memory");
  return old;
}

__device__ __forceinline__ void epi_bar() { group_bar(2, kEpiThreads); }

// Debug timeline: %globaltimer (ns) of event ev of layer l on CTA `cta`.
enum { EV_CONS_BEGIN = 0, EV_CONS_END, EV_EPI_ATTN, EV_MERGE, EV_SEL0, EV_ENTRY, EV_SEL2, EV_PDL,
       EV_C_PREFIX, EV_C_KEYS, EV_C_DONE, EV_F_PREFIX, EV_F_SCAN, EV_F_EMIT, EV_X0, EV_X1 };
__device__ __forceinline__ void stamp(const LycStepParams& p, int l, int ev, int cta) {
  if (p.trace) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    p.trace[((size_t)l * LYC_TRACE_EVENTS + ev) * p.n_ctas + cta] = t;
  }
}

// Per-launch runtime state of every thread: this launch's counter set (the
// launch parity) and the step's lengths from the plan header.
struct StepRt {
  uint32_t* ctr;     // LYC_CTR counters of this launch's set
  uint32_t* rowctr;  // [n_layers][max_sel][16] of this launch's set
  int n_keys;        // selection keys per row (max over the batch)
  int k_sel;         // ids kept per row
  int l_begin;       // first layer of this launch: earlier layers completed in earlier launches
  int ragged;        // batch items differ in (blocks, budget): per-row selection sizes
  const int32_t* seqs;  // [B] live lengths of the step (shared memory)
  const int32_t* nsel;  // [B] selection keys of each item's rows (shared memory)
  const int32_t* ksel;  // [B] ids kept per row of each item (shared memory)
};

// Every selection item signals CTR_SELDONE once after emitting its share of
// the index-cache row.
__device__ __forceinline__ uint32_t seldone_per_step(const LycStepParams& p, const StepRt& rt,
                                                     int l) {
  return (uint32_t)p.layers[l].n_sel * (uint32_t)((rt.n_keys + kItemKeys - 1) / kItemKeys);
}

struct StepWaits {
  const LycStepParams* p;
  const StepRt* rt;
  int layer;
  int pt;
  __device__ __forceinline__ void wait(const uint32_t* c, uint32_t target) const {
    if (pt == 0) spin_until(c, target);
    group_bar(3, kProducerThreads);
  }
  __device__ __forceinline__ void unit(const LycSlot& s) const {
    // every retrieval head of layer dep finished its selection (a layer of an
    // earlier launch has: stream order -- except a selection deferred into
    // this launch, counted in this launch's set)
    if (s.dep >= rt->l_begin - p->sel_defer_in)
      wait(LYC_CTR(rt->ctr, s.dep, CTR_SELDONE), seldone_per_step(*p, *rt, s.dep));
  }
  const uint32_t* clayer;  // shared: 1 + the layer this CTA's consumers started
  __device__ __forceinline__ bool needed() const { return layer > rt->l_begin; }
  // OR over the producer threads (barrier with reduction)
  __device__ __forceinline__ bool any(bool v) const {
    uint32_t r;
    asm volatile(
        "{\n .reg .pred p, q;\n setp.ne.u32 p, %1, 0;\n bar.red.or.pred q, 3, %2, p;\n"
        " selp.u32 %0, 1, 0, q;\n}"
        : "=r"(r)
        : "r"((uint32_t)v), "n"(kProducerThreads)
        : "memory");
    return r != 0;
  }
  // the previous layer's outputs are final once this CTA's consumers have
  // started this layer (they waited for it); otherwise wait for it here
  __device__ __forceinline__ void last_tile() const {
    if (layer == rt->l_begin) return;
    if (pt == 0 && (int)(ld_acquire_cta_shared(clayer) - (uint32_t)(layer + 1)) < 0)
      spin_until(LYC_CTR(rt->ctr, layer - 1, CTR_MERGE), (uint32_t)p->n_ctas);
    group_bar(3, kProducerThreads);
  }
};

__device__ __forceinline__ LycView layer_view(const LycStepParams& p, const StepRt& rt,
                                              const LycLayerDesc& L, int l, int esz) {
  LycView v;
  v.k = p.k;
  v.v = p.v;
  v.q = static_cast<const uint8_t*>(p.q) + (int64_t)(l - p.l_begin) * p.q_layer_stride * esz;
  v.out = static_cast<uint8_t*>(p.out) + (int64_t)(l - p.l_begin) * p.q_layer_stride * esz;
  v.slots = L.slots;
  v.units = L.units;
  v.unit_slots = L.unit_slots;
  v.split_off = L.split_off;
  v.part_o = p.part_o;
  v.part_lse = p.part_lse;
  v.sel_keys = p.sel_keys + (int64_t)(l & 1) * p.max_sel * p.sel_stride;
  v.hist1 = p.sel_mode == SEL_TOKEN_KEYS ? p.hist + (int64_t)(l & 1) * p.max_sel * LYC_H1_STRIDE
                                         : nullptr;
  v.exec_counts = nullptr;
  v.out_f32 = nullptr;  // single-unit slots write `out` directly
  v.out_lse = nullptr;
  v.sel_stride = p.sel_stride;
  v.counts_stride = 0;
  v.n_splits = p.n_splits;
  v.seq_len = rt.n_keys;
  v.block_size = p.block_size;
  v.group = p.group;
  v.sel_mode = p.sel_mode;
  v.scale = p.scale;
  v.scale_log2 = p.scale_log2;
  v.stages = p.stages;
  v.early_exit = 0;
  v.trace_l = p.trace ? p.trace + (size_t)l * LYC_TRACE_EVENTS * p.n_ctas : nullptr;
  v.slot_ctr = rt.rowctr + (size_t)l * p.max_sel * 16;
  v.trace_ctas = p.n_ctas;
  v.seq_of = rt.seqs;  // the live lengths (the plan's slot records may be up to 63 tokens old)
  return v;
}

// ---------------------------------------------------------------- selection
// Warp-level search of a histogram (from the top bin down) for the bin that
// holds the krem-th largest candidate (krem >= 1).  Two levels, no local
// arrays: every lane sums a contiguous run of nbins/32 bins, a warp scan picks
// the lane holding the target, then the warp splits that lane's run again.
// Returns (digit, count strictly above it).  nbins: power of two, 2..4096.
__device__ __forceinline__ uint32_t ld_bin(const uint32_t* a, bool global) {
  return global ? __ldcg(a) : *a;
}
__device__ __forceinline__ uint32_t warp_incl_scan(uint32_t v, int lane) {
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const uint32_t n = __shfl_up_sync(0xffffffffu, v, off);
    if (lane >= off) v += n;
  }
  return v;
}
__device__ __forceinline__ void find_digit(const uint32_t* h, int nbins, uint32_t krem,
                                           uint32_t& digit, uint32_t& above, int lane,
                                           bool global) {
  // bins per lane (1..128); histograms smaller than 32 bins: one bin per lane
  // for the first nbins lanes, none for the rest
  const int per = nbins >= 32 ? nbins / 32 : 1;
  const int hi = nbins - 1 - lane * per;  // lane owns bins (hi - per, hi], highest first
  uint32_t sum = 0;
  if (hi < 0) {
    // no bins
  } else if (per >= 4) {
    const uint4* src = reinterpret_cast<const uint4*>(h + hi - per + 1);
#pragma unroll 8
    for (int q = 0; q < per / 4; ++q) {
      const uint4 v = global ? __ldcg(src + q) : src[q];
      sum += v.x + v.y + v.z + v.w;
    }
  } else {
    for (int i = 0; i < per; ++i) sum += ld_bin(h + hi - i, global);
  }
  uint32_t incl = warp_incl_scan(sum, lane);
  unsigned who = __ballot_sync(0xffffffffu, incl - sum < krem && krem <= incl);
  const int L = __ffs(who) - 1;
  uint32_t run = __shfl_sync(0xffffffffu, incl - sum, L);  // keys above lane L's run
  const int top = nbins - 1 - L * per;                      // lane L's highest bin
  // second level: lane i takes `sub` consecutive bins of lane L's run, highest first
  const int sub = per >= 32 ? per / 32 : 1;
  const bool act = lane * sub < per;
  uint32_t s2 = 0;
  if (act) {
#pragma unroll 4
    for (int i = 0; i < sub; ++i) s2 += ld_bin(h + top - lane * sub - i, global);
  }
  incl = warp_incl_scan(s2, lane) + run;
  who = __ballot_sync(0xffffffffu, act && incl - s2 < krem && krem <= incl);
  const int M = __ffs(who) - 1;
  uint32_t d = 0, a = 0;
  if (lane == M) {
    uint32_t r = incl - s2;
    for (int i = 0; i < sub; ++i) {
      const int bin = top - lane * sub - i;
      const uint32_t c = ld_bin(h + bin, global);
      if (krem <= r + c) {
        d = (uint32_t)bin;
        a = r;
        break;
      }
      r += c;
    }
  }
  digit = __shfl_sync(0xffffffffu, d, M);
  above = __shfl_sync(0xffffffffu, a, M);
}

// Selection bitmaps (global and on chip) are stored in 64-word chunks at a
// 68-word stride: the finisher's thread t reads chunk t as 16-B vectors, and
// the 4-word skew makes those reads bank-conflict-free.
__host__ __device__ __forceinline__ int bm_pad(int w) { return w + (w >> 6) * 4; }
__host__ __device__ __forceinline__ int bm_padded_words(int nwords) { return (nwords + 63) / 64 * 68; }

// Epilogue scratch (inside AttnSmem::extra).
constexpr int kEpiBufWords = 8192;  // 32 KB: one classify item; finisher candidates
struct EpiSmem {
  // classify: one item's keys [kItemKeys]; finish: bitmap [nwords] followed by
  // the candidates' keys and indices
  uint32_t buf[kEpiBufWords];
  uint32_t hist[LYC_BINS];
  uint32_t scan[64];
  uint32_t seg[72];          // resolve: start of each item's block in the row's candidate array
  uint32_t cnt[72];          // resolve: candidates of each item
  uint32_t defc[72];         // resolve: definite keys of each item
  uint64_t bar;
  uint32_t digit, above, last, pad;
};

// 64-thread inclusive scan (2 warps).
__device__ __forceinline__ uint32_t epi_scan(uint32_t v, uint32_t* scan, int et, uint32_t& total) {
  const int lane = et & 31, w = et >> 5;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const uint32_t n = __shfl_up_sync(0xffffffffu, v, off);
    if (lane >= off) v += n;
  }
  if (lane == 31) scan[w] = v;
  epi_bar();
  const uint32_t before = w ? scan[0] : 0u;
  total = scan[0] + scan[1];
  epi_bar();
  return v + before;
}

// Digit of a histogram by warp 0 of the epilogue; result broadcast via smem.
__device__ __forceinline__ void epi_digit(EpiSmem& es, const uint32_t* h, bool global, int nbins,
                                          uint32_t krem, int et) {
  if (et < 32) {
    uint32_t d, a;
    find_digit(h, nbins, krem, d, a, et, global);
    if (et == 0) {
      es.digit = d;
      es.above = a;
    }
  }
  epi_bar();
}

struct SelRow {
  uint32_t k;         // ids kept (variable-length batch: this row's budget)
  int n;              // keys of this row's sequence (<= nk; the rest are masked)
  int nk;             // keys of the longest row (the padded row length)
  uint32_t* keys;     // keys of the row [n]
  uint32_t* h1;       // fused first-pass (12-bit) histogram (token mode) or nullptr
  uint32_t* bitmap;   // [n_words]
  uint32_t* ckey;     // [n] candidate keys, item q's segment at q*kItemKeys
  uint32_t* cidx;     // [n] candidate indices
  uint32_t* csub;     // [64 items][256] u16: each item's bucket starts of its boundary-bin
                      // candidates by their next 8 bits (descending: start[b] = #above b)
  uint32_t* ccnt;     // [n_items] candidates per item; +64: definite keys per item;
                      // +128: output offset of each item
  uint32_t* ctr;      // per-row words: [0] items classified, [8] items holding their copies
};

__device__ __forceinline__ SelRow sel_row(const LycStepParams& p, const StepRt& rt, int l, int r) {
  const int64_t pr = (int64_t)(l & 1) * p.max_sel + r;
  SelRow s;
  const LycLayerDesc& L = p.layers[l];
  if (rt.ragged) {  // this row's item: its own length and budget (policy.hpp:57-72)
    const int b = __ldcg(L.sel_rows + r) / p.plan.H;
    s.k = (uint32_t)rt.ksel[b];
    s.n = rt.nsel[b];
  } else {
    s.k = (uint32_t)rt.k_sel;
    s.n = rt.n_keys;
  }
  s.nk = rt.n_keys;
  s.keys = p.sel_keys + pr * p.sel_stride;
  s.h1 = p.sel_mode == SEL_TOKEN_KEYS ? p.hist + pr * LYC_H1_STRIDE : nullptr;
  s.bitmap = p.sel_bitmap + pr * p.bitmap_stride;
  s.ckey = p.sel_cand + pr * 2 * p.sel_stride;
  s.cidx = s.ckey + p.sel_stride;
  s.csub = p.sel_csub + pr * (64 * 128);
  s.ccnt = p.sel_ccnt + pr * 256;
  s.ctr = rt.rowctr + ((int64_t)l * p.max_sel + r) * 16;
  return s;
}

// The boundary prefix of a row.  Token mode: the 12-bit bin from the first
// radix pass the attention consumers fused into scoring (h1); block mode (one
// item): the 11-bit bin of the item's own histogram (es.hist).
// Sets es.digit = prefix, es.above = keys strictly above it, es.last = shift.
__device__ __forceinline__ void row_prefix(const LycStepParams& p, const SelRow& R, EpiSmem& es,
                                           int et) {
  if (R.h1) {
    // two coalesced L2 reads by warp 0: the 64 coarse bins, then the 64 fine
    // bins of the chosen coarse bin (lane i holds bins 2(31-i), 2(31-i)+1)
    if (et < 32) {
      uint32_t k = R.k, base = 0, above = 0;
      const uint32_t* h = R.h1 + LYC_H1_BINS;
#pragma unroll
      for (int level = 0; level < 2; ++level) {
        uint2 v = make_uint2(0u, 0u);
#pragma unroll
        for (int c = 0; c < LYC_H1_COPIES; ++c) {
          const uint2 w = __ldcg(reinterpret_cast<const uint2*>(h + c * LYC_H1_ROW) + (31 - et));
          v.x += w.x;
          v.y += w.y;
        }
        const uint32_t sum = v.x + v.y;
        const uint32_t incl = warp_incl_scan(sum, et);
        const unsigned who = __ballot_sync(0xffffffffu, incl - sum < k && k <= incl);
        const int L = who ? __ffs(who) - 1 : 31;
        const uint32_t ex = __shfl_sync(0xffffffffu, incl - sum, L);
        const uint32_t hi = __shfl_sync(0xffffffffu, v.y, L);
        const bool upper = k <= ex + hi;
        const uint32_t bin = 2u * (31u - (uint32_t)L) + (upper ? 1u : 0u);
        const uint32_t a = upper ? ex : ex + hi;
        above += a;
        k -= a;
        base = level == 0 ? bin * 64u : base + bin;
        h = R.h1 + bin * 64u;
      }
      if (et == 0) {
        es.digit = base;
        es.above = above;
      }
    }
    epi_bar();
  } else
    epi_digit(es, es.hist, false, LYC_BINS, R.k, et);
  if (et == 0) es.last = R.h1 ? 32u - LYC_H1_BITS : 21u;
  epi_bar();
}

// Classify item q of one row: keys above the row's boundary prefix set bitmap
// bits, keys inside it become candidates (index order) and are histogrammed by
// their next 8 bits into the row's 256-bin sub-histogram (global, atomics).
__device__ void classify_item(const LycStepParams& p, const SelRow& R, int q, EpiSmem& es,
                              uint32_t& bar_phase, int et, int l, int cta) {
  const int n = R.nk;
  const int lo = q * kItemKeys;
  const int cnt = min(kItemKeys, n - lo);
  // keys of this row's own sequence (a shorter item of a variable-length
  // batch: the rest of the padded row is masked out, never selected)
  const int vcnt = min(cnt, R.n - lo);
  if (et == 0) {
    fence_proxy_async();         // earlier generic use of es.buf -> TMA write
    fence_proxy_async_global();  // consumers' key stores (acquired) -> TMA read
    const uint32_t bytes = (uint32_t)((cnt + 3) & ~3) * 4u;  // key rows are padded to 4
    mbar_arrive_expect_tx(&es.bar, bytes);
    bulk_g2s(es.buf, R.keys + lo, bytes, &es.bar);
  }
  if (!R.h1) {  // block mode: the row is a single item -- histogram it here
    mbar_wait(&es.bar, bar_phase);
    for (int b = et; b < LYC_BINS; b += kEpiThreads) es.hist[b] = 0u;
    epi_bar();
    for (int i = et; i < vcnt; i += kEpiThreads) atomicAdd(&es.hist[es.buf[i] >> 21], 1u);
    epi_bar();
  }
  row_prefix(p, R, es, et);
  if (et == 0) stamp(p, l, EV_C_PREFIX, cta);
  const uint32_t P = es.digit;
  const uint32_t above = es.above;
  const int shift = (int)es.last;
  epi_bar();
  for (int b = et; b < 256; b += kEpiThreads) es.hist[b] = 0u;  // item sub-histogram
  mbar_wait(&es.bar, bar_phase);
  bar_phase ^= 1u;
  if (et == 0) stamp(p, l, EV_C_KEYS, cta);
  // thread et owns 128 consecutive keys = 4 bitmap words, read as rotated 16-B
  // vectors (conflict-free).  Threshold compares against the prefix's key
  // range [T0, T1m]; bits are set at static positions (predicated ORs) and the
  // words rotated once at the end; the tail item's words are masked after.
  const uint32_t T0 = P << shift;
  const uint32_t T1m = T0 | ((1u << shift) - 1u);  // largest key with prefix P
  uint32_t words[4], eqm[4];
  const int k0 = et * 128;
  const int rot = 4 * (et & 7);
#pragma unroll
  for (int w = 0; w < 4; ++w) {
    uint32_t ta = 0u, tg = 0u;
#pragma unroll
    for (int qv = 0; qv < 8; ++qv) {
      const uint4 v = reinterpret_cast<const uint4*>(es.buf + k0 + w * 32)[(qv + et) & 7];
      const uint32_t kv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        if (kv[e] > T1m) ta |= 1u << (qv * 4 + e);
        if (kv[e] >= T0) tg |= 1u << (qv * 4 + e);
      }
    }
    ta = __funnelshift_l(ta, ta, rot);
    tg = __funnelshift_l(tg, tg, rot);
    const int valid = vcnt - (k0 + w * 32);
    const uint32_t vm = valid >= 32 ? 0xffffffffu : valid <= 0 ? 0u : (1u << valid) - 1u;
    words[w] = ta & vm;
    eqm[w] = tg & ~ta & vm;
  }
#pragma unroll
  for (int w = 0; w < 4; ++w)
    if (k0 + w * 32 < cnt) R.bitmap[bm_pad((lo + k0) / 32 + w)] = words[w];
  const uint32_t c = __popc(eqm[0]) + __popc(eqm[1]) + __popc(eqm[2]) + __popc(eqm[3]);
  uint32_t total;
  epi_scan(c, es.scan, et, total);
  // this item's block of the row's contiguous candidate array (per-step
  // counter, reset by the row's last resolver); the reservation's round trip
  // overlaps the sub-histogram
  if (et == 0) es.pad = atomicAdd(R.ctr + 4, total);
#pragma unroll
  for (int w = 0; w < 4; ++w) {
    uint32_t m = eqm[w];
    while (m) {
      const int j = __ffs(m) - 1;
      m &= m - 1;
      atomicAdd(&es.hist[(es.buf[k0 + w * 32 + j] >> (shift - 8)) & 255u], 1u);
    }
  }
  uint32_t ndef = __popc(words[0]) + __popc(words[1]) + __popc(words[2]) + __popc(words[3]);
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) ndef += __shfl_xor_sync(0xffffffffu, ndef, off);
  if ((et & 31) == 0) es.scan[32 + (et >> 5)] = ndef;
  epi_bar();
  // descending bucket starts (thread et: bins 255-4et .. 252-4et): published
  // for the resolvers (u16) and used as scatter cursors here
  {
    uint32_t h4[4], hs = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      h4[j] = es.hist[255 - 4 * et - j];
      hs += h4[j];
    }
    uint32_t tot2;
    uint32_t run = epi_scan(hs, es.scan, et, tot2) - hs;
    uint32_t st[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      st[j] = run;
      es.hist[256 + 255 - 4 * et - j] = run;
      run += h4[j];
    }
    // u16 bins 252-4et .. 255-4et (ascending in memory)
    reinterpret_cast<uint2*>(R.csub + q * 128)[63 - et] =
        make_uint2(st[3] | (st[2] << 16), st[1] | (st[0] << 16));
  }
  epi_bar();
  // candidates scattered by bucket (order inside a bucket is free: survivors
  // are ranked by (key, index))
  {
    const uint32_t base = es.pad;
#pragma unroll
    for (int w = 0; w < 4; ++w) {
      uint32_t m = eqm[w];
      while (m) {
        const int j = __ffs(m) - 1;
        m &= m - 1;
        const int i = k0 + w * 32 + j;
        const uint32_t key = es.buf[i];
        const uint32_t pos = base + atomicAdd(&es.hist[256 + ((key >> (shift - 8)) & 255u)], 1u);
        R.ckey[pos] = key;
        R.cidx[pos] = (uint32_t)(lo + i);
      }
    }
  }
  if (et == 0) {
    R.ccnt[q] = total;
    R.ccnt[64 + q] = es.scan[32] + es.scan[33];
    R.ccnt[128 + q] = es.pad;
    // the row's boundary prefix (identical from every item) for the resolvers
    R.ccnt[192] = P;
    R.ccnt[193] = above;
    R.ccnt[194] = (uint32_t)shift;
  }
  epi_bar();
  if (et == 0) {
    stamp(p, l, EV_C_DONE, cta);
    signal(R.ctr);  // release this item's writes
  }
}

// Resolve the row and emit item q's share of the index-cache row.  Every item
// of the row resolves it redundantly (no hand-off to a finisher and back):
// once all items are classified, bulk-load the boundary-bin candidates (about
// k/4 keys) and the row's 256-bin sub-histogram; the sub-histogram narrows the
// boundary by 8 more bits, one scan takes everything above it and compacts the
// few survivors, which are ranked exactly (greater key, or equal key and lower
// index: attention.hpp:115-119).  Per-item selected counts give this item's
// output offset; its own words (definite keys + its selected candidates) are
// emitted with branch-free predicated stores.
__device__ void resolve_emit_item(const LycStepParams& p, const StepRt& rt, const SelRow& R, int q,
                                  int row, int32_t* out, EpiSmem& es, uint32_t& bar_phase, int et,
                                  int l, int cta) {
  constexpr uint32_t epoch1 = 1u;  // counters count from zero in every launch
  const int n = R.nk;
  const int items = (n + kItemKeys - 1) / kItemKeys;
  const int lo = q * kItemKeys;
  const int cnt = min(kItemKeys, n - lo);
  const int lane = et & 31, ew = et >> 5;
  if (et == 0) spin_until(R.ctr, epoch1 * (uint32_t)items);  // every item classified
  epi_bar();
  if (et == 0) stamp(p, l, EV_F_SCAN, cta);
  // one round: the row prefix and counts, this item's definite words, every
  // item's bucket starts and (speculatively) the first kSpec candidates
  const int bsw = items * 128;  // words of the items' u16 bucket starts
  const int cap = ((kEpiBufWords - bsw) / 2) & ~3;  // candidates that fit on chip
  const int spec = max(0, min(min(kSpec, cap), (int)(p.sel_stride & ~(int64_t)3)));
  const uint16_t* bs16 = reinterpret_cast<const uint16_t*>(es.buf);  // [items][256]
  uint32_t* skey = es.buf + bsw;
  uint32_t* sidx = skey + cap;
  if (et == 0) {
    fence_proxy_async();         // earlier generic use of es.buf / es.hist -> TMA write
    fence_proxy_async_global();  // other CTAs' generic writes -> this TMA read
    mbar_arrive_expect_tx(&es.bar, 4u * (uint32_t)bsw + 8u * (uint32_t)spec);
    bulk_g2s(es.buf, R.csub, 4u * (uint32_t)bsw, &es.bar);
    if (spec > 0) {
      bulk_g2s(skey, R.ckey, 4u * (uint32_t)spec, &es.bar);
      bulk_g2s(sidx, R.cidx, 4u * (uint32_t)spec, &es.bar);
    }
  }
  if (R.h1) {  // every item has read the row's first-pass histograms: item q re-zeroes its share
    constexpr int kVec = LYC_H1_STRIDE / 4;
    const int per = (kVec + items - 1) / items;
    const int b1 = min(kVec, (q + 1) * per);
    for (int b = q * per + et; b < b1; b += kEpiThreads)
      reinterpret_cast<uint4*>(R.h1)[b] = make_uint4(0u, 0u, 0u, 0u);
  }
  uint32_t P = __ldcg(R.ccnt + 192);
  int shift = (int)__ldcg(R.ccnt + 194);
  uint32_t krem = R.k - __ldcg(R.ccnt + 193);
  const int ns = (int)__ldcg(R.ctr + 4);  // candidates of the row
  const uint32_t d_mine = et < items ? __ldcg(R.ccnt + 64 + et) : 0u;
  if (et < items) {
    es.cnt[et] = __ldcg(R.ccnt + et);
    es.seg[et] = __ldcg(R.ccnt + 128 + et);
  }
  const int w0 = lo / 32 + et * 4;  // this thread's 4 words (128 keys)
  uint4 wv4 = make_uint4(0u, 0u, 0u, 0u);
  if (et * 128 < cnt) wv4 = __ldcg(reinterpret_cast<const uint4*>(R.bitmap + bm_pad(w0)));
  uint32_t* ws = es.hist + 1792;  // [256] this item's words on chip
  reinterpret_cast<uint4*>(ws)[et] = wv4;
  if (et < items) es.defc[et] = d_mine;
  if (et == 0) {
    es.scan[44] = 0u;
    es.scan[45] = 0u;
    es.scan[46] = 0u;
  }
  const bool on_chip = ns <= cap;
  mbar_wait(&es.bar, bar_phase);
  bar_phase ^= 1u;
  if (on_chip && ns > spec) {  // the rest of the candidates
    epi_bar();
    if (et == 0) {
      const uint32_t rest = (uint32_t)(((ns + 3) & ~3) - spec) * 4u;
      mbar_arrive_expect_tx(&es.bar, 2u * rest);
      bulk_g2s(skey + spec, R.ckey + spec, rest, &es.bar);
      bulk_g2s(sidx + spec, R.cidx + spec, rest, &es.bar);
    }
    mbar_wait(&es.bar, bar_phase);
    bar_phase ^= 1u;
  }
  if (et == 0) {
    stamp(p, l, EV_SEL2, cta);
  }
  auto get = [&](int i, uint32_t& key, uint32_t& idx) -> bool {
    if (i >= ns) return false;
    if (on_chip) {
      key = skey[i];
      idx = sidx[i];
    } else {
      key = __ldcg(R.ckey + i);
      idx = __ldcg(R.cidx + i);
    }
    return true;
  };
  // a selected candidate: counted when it precedes this item (output offset),
  // OR-ed into this item's words when inside it
  auto take = [&](uint32_t idx) {
    if ((int)idx < lo) atomicAdd(&es.scan[46], 1u);
    else if ((int)idx < lo + cnt) atomicOr(ws + ((idx - (uint32_t)lo) >> 5), 1u << (idx & 31));
  };
  // the row's sub-histogram from the items' bucket starts:
  // count[b] = start[b - 1] - start[b] (start[-1] = the item's candidates)
  epi_bar();
  {  // this item's output offset from the definite keys of the items before it
     // (known now; the taken candidates are added at emission)
    const uint32_t n_q = et < items ? es.defc[et] : 0u;
    uint32_t tot;
    const uint32_t end_q = epi_scan(n_q, es.scan, et, tot);
    if (et == q) es.pad = end_q - n_q;
  }
  {  // thread et: bins 4et .. 4et+3 (one 8-B load + the bin below per item)
    uint32_t h0 = 0, h1 = 0, h2 = 0, h3 = 0;
    for (int i = 0; i < items; ++i) {
      const uint2 v = reinterpret_cast<const uint2*>(bs16 + i * 256)[et];
      const uint32_t prev = et ? (uint32_t)bs16[i * 256 + 4 * et - 1] : es.cnt[i];
      const uint32_t s0 = v.x & 0xffffu, s1 = v.x >> 16, s2 = v.y & 0xffffu, s3 = v.y >> 16;
      h0 += prev - s0;
      h1 += s0 - s1;
      h2 += s1 - s2;
      h3 += s2 - s3;
    }
    reinterpret_cast<uint4*>(es.hist)[et] = make_uint4(h0, h1, h2, h3);
  }
  epi_bar();
  epi_digit(es, es.hist, false, 256, krem, et);
  // every thread's reads of the shared row state (count, sub-histogram; bulk
  // copies complete) are performed (barrier above): count this item's copy
  // taken.  The last item resets the state for the next use at the end
  // (before this CTA's CTR_SELDONE signal); the atomic's round trip overlaps
  // the scan.
  uint32_t copies = 0;
  if (et == 0) copies = atomicAdd(R.ctr + 8, 1u);
  P = (P << 8) | es.digit;
  shift -= 8;
  krem -= es.above;
  uint32_t live = es.hist[es.digit];
  if (et == 0) stamp(p, l, EV_F_PREFIX, cta);
  if (live <= (uint32_t)kRankMax) {
    // ---- fast path: the buckets above the digit are taken whole; the digit's
    // bucket of every item (the survivors, contiguous) is ranked exactly
    const uint32_t d = es.digit;
    uint32_t n_i = 0, off_i = 0;
    if (et < items) {
      const uint32_t above_i = bs16[et * 256 + d];
      n_i = (d ? (uint32_t)bs16[et * 256 + d - 1] : es.cnt[et]) - above_i;
      off_i = es.seg[et] + above_i;
      if (et < q) atomicAdd(&es.scan[44], above_i);  // taken above the bucket, before this item
    }
    uint32_t m;
    const uint32_t base_i = epi_scan(n_i, es.scan, et, m) - n_i;
    uint32_t* lk = es.hist + 256;  // survivors: keys [kRankMax] | ids [kRankMax]
    for (uint32_t j = 0; j < n_i; ++j) {
      uint32_t key = 0, idx = 0;
      get((int)(off_i + j), key, idx);
      lk[base_i + j] = key;
      lk[kRankMax + base_i + j] = idx;
    }
    {  // this item's candidates above the bucket
      const uint32_t a_q = bs16[q * 256 + d];
      const int s_q = (int)es.seg[q];
      for (int j = et; j < (int)a_q; j += kEpiThreads) {
        uint32_t key = 0, idx = 0;
        get(s_q + j, key, idx);
        atomicOr(ws + ((idx - (uint32_t)lo) >> 5), 1u << (idx & 31));
      }
    }
    epi_bar();
    if (et == 0) stamp(p, l, EV_X1, cta);
    for (uint32_t e = et; e < m; e += kEpiThreads) {
      const uint32_t ki = lk[e], xi = lk[kRankMax + e];
      uint32_t rank = 0;
      for (uint32_t j = 0; j < m; ++j) {
        const uint32_t kj = lk[j];
        rank += (kj > ki || (kj == ki && lk[kRankMax + j] < xi)) ? 1u : 0u;
      }
      if (rank < krem) take(xi);
    }
  } else {
  // (rare) keep narrowing while too many candidates share the prefix
  while (live > (uint32_t)kRankMax && shift > 0) {
    const int wbits = shift > 8 ? 8 : shift;
    shift -= wbits;
    const uint32_t mask = (1u << wbits) - 1u;
    epi_bar();
    for (int b = et; b < (1 << wbits); b += kEpiThreads) es.hist[b] = 0u;
    epi_bar();
    for (int i = et; i < ns; i += kEpiThreads) {
      uint32_t key, idx;
      if (get(i, key, idx) && (key >> (shift + wbits)) == P)
        atomicAdd(&es.hist[(key >> shift) & mask], 1u);
    }
    epi_bar();
    epi_digit(es, es.hist, false, 1 << wbits, krem, et);
    P = (P << wbits) | es.digit;
    krem -= es.above;
    live = es.hist[es.digit];
  }
  epi_bar();
  // one scan: take everything above the prefix (count the ones before this
  // item, OR in its own), compact the survivors (per-warp ballot lists at
  // es.hist + 256 + w * 3 * kRankMax: keys | ids); four loads in flight
  {
    uint32_t* lk = es.hist + 256 + ew * 3 * kRankMax;
    uint32_t mw = 0, before = 0;
    constexpr int U = 4;
    for (int i0 = ew * 32; i0 < ns; i0 += kEpiThreads * U) {
      uint32_t key[U], idx[U];
      bool ok[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        key[u] = 0u;
        idx[u] = 0u;
        ok[u] = get(i0 + u * kEpiThreads + lane, key[u], idx[u]);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint32_t pre = key[u] >> shift;  // shift < 32
        const bool tk = ok[u] && pre > P;
        before += (uint32_t)__popc(__ballot_sync(0xffffffffu, tk && (int)idx[u] < lo));
        if (tk && (int)idx[u] >= lo && (int)idx[u] < lo + cnt)
          atomicOr(ws + ((idx[u] - (uint32_t)lo) >> 5), 1u << (idx[u] & 31));
        const bool surv = ok[u] && pre == P;
        const unsigned bal = __ballot_sync(0xffffffffu, surv);
        const uint32_t at = mw + (uint32_t)__popc(bal & ((1u << lane) - 1u));
        if (surv && at < (uint32_t)kRankMax) {
          lk[at] = key[u];
          lk[kRankMax + at] = idx[u];
        }
        mw += (uint32_t)__popc(bal);
      }
    }
    if (lane == 0) {
      es.scan[40 + ew] = mw;
      es.scan[44 + ew] = before;
    }
  }
  epi_bar();
  const uint32_t m0 = es.scan[40], m1 = es.scan[41];
  if (et == 0) stamp(p, l, EV_X1, cta);
  if (m0 <= (uint32_t)kRankMax && m1 <= (uint32_t)kRankMax) {
    const uint32_t m = m0 + m1;
    const uint32_t* L0 = es.hist + 256;
    const uint32_t* L1 = es.hist + 256 + 3 * kRankMax;
    for (uint32_t e = et; e < m; e += kEpiThreads) {
      const uint32_t* Le = e < m0 ? L0 + e : L1 + (e - m0);
      const uint32_t ki = Le[0], xi = Le[kRankMax];
      uint32_t rank = 0;
      for (uint32_t j = 0; j < m0; ++j) {
        const uint32_t kj = L0[j];
        rank += (kj > ki || (kj == ki && L0[kRankMax + j] < xi)) ? 1u : 0u;
      }
      for (uint32_t j = 0; j < m1; ++j) {
        const uint32_t kj = L1[j];
        rank += (kj > ki || (kj == ki && L1[kRankMax + j] < xi)) ? 1u : 0u;
      }
      if (rank < krem) take(xi);
    }
  } else {
    // (only with shift == 0) more than kRankMax copies of one key: the krem
    // LOWEST indices among them (attention.hpp:117-118), by a radix select on
    // kp = 0xFFFFF - idx (largest kp = smallest index; idx < 2^20)
    uint32_t Pi = 0, kr = krem;
    int sh = 20;
    while (sh > 0) {
      const int wbits = sh > 8 ? 8 : sh;
      sh -= wbits;
      const uint32_t mask = (1u << wbits) - 1u;
      epi_bar();
      for (int b = et; b < (1 << wbits); b += kEpiThreads) es.hist[b] = 0u;
      epi_bar();
      for (int i = et; i < ns; i += kEpiThreads) {
        uint32_t key, idx;
        if (get(i, key, idx) && key == P) {
          const uint32_t kp = 0xFFFFFu - idx;
          if ((kp >> (sh + wbits)) == Pi) atomicAdd(&es.hist[(kp >> sh) & mask], 1u);
        }
      }
      epi_bar();
      epi_digit(es, es.hist, false, 1 << wbits, kr, et);
      Pi = (Pi << wbits) | es.digit;
      kr -= es.above;
    }
    for (int i = et; i < ns; i += kEpiThreads) {
      uint32_t key, idx;
      if (get(i, key, idx) && key == P && 0xFFFFFu - idx >= Pi) take(idx);
    }
  }
  }  // narrowing / scan path
  if (et == 0) es.last = copies == epoch1 * (uint32_t)items - 1u;
  epi_bar();
  if (et == 0) stamp(p, l, EV_SEL0, cta);
  // this item's output offset: definite keys + selected candidates of the
  // items before it
  const uint32_t taken_before = es.scan[44] + es.scan[45] + es.scan[46];
  const uint32_t out0 = es.pad + taken_before;
  const uint4 v = reinterpret_cast<const uint4*>(ws)[et];
  uint32_t wv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
  for (int i = 0; i < 4; ++i)
    if (et * 128 + i * 32 >= cnt) wv[i] = 0u;
  const uint32_t c = __popc(wv[0]) + __popc(wv[1]) + __popc(wv[2]) + __popc(wv[3]);
  uint32_t tot;
  uint32_t pos = epi_scan(c, es.scan, et, tot) - c + out0;
  const uint32_t pos0 = pos;
  if (et == 0) stamp(p, l, EV_X0, cta);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const uint32_t m0w = wv[i];
    const uint32_t base = (uint32_t)(w0 + i) * 32u;
    const uint32_t m1w = m0w & (m0w - 1u), m2w = m1w & (m1w - 1u), m3w = m2w & (m2w - 1u);
    uint32_t m4w = m3w & (m3w - 1u);
    st_global_pred(out + pos, base + (uint32_t)(__ffs(m0w) - 1), m0w != 0u);
    st_global_pred(out + pos + 1, base + (uint32_t)(__ffs(m1w) - 1), m1w != 0u);
    st_global_pred(out + pos + 2, base + (uint32_t)(__ffs(m2w) - 1), m2w != 0u);
    st_global_pred(out + pos + 3, base + (uint32_t)(__ffs(m3w) - 1), m3w != 0u);
    uint32_t p4 = pos + 4u;
    pos += __popc(m0w);
    while (m4w) {
      out[p4++] = (int32_t)(base + (uint32_t)(__ffs(m4w) - 1));
      m4w &= m4w - 1u;
    }
  }
  if (q == 0 && et == 0 && p.idx_count) p.idx_count[row] = (int32_t)R.k;
  if (p.set_trace) {  // debug: this layer's set (the StepTrace of decode_engine.hpp:144-147)
    int32_t* tr = p.set_trace + ((int64_t)l * p.max_sel + row) * p.idx_stride;
    for (uint32_t i = pos0; i < pos0 + c; ++i) tr[i] = out[i];
    if (q == 0 && et == 0) p.set_trace_count[(int64_t)l * p.max_sel + row] = (int32_t)R.k;
  }
  if (es.last) {
    if (et == 0) R.ctr[4] = 0u;
    if (p.sel_mode == SEL_BLOCK_KEYS)
      for (int i = et; i < n; i += kEpiThreads) R.keys[i] = 0u;
  }
  epi_bar();
  if (et == 0) {
    stamp(p, l, EV_F_EMIT, cta);
    signal(LYC_CTR(rt.ctr, l, CTR_SELDONE));
  }
}

// The step's lengths into shared memory (cold prologue code, kept out of the
// kernel body): per item its length, selection keys and budget; n_keys /
// k_sel of the longest item and the ragged flag into dyn[1..3].  Returns
// false (and flags the header) when a length is < 1 or > seq_cap.
__device__ __noinline__ bool step_lengths(const LycStepParams& p, int32_t* seqs, int32_t* nsel,
                                          int32_t* ksel, int32_t* dyn) {
  const LycPlanIn& pin = p.plan;
  __shared__ int32_t s_max, s_bad;
  if (threadIdx.x == 0) {
    s_max = 0;
    s_bad = INT_MAX;
  }
  __syncthreads();
  for (int b = threadIdx.x; b < pin.B; b += blockDim.x) {
    const int64_t v = pin.dlens ? __ldcg(pin.dlens + b) : pin.has_lens ? (int64_t)pin.lens[b] : pin.seq;
    const bool ok = v >= 1 && v <= pin.seq_cap;
    int32_t nb = 0, kb = 0;
    if (ok) {
      plan_item_key(pin, v, nb, kb);
      atomicMax(&s_max, (int32_t)v);
    } else {
      atomicMin(&s_bad, b);
    }
    seqs[b] = ok ? (int32_t)v : 0;
    nsel[b] = p.sel_mode == SEL_BLOCK_KEYS ? nb : (int32_t)v;
    ksel[b] = kb;
  }
  __syncthreads();
  if (s_bad != INT_MAX) {
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      p.hdr->bad_item = s_bad;
      p.hdr->status = 1;
    }
    return false;
  }
  int rag = 0;
  for (int b = threadIdx.x; b < pin.B; b += blockDim.x)
    rag |= (nsel[b] != nsel[0] || ksel[b] != ksel[0]) ? 1 : 0;
  const int ragged = __syncthreads_or(rag);
  if (threadIdx.x == 0) {
    int32_t nb, kb;
    plan_item_key(pin, s_max, nb, kb);
    dyn[1] = p.sel_mode == SEL_BLOCK_KEYS ? nb : s_max;
    dyn[2] = kb;
    dyn[3] = ragged;
  }
  __syncthreads();
  return true;
}

// ---------------------------------------------------------------- kernel
template <typename T, int D>
__global__ void __launch_bounds__(kStepThreads, 1) hybrid_step_kernel(const __grid_constant__ LycStepParams p) {
  using C = AttnCfg<T, D>;
  static_assert(sizeof(EpiSmem) <= C::kExtraBytes, "epilogue scratch does not fit");
  extern __shared__ uint8_t smem_raw[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int cta = blockIdx.x;
  const size_t set_words = LYC_CTR_SET_WORDS(p.n_layers);
  uint32_t* ctrl = p.ctr + 2 * set_words;  // [0] launch parity, [LYC_CTR_STRIDE] exits
  __shared__ int32_t s_dyn[4];             // parity, n_keys, k_sel, ragged
  __shared__ int32_t s_seq[LYC_PLAN_MAX_B];  // the step's lengths, per batch item
  __shared__ int32_t s_nsel[LYC_PLAN_MAX_B]; //   selection keys of its rows
  __shared__ int32_t s_ksel[LYC_PLAN_MAX_B]; //   ids kept per row
  const AttnSmem<T, D> sm = AttnSmem<T, D>::carve(smem_raw);
  EpiSmem& es = *reinterpret_cast<EpiSmem*>(sm.extra);
  const LycPlanIn& pin = p.plan;
  if (threadIdx.x == 0) stamp(p, p.l_begin, EV_ENTRY, cta);
  // on-chip setup before the wait for the previous launch (it touches no
  // global memory): barriers, the layer mark, the first-pass histogram
  if (threadIdx.x == 0) {
    for (int s = 0; s < C::kStages; ++s) {
      mbar_init(&sm.full[s], kProducerThreads + 1);  // + the tile-info arrival
      mbar_init(&sm.empty[s], kConsumerWarps);
    }
    mbar_init(&es.bar, 1);
    fence_mbar_init();
    *sm.clayer = 0u;
  }
  for (int b = threadIdx.x; b < LYC_H1_BINS; b += kStepThreads) sm.hist[b] = 0u;
  pdl_wait();     // the previous launch of the stream has completed and its writes are visible
  pdl_trigger();  // the next launch in the stream may begin its launch while this one runs
  if (threadIdx.x == 0) stamp(p, p.l_begin, EV_PDL, cta);
  if (threadIdx.x == 0) s_dyn[0] = (int32_t)__ldcg(ctrl);
  __syncthreads();
  if (threadIdx.x == 0) stamp(p, p.l_begin, 23, cta);  // barriers initialised
  // ---- the step's lengths (host values by value, or a device array read now);
  // one host length for the whole batch arrives pre-digested (no prologue pass)
  if (p.uniform) {
    for (int b = threadIdx.x; b < pin.B; b += kStepThreads) {
      s_seq[b] = (int32_t)pin.seq;
      s_nsel[b] = p.uni_nsel;
      s_ksel[b] = p.uni_ksel;
    }
    if (threadIdx.x == 0) {
      s_dyn[1] = p.uni_nsel;
      s_dyn[2] = p.uni_ksel;
      s_dyn[3] = 0;
    }
    __syncthreads();
  } else if (!step_lengths(p, s_seq, s_nsel, s_ksel, s_dyn)) {
    return;  // invalid: no work, no counter touched
  }
  const int par = s_dyn[0] & 1;
  StepRt rt;
  rt.ctr = p.ctr + (size_t)par * set_words;
  rt.rowctr = p.sel_rowctr + par * p.rowctr_set;
  rt.n_keys = s_dyn[1];
  rt.k_sel = s_dyn[2];
  rt.l_begin = p.l_begin;
  rt.ragged = s_dyn[3];
  rt.seqs = s_seq;
  rt.nsel = s_nsel;
  rt.ksel = s_ksel;
  if (threadIdx.x == 0) stamp(p, p.l_begin, 17, cta);  // prologue done
  if (cta == 0 && threadIdx.x == 0) p.hdr->status = 0;
  {  // zero the other set for the next launch (nobody uses it in this one)
    uint32_t* oc = p.ctr + (size_t)(par ^ 1) * set_words;
    uint32_t* orc = p.sel_rowctr + (par ^ 1) * p.rowctr_set;
    const int64_t stride = (int64_t)p.n_ctas * kStepThreads;
    for (int64_t i = (int64_t)cta * kStepThreads + threadIdx.x; i < (int64_t)set_words; i += stride)
      oc[i] = 0u;
    for (int64_t i = (int64_t)cta * kStepThreads + threadIdx.x; i < p.rowctr_set; i += stride)
      orc[i] = 0u;
  }
  constexpr uint32_t epoch1 = 1u;
  const uint32_t t_attn = (uint32_t)p.n_ctas;
  constexpr int esz = (int)sizeof(T);
  const int cell = cta;  // = b * n_splits + split

  if (warp < kConsumerWarps) {
    // ---------------- consumers
    const int tid = threadIdx.x;
    int stage = 0;
    uint32_t phase = 0;
    for (int l = p.l_begin; l < p.l_end; ++l) {
      if (l > p.l_begin) {
        if (tid == 0) {
          // the previous layer's outputs are final, and the key / histogram
          // buffers of this parity are free once layer l-2's selection (if
          // any) finished: both counters polled together (one round trip)
          const bool sel2 = l - 2 >= p.l_begin && p.layers[l - 2].n_sel > 0 && p.sel_mode != SEL_NONE;
          spin_until2(LYC_CTR(rt.ctr, l - 1, CTR_MERGE), t_attn,
                      sel2 ? LYC_CTR(rt.ctr, l - 2, CTR_SELDONE) : nullptr,
                      sel2 ? seldone_per_step(p, rt, l - 2) : 0u);
        }
        consumer_bar();
      }
      if (tid == 0) {
        st_release_cta_shared(sm.clayer, (uint32_t)(l + 1));
        stamp(p, l, EV_CONS_BEGIN, cta);
      }
      const LycLayerDesc L = p.layers[l];
      const LycView v = layer_view(p, rt, L, l, esz);
      consume_units<T, D>(v, sm, L.split_off[cell], L.split_off[cell + 1], warp, lane, stage,
                          phase, l > p.l_begin ? (l & 1) : -1);
      consumer_bar();
      if (tid == 0) {
        stamp(p, l, EV_CONS_END, cta);
        signal(LYC_CTR(rt.ctr, l, CTR_ATTN));
      }
      // while the grid finishes layer l: stage layer l + 1's unit records
      // (static plan data) into the other record buffer
      if constexpr (sizeof(T) == 2) {
        if (l + 1 < p.l_end) {
          const LycLayerDesc Ln = p.layers[l + 1];
          const LycView vn = layer_view(p, rt, Ln, l + 1, esz);
          UnitRec* rec = reinterpret_cast<UnitRec*>(sm.ustage) + ((l + 1) & 1) * C::kQUnits;
          stage_unit_records(vn, rec, Ln.split_off[cell], Ln.split_off[cell + 1], tid, C::kQUnits);
        }
      }
    }
  } else if (warp < kConsumerWarps + kProducerWarps) {
    // ---------------- producers
    const int pt = threadIdx.x - kConsumerWarps * 32;
    if (pt == 0) {
      prefetch_tensormap(&p.tmap_k);
      prefetch_tensormap(&p.tmap_v);
    }
    int stage = 0;
    uint32_t phase = 0;
    for (int l = p.l_begin; l < p.l_end; ++l) {
      const LycLayerDesc L = p.layers[l];
      const LycView v = layer_view(p, rt, L, l, esz);
      StepWaits waits{&p, &rt, l, pt, sm.clayer};
      produce_units<T, D>(v, &p.tmap_k, &p.tmap_v, sm.ring, sm.full, sm.empty, sm.tinfo,
                          L.split_off[cell], L.split_off[cell + 1], pt, stage, phase, waits);
    }
  } else {
    // ---------------- epilogue: merge + pooled selection
    const int et = threadIdx.x - (kConsumerWarps + kProducerWarps) * 32;
    const int ew = et >> 5;
    const int chunks = (D + 31) / 32;
    const int items = (rt.n_keys + kItemKeys - 1) / kItemKeys;
    uint32_t bar_phase = 0;
    // the selection items of layer l: classify every own item, then resolve
    // the rows and emit the items.  A deferred selection (the previous
    // layer's, carried into this launch) finds its slots complete already.
    auto run_items = [&](int l, int n_items, int item_base, bool split_roles, bool deferred) {
      const LycLayerDesc& L = p.layers[l];
      uint32_t* slot_ctr = rt.rowctr + (size_t)l * p.max_sel * 16 + 12;
      const int i0 = cta - item_base, istep = split_roles ? n_items : p.n_ctas;
      for (int it = i0; it < n_items; it += istep) {
        const int r = it / items, q = it - r * items;
        if (et == 0) {  // the row's retrieval slot is complete
          if (!deferred) {
            const int slot = __ldg(L.sel_rows + r);
            spin_until(slot_ctr + (size_t)slot * 16, epoch1 * (uint32_t)L.slots[slot].n_units);
          }
          stamp(p, l, EV_EPI_ATTN, cta);
        }
        epi_bar();
        classify_item(p, sel_row(p, rt, l, r), q, es, bar_phase, et, l, cta);
      }
      for (int it = i0; it < n_items; it += istep) {
        const int r = it / items, q = it - r * items;
        const int row = __ldg(L.sel_rows + r);
        resolve_emit_item(p, rt, sel_row(p, rt, l, r), q, row, p.idx + (int64_t)row * p.idx_stride,
                          es, bar_phase, et, l, cta);
      }
    };
    auto layer_items = [&](int l) {
      const LycLayerDesc& L = p.layers[l];
      return (L.n_sel > 0 && p.sel_mode != SEL_NONE) ? L.n_sel * items : 0;
    };
    if (p.sel_defer_in) {
      // the previous layer's selection, deferred from the previous launch
      // (one launch per layer): it runs while this layer's attention streams;
      // only this layer's units that read its sets wait for it
      const int l = p.l_begin - 1;
      const int n_items = layer_items(l);
      const bool split_roles = n_items > 0 && 2 * n_items <= p.n_ctas;
      const int item_base = split_roles ? p.n_ctas - n_items : 0;
      if (n_items > 0 && cta >= item_base) run_items(l, n_items, item_base, split_roles, true);
    }
    for (int l = p.l_begin; l < p.l_end; ++l) {
      const LycLayerDesc L = p.layers[l];
      // Roles of this layer's epilogue: when the selection items fit in half
      // the grid they go to the LAST n_items CTAs, which start classifying a
      // row as soon as its retrieval slot's units are all done (per-row unit
      // counter; retrieval units come first in every split) -- without waiting
      // for the rest of the layer -- while the other CTAs merge; otherwise
      // every CTA merges, then classifies.  The last layer's selection of a
      // launch with sel_defer_out is left to the next launch.
      const bool defer = p.sel_defer_out && l == p.l_end - 1;
      const int n_items = defer ? 0 : layer_items(l);
      const bool split_roles = n_items > 0 && 2 * n_items <= p.n_ctas;
      const int item_base = split_roles ? p.n_ctas - n_items : 0;
      const int merge_ctas = split_roles ? item_base : p.n_ctas;
      // no layer barrier: every merge task waits for its own slot's units,
      // every selection item for its row's retrieval slot (per-slot counters)
      uint32_t* slot_ctr = rt.rowctr + (size_t)l * p.max_sel * 16 + 12;
      // (a) split-KV merge
      const int total = L.n_merges * chunks;
      uint8_t* outl = static_cast<uint8_t*>(p.out) + (int64_t)(l - p.l_begin) * p.q_layer_stride * esz;
      if (cta < merge_ctas)
        for (int t = ew * merge_ctas + cta; t < total; t += merge_ctas * kEpiWarps) {
          const LycMergeTask tk = L.merges[t / chunks];
          if (lane == 0) spin_until(slot_ctr + (size_t)tk.slot * 16, epoch1 * (uint32_t)tk.n_units);
          __syncwarp();
          merge_task<T>(p.part_o, p.part_lse, tk, t % chunks, p.group, D, outl, lane);
        }
      epi_bar();
      if (et == 0) {
        stamp(p, l, EV_MERGE, cta);
        signal(LYC_CTR(rt.ctr, l, CTR_MERGE));
      }
      // (b) selection items of this layer's retrieval heads
      if (n_items > 0 && cta >= item_base) run_items(l, n_items, item_base, split_roles, false);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) stamp(p, max(p.l_begin, p.l_end - 1), 19, cta);  // CTA exit
  if (threadIdx.x == 0) {
    const uint32_t done = atomicAdd(ctrl + LYC_CTR_STRIDE, 1u);
    if (done == (uint32_t)p.n_ctas - 1u) {  // last CTA out: the next launch uses the other set
      ctrl[LYC_CTR_STRIDE] = 0u;
      ctrl[0] = (uint32_t)(par ^ 1);
    }
  }
}

template <typename T, int D>
static cudaError_t launch_step_t(const LycStepParams& p, cudaStream_t st, bool pdl) {
  using C = AttnCfg<T, D>;
  static bool configured[64] = {};
  bool& done = device_flag(configured);
  if (!done) {
    cudaError_t e = cudaFuncSetAttribute(hybrid_step_kernel<T, D>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmem);
    if (e != cudaSuccess) return e;
    done = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(p.n_ctas);
  cfg.blockDim = dim3(kStepThreads);
  cfg.dynamicSmemBytes = C::kSmem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 2 : 1;
  return cudaLaunchKernelEx(&cfg, hybrid_step_kernel<T, D>, p);
}

cudaError_t launch_step(const LycStepParams& p, int dtype, int d, cudaStream_t st, bool pdl) {
  if (dtype == 1) {
    switch (d) {
      case 64: return launch_step_t<__nv_bfloat16, 64>(p, st, pdl);
      case 128: return launch_step_t<__nv_bfloat16, 128>(p, st, pdl);
    }
  } else {
    switch (d) {
      case 16: return launch_step_t<float, 16>(p, st, pdl);
      case 32: return launch_step_t<float, 32>(p, st, pdl);
      case 64: return launch_step_t<float, 64>(p, st, pdl);
      case 128: return launch_step_t<float, 128>(p, st, pdl);
    }
  }
  return cudaErrorInvalidValue;
}

// Largest selection row (keys) the fused step supports.
int64_t step_max_keys() {
  return (int64_t)64 * kItemKeys;  // <= 64 items per row (one epilogue thread per item)
}
// Bytes of the step kernel's K/V ring (the in-kernel planner's scratch).
int64_t step_ring_bytes(int dtype, int d) {
  if (dtype == 1) {
    if (d == 64) return (int64_t)AttnCfg<__nv_bfloat16, 64>::kStages * AttnCfg<__nv_bfloat16, 64>::kStageBytes;
    if (d == 128) return (int64_t)AttnCfg<__nv_bfloat16, 128>::kStages * AttnCfg<__nv_bfloat16, 128>::kStageBytes;
    return 0;
  }
  switch (d) {
    case 16: return (int64_t)AttnCfg<float, 16>::kStages * AttnCfg<float, 16>::kStageBytes;
    case 32: return (int64_t)AttnCfg<float, 32>::kStages * AttnCfg<float, 32>::kStageBytes;
    case 64: return (int64_t)AttnCfg<float, 64>::kStages * AttnCfg<float, 64>::kStageBytes;
    case 128: return (int64_t)AttnCfg<float, 128>::kStages * AttnCfg<float, 128>::kStageBytes;
  }
  return 0;
}

int64_t step_bitmap_words(int64_t n_keys) { return bm_padded_words((int)((n_keys + 31) / 32)); }
int step_item_keys() { return kItemKeys; }

bool step_supported(int dtype, int d) {
  return dtype == 1 ? (d == 64 || d == 128) : (d == 16 || d == 32 || d == 64 || d == 128);
}

}  // namespace lyc
