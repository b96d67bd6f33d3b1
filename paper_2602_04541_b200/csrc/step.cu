// step.cu -- the persistent decode-step kernel: every layer of one decode step
// (decode_engine.hpp:109-151) in ONE launch, one CTA per SM.
//
// Warp roles per CTA (256 threads):
//   0-3 consumers  attention of this CTA's split of layer l (attn_core.cuh);
//                  layer l+1 starts only after layer l's outputs are final
//                  (device counter), emulating the model's layer dependency.
//   4-5 producers  stream the K/V tiles of layer l, l+1, ... continuously
//                  through the smem ring: the next layer's history rows are in
//                  flight while layer l is still being merged.  Tiles whose
//                  index list comes from a selection wait for that selection;
//                  the tile holding the current token waits for the previous
//                  layer (its K/V row is produced after it).
//   6-7 epilogue   after the whole grid finishes layer l's attention:
//                  (a) the split-KV LSE merge (kernel_sim.hpp:205-225), work
//                      spread over every CTA;
//                  (b) exact top-k selection for the layer's retrieval heads
//                      (args_top_k, attention.hpp:108-123: largest k, ties to
//                      the lower index, ascending) as a grid-wide radix select:
//                      the consumers already built the first 11-bit histogram
//                      while scoring; three more passes over each CTA's key
//                      slice, separated by grid barriers, fix the k-th key T
//                      exactly; an ordered compaction writes the index cache.
//                  Selection runs concurrently with the next layer's attention
//                  (Algorithm 2's workload pooling applied to selection).
// Grid-wide coordination uses monotonic per-layer counters in global memory
// (a step adds n_ctas to each); the launch is cooperative so every CTA is
// co-resident.
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
    __nanosleep(40);
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

struct StepWaits {
  const uint32_t* ctr;
  uint32_t target;
  int layer;
  int pt;
  __device__ __forceinline__ void wait(const uint32_t* c) const {
    if (pt == 0) spin_until(c, target);
    group_bar(3, kProducerThreads);
  }
  __device__ __forceinline__ void unit(const LycSlot& s) const {
    if (s.dep >= 0) wait(ctr + s.dep * CTR_PER_LAYER + CTR_SELDONE);
  }
  __device__ __forceinline__ void last_tile() const {
    if (layer > 0) wait(ctr + (layer - 1) * CTR_PER_LAYER + CTR_MERGE);
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
  v.hist1 = p.sel_mode == SEL_TOKEN_KEYS
                ? p.hist + (int64_t)((l & 1) * 3) * p.max_sel * LYC_BINS
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
// Warp-level search of a 2048-bin histogram (from the top bin down) for the
// bin holding the krem-th largest candidate.  Returns (digit, count above).
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
    const uint4 v = __ldcg(src + q);
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

struct SelScratch {      // per selection row, in the epilogue smem scratch
  uint32_t prefix;       // key bits fixed so far
  uint32_t krem;         // candidates still to take among keys matching prefix
  uint32_t take_eq;      // phase E: ties this CTA takes
  uint32_t out_base;     // phase E: output offset of this CTA
};

__device__ __forceinline__ void grid_barrier_epi(uint32_t* ctr, uint32_t target, int et) {
  group_bar(2, kEpiThreads);
  if (et == 0) {
    signal(ctr);
    spin_until(ctr, target);
  }
  group_bar(2, kEpiThreads);
}

template <typename T, int D>
__device__ void select_layer(const LycStepParams& p, const LycLayerDesc& L, int l, int cta,
                             uint32_t target, int et, SelScratch* ss, uint32_t* scan) {
  const int lane = et & 31, w = et >> 5;
  const int n = p.n_keys;
  const int lo = (int)((int64_t)cta * n / p.n_ctas);
  const int hi = (int)((int64_t)(cta + 1) * n / p.n_ctas);
  uint32_t* lc = p.ctr + l * CTR_PER_LAYER;
  auto keys_of = [&](int r) {
    return p.sel_keys + ((int64_t)(l & 1) * p.max_sel + r) * p.sel_stride;
  };
  auto hist_of = [&](int r, int pass) {
    return p.hist + ((int64_t)((l & 1) * 3 + pass) * p.max_sel + r) * LYC_BINS;
  };
  const int nsel = L.n_sel;

  if (p.sel_mode == SEL_BLOCK_KEYS) {
    // block keys were max-folded by atomics: build the first-pass histogram here
    for (int r = 0; r < nsel; ++r) {
      const uint32_t* kr = keys_of(r);
      uint32_t* h = hist_of(r, 0);
      for (int i0 = lo; i0 < hi; i0 += kEpiThreads) {
        const int i = i0 + et;
        const bool ok = i < hi;
        const uint32_t key = ok ? __ldcg(kr + i) : 0u;
        hist_add(h, key >> 21, ok, 0xffffffffu, lane);
      }
    }
    grid_barrier_epi(lc + CTR_SEL3, target, et);
  }
  // ---- pass 1 digit (bits 31..21) from the fused histogram; pass 2 histogram
  for (int r = w; r < nsel; r += kEpiWarps) {
    uint32_t d, a;
    find_digit(hist_of(r, 0), 2048, (uint32_t)p.k_sel, d, a, lane);
    if (lane == 0) {
      ss[r].prefix = d << 21;
      ss[r].krem = (uint32_t)p.k_sel - a;
    }
  }
  group_bar(2, kEpiThreads);
  for (int r = 0; r < nsel; ++r) {
    const uint32_t* kr = keys_of(r);
    uint32_t* h = hist_of(r, 1);
    const uint32_t pre = ss[r].prefix >> 21;
    for (int i0 = lo; i0 < hi; i0 += kEpiThreads) {
      const int i = i0 + et;
      const uint32_t key = i < hi ? __ldcg(kr + i) : 0u;
      const bool ok = i < hi && (key >> 21) == pre;
      hist_add(h, (key >> 10) & 0x7ffu, ok, 0xffffffffu, lane);
    }
  }
  grid_barrier_epi(lc + CTR_SEL0, target, et);
  // ---- pass 2 digit (bits 20..10); pass 3 histogram
  for (int r = w; r < nsel; r += kEpiWarps) {
    uint32_t d, a;
    find_digit(hist_of(r, 1), 2048, ss[r].krem, d, a, lane);
    if (lane == 0) {
      ss[r].prefix |= d << 10;
      ss[r].krem -= a;
    }
  }
  group_bar(2, kEpiThreads);
  for (int r = 0; r < nsel; ++r) {
    const uint32_t* kr = keys_of(r);
    uint32_t* h = hist_of(r, 2);
    const uint32_t pre = ss[r].prefix >> 10;
    for (int i0 = lo; i0 < hi; i0 += kEpiThreads) {
      const int i = i0 + et;
      const uint32_t key = i < hi ? __ldcg(kr + i) : 0u;
      const bool ok = i < hi && (key >> 10) == pre;
      hist_add(h, key & 0x3ffu, ok, 0xffffffffu, lane);
    }
  }
  grid_barrier_epi(lc + CTR_SEL1, target, et);
  // ---- pass 3 digit (bits 9..0): T exact; count > T and == T in this slice
  for (int r = w; r < nsel; r += kEpiWarps) {
    uint32_t d, a;
    find_digit(hist_of(r, 2), 1024, ss[r].krem, d, a, lane);
    if (lane == 0) {
      ss[r].prefix |= d;
      ss[r].krem -= a;  // ties of T to take, grid-wide
    }
  }
  group_bar(2, kEpiThreads);
  for (int r = 0; r < nsel; ++r) {
    const uint32_t* kr = keys_of(r);
    const uint32_t T = ss[r].prefix;
    uint32_t gt = 0, eq = 0;
    for (int i = lo + et; i < hi; i += kEpiThreads) {
      const uint32_t key = __ldcg(kr + i);
      gt += key > T;
      eq += key == T;
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      gt += __shfl_xor_sync(0xffffffffu, gt, off);
      eq += __shfl_xor_sync(0xffffffffu, eq, off);
    }
    if (lane == 0) {
      scan[2 * w] = gt;
      scan[2 * w + 1] = eq;
    }
    group_bar(2, kEpiThreads);
    if (et == 0) {
      uint32_t* tm = p.team + (((int64_t)(l & 1) * p.max_sel + r) * p.n_ctas + cta) * 2;
      tm[0] = scan[0] + scan[2];
      tm[1] = scan[1] + scan[3];
    }
    group_bar(2, kEpiThreads);
  }
  grid_barrier_epi(lc + CTR_SEL2, target, et);
  // ---- ordered compaction of this slice into the index cache
  for (int r = w; r < nsel; r += kEpiWarps) {
    const uint32_t* tm = p.team + ((int64_t)(l & 1) * p.max_sel + r) * p.n_ctas * 2;
    uint32_t base = 0, eqb = 0;
    for (int c = lane; c < cta; c += 32) {
      base += __ldcg(tm + 2 * c);
      eqb += __ldcg(tm + 2 * c + 1);
    }
    // the ties taken by earlier CTAs are min(their ties, remaining) in order:
    // sum_{c<cta} take_c = min(eq_before, krem)
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      base += __shfl_xor_sync(0xffffffffu, base, off);
      eqb += __shfl_xor_sync(0xffffffffu, eqb, off);
    }
    if (lane == 0) {
      const uint32_t krem = ss[r].krem;
      const uint32_t mine_eq = __ldcg(tm + 2 * cta + 1);
      ss[r].out_base = base + min(eqb, krem);
      ss[r].take_eq = krem > eqb ? min(mine_eq, krem - eqb) : 0u;
    }
  }
  group_bar(2, kEpiThreads);
  for (int r = 0; r < nsel; ++r) {
    const uint32_t* kr = keys_of(r);
    const uint32_t T = ss[r].prefix, take_eq = ss[r].take_eq;
    int32_t* out = p.idx + (int64_t)__ldg(L.sel_rows + r) * p.idx_stride + ss[r].out_base;
    uint32_t run_gt = 0, run_eq = 0;
    constexpr int kPer = 4;
    for (int base = lo; base < hi; base += kEpiThreads * kPer) {
      const int i0 = base + et * kPer;
      uint32_t kv[kPer];
      uint32_t g = 0, e = 0;
#pragma unroll
      for (int q = 0; q < kPer; ++q) {
        const bool ok = i0 + q < hi;
        kv[q] = ok ? __ldcg(kr + i0 + q) : 0u;
        g += ok && kv[q] > T;
        e += ok && kv[q] == T;
      }
      const uint32_t mine = (e << 16) | g;
      uint32_t incl = mine;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const uint32_t t = __shfl_up_sync(0xffffffffu, incl, off);
        if (lane >= off) incl += t;
      }
      if (lane == 31) scan[w] = incl;
      group_bar(2, kEpiThreads);
      const uint32_t wbefore = w == 0 ? 0u : scan[0];
      const uint32_t total = scan[0] + scan[1];
      group_bar(2, kEpiThreads);
      const uint32_t excl = incl - mine + wbefore;
      uint32_t gb = run_gt + (excl & 0xffffu);
      uint32_t eb = run_eq + (excl >> 16);
#pragma unroll
      for (int q = 0; q < kPer; ++q) {
        if (i0 + q >= hi) break;
        const bool is_gt = kv[q] > T, is_eq = kv[q] == T;
        if (is_gt || (is_eq && eb < take_eq)) out[gb + min(eb, take_eq)] = i0 + q;
        gb += is_gt;
        eb += is_eq;
      }
      run_gt += total & 0xffffu;
      run_eq += total >> 16;
    }
    // reset this CTA's share of the histograms (and block keys) for reuse
    for (int pass = 0; pass < 3; ++pass) {
      uint32_t* h = hist_of(r, pass);
      const int b0 = (int)((int64_t)cta * LYC_BINS / p.n_ctas);
      const int b1 = (int)((int64_t)(cta + 1) * LYC_BINS / p.n_ctas);
      for (int b = b0 + et; b < b1; b += kEpiThreads) h[b] = 0u;
    }
    if (p.sel_mode == SEL_BLOCK_KEYS) {
      uint32_t* kw = p.sel_keys + ((int64_t)(l & 1) * p.max_sel + r) * p.sel_stride;
      for (int i = lo + et; i < hi; i += kEpiThreads) kw[i] = 0u;
    }
    if (cta == 0 && et == 0 && p.idx_count) p.idx_count[__ldg(L.sel_rows + r)] = p.k_sel;
  }
  group_bar(2, kEpiThreads);
  if (et == 0) signal(lc + CTR_SELDONE);
}

// ---------------------------------------------------------------- kernel
template <typename T, int D>
__global__ void __launch_bounds__(kStepThreads, 1) hybrid_step_kernel(const __grid_constant__ LycStepParams p) {
  using C = AttnCfg<T, D>;
  extern __shared__ uint8_t smem_raw[];
  const AttnSmem<T, D> sm = AttnSmem<T, D>::carve(smem_raw);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int cta = blockIdx.y * p.n_splits + blockIdx.x;
  uint32_t* ctrl = p.ctr + p.n_layers * CTR_PER_LAYER;  // [0] completed steps, [1] exits

  if (threadIdx.x == 0) {
    for (int s = 0; s < C::kStages; ++s) {
      mbar_init(&sm.full[s], kProducerThreads);
      mbar_init(&sm.empty[s], kConsumerWarps);
    }
    fence_mbar_init();
    reinterpret_cast<uint32_t*>(sm.extra)[0] = ld_acquire(ctrl);
  }
  __syncthreads();
  const uint32_t target = (reinterpret_cast<uint32_t*>(sm.extra)[0] + 1u) * (uint32_t)p.n_ctas;
  __syncthreads();
  constexpr int esz = (int)sizeof(T);

  if (warp < kConsumerWarps) {
    const int tid = threadIdx.x;
    int stage = 0;
    uint32_t phase = 0;
    for (int l = 0; l < p.n_layers; ++l) {
      if (l > 0) {
        if (tid == 0) {
          spin_until(p.ctr + (l - 1) * CTR_PER_LAYER + CTR_MERGE, target);
          // key / histogram buffers of this parity are free once layer l-2's
          // selection (if any) finished
          if (l >= 2 && p.layers[l - 2].n_sel > 0)
            spin_until(p.ctr + (l - 2) * CTR_PER_LAYER + CTR_SELDONE, target);
          __threadfence();
        }
        consumer_bar();
      }
      const LycLayerDesc L = p.layers[l];
      const LycView v = layer_view(p, L, l, esz);
      const int cell = blockIdx.y * p.n_splits + blockIdx.x;
      consume_units<T, D>(v, sm, L.split_off[cell], L.split_off[cell + 1], warp, lane, stage,
                          phase);
      consumer_bar();
      if (tid == 0) signal(p.ctr + l * CTR_PER_LAYER + CTR_ATTN);
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
      const int cell = blockIdx.y * p.n_splits + blockIdx.x;
      StepWaits waits{p.ctr, target, l, pt};
      produce_units<T, D>(v, &p.tmap_k, &p.tmap_v, sm.ring, sm.full, sm.empty,
                          L.split_off[cell], L.split_off[cell + 1], pt, stage, phase, waits);
    }
  } else {
    const int et = threadIdx.x - (kConsumerWarps + kProducerWarps) * 32;
    const int ew = et >> 5;
    SelScratch* ss = reinterpret_cast<SelScratch*>(sm.extra + 64);
    uint32_t* scan = reinterpret_cast<uint32_t*>(sm.extra + 16);
    const int chunks = (D + 31) / 32;
    for (int l = 0; l < p.n_layers; ++l) {
      const LycLayerDesc L = p.layers[l];
      uint32_t* lc = p.ctr + l * CTR_PER_LAYER;
      if (et == 0) {
        spin_until(lc + CTR_ATTN, target);
        __threadfence();
      }
      group_bar(2, kEpiThreads);
      // (a) split-KV merge, spread over all CTAs' epilogue warps
      const int total = L.n_merges * chunks;
      const uint8_t* outl = static_cast<const uint8_t*>(p.out) + (int64_t)l * p.q_layer_stride * esz;
      for (int t = cta * kEpiWarps + ew; t < total; t += p.n_ctas * kEpiWarps) {
        const LycMergeTask tk = L.merges[t / chunks];
        const LycSlot s = L.slots[tk.slot];
        merge_task<T>(p.part_o, p.part_lse, s, tk.j, t % chunks, p.group, D,
                      const_cast<uint8_t*>(outl), lane);
      }
      group_bar(2, kEpiThreads);
      if (et == 0) signal(lc + CTR_MERGE);
      // (b) selection for this layer's retrieval heads
      if (L.n_sel > 0 && p.sel_mode != SEL_NONE)
        select_layer<T, D>(p, L, l, cta, target, et, ss, scan);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const uint32_t done = atomicAdd(ctrl + 1, 1u);
    if (done == target - 1u) atomicAdd(ctrl, 1u);  // last CTA out: one more completed step
  }
}

template <typename T, int D>
static cudaError_t launch_step_t(const LycStepParams& p, int batch, cudaStream_t st) {
  using C = AttnCfg<T, D>;
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(hybrid_step_kernel<T, D>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmem);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(p.n_splits, batch);
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

cudaError_t launch_step(const LycStepParams& p, int dtype, int d, int batch, cudaStream_t st) {
  if (dtype == 1) {
    switch (d) {
      case 64: return launch_step_t<__nv_bfloat16, 64>(p, batch, st);
      case 128: return launch_step_t<__nv_bfloat16, 128>(p, batch, st);
    }
  } else {
    switch (d) {
      case 16: return launch_step_t<float, 16>(p, batch, st);
      case 32: return launch_step_t<float, 32>(p, batch, st);
      case 64: return launch_step_t<float, 64>(p, batch, st);
      case 128: return launch_step_t<float, 128>(p, batch, st);
    }
  }
  return cudaErrorInvalidValue;
}

bool step_supported(int dtype, int d) {
  return dtype == 1 ? (d == 64 || d == 128) : (d == 16 || d == 32 || d == 64 || d == 128);
}

}  // namespace lyc
