// attn.cu -- per-launch kernels of the hybrid-head decode attention:
//   hybrid_attn_kernel  one layer's pooled split-KV attention (Algorithm 2,
//                       PAPER.md:543-557; kernel_sim.hpp:169-201 run_split),
//                       used by lyc_workload_run (hh::kernel::run) and
//                       lyc_decoder_layer;
//   split_merge_kernel  the LSE merge (kernel_sim.hpp:205-225 combine).
// The device building blocks live in attn_core.cuh; the persistent whole-step
// kernel is step.cu.
#include "attn_core.cuh"

namespace lyc {

constexpr int kAttnThreads = (kConsumerWarps + kProducerWarps) * 32;

template <typename T, int D, bool kEarlyExit>
__global__ void __launch_bounds__(kAttnThreads, 1) hybrid_attn_kernel(const __grid_constant__ LycAttnParams p) {
  using C = AttnCfg<T, D>;
  extern __shared__ uint8_t smem_raw[];
  const AttnSmem<T, D> sm = AttnSmem<T, D>::carve(smem_raw);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int cell = blockIdx.y * p.v.n_splits + blockIdx.x;
  const int ub = p.v.split_off[cell], ue = p.v.split_off[cell + 1];

  if (threadIdx.x == 0) {
    for (int s = 0; s < C::kStages; ++s) {
      mbar_init(&sm.full[s], kProducerThreads + 1);  // + the tile-info arrival
      mbar_init(&sm.empty[s], kConsumerWarps);
    }
    fence_mbar_init();
  }
  __syncthreads();
  int stage = 0;
  uint32_t phase = 0;
  if (warp >= kConsumerWarps) {
    const int pt = threadIdx.x - kConsumerWarps * 32;
    if (pt == 0) {
      prefetch_tensormap(&p.tmap_k);
      prefetch_tensormap(&p.tmap_v);
    }
    produce_units<T, D>(p.v, &p.tmap_k, &p.tmap_v, sm.ring, sm.full, sm.empty, sm.tinfo, ub, ue, pt, stage,
                        phase, NoWaits{});
  } else {
    consume_units<T, D, kEarlyExit>(p.v, sm, ub, ue, warp, lane, stage, phase);
  }
}

template <typename T>
__global__ void __launch_bounds__(128) split_merge_kernel(const __grid_constant__ LycMergeParams p) {
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int task = gw / p.chunks, chunk = gw - task * p.chunks;
  if (task >= p.n_tasks) return;
  const LycMergeTask tk = p.tasks[task];
  merge_task<T>(p.part_o, p.part_lse, tk, chunk, p.group, p.d, p.out, lane, p.out_f32, p.out_lse);
}

// ---------------------------------------------------------------- launchers
template <typename T, int D, bool kEarlyExit>
static cudaError_t launch_attn_tt(const LycAttnParams& p, int batch, cudaStream_t st) {
  using C = AttnCfg<T, D>;
  static bool configured_[64] = {};
  bool& configured = device_flag(configured_);
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(hybrid_attn_kernel<T, D, kEarlyExit>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmem);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  dim3 grid(p.v.n_splits, batch);
  hybrid_attn_kernel<T, D, kEarlyExit><<<grid, kAttnThreads, C::kSmem, st>>>(p);
  return cudaGetLastError();
}

template <typename T, int D>
static cudaError_t launch_attn_t(const LycAttnParams& p, int batch, cudaStream_t st) {
  return p.v.early_exit ? launch_attn_tt<T, D, true>(p, batch, st)
                        : launch_attn_tt<T, D, false>(p, batch, st);
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
