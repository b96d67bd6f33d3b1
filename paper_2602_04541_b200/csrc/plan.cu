// plan.cu -- the device planner of the fused decode step (plan.cuh).  One CTA
// per layer turns the static role map and the step's lengths (by value, or a
// device array) into the per-layer unit / merge / selection arrays the step
// kernel reads.  The plan depends on the lengths only through its key (per
// item: dense blocks and sparse budget; selection items per row, lyc_plan.h),
// so a growing sequence re-plans once per 64 tokens:
//   * host lengths: the host tracks the key and launches the planner only when
//     it changes (stream-ordered before the step kernel);
//   * device lengths (a captured graph replaying t, t+1, ...): the planner
//     runs every step and returns at once when a layer's stored key matches.
// The same plan_layer also runs sequentially on the host (lyc_plan_selftest).
#include <cuda_runtime.h>

#include <climits>
#include <vector>

#include "lyc_common.cuh"
#include "plan.cuh"

namespace lyc {

__global__ void __launch_bounds__(LYC_PLAN_THREADS) plan_kernel(const __grid_constant__ LycPlanIn in) {
  extern __shared__ int32_t plan_smem[];
  __shared__ int32_t s_max, s_bad;
  pdl_trigger();  // the step kernel may launch now (it waits for this grid)
  pdl_wait();     // the previous step kernel has stopped reading the plan
  const int l = blockIdx.x, B = in.B;
  int32_t* key = in.keys + (size_t)l * LYC_PLAN_KEY_INTS(B);
  if (threadIdx.x == 0) {
    s_max = 0;
    s_bad = 0;
  }
  __syncthreads();
  // this step's key (lengths from the device array or by value)
  for (int b = threadIdx.x; b < B; b += blockDim.x) {
    const int64_t v = in.dlens ? __ldcg(in.dlens + b) : in.has_lens ? (int64_t)in.lens[b] : in.seq;
    if (v < 1 || v > in.seq_cap) s_bad = 1;
    else atomicMax(&s_max, (int32_t)v);
  }
  __syncthreads();
  int diff = s_bad;
  if (!s_bad) {
    for (int b = threadIdx.x; b < B; b += blockDim.x) {
      const int64_t v = in.dlens ? __ldcg(in.dlens + b) : in.has_lens ? (int64_t)in.lens[b] : in.seq;
      int32_t nb, kb;
      plan_item_key(in, v, nb, kb);
      diff |= (key[2 + b] != nb || key[2 + B + b] != kb) ? 1 : 0;
    }
    if (threadIdx.x == 0) diff |= (key[0] != 1 || key[1] != plan_items(in, s_max)) ? 1 : 0;
  }
  if (!__syncthreads_or(diff)) return;  // this layer's plan already fits
  const PlanScratch s = plan_carve(plan_smem, in.B, in.H, in.S, in.NL);
  DevX x;
  plan_layer(x, in, l, s, plan_out_of(in.layers + l));
  __syncthreads();
  // the key this layer's plan was made for (invalid lengths: none)
  for (int b = threadIdx.x; b < B; b += blockDim.x) {
    const int64_t v = in.dlens ? __ldcg(in.dlens + b) : in.has_lens ? (int64_t)in.lens[b] : in.seq;
    int32_t nb = 0, kb = 0;
    if (!s_bad) plan_item_key(in, v, nb, kb);
    key[2 + b] = nb;
    key[2 + B + b] = kb;
  }
  if (threadIdx.x == 0) {
    key[0] = s_bad ? 0 : 1;
    key[1] = s_bad ? 0 : plan_items(in, s_max);
  }
}

size_t plan_smem_bytes(int B, int H, int S, int NL) {
  return (size_t)plan_scratch_ints(B, H, S, NL) * 4;
}

cudaError_t launch_plan(const LycPlanIn& in, cudaStream_t st, bool pdl) {
  const size_t smem = plan_smem_bytes(in.B, in.H, in.S, in.NL);
  static bool configured[64] = {};
  bool& done = device_flag(configured);
  if (!done) {  // up to the largest plan a decoder may create (capi.cu: B*H <= 2048)
    cudaError_t e = cudaFuncSetAttribute(plan_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         160 * 1024);
    if (e != cudaSuccess) return e;
    done = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(in.NL);
  cfg.blockDim = dim3(LYC_PLAN_THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, plan_kernel, in);
}

// The same planner, sequentially on the host (self-test; in.roles, in.hdr and
// the PlanOut targets are host memory).
void plan_layer_host(const LycPlanIn& in, int l, const PlanOut& o) {
  std::vector<int32_t> scratch((size_t)plan_scratch_ints(in.B, in.H, in.S, in.NL));
  const PlanScratch s = plan_carve(scratch.data(), in.B, in.H, in.S, in.NL);
  HostX x;
  plan_layer(x, in, l, s, o);
}

}  // namespace lyc
