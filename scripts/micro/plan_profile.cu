// Micro-benchmark of the device planner (plan.cuh) on the qwen3-8b-128k shape:
// per-phase %globaltimer stamps of one CTA (build: nvcc -arch=sm_100a -O3 -I..).
#include <cstdio>
#include <vector>
#include <cuda_runtime.h>
#define LYC_PLAN_STAMP(k) do { LYC_PLAN_STAMP_DEV(k) } while (0)
#ifdef __CUDA_ARCH__
#define LYC_PLAN_STAMP_DEV(k) if (threadIdx.x == 0 && g_stamps) { unsigned long long t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); g_stamps[blockIdx.x * 16 + (k)] = t; }
#else
#define LYC_PLAN_STAMP_DEV(k)
#endif
__device__ unsigned long long* g_stamps;
#include "../../paper_2602_04541_b200/csrc/lyc_common.cuh"
#include "../../paper_2602_04541_b200/csrc/plan.cuh"
#include "../../paper_2602_04541_b200/csrc/plan.cu"

int main() {
  const int NL = 36, B = 1, H = 8, G = 4, D = 128, S = 148;
  std::vector<uint8_t> roles(NL * H, 1);
  for (int g = 0; g < H; ++g) roles[g] = 0;
  for (int l = 1; l < NL; l += 2) roles[l * H + (l % H)] = 0;
  uint8_t* d_roles; cudaMalloc(&d_roles, roles.size()); cudaMemcpy(d_roles, roles.data(), roles.size(), cudaMemcpyHostToDevice);
  const int BH = B * H, cells = B * S, max_units = BH + 3 * cells + 3, max_merges = BH * G;
  std::vector<LycLayerDesc> descs(NL);
  for (int l = 0; l < NL; ++l) {
    LycLayerDesc& d = descs[l];
    LycSlot* p; cudaMalloc(&p, BH * sizeof(LycSlot)); d.slots = p;
    LycUnit* u; cudaMalloc(&u, max_units * sizeof(LycUnit)); d.units = u;
    cudaMalloc(&p, max_units * sizeof(LycSlot)); d.unit_slots = p;
    int32_t* i; cudaMalloc(&i, (cells + 1) * 4); d.split_off = i;
    LycMergeTask* m; cudaMalloc(&m, max_merges * sizeof(LycMergeTask)); d.merges = m;
    cudaMalloc(&i, BH * 4); d.sel_rows = i; cudaMalloc(&i, BH * 4); d.sel_n = i; cudaMalloc(&i, BH * 4); d.sel_k = i;
  }
  LycLayerDesc* d_layers; cudaMalloc(&d_layers, NL * sizeof(LycLayerDesc));
  cudaMemcpy(d_layers, descs.data(), NL * sizeof(LycLayerDesc), cudaMemcpyHostToDevice);
  LycPlanHdr* hdr; cudaMalloc(&hdr, sizeof(LycPlanHdr));
  int32_t* idx; cudaMalloc(&idx, BH * 4096 * 4);
  unsigned long long* st; cudaMalloc(&st, NL * 16 * 8); cudaMemset(st, 0, NL * 16 * 8);
  cudaMemcpyToSymbol(g_stamps, &st, sizeof(st));
  LycPlanIn in{};
  in.NL = NL; in.B = B; in.H = H; in.G = G; in.D = D; in.S = S; in.bs = 64; in.select_mode = 0;
  in.policy_kind = 0; in.item_keys = 8192; in.seq_cap = 131072; in.k_cap = 4096; in.top_k = 4096;
  in.roles = d_roles; in.idx = idx; in.layers = d_layers; in.hdr = hdr; in.max_units = max_units;
  in.max_merges = max_merges; in.seq = 131072;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int it = 0; it < 5; ++it) lyc::launch_plan(in, 0, false);
  cudaEventRecord(e0);
  for (int it = 0; it < 100; ++it) lyc::launch_plan(in, 0, false);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  printf("plan kernel: %.2f us per launch (back to back), err=%s\n", ms * 10, cudaGetErrorString(cudaGetLastError()));
  std::vector<unsigned long long> h(NL * 16);
  cudaMemcpy(h.data(), st, h.size() * 8, cudaMemcpyDeviceToHost);
  for (int l = 0; l < 3; ++l) {
    printf("layer %d:", l);
    for (int k = 1; k < 16; ++k) if (h[l * 16 + k]) printf(" %d:%.2f", k, (h[l * 16 + k] - h[l * 16]) / 1e3);
    printf("\n");
  }
  return 0;
}
