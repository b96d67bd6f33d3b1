// Micro-benchmark: mma.sync m16n8k16 bf16 throughput/latency on sm_100a.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ void mma(float* c, uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0, uint32_t b1) {
  asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
               : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3]) : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
template <int CHAINS>
__global__ void k(long long* out, float* sink, int iters) {
  float c[CHAINS][4] = {};
  uint32_t a = threadIdx.x * 0x3c003c00u, b = 0x3c003c00u;
  const long long t0 = clock64();
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int j = 0; j < CHAINS; ++j) mma(c[j], a, a ^ j, a, a, b, b ^ i);
  const long long t1 = clock64();
  float s = 0;
  for (int j = 0; j < CHAINS; ++j) s += c[j][0] + c[j][1] + c[j][2] + c[j][3];
  sink[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = t1 - t0;
}
int main() {
  long long* o; float* s; cudaMalloc(&o, 8); cudaMalloc(&s, 1 << 24);
  const int iters = 4096;
  for (int warps : {1, 4, 8}) {
    long long c;
    k<1><<<1, 32 * warps>>>(o, s, iters); cudaMemcpy(&c, o, 8, cudaMemcpyDeviceToHost);
    printf("warps %d chains 1: %.1f cycles/mma per warp\n", warps, (double)c / iters);
    k<4><<<1, 32 * warps>>>(o, s, iters); cudaMemcpy(&c, o, 8, cudaMemcpyDeviceToHost);
    printf("warps %d chains 4: %.1f cycles/mma per warp\n", warps, (double)c / iters / 4);
    k<8><<<1, 32 * warps>>>(o, s, iters); cudaMemcpy(&c, o, 8, cudaMemcpyDeviceToHost);
    printf("warps %d chains 8: %.1f cycles/mma per warp\n", warps, (double)c / iters / 8);
  }
}
