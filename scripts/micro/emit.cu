// Micro-benchmark: ascending emission of the set bits of a 4096-word smem
// bitmap by 64 threads (the selection finisher's last phase), two variants.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void emit_warp_rounds(const uint32_t* gbm, int nwords, int* out, long long* cyc) {
  __shared__ uint32_t bmp[4096];
  __shared__ uint32_t scan[64];
  const int et = threadIdx.x, lane = et & 31, ew = et >> 5;
  for (int i = et; i < nwords; i += 64) bmp[i] = gbm[i];
  __syncthreads();
  const long long c0 = clock64();
  const int hw = (((nwords + 1) / 2) + 31) & ~31;
  const int wb = min(nwords, ew * hw), we = min(nwords, wb + hw);
  uint32_t c = 0;
  for (int w = wb + lane; w < we; w += 32) c += __popc(bmp[w]);
  for (int off = 16; off > 0; off >>= 1) c += __shfl_xor_sync(0xffffffffu, c, off);
  if (lane == 0) scan[32 + ew] = c;
  __syncthreads();
  uint32_t base = ew ? scan[32] : 0u;
  for (int w0 = wb; w0 < we; w0 += 32) {
    const int w = w0 + lane;
    uint32_t m = w < we ? bmp[w] : 0u;
    const uint32_t cw = __popc(m);
    uint32_t incl = cw;
    for (int off = 1; off < 32; off <<= 1) {
      const uint32_t t = __shfl_up_sync(0xffffffffu, incl, off);
      if (lane >= off) incl += t;
    }
    uint32_t pos = base + incl - cw;
    base += __shfl_sync(0xffffffffu, incl, 31);
    while (m) {
      const int j = __ffs(m) - 1;
      m &= m - 1;
      out[pos++] = w * 32 + j;
    }
  }
  __syncthreads();
  if (et == 0) cyc[0] = clock64() - c0;
}

__global__ void emit_chunks(const uint32_t* gbm, int nwords, int* out, long long* cyc) {
  __shared__ uint32_t bmp[4096];
  __shared__ uint32_t scan[64];
  __shared__ int stage[6144];
  const int et = threadIdx.x, lane = et & 31, ew = et >> 5;
  for (int i = et; i < nwords; i += 64) bmp[i] = gbm[i];
  __syncthreads();
  const long long c0 = clock64();
  const int per = (nwords + 63) / 64;
  const int w0 = min(nwords, et * per), w1 = min(nwords, w0 + per);
  uint32_t c = 0;
  for (int i = 0; i < per; ++i) {  // rotated: conflict-free
    const int w = w0 + ((i + et) % per);
    if (w < w1) c += __popc(bmp[w]);
  }
  const long long c1 = clock64();
  uint32_t incl = c;
  for (int off = 1; off < 32; off <<= 1) {
    const uint32_t t = __shfl_up_sync(0xffffffffu, incl, off);
    if (lane >= off) incl += t;
  }
  if (lane == 31) scan[ew] = incl;
  __syncthreads();
  uint32_t pos = incl - c + (ew ? scan[0] : 0u);
  const uint32_t total = scan[0] + scan[1];
  for (int w = w0; w < w1; ++w) {
    uint32_t m = bmp[w];
    while (m) {
      const int j = __ffs(m) - 1;
      m &= m - 1;
      stage[pos++] = w * 32 + j;
    }
  }
  const long long c2 = clock64();
  __syncthreads();
  const long long c3 = clock64();
  for (uint32_t i = et; i < total; i += 64) out[i] = stage[i];
  __syncthreads();
  if (et == 0) { cyc[0] = clock64() - c0; cyc[1] = c1 - c0; cyc[2] = c2 - c0; cyc[3] = c3 - c0; }
}

int main() {
  const int nwords = 4096;
  uint32_t h[nwords] = {};
  unsigned s = 12345;
  int nb = 0;
  while (nb < 4096) {
    s = s * 1103515245u + 12345u;
    const int b = (s >> 8) % (nwords * 32);
    if (!(h[b / 32] >> (b % 32) & 1)) { h[b / 32] |= 1u << (b % 32); ++nb; }
  }
  uint32_t* d; int* o; long long* cyc;
  cudaMalloc(&d, sizeof(h)); cudaMalloc(&o, 8192 * 4); cudaMalloc(&cyc, 32);
  cudaMemcpy(d, h, sizeof(h), cudaMemcpyHostToDevice);
  for (int v = 0; v < 2; ++v) {
    for (int r = 0; r < 3; ++r) {
      if (v == 0) emit_warp_rounds<<<1, 64>>>(d, nwords, o, cyc);
      else emit_chunks<<<1, 64>>>(d, nwords, o, cyc);
      long long cc[4]; cudaMemcpy(cc, cyc, 32, cudaMemcpyDeviceToHost); long long c = cc[0];
      if (v == 1) printf("  count %lld  emit-to-smem %lld  bar %lld\n", cc[1], cc[2], cc[3]);
      int first[4]; cudaMemcpy(first, o, 16, cudaMemcpyDeviceToHost);
      printf("variant %d rep %d: %lld cycles (first ids %d %d %d)\n", v, r, c, first[0], first[1], first[2]);
    }
  }
  return 0;
}
