// Micro-benchmark of the finisher's emission building blocks (64 threads).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ int bm_pad(int w) { return w + (w >> 6) * 4; }

template <int MODE>
__global__ void k(const uint32_t* gbm, int nwords, int* out, long long* cyc) {
  __shared__ __align__(16) uint32_t bmp[64 * 68];
  __shared__ uint32_t stg[4096 + 64];
  __shared__ uint32_t scan[64];
  __shared__ uint32_t tab[32];
  const int et = threadIdx.x, lane = et & 31, ew = et >> 5;
  if (et < 32) tab[(0x077CB531u << et) >> 27] = et;
  for (int i = et; i < nwords; i += 64) bmp[bm_pad(i)] = gbm[i];
  __syncthreads();
  const long long c0 = clock64();
  uint32_t cnt = 0;
  for (int qq = 0; qq < 4; ++qq) {
    const uint4* src = reinterpret_cast<const uint4*>(bmp + et * 68 + qq * 16);
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      const uint4 x = src[v];
      cnt += __popc(x.x) + __popc(x.y) + __popc(x.z) + __popc(x.w);
    }
  }
  uint32_t incl = cnt;
  for (int off = 1; off < 32; off <<= 1) {
    const uint32_t t = __shfl_up_sync(0xffffffffu, incl, off);
    if (lane >= off) incl += t;
  }
  if (lane == 31) scan[ew] = incl;
  __syncthreads();
  const long long c1 = clock64();
  uint32_t pos = incl - cnt + (ew ? scan[0] : 0u);
  if (MODE >= 1) {
    for (int qq = 0; qq < 4; ++qq) {
      uint32_t wv[16];
      const uint4* src = reinterpret_cast<const uint4*>(bmp + et * 68 + qq * 16);
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        const uint4 x = src[v];
        wv[4 * v] = x.x; wv[4 * v + 1] = x.y; wv[4 * v + 2] = x.z; wv[4 * v + 3] = x.w;
      }
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        uint32_t m = wv[i];
        const uint32_t base = (uint32_t)(et * 64 + qq * 16 + i) * 32u;
        if (MODE == 1) {
#pragma unroll
          for (int u = 0; u < 2; ++u)
            if (m) { stg[pos++] = base + (uint32_t)(__ffs(m) - 1); m &= m - 1; }
          while (m) { stg[pos++] = base + (uint32_t)(__ffs(m) - 1); m &= m - 1; }
        } else if (MODE == 4) {
          const uint32_t sb = (uint32_t)__cvta_generic_to_shared(stg);
          while (m) {
            const uint32_t v = base + (uint32_t)(__ffs(m) - 1);
            asm volatile("st.shared.u32 [%0], %1;" :: "r"(sb + 4u * pos), "r"(v) : "memory");
            ++pos; m &= m - 1;
          }
        } else if (MODE == 6) {
          const uint32_t sb = (uint32_t)__cvta_generic_to_shared(stg);
          const uint32_t a = sb + 4u * pos;
          const uint32_t m1 = m & (m - 1u), m2 = m1 & (m1 - 1u), m3 = m2 & (m2 - 1u);
          uint32_t m4 = m3 & (m3 - 1u);
          asm volatile("{.reg .pred p; setp.ne.u32 p, %2, 0; @p st.shared.u32 [%0], %1;}" :: "r"(a), "r"(base + (uint32_t)(__ffs(m) - 1)), "r"(m) : "memory");
          asm volatile("{.reg .pred p; setp.ne.u32 p, %2, 0; @p st.shared.u32 [%0], %1;}" :: "r"(a + 4u), "r"(base + (uint32_t)(__ffs(m1) - 1)), "r"(m1) : "memory");
          asm volatile("{.reg .pred p; setp.ne.u32 p, %2, 0; @p st.shared.u32 [%0], %1;}" :: "r"(a + 8u), "r"(base + (uint32_t)(__ffs(m2) - 1)), "r"(m2) : "memory");
          asm volatile("{.reg .pred p; setp.ne.u32 p, %2, 0; @p st.shared.u32 [%0], %1;}" :: "r"(a + 12u), "r"(base + (uint32_t)(__ffs(m3) - 1)), "r"(m3) : "memory");
          uint32_t p2 = pos + 4u;
          pos += __popc(m);
          while (m4) {
            asm volatile("st.shared.u32 [%0], %1;" :: "r"(sb + 4u * p2), "r"(base + (uint32_t)(__ffs(m4) - 1)) : "memory");
            ++p2; m4 &= m4 - 1u;
          }
        } else if (MODE == 7) {
          const uint32_t sb = (uint32_t)__cvta_generic_to_shared(stg);
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const uint32_t lb = m & (0u - m);
            m ^= lb;
            const uint32_t j = tab[(lb * 0x077CB531u) >> 27];
            asm volatile("{.reg .pred p; setp.ne.u32 p, %2, 0; @p st.shared.u32 [%0], %1;}" :: "r"(sb + 4u * pos), "r"(base + j), "r"(lb) : "memory");
            pos += lb != 0u;
          }
          while (m) {
            const uint32_t lb = m & (0u - m);
            m ^= lb;
            asm volatile("st.shared.u32 [%0], %1;" :: "r"(sb + 4u * pos), "r"(base + tab[(lb * 0x077CB531u) >> 27]) : "memory");
            ++pos;
          }
        } else if (MODE == 5) {
          while (m) { out[pos++] = base + (uint32_t)(__ffs(m) - 1); m &= m - 1; }
        } else if (MODE == 2) {
          while (m) { const uint32_t lb = m & (0u - m); stg[pos++] = base + __popc(lb - 1u); m ^= lb; }
        } else {  // MODE 3: no stores, just count iterations
          while (m) { pos += 1; m &= m - 1; }
        }
      }
    }
  }
  const long long c2 = clock64();
  __syncthreads();
  for (int i = et; i < 4096; i += 64) out[i] = stg[i];
  __syncthreads();
  if (et == 0) { cyc[0] = c1 - c0; cyc[1] = c2 - c1; cyc[2] = clock64() - c0; cyc[3] = pos; }
}

int main() {
  const int nwords = 4096;
  static uint32_t h[nwords] = {};
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
  for (int mode = 0; mode < 8; ++mode)
    for (int r = 0; r < 2; ++r) {
      switch (mode) {
        case 0: k<0><<<1, 64>>>(d, nwords, o, cyc); break;
        case 1: k<1><<<1, 64>>>(d, nwords, o, cyc); break;
        case 2: k<2><<<1, 64>>>(d, nwords, o, cyc); break;
        case 3: k<3><<<1, 64>>>(d, nwords, o, cyc); break;
        case 4: k<4><<<1, 64>>>(d, nwords, o, cyc); break;
        case 7: k<7><<<1, 64>>>(d, nwords, o, cyc); break;
        case 6: k<6><<<1, 64>>>(d, nwords, o, cyc); break;
        case 5: k<5><<<1, 64>>>(d, nwords, o + 4096, cyc); break;
      }
      long long c[4]; cudaMemcpy(c, cyc, 32, cudaMemcpyDeviceToHost);
      int f[3]; cudaMemcpy(f, o, 12, cudaMemcpyDeviceToHost);
      printf("mode %d: count+scan %lld  emit %lld  total %lld  (first %d %d %d)\n", mode, c[0], c[1], c[2], f[0], f[1], f[2]);
    }
  return 0;
}
