// gather_bench.cu -- throughput of the sparse heads' access pattern on B200:
// tiles of 64 token rows of K and V (256 B per row, bf16 d = 128) gathered
// from sorted random row ids into a shared-memory ring, with three copy paths:
//   mode 0: 16-B cp.async (LDGSTS) by P producer threads  (the step kernel's path)
//   mode 1: one 256-B cp.async.bulk per row (TMA engine), rows spread over P threads
//   mode 2: LDG.128 into registers by all threads (no shared memory)
// Two sizes: one sparse layer (8 heads x 64 tiles = 512 tiles, latency-bound)
// and 64 such layers back to back (throughput).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/gather_bench scripts/micro/gather_bench.cu
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <vector>

constexpr int kTile = 64, kRowBytes = 256, kStages = 4;
constexpr int kTileBytes = 2 * kTile * kRowBytes;  // K then V

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t ph) {
  asm volatile(
      "{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W;\n}" ::"r"(
          smem_u32(b)),
      "r"(ph)
      : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_expect(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes)
               : "memory");
}

template <int MODE, int P>
__global__ void __launch_bounds__(P + 32) gather_kernel(const uint8_t* __restrict__ K,
                                                        const uint8_t* __restrict__ V,
                                                        const int32_t* __restrict__ ids, int n_tiles,
                                                        int tiles_per_head, int64_t head_rows,
                                                        uint32_t* sink) {
  extern __shared__ __align__(128) uint8_t ring[];
  __shared__ __align__(8) uint64_t full[kStages], empty[kStages];
  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], MODE == 0 ? P : 1);
      mbar_init(&empty[s], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  int stage = 0;
  uint32_t phase = 0;
  if (tid < P) {
    for (int t = blockIdx.x; t < n_tiles; t += gridDim.x) {
      const int head = (t / tiles_per_head) % 8, tile = t % tiles_per_head;
      const int32_t* tid_ids = ids + (int64_t)head * tiles_per_head * kTile + tile * kTile;
      const uint8_t* kb = K + head * head_rows * kRowBytes;
      const uint8_t* vb = V + head * head_rows * kRowBytes;
      mbar_wait(&empty[stage], phase ^ 1);
      uint8_t* dst = ring + stage * kTileBytes;
      if constexpr (MODE == 0) {
        for (int c = tid; c < 2 * kTile * 16; c += P) {  // (row, 16-B chunk) of K then V
          const int kv = c / (kTile * 16), r = (c / 16) % kTile, ch = c % 16;
          const int64_t row = __ldg(tid_ids + r);
          const uint8_t* src = (kv ? vb : kb) + row * kRowBytes + ch * 16;
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst + c * 16)),
                       "l"(src)
                       : "memory");
        }
        asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(&full[stage]))
                     : "memory");
      } else {
        if (tid == 0) mbar_expect(&full[stage], kTileBytes);
        asm volatile("bar.sync 1, %0;" ::"n"(P) : "memory");
        for (int c = tid; c < 2 * kTile; c += P) {
          const int kv = c / kTile, r = c % kTile;
          const int64_t row = __ldg(tid_ids + r);
          const uint8_t* src = (kv ? vb : kb) + row * kRowBytes;
          asm volatile(
              "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                  smem_u32(dst + c * kRowBytes)),
              "l"(src), "r"(kRowBytes), "r"(smem_u32(&full[stage]))
              : "memory");
        }
      }
      if (++stage == kStages) {
        stage = 0;
        phase ^= 1;
      }
    }
  } else {
    // one consumer warp: touch every row of the tile, release the stage
    uint32_t acc = 0;
    const int lane = tid - P;
    for (int t = blockIdx.x; t < n_tiles; t += gridDim.x) {
      mbar_wait(&full[stage], phase);
      const uint8_t* src = ring + stage * kTileBytes;
      for (int r = lane; r < 2 * kTile; r += 32) acc ^= *reinterpret_cast<const uint32_t*>(src + r * kRowBytes);
      __syncwarp();
      if (lane == 0 && acc != 0xdeadbeefu) mbar_arrive(&empty[stage]);
      if (++stage == kStages) {
        stage = 0;
        phase ^= 1;
      }
    }
    if (acc == 0x12345678u) sink[0] = acc;
  }
}

// mode 2: every thread streams 16-B chunks of the tile's rows into registers
__global__ void __launch_bounds__(256) ldg_kernel(const uint8_t* __restrict__ K, const uint8_t* __restrict__ V,
                                                  const int32_t* __restrict__ ids, int n_tiles,
                                                  int tiles_per_head, int64_t head_rows, uint32_t* sink) {
  uint32_t acc = 0;
  for (int t = blockIdx.x; t < n_tiles; t += gridDim.x) {
    const int head = (t / tiles_per_head) % 8, tile = t % tiles_per_head;
    const int32_t* tid_ids = ids + (int64_t)head * tiles_per_head * kTile + tile * kTile;
    const uint8_t* kb = K + head * head_rows * kRowBytes;
    const uint8_t* vb = V + head * head_rows * kRowBytes;
    uint4 v[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int c = threadIdx.x + i * 256;
      const int kv = c / (kTile * 16), r = (c / 16) % kTile, ch = c % 16;
      const int64_t row = __ldg(tid_ids + r);
      v[i] = __ldcs(reinterpret_cast<const uint4*>((kv ? vb : kb) + row * kRowBytes + ch * 16));
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) acc ^= v[i].x ^ v[i].w;
  }
  if (acc == 0x12345678u) sink[0] = acc;
}

int main() {
  const int H = 8, tiles_per_head = 64;
  const int64_t L = 131072;
  const size_t bytes = (size_t)H * L * kRowBytes;
  uint8_t *K, *V;
  int32_t* ids;
  uint32_t* sink;
  cudaMalloc(&K, bytes);
  cudaMalloc(&V, bytes);
  cudaMemset(K, 1, bytes);
  cudaMemset(V, 2, bytes);
  std::vector<int32_t> h((size_t)H * tiles_per_head * kTile);
  uint64_t s = 2602;
  for (int g = 0; g < H; ++g) {
    std::vector<int32_t> all(L);
    for (int64_t i = 0; i < L; ++i) all[i] = (int32_t)i;
    for (int64_t i = L - 1; i > 0; --i) {  // partial Fisher-Yates: a random 4096-subset
      s = s * 6364136223846793005ull + 1442695040888963407ull;
      std::swap(all[i], all[(s >> 33) % (i + 1)]);
    }
    std::sort(all.end() - tiles_per_head * kTile, all.end());
    std::copy(all.end() - tiles_per_head * kTile, all.end(), h.begin() + (size_t)g * tiles_per_head * kTile);
  }
  cudaMalloc(&ids, h.size() * 4);
  cudaMemcpy(ids, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
  cudaMalloc(&sink, 4);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int smem = kStages * kTileBytes;
  cudaFuncSetAttribute(gather_kernel<0, 64>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(gather_kernel<0, 128>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(gather_kernel<0, 256>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(gather_kernel<1, 64>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(gather_kernel<1, 128>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int layers : {1, 64}) {
    const int n_tiles = layers * H * tiles_per_head;
    auto run = [&](const char* name, auto launch) {
      for (int i = 0; i < 3; ++i) launch();
      cudaEventRecord(e0);
      const int reps = layers == 1 ? 200 : 10;
      for (int i = 0; i < reps; ++i) launch();
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms = 0.f;
      cudaEventElapsedTime(&ms, e0, e1);
      const double us = ms * 1e3 / reps;
      std::printf("layers %2d  %-34s %8.2f us  %7.0f GB/s\n", layers, name, us,
                  (double)n_tiles * kTileBytes / us / 1e3);
    };
    run("cp.async 16 B, 64 producers", [&] {
      gather_kernel<0, 64><<<sms, 96, smem>>>(K, V, ids, n_tiles, tiles_per_head, L, sink);
    });
    run("cp.async 16 B, 128 producers", [&] {
      gather_kernel<0, 128><<<sms, 160, smem>>>(K, V, ids, n_tiles, tiles_per_head, L, sink);
    });
    run("cp.async 16 B, 256 producers", [&] {
      gather_kernel<0, 256><<<sms, 288, smem>>>(K, V, ids, n_tiles, tiles_per_head, L, sink);
    });
    run("cp.async.bulk 256 B/row, 64 thr", [&] {
      gather_kernel<1, 64><<<sms, 96, smem>>>(K, V, ids, n_tiles, tiles_per_head, L, sink);
    });
    run("cp.async.bulk 256 B/row, 128 thr", [&] {
      gather_kernel<1, 128><<<sms, 160, smem>>>(K, V, ids, n_tiles, tiles_per_head, L, sink);
    });
    run("LDG.128 to registers, 256 thr x2/SM", [&] {
      ldg_kernel<<<2 * sms, 256>>>(K, V, ids, n_tiles, tiles_per_head, L, sink);
    });
  }
  const cudaError_t e = cudaDeviceSynchronize();
  std::printf("status: %s\n", cudaGetErrorString(e));
  return e == cudaSuccess ? 0 : 1;
}
