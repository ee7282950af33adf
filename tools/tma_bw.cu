// Microbenchmark: read bandwidth of (a) a persistent TMA bulk-copy ring with
// consumers that only touch the data lightly, (b) a plain LDG.128 grid-stride read.
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int TILE, int STAGES, int CW>
__global__ void __launch_bounds__((CW + 1) * 32, 1) tma_ring(const uint8_t* __restrict__ src, uint64_t n, uint32_t* out) {
  extern __shared__ __align__(128) uint8_t sm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + STAGES * TILE);
  uint64_t* empty = full + STAGES;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&full[s])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(&empty[s])), "r"(CW));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const uint64_t ntiles = n / TILE;
  if (warp == 0) {
    uint32_t st = 0, ph = 0;
    for (uint64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
      asm volatile("{.reg .pred P; W: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1; @!P bra W;}" ::"r"(sa(&empty[st])), "r"(ph ^ 1) : "memory");
      if (lane == 0) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&full[st])), "r"(TILE) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     ::"r"(sa(sm + st * TILE)), "l"(src + t * TILE), "r"(TILE), "r"(sa(&full[st])) : "memory");
      }
      if (++st == STAGES) { st = 0; ph ^= 1; }
    }
  } else {
    uint32_t st = 0, ph = 0, acc = 0;
    const int c = tid - 32;
    for (uint64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
      asm volatile("{.reg .pred P; W: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1; @!P bra W;}" ::"r"(sa(&full[st])), "r"(ph) : "memory");
      const uint4* p = reinterpret_cast<const uint4*>(sm + st * TILE);
      for (int i = c; i < TILE / 16; i += CW * 32) { uint4 v = p[i]; acc ^= v.x ^ v.y ^ v.z ^ v.w; }
      __syncwarp();
      if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(&empty[st])) : "memory");
      if (++st == STAGES) { st = 0; ph ^= 1; }
    }
    if (acc == 0x12345678u) out[0] = acc;
  }
}

// two "planes" per stage: copies of TILE/2 + 16 bytes from two distant regions at a 16-byte
// (not 128-byte) offset, as the index variant streams them
template <int TILE, int STAGES, int CW>
__global__ void __launch_bounds__((CW + 1) * 32, 1) tma_ring2(const uint8_t* __restrict__ src, uint64_t n, uint32_t* out) {
  extern __shared__ __align__(128) uint8_t sm[];
  constexpr int SB = TILE + 32;
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + STAGES * SB);
  uint64_t* empty = full + STAGES;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&full[s])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(&empty[s])), "r"(CW));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const uint64_t half = n / 2;
  const uint64_t ntiles = (half - 4096) / (TILE / 2);
  if (warp == 0) {
    uint32_t st = 0, ph = 0;
    for (uint64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
      asm volatile("{.reg .pred P; W: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1; @!P bra W;}" ::"r"(sa(&empty[st])), "r"(ph ^ 1) : "memory");
      if (lane == 0) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&full[st])), "r"(TILE + 32) : "memory");
        for (int k = 0; k < 2; ++k)
          asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                       ::"r"(sa(sm + st * SB + k * (TILE / 2 + 16))), "l"(src + k * half + 16 + t * (TILE / 2)), "r"(TILE / 2 + 16), "r"(sa(&full[st])) : "memory");
      }
      if (++st == STAGES) { st = 0; ph ^= 1; }
    }
  } else {
    uint32_t st = 0, ph = 0, acc = 0;
    const int c = tid - 32;
    for (uint64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
      asm volatile("{.reg .pred P; W: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1; @!P bra W;}" ::"r"(sa(&full[st])), "r"(ph) : "memory");
      const uint2* p = reinterpret_cast<const uint2*>(sm + st * SB);
      acc ^= p[c].x ^ p[c + 514].y;
      __syncwarp();
      if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(&empty[st])) : "memory");
      if (++st == STAGES) { st = 0; ph ^= 1; }
    }
    if (acc == 0x12345678u) out[0] = acc;
  }
}

template <int TILE, int STAGES, int CW>
void run_tma2(const uint8_t* d, uint64_t n, uint32_t* o, int sms) {
  auto k = tma_ring2<TILE, STAGES, CW>;
  size_t smem = STAGES * (TILE + 32) + 2 * STAGES * 8;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int it = 0; it < 3; ++it) k<<<sms, (CW + 1) * 32, smem>>>(d, n, o);
  cudaEventRecord(a);
  const int R = 10;
  for (int it = 0; it < R; ++it) k<<<sms, (CW + 1) * 32, smem>>>(d, n, o);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  printf("tma2 (2 planes) tile=%6d stages=%2d : %8.1f GB/s  (%s)\n", TILE, STAGES,
         (n - 8192) * (double)R / (ms * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
}

__global__ void ldg_read(const uint4* __restrict__ src, uint64_t n16, uint32_t* out) {
  uint32_t acc = 0;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n16; i += (uint64_t)gridDim.x * blockDim.x) {
    uint4 v = __ldcs(src + i); acc ^= v.x ^ v.y ^ v.z ^ v.w;
  }
  if (acc == 0x12345678u) out[0] = acc;
}

template <int TILE, int STAGES, int CW>
void run_tma(const uint8_t* d, uint64_t n, uint32_t* o, int sms, int ctas_per_sm) {
  auto k = tma_ring<TILE, STAGES, CW>;
  size_t smem = STAGES * TILE + 2 * STAGES * 8;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int it = 0; it < 3; ++it) k<<<sms * ctas_per_sm, (CW + 1) * 32, smem>>>(d, n, o);
  cudaEventRecord(a);
  const int R = 10;
  for (int it = 0; it < R; ++it) k<<<sms * ctas_per_sm, (CW + 1) * 32, smem>>>(d, n, o);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  printf("tma tile=%6d stages=%d cw=%2d ctas/sm=%d : %8.1f GB/s  (%s)\n", TILE, STAGES, CW, ctas_per_sm,
         n * (double)R / (ms * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
}

int main(int argc, char** argv) {
  const uint64_t n = argc > 1 ? strtoull(argv[1], 0, 0) : (1ull << 30);
  uint8_t* d; uint32_t* o;
  cudaMalloc(&d, n); cudaMalloc(&o, 64); cudaMemset(d, 1, n);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run_tma<32768, 4, 16>(d, n, o, sms, 1);
  run_tma<32768, 5, 16>(d, n, o, sms, 1);
  run_tma<32768, 6, 16>(d, n, o, sms, 1);
  run_tma<16384, 8, 16>(d, n, o, sms, 1);
  run_tma<16384, 12, 16>(d, n, o, sms, 1);
  run_tma<16384, 6, 8>(d, n, o, sms, 2);
  run_tma<8192, 12, 8>(d, n, o, sms, 2);
  run_tma<65536, 3, 16>(d, n, o, sms, 1);
  // small stages (the index variant streams 2 planes x 4 KiB per 32K-position tile)
  run_tma<8192, 5, 16>(d, n, o, sms, 1);
  run_tma<8192, 10, 16>(d, n, o, sms, 1);
  run_tma<8192, 20, 16>(d, n, o, sms, 1);
  run_tma<16384, 10, 16>(d, n, o, sms, 1);
  run_tma2<8192, 5, 16>(d, n, o, sms);
  run_tma2<8192, 10, 16>(d, n, o, sms);
  run_tma2<32768, 5, 16>(d, n, o, sms);
  {
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    for (int bs : {256, 512, 1024}) for (int per : {4, 8}) {
      int grid = sms * (2048 / bs) * per / 4;
      for (int it = 0; it < 3; ++it) ldg_read<<<grid, bs>>>((const uint4*)d, n / 16, o);
      cudaEventRecord(a);
      for (int it = 0; it < 10; ++it) ldg_read<<<grid, bs>>>((const uint4*)d, n / 16, o);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      printf("ldg bs=%4d grid=%6d : %8.1f GB/s\n", bs, grid, n * 10.0 / (ms * 1e-3) / 1e9);
    }
  }
  return 0;
}
