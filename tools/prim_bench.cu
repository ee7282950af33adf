// Microbenchmark: SM-wide throughput of the warp primitives a group-search ranking can be built
// from (match.any, shared atomics, private shared counters, random / lane-replicated byte tables).
// Prints warp-instructions per SM clock for each.  nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kIters = 4096;

__device__ __forceinline__ uint32_t rnd(uint32_t& s) {
  s = s * 1664525u + 1013904223u;
  return s >> 8;
}

template <int MODE>
__global__ void __launch_bounds__(512) prim(uint32_t* out, uint32_t nid) {
  __shared__ __align__(16) uint8_t tab[32768];
  __shared__ uint32_t cnt[512];
  const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
  for (uint32_t i = threadIdx.x; i < 32768; i += blockDim.x) tab[i] = static_cast<uint8_t>(i * 7u);
  for (uint32_t i = threadIdx.x; i < 512; i += blockDim.x) cnt[i] = 0;
  __syncthreads();
  uint32_t s = threadIdx.x * 747796405u + blockIdx.x, acc = 0;
#pragma unroll 8
  for (int it = 0; it < kIters; ++it) {
    const uint32_t r = rnd(s);
    const uint32_t id = r & (nid - 1u);
    if constexpr (MODE == 0) {            // match.any on ids
      acc += __match_any_sync(0xffffffffu, id);
    } else if constexpr (MODE == 1) {     // shared atomics, spread
      atomicAdd(&cnt[id & 511u], 1u);
    } else if constexpr (MODE == 2) {     // LDS.U8 random in a 16 KB table
      acc += tab[r & 16383u];
    } else if constexpr (MODE == 3) {     // LDS.U8 lane-replicated (b * 32 + lane), 8 KB
      acc += tab[((r & 255u) << 5) | lane];
    } else if constexpr (MODE == 4) {     // private byte counter per (id, lane): LDS.U8 + STS.U8
      uint8_t* p = &tab[((id & 255u) << 5) | lane];
      *p = static_cast<uint8_t>(*p + 1);
    } else if constexpr (MODE == 5) {     // ballot x8 + lop (multisplit rank on 8 id bits)
      uint32_t eq = 0xffffffffu;
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const uint32_t b = __ballot_sync(0xffffffffu, (id >> k) & 1u);
        eq &= ((id >> k) & 1u) ? b : ~b;
      }
      acc += __popc(eq & ((1u << lane) - 1u));
    } else if constexpr (MODE == 6) {     // baseline: the rnd loop only
      acc += id;
    } else if constexpr (MODE == 7) {     // LDS.U8 random in a 256 B table
      acc += tab[r & 255u];
    } else if constexpr (MODE == 8) {     // shared atomics with the old value used (ATOMS)
      acc += atomicAdd(&cnt[id & 511u], 1u);
    } else if constexpr (MODE == 9) {     // shared atomics, 40% of lanes active
      if ((r >> 20) % 5u < 2u) atomicAdd(&cnt[id & 511u], 1u);
    }
  }
  if (acc == 0x12345678u) out[0] = acc + cnt[lane] + tab[warp];
}

template <int MODE>
void run(const char* name, uint32_t nid) {
  uint32_t* out;
  cudaMalloc(&out, 4);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  prim<MODE><<<148, 512>>>(out, nid);
  cudaEventRecord(a);
  prim<MODE><<<148, 512>>>(out, nid);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  int clk;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const double clocks = ms * 1e-3 * clk * 1e3;
  const double ops_per_sm = 16.0 * kIters;   // warp-ops per SM
  printf("%-28s nid=%4u  %8.3f ms  %6.2f clk per warp-op per SM\n", name, nid, ms, clocks / ops_per_sm);
  cudaFree(out);
}

int main() {
  run<6>("baseline rnd", 128);
  run<8>("atomicAdd shared, old used", 128);
  run<9>("atomicAdd shared 40% lanes", 128);
  run<1>("atomicAdd shared spread", 8);
  run<0>("match.any", 128);
  run<0>("match.any", 8);
  run<1>("atomicAdd shared spread", 128);
  run<2>("LDS.U8 random 16KB", 128);
  run<7>("LDS.U8 random 256B", 128);
  run<3>("LDS.U8 replicated b*32+l", 128);
  run<4>("private ctr LDS+STS", 128);
  run<5>("ballot x8 multisplit", 128);
  return 0;
}
