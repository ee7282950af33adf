// Microbenchmark: HBM write bandwidth of fan-out styles (one source chunk written to K outputs).
//   bulk: a 32 KiB shared-memory chunk leaves as one cp.async.bulk store per output (the
//         replicate kernel's style), CHUNK-sized pieces, K outputs per chunk;
//   reg:  each warp holds 512 B of the chunk in registers and stores it with st.global.v4
//         (coalesced) to each of the K outputs;
//   fill: plain st.global.v4 of a constant over one buffer (the write ceiling).
// Prints TB/s of bytes written.  nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t sa(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

template <int CHUNK>
__global__ void __launch_bounds__(128) bulk_fan(uint8_t* const* outs, int K, uint64_t bytes_per_out) {
  extern __shared__ __align__(128) uint8_t buf[];
  for (int i = threadIdx.x; i < CHUNK / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(buf)[i] = make_uint4(i, i + 1, i + 2, i + 3);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  const uint64_t nch = bytes_per_out / CHUNK;
  if (threadIdx.x == 0) {
    for (uint64_t c = blockIdx.x; c < nch; c += gridDim.x) {
      for (int k = 0; k < K; ++k)
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(outs[k] + c * CHUNK),
                     "r"(sa(buf)), "r"(CHUNK)
                     : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      asm volatile("cp.async.bulk.wait_group.read 2;" ::: "memory");
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
}

__global__ void __launch_bounds__(256) reg_fan(uint8_t* const* outs, int K, uint64_t bytes_per_out) {
  // each thread: 16 B per 4 KiB block row, block of 256 threads covers 4 KiB per step
  const uint64_t step = static_cast<uint64_t>(gridDim.x) * 4096;
  for (uint64_t base = static_cast<uint64_t>(blockIdx.x) * 4096; base < bytes_per_out; base += step) {
    const uint4 v = make_uint4(base, base + 1, threadIdx.x, 7);
    for (int k = 0; k < K; ++k) {
      uint4* d = reinterpret_cast<uint4*>(outs[k] + base) + threadIdx.x;
      asm volatile("st.global.cs.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(d), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
                   : "memory");
    }
  }
}

__global__ void __launch_bounds__(256) fill(uint4* p, uint64_t n16) {
  for (uint64_t i = blockIdx.x * 256ull + threadIdx.x; i < n16; i += gridDim.x * 256ull) p[i] = make_uint4(1, 2, 3, 4);
}

int main() {
  const uint64_t total = 24ull << 30;                 // bytes written per run
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  uint8_t* pool;
  if (cudaMalloc(&pool, total) != cudaSuccess) { printf("alloc failed\n"); return 1; }
  uint8_t** d_outs;
  cudaMalloc(&d_outs, 64 * sizeof(uint8_t*));
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  auto timeit = [&](auto fn) {
    fn();
    cudaEventRecord(a);
    for (int r = 0; r < 3; ++r) fn();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    return 3.0 * total / (ms * 1e-3) / 1e12;
  };
  printf("fill                 %.2f TB/s\n",
         timeit([&] { fill<<<sms * 8, 256>>>(reinterpret_cast<uint4*>(pool), total / 16); }));
  for (int K : {1, 4, 8, 24}) {
    const uint64_t per = total / K / 32768 * 32768;
    uint8_t* h[64];
    for (int k = 0; k < K; ++k) h[k] = pool + k * per;
    cudaMemcpy(d_outs, h, K * sizeof(uint8_t*), cudaMemcpyHostToDevice);
    cudaFuncSetAttribute(bulk_fan<32768>, cudaFuncAttributeMaxDynamicSharedMemorySize, 32768);
    for (int cps : {1, 2, 4}) {
      const double tb = timeit([&] { bulk_fan<32768><<<sms * cps, 128, 32768>>>(d_outs, K, per); }) * (double)(per * K) / total;
      printf("bulk K=%2d ctas/sm=%d  %.2f TB/s\n", K, cps, tb);
    }
    for (int cps : {2, 8}) {
      const double tb = timeit([&] { reg_fan<<<sms * cps, 256>>>(d_outs, K, per); }) * (double)(per * K) / total;
      printf("reg  K=%2d ctas/sm=%d  %.2f TB/s\n", K, cps, tb);
    }
  }
  return 0;
}
