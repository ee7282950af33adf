// epsm_long.cuh -- sm_100a kernels for long patterns at EPSMc's sampling stride.
//
// EPSMc (Fig. 1 lines 1-13) hashes one 16-byte text block every
// (floor(m/16) - 1) * 16 bytes and naively checks the starts that the
// block's fingerprint names through the table L of the pattern's 16-byte substrings.
// A sampled 16-byte block costs a whole 128-byte line of DRAM traffic on B200 (measured: 1 GiB
// of reads for L = 112), so the path starts at m = 208 (L = 192): 53% of the text read at
// m = 256, 13% at m = 1024, 3% at m = 4096 (shorter long patterns keep the
// full-text sampled kernel).
//
// Every start s is examined exactly once, through the FIRST sampled block at or after it,
// x = ceil(s / L) * L: the block [x, x + 16) lies inside the window because L <= m - 16, and the
// table holds the pattern's substrings at offsets j = x - s in [0, L) (R17).  The
// starts of one block come out in ascending order (the table lists each bucket's offsets in
// descending j), and blocks are visited in text order, so positions are written sorted.
//
// Kernels (host: epsm_long.cu), per search:
//   1. epsm_long_count_kernel   per chunk of 1024 samples: matches (bitmap -> bucket -> check);
//   2. epsm_long_scan_kernel    exclusive prefix over the chunks, occ;
//   3. epsm_long_write_kernel   chunks with matches again: positions at prefix + rank.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "epsm_ptx.cuh"

namespace epsm {
namespace lg {

constexpr int kThreads = 256;
constexpr int kPerThread = 8;                       // consecutive samples per thread
constexpr int kChunk = kThreads * kPerThread;       // samples per chunk
constexpr int kBitmapWords = 2048;                  // 2^16-bit two-probe filter
constexpr int kBucketLog = 12;
constexpr int kMaxEnt = 4096;                       // offsets j < L <= 4080

// The pattern's table (host-built at plan time, device copy per plan).
struct __align__(16) LongDesc {
  uint32_t bitmap[kBitmapWords];
  uint16_t boff[(1 << kBucketLog) + 8];             // CSR offsets of the buckets into ent
  uint16_t ent[kMaxEnt];                            // j << 4 | 4-bit fingerprint, descending j
};

struct LParams {
  const uint8_t* text;          // 16-byte aligned virtual base
  uint64_t nbytes;              // readable bytes from text
  uint64_t s_lo, s_hi;          // valid virtual starts
  uint64_t pos_bias;            // reported = virtual start + pos_bias
  uint64_t nsamples;            // sampled blocks x = i * L, i < nsamples
  uint64_t nchunks;
  uint32_t L;                   // sampling stride (bytes, multiple of 16)
  uint32_t m;
  const LongDesc* desc;
  const uint32_t* dpat;         // zero-padded pattern words
  uint32_t* counts;             // [nchunks]
  unsigned long long* prefix;   // [nchunks]
  unsigned long long* occ;      // the search's occ
  uint64_t* pos;
  uint64_t cap;
};

__host__ __device__ __forceinline__ uint32_t long_hash(uint32_t w0, uint32_t w1, uint32_t w2, uint32_t w3) {
  return w0 * 0x9E3779B1u + w1 * 0x85EBCA77u + w2 * 0xC2B2AE3Du + w3 * 0x27D4EB2Fu;
}
__host__ __device__ __forceinline__ uint32_t long_bloom2(uint32_t h) { return (h ^ (h >> 15)) * 0x2C1B3C6Du; }

// only the bitmap goes to shared memory (8 KiB per CTA); the buckets are read through L1 on the
// rare bitmap hits
__device__ __forceinline__ void load_bitmap(uint32_t* bm, const LongDesc* src) {
  const uint4* s = reinterpret_cast<const uint4*>(src->bitmap);
  uint4* d = reinterpret_cast<uint4*>(bm);
  for (uint32_t i = threadIdx.x; i < kBitmapWords / 4; i += blockDim.x) d[i] = s[i];
  __syncthreads();
}

// the naive check of the window at virtual start s against the pattern, 16 words
// (64 bytes) per step with all of a step's loads issued first: a true match of m = 4096 costs
// 64 memory round trips, not 1024
__device__ __forceinline__ bool check_window(const LParams& P, uint64_t s) {
  constexpr uint32_t kStep = 16;
  const uint32_t* t32 = reinterpret_cast<const uint32_t*>(P.text);
  const uint64_t last_word = (P.nbytes - 1) >> 2;
  const uint32_t nw = (P.m + 3) >> 2;
  const uint32_t tail = (P.m & 3u) ? (0xFFFFFFFFu >> (8u * (4u - (P.m & 3u)))) : 0xFFFFFFFFu;
  const uint64_t w0 = s >> 2;
  const uint32_t sh = static_cast<uint32_t>(s & 3u) * 8u;
  for (uint32_t q0 = 0; q0 < nw; q0 += kStep) {
    uint32_t tw[kStep + 1], pw[kStep];
#pragma unroll
    for (uint32_t r = 0; r <= kStep; ++r) {
      const uint64_t wi = w0 + q0 + r;
      tw[r] = (q0 + r <= nw && wi <= last_word) ? __ldg(t32 + wi) : 0u;
    }
#pragma unroll
    for (uint32_t r = 0; r < kStep; ++r) pw[r] = q0 + r < nw ? __ldg(P.dpat + q0 + r) : 0u;
    uint32_t diff = 0;
#pragma unroll
    for (uint32_t r = 0; r < kStep; ++r) {
      const uint32_t q = q0 + r;
      const uint32_t pm = q + 1 < nw ? 0xFFFFFFFFu : (q + 1 == nw ? tail : 0u);
      diff |= (__funnelshift_r(tw[r], tw[r + 1], sh) ^ pw[r]) & pm;
    }
    if (diff) return false;
  }
  return true;
}

// The matches named by sample i (block at x = i*L): calls emit(s) for every matching start, in
// ascending order.  Returns their number.
template <class Emit>
__device__ __forceinline__ uint32_t sample_matches(const LParams& P, const uint32_t* bm, uint64_t i, uint4 blk,
                                                   Emit&& emit) {
  const uint32_t h = long_hash(blk.x, blk.y, blk.z, blk.w);
  const uint32_t h2 = long_bloom2(h);
  const uint32_t b1 = bm[h >> 21] >> ((h >> 16) & 31u);
  const uint32_t b2 = bm[h2 >> 21] >> ((h2 >> 16) & 31u);
  if (((b1 & b2) & 1u) == 0) return 0;
  const LongDesc& D = *P.desc;
  const uint64_t x = i * P.L;
  const uint32_t bk = h >> (32 - kBucketLog), fp = (h >> 16) & 15u;
  uint32_t n = 0;
  const uint32_t e1 = __ldg(&D.boff[bk + 1]);
  for (uint32_t e = __ldg(&D.boff[bk]); e < e1; ++e) {
    const uint32_t v = __ldg(&D.ent[e]);
    if ((v & 15u) != fp) continue;
    const uint32_t j = v >> 4;
    if (j > x) continue;
    const uint64_t s = x - j;
    if (s < P.s_lo || s >= P.s_hi) continue;
    if (check_window(P, s)) {
      emit(s);
      ++n;
    }
  }
  return n;
}

__device__ __forceinline__ uint4 load_block(const LParams& P, uint64_t i) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(P.text + i * P.L));
  return v;
}

__global__ void __launch_bounds__(kThreads) epsm_long_count_kernel(const __grid_constant__ LParams P) {
  __shared__ __align__(16) uint32_t bm[kBitmapWords];
  __shared__ uint32_t wsum[kThreads / 32];
  load_bitmap(bm, P.desc);
  const uint32_t lane = threadIdx.x & 31u, w = threadIdx.x >> 5;
  for (uint64_t c = blockIdx.x; c < P.nchunks; c += gridDim.x) {
    const uint64_t i0 = c * kChunk + threadIdx.x * kPerThread;
    uint4 blk[kPerThread];
#pragma unroll
    for (int k = 0; k < kPerThread; ++k)              // all loads in flight first
      if (i0 + k < P.nsamples) blk[k] = load_block(P, i0 + k);
    uint32_t cnt = 0;
#pragma unroll
    for (int k = 0; k < kPerThread; ++k)
      if (i0 + k < P.nsamples) cnt += sample_matches(P, bm, i0 + k, blk[k], [](uint64_t) {});
    cnt = __reduce_add_sync(0xffffffffu, cnt);
    if (lane == 0) wsum[w] = cnt;
    __syncthreads();
    if (threadIdx.x < 32) {
      uint32_t t = lane < kThreads / 32 ? wsum[lane] : 0u;
      t = __reduce_add_sync(0xffffffffu, t);
      if (lane == 0) P.counts[c] = t;
    }
    __syncthreads();
  }
}

// exclusive prefix over the chunk counts (one block), and occ
__global__ void __launch_bounds__(1024) epsm_long_scan_kernel(const __grid_constant__ LParams P) {
  __shared__ unsigned long long ws[32];
  __shared__ unsigned long long carry_s;
  const uint32_t lane = threadIdx.x & 31u, w = threadIdx.x >> 5;
  unsigned long long carry = 0;
  for (uint64_t c0 = 0; c0 < P.nchunks; c0 += 1024) {
    const uint64_t c = c0 + threadIdx.x;
    const unsigned long long v = c < P.nchunks ? P.counts[c] : 0ull;
    unsigned long long x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned long long y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= static_cast<uint32_t>(o)) x += y;
    }
    if (lane == 31) ws[w] = x;
    __syncthreads();
    if (w == 0) {
      const unsigned long long s0 = ws[lane];
      unsigned long long t = s0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long y = __shfl_up_sync(0xffffffffu, t, o);
        if (lane >= static_cast<uint32_t>(o)) t += y;
      }
      ws[lane] = t - s0;
      if (lane == 31) carry_s = t;
    }
    __syncthreads();
    if (c < P.nchunks) P.prefix[c] = carry + ws[w] + (x - v);
    carry += carry_s;
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    griddep_wait();                                     // (the previous grid may write the same occ)
    *P.occ = carry;
  }
}

__global__ void __launch_bounds__(kThreads) epsm_long_write_kernel(const __grid_constant__ LParams P) {
  __shared__ __align__(16) uint32_t bm[kBitmapWords];
  __shared__ uint32_t wsum[kThreads / 32];
  bool loaded = false;
  const uint32_t lane = threadIdx.x & 31u, w = threadIdx.x >> 5;
  for (uint64_t c = blockIdx.x; c < P.nchunks; c += gridDim.x) {
    if (P.counts[c] == 0) continue;                   // (block-uniform)
    const unsigned long long base = P.prefix[c];
    if (base >= P.cap) continue;
    if (!loaded) {
      load_bitmap(bm, P.desc);
      loaded = true;
    }
    const uint64_t i0 = c * kChunk + threadIdx.x * kPerThread;
    uint4 blk[kPerThread];
#pragma unroll
    for (int k = 0; k < kPerThread; ++k)
      if (i0 + k < P.nsamples) blk[k] = load_block(P, i0 + k);
    uint32_t cnt = 0;
#pragma unroll
    for (int k = 0; k < kPerThread; ++k)
      if (i0 + k < P.nsamples) cnt += sample_matches(P, bm, i0 + k, blk[k], [](uint64_t) {});
    // exclusive offset of this thread's matches inside the chunk (text order = thread order)
    uint32_t incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= static_cast<uint32_t>(o)) incl += y;
    }
    if (lane == 31) wsum[w] = incl;
    __syncthreads();
    uint32_t woff = 0;
    for (uint32_t q = 0; q < w; ++q) woff += wsum[q];
    uint64_t g = base + woff + incl - cnt;
    if (cnt) {
      griddep_wait();                                   // (outputs of the previous grid)
#pragma unroll
      for (int k = 0; k < kPerThread; ++k)
        if (i0 + k < P.nsamples)
          sample_matches(P, bm, i0 + k, blk[k], [&](uint64_t s) {
            if (g < P.cap) P.pos[g] = s + P.pos_bias;
            ++g;
          });
    }
    __syncthreads();
  }
}

}  // namespace lg
}  // namespace epsm
