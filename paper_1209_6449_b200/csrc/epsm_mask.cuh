// epsm_mask.cuh -- the DENSE patterns of a group in one pass over the equality-mask index.
//
// EPSMa computes r = s_0 & (s_1 >> 1) & ... from the byte-equality masks
// s_j = wscmp(T_i, B[j]); the index holds those masks per byte value (planes), so every pattern
// of a set is a few ANDs of shifted plane words.  The group search sends its dense patterns
// (>= 2^-7 occurrences per text byte: short patterns over small alphabets -- their positions are
// the traffic) here when they fit: m <= 8, at most 8 distinct bytes among them, m * (distinct
// bytes) <= 16 shifted plane words, at most 64 patterns.  Per warp task of 128 plane words
// (8192 starts; a block = 8 tasks):
//   1. epsm_mask_count_kernel   the shifted planes of a round of 32 words go to shared memory,
//                               every pattern's mask is m loads + ANDs; per-task count per pattern;
//   2. epsm_mask_scan_kernel    per pattern: exclusive prefix over the tasks (text order) and occ;
//   3. epsm_mask_write_kernel   the masks again; a pattern's positions of a round are ranked by a
//                               warp scan over the lanes (text order) and stored at prefix + rank.
// Each pattern's FIRST search gets the positions; its duplicates are copied by the replicate
// kernel.  Every start in [0, nstarts) is bit s % 64 of plane word s / 64.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "epsm_ptx.cuh"

namespace epsm {
namespace mk {

constexpr int kWarps = 8;
constexpr int kThreads = 32 * kWarps;
constexpr int kRounds = 4;                          // 32-word rounds per warp task
constexpr int kTaskWords = 32 * kRounds;            // 128 words = 8192 starts per task
constexpr int kMaxVals = 8;                         // distinct bytes (planes)
constexpr int kMaxM = 8;
constexpr int kMaxSh = 16;                          // m * vals shifted words per lane
constexpr int kMaxD = 64;

struct MaskParams {
  const uint64_t* planes;
  uint64_t pstride;
  uint32_t nval, m, D, pad;
  uint32_t pid[kMaxVals];                           // plane of value slot s
  uint8_t sh[kMaxD][kMaxM];                         // shifted-word index (i * nval + slot) of byte i of pattern d
  uint64_t nstarts;
  uint64_t pos_bias;
  uint64_t nwords;
  uint64_t ntasks;
  uint16_t* counts;                                 // [D][ntasks]
  unsigned long long* prefix;                       // [D][ntasks]
  uint64_t* pos[kMaxD];                             // the first output of pattern d
  uint64_t cap[kMaxD];
  unsigned long long* occ[kMaxD];
};

// Round r of a task: the shifted plane words of this lane's word into SH[.][lane]; returns the
// word index (or ~0 past the text).
__device__ __forceinline__ uint64_t stage_round(const MaskParams& P, uint64_t task, int r, uint32_t lane,
                                                uint64_t (*SH)[32]) {
  const uint64_t w = task * kTaskWords + static_cast<uint64_t>(r) * 32 + lane;
  uint64_t lo[kMaxVals], hi[kMaxVals];
#pragma unroll
  for (int s = 0; s < kMaxVals; ++s) {
    if (s >= static_cast<int>(P.nval)) break;
    const uint64_t* pl = P.planes + static_cast<uint64_t>(P.pid[s]) * P.pstride;
    lo[s] = w <= P.nwords ? __ldg(pl + w) : 0ull;      // (word nwords: the last windows' tail)
  }
#pragma unroll
  for (int s = 0; s < kMaxVals; ++s) {
    if (s >= static_cast<int>(P.nval)) break;
    hi[s] = __shfl_down_sync(0xffffffffu, lo[s], 1);
    if (lane == 31) hi[s] = w < P.nwords ? __ldg(P.planes + static_cast<uint64_t>(P.pid[s]) * P.pstride + w + 1) : 0ull;
  }
#pragma unroll
  for (int i = 0; i < kMaxM; ++i) {
    if (i >= static_cast<int>(P.m)) break;
#pragma unroll
    for (int s = 0; s < kMaxVals; ++s) {
      if (s >= static_cast<int>(P.nval)) break;
      SH[i * P.nval + s][lane] = i ? ((lo[s] >> i) | (hi[s] << (64 - i))) : lo[s];
    }
  }
  __syncwarp();
  return w;
}

__device__ __forceinline__ uint64_t pattern_mask(const MaskParams& P, const uint8_t (*shs)[kMaxM], uint32_t d,
                                                 uint64_t w, uint32_t lane, uint64_t (*SH)[32]) {
  uint64_t M = ~0ull;
#pragma unroll
  for (int i = 0; i < kMaxM; ++i) {
    if (i >= static_cast<int>(P.m)) break;
    M &= SH[shs[d][i]][lane];
  }
  const uint64_t s0 = w * 64;
  if (s0 + 64 > P.nstarts) M &= P.nstarts > s0 ? (~0ull >> (64 - (P.nstarts - s0))) : 0ull;
  return M;
}

__device__ __forceinline__ void load_sh(const MaskParams& P, uint8_t (*shs)[kMaxM]) {
  for (uint32_t i = threadIdx.x; i < kMaxD * kMaxM; i += blockDim.x) (&shs[0][0])[i] = (&P.sh[0][0])[i];
  __syncthreads();
}

__global__ void __launch_bounds__(kThreads) epsm_mask_count_kernel(const __grid_constant__ MaskParams P) {
  __shared__ uint64_t SH[kWarps][kMaxSh][32];
  __shared__ uint8_t shs[kMaxD][kMaxM];
  load_sh(P, shs);
  const uint32_t lane = threadIdx.x & 31u, wp = threadIdx.x >> 5;
  for (uint64_t task = static_cast<uint64_t>(blockIdx.x) * kWarps + wp; task < P.ntasks;
       task += static_cast<uint64_t>(gridDim.x) * kWarps) {
    uint32_t cnt = 0;                                   // lane d (and d + 32): pattern d's count
    uint32_t cnt2 = 0;
    for (int r = 0; r < kRounds; ++r) {
      const uint64_t w = stage_round(P, task, r, lane, SH[wp]);
#pragma unroll 4
      for (uint32_t d = 0; d < P.D; ++d) {
        const uint32_t c = __reduce_add_sync(0xffffffffu, __popcll(pattern_mask(P, shs, d, w, lane, SH[wp])));
        if (lane == (d & 31u)) {
          if (d < 32) cnt += c;
          else cnt2 += c;
        }
      }
      __syncwarp();
    }
    if (lane < P.D) P.counts[static_cast<uint64_t>(lane) * P.ntasks + task] = static_cast<uint16_t>(cnt);
    if (lane + 32 < P.D) P.counts[static_cast<uint64_t>(lane + 32) * P.ntasks + task] = static_cast<uint16_t>(cnt2);
  }
}

// per pattern (block d): exclusive prefix over the tasks, and occ (the first search's slot)
__global__ void __launch_bounds__(1024) epsm_mask_scan_kernel(const __grid_constant__ MaskParams P) {
  __shared__ unsigned long long ws[32];
  __shared__ unsigned long long carry_s;
  const uint32_t lane = threadIdx.x & 31u, w = threadIdx.x >> 5;
  const uint32_t d = blockIdx.x;
  const uint16_t* row = P.counts + static_cast<uint64_t>(d) * P.ntasks;
  unsigned long long* prow = P.prefix + static_cast<uint64_t>(d) * P.ntasks;
  unsigned long long carry = 0;
  for (uint64_t c0 = 0; c0 < P.ntasks; c0 += 1024) {
    const uint64_t c = c0 + threadIdx.x;
    const unsigned long long v = c < P.ntasks ? row[c] : 0ull;
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
    if (c < P.ntasks) prow[c] = carry + ws[w] + (x - v);
    carry += carry_s;
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    griddep_wait();
    *P.occ[d] = carry;
  }
}

// a lane's run of positions: the set bits of M (starts pb + bit) to out[g ..]; cap checked once
// per run (all of it fits: no per-element test)
__device__ __forceinline__ void write_run(uint64_t M, uint64_t* out, uint64_t g, uint64_t cap, uint64_t pb, uint32_t c) {
  uint64_t* o = out + g;
  if (g + c <= cap) {
    for (uint32_t lo = static_cast<uint32_t>(M); lo; lo &= lo - 1) st_stream_u64(o++, pb + (__ffs(lo) - 1));
    for (uint32_t hi = static_cast<uint32_t>(M >> 32); hi; hi &= hi - 1) st_stream_u64(o++, pb + 31 + __ffs(hi));
  } else {
    while (M) {
      const uint32_t bit = __ffsll(static_cast<long long>(M)) - 1;
      M &= M - 1;
      if (g < cap) st_stream_u64(out + g, pb + bit);
      ++g;
    }
  }
}

__global__ void __launch_bounds__(kThreads) epsm_mask_write_kernel(const __grid_constant__ MaskParams P) {
  __shared__ uint64_t SH[kWarps][kMaxSh][32];
  __shared__ unsigned long long base[kWarps][kMaxD];   // the task's next output slot per pattern
  __shared__ uint8_t shs[kMaxD][kMaxM];
  __shared__ uint64_t* spos[kMaxD];
  __shared__ uint64_t scap[kMaxD];
  for (uint32_t d = threadIdx.x; d < kMaxD; d += blockDim.x) {
    spos[d] = P.pos[d];
    scap[d] = P.cap[d];
  }
  load_sh(P, shs);
  const uint32_t lane = threadIdx.x & 31u, wp = threadIdx.x >> 5;
  bool waited = false;
  for (uint64_t task = static_cast<uint64_t>(blockIdx.x) * kWarps + wp; task < P.ntasks;
       task += static_cast<uint64_t>(gridDim.x) * kWarps) {
    for (uint32_t d = lane; d < P.D; d += 32) base[wp][d] = P.prefix[static_cast<uint64_t>(d) * P.ntasks + task];
    __syncwarp();
    if (!waited) {
      griddep_wait();
      waited = true;
    }
    for (int r = 0; r < kRounds; ++r) {
      const uint64_t w = stage_round(P, task, r, lane, SH[wp]);
      const uint64_t pb = w * 64 + P.pos_bias;
      for (uint32_t d = 0; d < P.D; d += 2) {
        // two patterns per warp scan (their counts as the u16 halves of one word: <= 64 per lane,
        // <= 2048 per round, no carry between the halves)
        const bool two = d + 1 < P.D;
        const uint64_t M0 = pattern_mask(P, shs, d, w, lane, SH[wp]);
        const uint64_t M1 = two ? pattern_mask(P, shs, d + 1, w, lane, SH[wp]) : 0ull;
        const uint32_t c0 = __popcll(M0), c1 = __popcll(M1);
        // exclusive offset of this lane's matches among the round's (lanes in text order); each
        // lane stores its own run (the runs of consecutive lanes are adjacent in the output)
        uint32_t incl = c0 | (c1 << 16);
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
          if (lane >= static_cast<uint32_t>(o)) incl += y;
        }
        const uint32_t i0 = incl & 0xFFFFu, i1 = incl >> 16;
        write_run(M0, spos[d], base[wp][d] + i0 - c0, scap[d], pb, c0);
        if (two) write_run(M1, spos[d + 1], base[wp][d + 1] + i1 - c1, scap[d + 1], pb, c1);
        __syncwarp();
        if (lane == 31) {
          base[wp][d] += i0;
          if (two) base[wp][d + 1] += i1;
        }
        __syncwarp();
      }
    }
  }
}

}  // namespace mk
}  // namespace epsm
