// epsm_kernels.cuh -- sm_100a kernels of the exact packed string matcher.
//
// One CTA scans one 16 KiB tile of text (1024 "units" of alpha = 16 bytes,
// PAPER.md:166-168, Sec. 3.1).  The tile plus a 32-byte halo (>= m-1 for every
// m <= 32) is staged into shared memory by ONE TMA bulk copy
// (cp.async.bulk ... mbarrier::complete_tx) -- the GPU analogue of EPSMb's
// wsblend, which exists only to avoid unaligned loads; shared
// memory is byte addressable, so every alignment is read directly.
//
// Per thread and unit (16 candidate starts u..u+15):
//   filter  (EPSMa's shift-AND, PAPER.md:461-469 / Fig. 1 lines 5-9):
//           Z_k = OR_{i<F} ( S_i[k] XOR B_i ),  S_i = the text shifted by i bytes
//           (funnel shifts of the unit's words), B_i = p_i * 0x01010101.
//           A zero byte j of Z_k  <=>  t[u+4k+j+i] = p_i for all i < F.
//   verify  (the "naive check"): for m > F each candidate
//           window is compared word by word with the zero-padded pattern P_i
//           (PAPER.md:124-128), masking the last partial word.
//   count   popcount of the 16-bit mask r.
//   report  positions tile_base + unit + {r} (Fig. 1 line 11),
//           ordered across tiles by a decoupled look-back over 64-bit epoch-tagged
//           status words, staged in shared memory and stored coalesced.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace epsm {

constexpr int kThreads = 256;
constexpr int kUnitsPerThread = 4;
constexpr int kUnitBytes = 16;                                            // alpha
constexpr int kTileBytes = kThreads * kUnitsPerThread * kUnitBytes;      // 16 KiB
constexpr int kHaloBytes = 32;                                            // >= m-1, x16
constexpr int kSmemBytes = kTileBytes + kHaloBytes + 32;                  // + verify slack
constexpr int kStageCap = kTileBytes / 8;                                 // u64 per round
constexpr int kWarps = kThreads / 32;

// Tile status word: [63:40] epoch, [39:38] flag, [37:0] value.
constexpr int kEpochShift = 40;
constexpr unsigned long long kFlagAgg = 1ull << 38;
constexpr unsigned long long kFlagInc = 2ull << 38;
constexpr unsigned long long kFlagMask = 3ull << 38;
constexpr unsigned long long kValueMask = (1ull << 38) - 1;
constexpr unsigned long long kEpochMask = ~((1ull << kEpochShift) - 1);

struct KParams {
  const uint8_t* text;          // 16-byte aligned virtual base
  uint64_t nbytes;              // readable bytes from text
  uint64_t s_lo, s_hi;          // valid virtual starts [s_lo, s_hi)
  uint64_t pos_bias;            // reported = virtual start + pos_bias (mod 2^64)
  uint64_t* pos;                // output positions (search)
  uint64_t cap;                 // capacity of pos
  unsigned long long* occ;      // device occ (search: written by the last tile; count: atomics)
  unsigned long long* status;   // one word per tile (search)
  unsigned long long tag;       // epoch << 40
  uint32_t bcast[4];            // B_i = p_i * 0x01010101
  uint32_t pat[9];              // pattern, little-endian u32 words, zero padded
  uint32_t pmask[9];            // per-word byte masks (partial last word)
};

// ------------------------------------------------------------------ PTX helpers

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "LAB_WAIT:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@P1 bra DONE;\n"
      "bra LAB_WAIT;\n"
      "DONE:\n"
      "}\n" ::"r"(smem_addr(bar)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}

// TMA bulk copy global -> shared, completion counted on an mbarrier (UBLKCP in SASS).
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                         uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1], %2, [%3], %4;" ::"r"(smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar)), "l"(policy)
      : "memory");
}

__device__ __forceinline__ unsigned long long ld_relaxed(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void st_relaxed(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ void st_stream_u64(uint64_t* p, uint64_t v) {
  asm volatile("st.global.cs.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// ------------------------------------------------------------------ packed filter

// Exact "byte is zero" flags: bit 8j+7 set iff byte j of z is 0x00.
__device__ __forceinline__ uint32_t zero_byte_flags(uint32_t z) {
  return ~(((z | 0x80808080u) - 0x01010101u) | z) & 0x80808080u;
}

// Nonzero iff some byte of z is zero (the classic has-zero test; exact as a boolean).
__device__ __forceinline__ uint32_t has_zero_byte(uint32_t z) {
  return (z - 0x01010101u) & ~z & 0x80808080u;
}

// movemask: flags at bits 7,15,23,31 -> 4-bit mask, bit j <=> byte j.
__device__ __forceinline__ uint32_t movemask4(uint32_t flags) {
  return (((flags >> 7) * 0x00204081u) >> 21) & 0xFu;
}

// Z words of one unit for an F-byte filter: byte j of Z[k] is zero iff the
// F bytes starting at unit offset 4k+j equal p_0..p_{F-1}.
template <int F>
__device__ __forceinline__ void filter_words(const uint32_t (&w)[5], const uint32_t (&B)[4], uint32_t (&Z)[4]) {
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    uint32_t z = w[k] ^ B[0];
    if (F > 1) z |= __funnelshift_r(w[k], w[k + 1], 8) ^ B[1];
    if (F > 2) z |= __funnelshift_r(w[k], w[k + 1], 16) ^ B[2];
    if (F > 3) z |= __funnelshift_r(w[k], w[k + 1], 24) ^ B[3];
    Z[k] = z;
  }
}

// Bits j of a 16-bit unit mask whose start (ustart + j) lies in [lo, hi).
__device__ __forceinline__ uint32_t range_mask(uint64_t ustart, uint64_t lo, uint64_t hi) {
  uint32_t m = 0xFFFFu;
  if (lo > ustart) {
    const uint64_t c = lo - ustart;
    m = c >= 16 ? 0u : (m << c) & 0xFFFFu;
  }
  if (hi < ustart + 16) {
    const uint64_t c = hi > ustart ? hi - ustart : 0;
    m &= (1u << c) - 1u;
  }
  return m;
}

// Naive check of every candidate bit of r: words 1..MW-1 of the
// window starting at shared byte offset o+b against the zero-padded pattern.
template <int MW>
__device__ __forceinline__ uint32_t verify_candidates(uint32_t r, const uint8_t* tile, uint32_t o,
                                                      const KParams& P) {
  uint32_t keep = r;
  while (r) {
    const int b = __ffs(r) - 1;
    r &= r - 1;
    const uint32_t so = o + b;
    const uint32_t* wp = reinterpret_cast<const uint32_t*>(tile + (so & ~3u));
    const uint32_t sh = (so & 3u) * 8u;
    uint32_t lo = wp[1];
#pragma unroll
    for (int q = 1; q < MW; ++q) {
      const uint32_t hi = wp[q + 1];
      const uint32_t win = __funnelshift_r(lo, hi, sh);
      if ((win ^ P.pat[q]) & P.pmask[q]) {
        keep &= ~(1u << b);
        break;
      }
      lo = hi;
    }
  }
  return keep;
}

__device__ __forceinline__ unsigned long long warp_sum_u64(unsigned long long v) {
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) v += __shfl_xor_sync(0xffffffffu, v, d);
  return v;
}

// Decoupled look-back (single pass): publish this tile's aggregate, walk the
// predecessors 32 at a time until an inclusive prefix is found, publish the
// inclusive prefix.  Called by one full warp; returns the exclusive prefix.
__device__ __forceinline__ unsigned long long lookback(const KParams& P, uint64_t tile, uint32_t total,
                                                       uint32_t lane) {
  const unsigned long long tag = P.tag;
  if (tile == 0) {
    if (lane == 0) st_relaxed(P.status, tag | kFlagInc | total);
    return 0;
  }
  if (lane == 0) st_relaxed(P.status + tile, tag | kFlagAgg | total);
  unsigned long long prefix = 0;
  long long pred = static_cast<long long>(tile) - 1;
  uint32_t spins = 0;
  while (true) {
    const long long idx = pred - static_cast<long long>(lane);
    unsigned long long s;
    while (true) {
      s = idx >= 0 ? ld_relaxed(P.status + idx) : (tag | kFlagInc);
      const bool valid = ((s & kEpochMask) == tag) && (s & kFlagMask);
      if (__all_sync(0xffffffffu, valid)) break;
      __nanosleep(64);
      if (++spins > (1u << 24)) __trap();   // a predecessor never published: fail loudly, never hang
    }
    const uint32_t inc = __ballot_sync(0xffffffffu, (s & kFlagMask) == kFlagInc);
    unsigned long long v = s & kValueMask;
    if (inc) {
      const uint32_t k = __ffs(inc) - 1;
      prefix += warp_sum_u64(lane <= k ? v : 0ull);
      break;
    }
    prefix += warp_sum_u64(v);
    pred -= 32;
  }
  if (lane == 0) st_relaxed(P.status + tile, tag | kFlagInc | (prefix + total));
  return prefix;
}

// ------------------------------------------------------------------ the scan kernel

// F  = filter bytes (min(m, 4));  MW = ceil(m/4) pattern words (MW <= 1: no verify);
// SEARCH = report positions (else count only).
template <int F, int MW, bool SEARCH>
__global__ void __launch_bounds__(kThreads) epsm_scan_kernel(const __grid_constant__ KParams P) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t warp_cnt[kWarps];
  __shared__ uint32_t warp_tot[kUnitsPerThread * kWarps];
  __shared__ unsigned long long s_prefix;

  const uint32_t tid = threadIdx.x;
  const uint32_t lane = tid & 31u;
  const uint32_t warp = tid >> 5;
  const uint64_t tile = blockIdx.x;
  const uint64_t base = tile * static_cast<uint64_t>(kTileBytes);
  const uint64_t want_end = base + static_cast<uint64_t>(kTileBytes + kHaloBytes);
  const uint64_t end = want_end < P.nbytes ? want_end : P.nbytes;
  const uint32_t bulk = static_cast<uint32_t>((end & ~15ull) - base);   // 16-byte multiple

  // ---- stage tile + halo: one TMA bulk copy, scalar tail, zero fill beyond `end`
  if (tid == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (tid == 0 && bulk) {
    mbar_arrive_expect_tx(&bar, bulk);
    bulk_g2s(smem, P.text + base, bulk, &bar, policy_evict_first());
  }
  for (uint32_t i = bulk + tid; i < static_cast<uint32_t>(kSmemBytes); i += kThreads) {
    const uint64_t g = base + i;
    smem[i] = g < end ? P.text[g] : static_cast<uint8_t>(0);
  }
  if (bulk) mbar_wait(&bar, 0);
  __syncthreads();

  // ---- filter + verify: 16 alignments per unit, 4 units per thread
  const uint32_t B[4] = {P.bcast[0], P.bcast[1], P.bcast[2], P.bcast[3]};
  uint32_t r[kUnitsPerThread];
  uint32_t cnt = 0;
#pragma unroll
  for (int j = 0; j < kUnitsPerThread; ++j) {
    const uint32_t o = (j * kThreads + tid) * kUnitBytes;
    const uint4 v = *reinterpret_cast<const uint4*>(smem + o);
    const uint32_t w[5] = {v.x, v.y, v.z, v.w, *reinterpret_cast<const uint32_t*>(smem + o + 16)};
    uint32_t Z[4];
    filter_words<F>(w, B, Z);
    const uint32_t hz = has_zero_byte(Z[0]) | has_zero_byte(Z[1]) | has_zero_byte(Z[2]) | has_zero_byte(Z[3]);
    uint32_t mask = 0;
    if (__any_sync(0xffffffffu, hz)) {
      mask = movemask4(zero_byte_flags(Z[0])) | (movemask4(zero_byte_flags(Z[1])) << 4) |
             (movemask4(zero_byte_flags(Z[2])) << 8) | (movemask4(zero_byte_flags(Z[3])) << 12);
      const uint64_t us = base + o;
      if (us < P.s_lo || us + 16 > P.s_hi) mask &= range_mask(us, P.s_lo, P.s_hi);
      if (MW > 1 && mask) mask = verify_candidates<MW>(mask, smem, o, P);
    }
    r[j] = mask;
    cnt += __popc(mask);
  }

  // ---- tile total
  const uint32_t wsum = __reduce_add_sync(0xffffffffu, cnt);
  if (lane == 0) warp_cnt[warp] = wsum;
  __syncthreads();
  uint32_t total = 0;
#pragma unroll
  for (int i = 0; i < kWarps; ++i) total += warp_cnt[i];

  if (!SEARCH) {
    if (tid == 0 && total) atomicAdd(P.occ, static_cast<unsigned long long>(total));
    return;
  }

  const bool last_tile = tile + 1 == gridDim.x;
  if (total == 0) {
    // nothing to write: warp 0 still resolves the inclusive prefix for successors
    if (warp == 0) {
      const unsigned long long pre = lookback(P, tile, 0, lane);
      if (last_tile && lane == 0) *P.occ = pre;
    }
    return;
  }

  // ---- ordered offsets within the tile (unit order u = j*256 + tid)
  uint32_t off[kUnitsPerThread];
#pragma unroll
  for (int j = 0; j < kUnitsPerThread; ++j) {
    const uint32_t c = __popc(r[j]);
    uint32_t x = c;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, x, d);
      if (lane >= static_cast<uint32_t>(d)) x += y;
    }
    off[j] = x - c;   // exclusive within the warp
    if (lane == 31) warp_tot[j * kWarps + warp] = x;
  }
  if (warp == 0) {
    const unsigned long long pre = lookback(P, tile, total, lane);
    if (lane == 0) {
      s_prefix = pre;
      if (last_tile) *P.occ = pre + total;
    }
  }
  __syncthreads();
  if (warp == 0) {   // exclusive scan of the 32 (unit-slot, warp) totals in unit order
    const uint32_t c = warp_tot[lane];
    uint32_t x = c;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, x, d);
      if (lane >= static_cast<uint32_t>(d)) x += y;
    }
    warp_tot[lane] = x - c;
  }
  __syncthreads();
#pragma unroll
  for (int j = 0; j < kUnitsPerThread; ++j) off[j] += warp_tot[j * kWarps + warp];

  // ---- staged, coalesced stores of this tile's positions into pos[prefix ...]
  const unsigned long long prefix = s_prefix;
  if (prefix >= P.cap) return;
  const uint64_t room = P.cap - prefix;
  const uint64_t limit = room < total ? room : static_cast<uint64_t>(total);
  uint64_t* stage = reinterpret_cast<uint64_t*>(smem);   // text is no longer needed
  for (uint64_t R = 0; R < limit; R += kStageCap) {
#pragma unroll
    for (int j = 0; j < kUnitsPerThread; ++j) {
      const uint32_t c = __popc(r[j]);
      if (c && off[j] < R + kStageCap && off[j] + c > R) {
        uint32_t mm = r[j];
        uint32_t idx = off[j];
        const uint64_t ubase = base + (j * kThreads + tid) * kUnitBytes + P.pos_bias;
        while (mm) {
          const int b = __ffs(mm) - 1;
          mm &= mm - 1;
          if (idx >= R && idx < R + kStageCap) stage[idx - R] = ubase + b;
          ++idx;
        }
      }
    }
    __syncthreads();
    const uint64_t left = limit - R;
    const uint32_t n_out = left < kStageCap ? static_cast<uint32_t>(left) : static_cast<uint32_t>(kStageCap);
    uint64_t* dst = P.pos + prefix + R;
    for (uint32_t i = tid; i < n_out; i += kThreads) st_stream_u64(dst + i, stage[i]);
    __syncthreads();
  }
}

}  // namespace epsm
