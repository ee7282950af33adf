// epsm_code.cuh -- sm_100a kernels of the group search's CODE MODE: dense groups of D <= 127
// distinct patterns of one length m <= 8 over a small pattern alphabet, every start keyed
// exactly (EPSMa's per-position compare, for all patterns of the group at
// once).  Same three passes as epsm_multi.cuh (counts per (chunk, pattern) -> prefix scan ->
// ranked write-out, PAPER.md:470 / Fig. 1 line 11: the positions i*alpha + {r} in text order), but
// built for groups whose matches are MANY (up to one start in three):
//
//   * per start: byte -> symbol code (cmap), rolling key of the window's m codes, key -> pattern
//     (a table of 2^(m*cb) bytes) -- two shared-memory loads and four ALU instructions per start;
//   * pass 1 counts every start with one warp-aggregated shared atomic (ATOMS.POPC.INC: the
//     non-matching lanes share a dummy counter);
//   * pass 3 ranks the matches WITHOUT warp-wide match_any (measured ~55 clk per round): every
//     lane counts its own matches per pattern in a private counter column (one shared atomic per
//     match, lane-distinct banks), a rotated (bank-conflict-free) scan turns the columns into
//     each lane's exclusive offsets inside the warp's per-pattern runs, a second walk places every
//     match into a per-warp staging buffer sorted by (pattern, text order), and the warp flushes
//     the buffer with coalesced stores (consecutive lanes -> consecutive output slots).
//
// Bytes outside the patterns' alphabet: with a spare code (cmap -> a code no pattern holds) the
// key never names a pattern; without one (cmap -> 0x80) the fast path's keys of windows holding
// such a byte are garbage, so a lane that met one re-derives which of its windows are valid and
// drops the others (counts subtracted in pass 1, ids cleared in pass 3).
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

#include "epsm_multi.cuh"
#include "epsm_ptx.cuh"

namespace epsm {
namespace cg {

using mp::kStageBytes;
using mp::kTile;
constexpr int kSeg = 64;                          // starts per lane
constexpr int kSlice = 32 * kSeg;                 // starts per warp slice (2048)
constexpr int kCntWarps = 16;                     // pass 1: 16 slices = one chunk
constexpr int kWrWarps = 8;                       // pass 3: 8 slices = half a chunk, twice
constexpr int kHalf = kWrWarps * kSlice;          // 16384
constexpr int kCntStages = 4;
constexpr int kWrStages = 2;
constexpr int kMaxD = 127;                        // ids 0..126; 0xFF: no pattern
constexpr int kMaxM = 8;
#ifndef EPSM_CG_CHAINS
#define EPSM_CG_CHAINS 2                          // key chains per lane in pass 1
#endif
constexpr int kTab = 1 << mp::kCodeKeyBits;       // key table bytes (16 KiB)
constexpr int kIdsLane = 80;                      // id bytes per lane (16-B aligned, STS.128 conflict-free)
constexpr int kRows = (kMaxD + 1) / 2;            // counter rows: ids 2r (low half), 2r+1 (high half)
constexpr int kCntThreads = 32 * (1 + kCntWarps);
constexpr int kWrThreads = 32 * (1 + kWrWarps);
static_assert(kCntWarps * kSlice == kTile && 2 * kHalf == kTile, "slices tile the chunk");

struct CParams {
  const uint8_t* text;          // 16-byte aligned virtual base
  uint64_t nbytes;              // readable bytes from text
  uint64_t s_lo, s_hi;          // valid virtual starts [s_lo, s_hi)
  uint64_t pos_bias;            // reported = virtual start + pos_bias
  uint32_t nchunks;             // tiles covering [0, s_hi)
  uint32_t it_lo, it_hi;        // interior tiles: every start in [s_lo, s_hi)
  uint32_t cb;                  // bits per symbol code
  uint32_t kmask;               // 2^(m * cb) - 1
  uint32_t D;                   // distinct patterns (<= kMaxD)
  uint32_t invmask;             // code bits that mark a byte outside the alphabet (IDENT: the byte's
                                // bits above cb; else cmap's 0x80)
  const mp::GroupDesc* desc;    // cmap, key table (overlaying bitmap + boff), dup lists
  uint16_t* counts;             // [D][nchunks]: pass 1 out
  uint32_t* listlen;            // [nchunks]: nonzero <=> the chunk holds a match (pass 1 out)
  const unsigned long long* prefix;   // [D][nchunks]: pass 3 in
  uint32_t* work;               // [0] chunks with matches, [1 ..] their ids (pass 1 zeroes
                                // [0]; the scan appends)
  const mp::JobOut* jobs;       // output of (local) search j
};

struct __align__(128) CntSmem {
  uint8_t ring[kCntStages][kStageBytes];
  uint8_t tab[kTab];
  uint8_t cmap[256];
  uint32_t hist[kCntWarps][256];                  // per warp: matches per id (255: the dummy)
  alignas(8) uint64_t full[kCntStages];
  uint64_t empty[kCntStages];
  uint32_t info[kCntStages];
  uint32_t any;
};

struct __align__(128) WrSmem {
  uint8_t ring[kWrStages][kStageBytes];
  uint8_t tab[kTab];
  uint8_t cmap[256];
  alignas(16) uint8_t ids[kWrWarps][32 * kIdsLane];   // id of each start (by lane, start)
  uint32_t ctr[kWrWarps][kRows * 32];             // [row][lane]: two u16 counters per word
  uint16_t stg[kWrWarps][kSlice];                 // staged matches: chunk offset ...
  uint8_t sid[kWrWarps][kSlice];                  // ... and pattern, sorted by (pattern, text order)
  alignas(16) uint16_t tot[2][kMaxD + 1][kWrWarps];   // per half: matches of (pattern, warp slice)
  int32_t wofs[kWrWarps][kMaxD + 1];              // per warp: output index - staging index
  uint64_t* cdst[2][kMaxD + 1];                   // per chunk parity: first slot of the chunk
  uint64_t* oend[kMaxD + 1];                      // end of each pattern's first output
  alignas(8) uint64_t full[kWrStages];
  uint64_t empty[kWrStages];
  uint32_t info[kWrStages];
};
static_assert(sizeof(CntSmem) <= 232448 && sizeof(WrSmem) <= 232448, "fits 227 KB of shared memory");
constexpr uint32_t kEnd = 0xFFFFFFFFu;

__device__ __forceinline__ void bar_cg(int nwarps) {   // named barrier over the consumer warps
  asm volatile("bar.sync 1, %0;" ::"r"(32 * nwarps) : "memory");
}

// cmap and key table into shared memory (16-byte pieces; the table overlays bitmap + boff)
__device__ __forceinline__ void load_tables(const mp::GroupDesc* g, uint8_t* tab, uint8_t* cmap, uint32_t tid,
                                            uint32_t nthr) {
  const uint4* src = reinterpret_cast<const uint4*>(g->bitmap);
  for (uint32_t i = tid; i < kTab / 16; i += nthr) reinterpret_cast<uint4*>(tab)[i] = src[i];
  for (uint32_t i = tid; i < 256; i += nthr) cmap[i] = g->cmap[i];
}

// The lane's 80 bytes: its 64 starts' first bytes + 16 of halo (the next lane's first 16; lane 31:
// the next slice's / the stage halo)
__device__ __forceinline__ void load_window(const uint8_t* ts, uint32_t seg, uint32_t lane, uint32_t (&W)[20]) {
  const uint4* src = reinterpret_cast<const uint4*>(ts + seg);
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const uint4 v = src[r];
    W[4 * r] = v.x;
    W[4 * r + 1] = v.y;
    W[4 * r + 2] = v.z;
    W[4 * r + 3] = v.w;
  }
#pragma unroll
  for (int r = 0; r < 4; ++r) W[16 + r] = __shfl_down_sync(0xffffffffu, W[r], 1);
  if (lane == 31) {
    const uint4 v = src[4];
    W[16] = v.x;
    W[17] = v.y;
    W[18] = v.z;
    W[19] = v.w;
  }
}

// Starts s of the lane (virtual ub + s) inside [s_lo, s_hi) -- only at the text's two ends
__device__ __forceinline__ uint64_t keep_mask(uint64_t ub, const CParams& P) {
  uint64_t keep = ~0ull;
  if (ub + 64 > P.s_hi) keep = P.s_hi <= ub ? 0ull : (~0ull >> (64 - (P.s_hi - ub)));
  if (ub < P.s_lo) keep &= P.s_lo >= ub + 64 ? 0ull : (~0ull << (P.s_lo - ub));
  return keep;
}

// Starts of the lane whose window holds a byte outside the patterns' alphabet (no spare code)
template <int M, bool IDENT>
__device__ uint64_t invalid_starts(const uint8_t* ts, uint32_t seg, const uint8_t* cmap, uint32_t invmask) {
  uint64_t bad = 0;
  int last = -64;
#pragma unroll 1
  for (int t = 0; t < kSeg + M - 1; ++t) {
    const uint32_t b = ts[seg + t];
    if ((IDENT ? b : cmap[b]) & invmask) last = t;
    if (t >= M - 1 && t - last < M) bad |= 1ull << (t - (M - 1));
  }
  return bad;
}

// The fast path's id of start s (same arithmetic as the unrolled filters: garbage for windows
// with an invalid byte, which is exactly what has to be undone)
template <int M, bool IDENT>
__device__ __forceinline__ uint32_t fast_id(const uint8_t* ts, uint32_t st, const uint8_t* cmap, const uint8_t* tab,
                                            uint32_t cb, uint32_t kmask) {
  uint32_t key = 0;
#pragma unroll
  for (int j = 0; j < M; ++j) {
    const uint32_t b = ts[st + j];
    key = ((key << cb) | (IDENT ? b : cmap[b])) & kmask;
  }
  return tab[key];
}

// IDENT: every pattern byte is below 2^cb and is its own code (the byte values of small symbol
// alphabets): no cmap load per start; a byte with a bit at or above cb marks an invalid window.
// ===================================================================================== pass 1
template <int M, bool IDENT>
__global__ void __launch_bounds__(kCntThreads, 1) cg_count_kernel(const __grid_constant__ CParams P) {
  extern __shared__ __align__(128) uint8_t smem_raw[];
  CntSmem& S = *reinterpret_cast<CntSmem*>(smem_raw);
  const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
  if (tid < static_cast<uint32_t>(kCntStages)) {
    mbar_init(&S.full[tid], 1);
    mbar_init(&S.empty[tid], kCntWarps);
    fence_mbar_init();
  }
  load_tables(P.desc, S.tab, S.cmap, tid, blockDim.x);
  for (uint32_t i = tid; i < kCntWarps * 256; i += blockDim.x) (&S.hist[0][0])[i] = 0;
  if (tid == 0) S.any = 0;
  if (blockIdx.x == 0 && tid == 0) P.work[0] = 0;   // (the scan kernel appends; it runs after)
  __syncthreads();

  if (warp == 0) {
    // ---------------------------------------------------------------- producer (TMA ring)
    const uint64_t policy = policy_evict_first();
    uint32_t stage = 0, phase = 0;
    for (uint32_t c = blockIdx.x; c < P.nchunks; c += gridDim.x) {
      mbar_wait_sleep(&S.empty[stage], phase ^ 1u, 256);
      const uint64_t base = static_cast<uint64_t>(c) * kTile;
      const uint64_t want_end = base + kTile + mp::kHalo;
      const uint64_t end = want_end < P.nbytes ? want_end : P.nbytes;
      const uint32_t bulk = static_cast<uint32_t>((end & ~15ull) - base);
      const uint32_t tail = static_cast<uint32_t>(end - base) - bulk;
      if (lane < tail) S.ring[stage][bulk + lane] = P.text[base + bulk + lane];
      __syncwarp();
      if (lane == 0) {
        S.info[stage] = c;
        if (bulk) {
          mbar_arrive_expect_tx(&S.full[stage], bulk);
          bulk_g2s(S.ring[stage], P.text + base, bulk, &S.full[stage], policy);
        } else {
          mbar_arrive(&S.full[stage]);
        }
      }
      if (++stage == kCntStages) {
        stage = 0;
        phase ^= 1u;
      }
    }
    mbar_wait_sleep(&S.empty[stage], phase ^ 1u, 256);
    if (lane == 0) {
      S.info[stage] = kEnd;
      mbar_arrive(&S.full[stage]);
    }
    return;
  }

  // ------------------------------------------------------------------ consumers
  const uint32_t cw = warp - 1;
  const uint32_t seg = cw * kSlice + lane * kSeg;
  const uint32_t cb = P.cb, kmask = P.kmask;
  uint32_t* const h = S.hist[cw];
  uint32_t stage = 0, phase = 0;
  while (true) {
    mbar_wait(&S.full[stage], phase);
    const uint32_t c = S.info[stage];
    if (c == kEnd) break;
    const uint8_t* ts = S.ring[stage];
    uint32_t W[20];
    load_window(ts, seg, lane, W);
    // every start of the lane: key -> id, counted (no pattern: the dummy counter 255); kChains
    // independent key chains (starts q*64/kChains ..) for instruction-level parallelism
    constexpr int kChains = EPSM_CG_CHAINS;
    constexpr int kPer = kSeg / kChains;
    uint32_t kc[kChains], inv = 0;
#pragma unroll
    for (int q = 0; q < kChains; ++q) kc[q] = 0;
#pragma unroll
    for (int t = 0; t < kPer + M - 1; ++t) {
#pragma unroll
      for (int q = 0; q < kChains; ++q) {
        const int tq = t + q * kPer;
        const uint32_t bq = __byte_perm(W[tq >> 2], 0u, 0x4440u | (tq & 3));
        const uint32_t cq = IDENT ? bq : S.cmap[bq];
        inv |= cq;
        kc[q] = ((kc[q] << cb) | cq) & kmask;
      }
      if (t >= M - 1) {
#pragma unroll
        for (int q = 0; q < kChains; ++q) atomicAdd(&h[S.tab[kc[q]]], 1u);
      }
    }
    // undo the starts that do not count: outside [s_lo, s_hi) (the text's ends) or whose window
    // holds a byte outside the alphabet (no spare code)
    uint64_t sub = 0;
    if (!(c >= P.it_lo && c < P.it_hi)) sub = ~keep_mask(static_cast<uint64_t>(c) * kTile + seg, P);
    if (inv & P.invmask) sub |= invalid_starts<M, IDENT>(ts, seg, S.cmap, P.invmask);
    while (sub) {
      const uint32_t s = __ffsll(static_cast<long long>(sub)) - 1;
      sub &= sub - 1;
      atomicSub(&h[fast_id<M, IDENT>(ts, seg + s, S.cmap, S.tab, cb, kmask)], 1u);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&S.empty[stage]);
    bar_cg(kCntWarps);
    // the chunk's counts: sum of the warps' (and the counters zeroed for the next chunk)
    for (uint32_t d = tid - 32; d < 256; d += 32 * kCntWarps) {
      uint32_t sum = 0;
#pragma unroll
      for (int w = 0; w < kCntWarps; ++w) {
        sum += S.hist[w][d];
        S.hist[w][d] = 0;
      }
      if (d < P.D) {
        P.counts[static_cast<uint64_t>(d) * P.nchunks + c] = static_cast<uint16_t>(sum);
        if (sum) S.any = 1;
      }
    }
    bar_cg(kCntWarps);
    if (tid == 32) {
      P.listlen[c] = S.any;
      S.any = 0;
    }
    if (++stage == kCntStages) {
      stage = 0;
      phase ^= 1u;
    }
  }
}

// ===================================================================================== pass 3
template <int M, bool IDENT>
__global__ void __launch_bounds__(kWrThreads, 1) cg_write_kernel(const __grid_constant__ CParams P) {
  extern __shared__ __align__(128) uint8_t smem_raw[];
  WrSmem& S = *reinterpret_cast<WrSmem*>(smem_raw);
  const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
  if (tid < static_cast<uint32_t>(kWrStages)) {
    mbar_init(&S.full[tid], 1);
    mbar_init(&S.empty[tid], kWrWarps);
    fence_mbar_init();
  }
  load_tables(P.desc, S.tab, S.cmap, tid, blockDim.x);
  for (uint32_t i = tid; i < kWrWarps * kRows * 32; i += blockDim.x) (&S.ctr[0][0])[i] = 0;
  for (uint32_t d = tid; d <= static_cast<uint32_t>(kMaxD); d += blockDim.x) {
    // the first output of every pattern (the others are copied from it after the pass)
    uint64_t* o = nullptr;
    uint64_t cap = 0;
    if (d < P.D) {
      const mp::JobOut J = P.jobs[P.desc->dup_list[P.desc->dup_off[d]]];
      o = J.pos;
      cap = J.pos ? J.cap : 0;
    }
    S.oend[d] = o + cap;
    S.cdst[0][d] = o;   // (pointer base; the chunk prefix is added per chunk)
    S.cdst[1][d] = o;
  }
  __syncthreads();

  if (warp == 0) {
    // ---------------------------------------------------------------- producer (TMA ring)
    const uint64_t policy = policy_evict_first();
    uint32_t stage = 0, phase = 0;
    const uint32_t nwork = *reinterpret_cast<volatile const uint32_t*>(P.work);
    for (uint32_t w = blockIdx.x; w < nwork; w += gridDim.x) {
      const uint32_t c = P.work[1 + w];
      mbar_wait_sleep(&S.empty[stage], phase ^ 1u, 256);
      const uint64_t base = static_cast<uint64_t>(c) * kTile;
      const uint64_t want_end = base + kTile + mp::kHalo;
      const uint64_t end = want_end < P.nbytes ? want_end : P.nbytes;
      const uint32_t bulk = static_cast<uint32_t>((end & ~15ull) - base);
      const uint32_t tail = static_cast<uint32_t>(end - base) - bulk;
      if (lane < tail) S.ring[stage][bulk + lane] = P.text[base + bulk + lane];
      __syncwarp();
      if (lane == 0) {
        S.info[stage] = c;
        if (bulk) {
          mbar_arrive_expect_tx(&S.full[stage], bulk);
          bulk_g2s(S.ring[stage], P.text + base, bulk, &S.full[stage], policy);
        } else {
          mbar_arrive(&S.full[stage]);
        }
      }
      if (++stage == kWrStages) {
        stage = 0;
        phase ^= 1u;
      }
    }
    mbar_wait_sleep(&S.empty[stage], phase ^ 1u, 256);
    if (lane == 0) {
      S.info[stage] = kEnd;
      mbar_arrive(&S.full[stage]);
    }
    return;
  }

  // ------------------------------------------------------------------ consumers
  const uint32_t cw = warp - 1;
  const uint32_t cb = P.cb, kmask = P.kmask;
  const uint32_t nrows = (P.D + 1) >> 1;
  uint8_t* const idl = S.ids[cw] + lane * kIdsLane;
  uint32_t* const ctr = S.ctr[cw];
  uint16_t* const stg = S.stg[cw];
  uint8_t* const sid = S.sid[cw];
  uint32_t stage = 0, phase = 0, par = 0;
  while (true) {
    mbar_wait(&S.full[stage], phase);
    const uint32_t c = S.info[stage];
    if (c == kEnd) break;
    const uint8_t* ts = S.ring[stage];
    const bool interior = c >= P.it_lo && c < P.it_hi;
    // the chunk's first output slot of each pattern (by chunk parity: the previous chunk's
    // flushes may still read the other copy; the next half's barrier orders this one)
    if (lane < 16) {
      const uint32_t d = cw + kWrWarps * lane;
      if (d < P.D) {
        const mp::JobOut* J = &P.jobs[P.desc->dup_list[P.desc->dup_off[d]]];
        S.cdst[par][d] = J->pos + P.prefix[static_cast<uint64_t>(d) * P.nchunks + c];
      }
    }
    const uint64_t cbase = static_cast<uint64_t>(c) * kTile + P.pos_bias;
#pragma unroll 1
    for (uint32_t hf = 0; hf < 2; ++hf) {
      const uint32_t soff = hf * kHalf + cw * kSlice;     // the warp slice's chunk offset
      const uint32_t seg = soff + lane * kSeg;
      // ---- filter: the id of every start (packed, 4 per word; 0xFF: none)
      uint32_t idw[16];
      uint32_t inv = 0;
      {
        uint32_t W[20];
        load_window(ts, seg, lane, W);
        uint32_t ka = 0, kb = 0;
#pragma unroll
        for (int t = 0; t < kSeg / 2 + M - 1; ++t) {
          // two independent key chains: starts 0..31 (bytes t) and 32..63 (bytes t + 32)
          const int tb = t + kSeg / 2;
          const uint32_t ba = __byte_perm(W[t >> 2], 0u, 0x4440u | (t & 3));
          const uint32_t bb = __byte_perm(W[tb >> 2], 0u, 0x4440u | (tb & 3));
          const uint32_t ca = IDENT ? ba : S.cmap[ba];
          const uint32_t cbb = IDENT ? bb : S.cmap[bb];
          inv |= ca | cbb;
          ka = ((ka << cb) | ca) & kmask;
          kb = ((kb << cb) | cbb) & kmask;
          if (t >= M - 1) {
            const int sa = t - (M - 1), sb = sa + kSeg / 2;
            const uint32_t ia = S.tab[ka], ib = S.tab[kb];
            if ((sa & 3) == 0) {
              idw[sa >> 2] = ia;
              idw[sb >> 2] = ib;
            } else {
              const uint32_t sel = (sa & 3) == 1 ? 0x3240u : ((sa & 3) == 2 ? 0x3410u : 0x4210u);
              idw[sa >> 2] = __byte_perm(idw[sa >> 2], ia, sel);
              idw[sb >> 2] = __byte_perm(idw[sb >> 2], ib, sel);
            }
          }
        }
      }
      // starts that do not count get 0xFF: outside [s_lo, s_hi), or windows with an invalid byte
      uint64_t drop = 0;
      if (!interior) drop = ~keep_mask(static_cast<uint64_t>(c) * kTile + seg, P);
      if (inv & P.invmask) drop |= invalid_starts<M, IDENT>(ts, seg, S.cmap, P.invmask);
      if (drop) {
#pragma unroll
        for (int w = 0; w < 16; ++w) {
          const uint32_t nib = static_cast<uint32_t>(drop >> (4 * w)) & 15u;
          idw[w] |= ((nib * 0x00204081u) & 0x01010101u) * 0xFFu;   // nibble bit k -> byte k
        }
      }
      if (hf == 1) {
        __syncwarp();
        if (lane == 0) mbar_arrive(&S.empty[stage]);      // (the text of both halves is read)
      }
      // the lane's match mask (bit s: start s has a pattern) and its ids into shared memory
      uint32_t mlo = 0, mhi = 0;
#pragma unroll
      for (int w = 0; w < 16; ++w) {
        const uint32_t nib = ((~idw[w] & 0x80808080u) * 0x00204081u) >> 28;   // byte k's top bit -> bit k
        if (w < 8) mlo |= nib << (4 * w);
        else mhi |= nib << (4 * (w - 8));
      }
#pragma unroll
      for (int r = 0; r < 4; ++r)
        reinterpret_cast<uint4*>(idl)[r] = make_uint4(idw[4 * r], idw[4 * r + 1], idw[4 * r + 2], idw[4 * r + 3]);
      __syncwarp();
      // ---- walk 1: the lane's count of every pattern (its private column: lane-distinct banks);
      // four matches per step, so that their loads and reductions are in flight together
      const uint64_t mall = (static_cast<uint64_t>(mhi) << 32) | mlo;
      for (uint64_t mm = mall; mm;) {
        uint32_t sk[4], id[4];
        bool v[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          v[k] = mm != 0;
          sk[k] = static_cast<uint32_t>(__ffsll(static_cast<long long>(mm)) - 1);
          mm &= mm - 1;
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) id[k] = v[k] ? idl[sk[k]] : 0u;
#pragma unroll
        for (int k = 0; k < 4; ++k)
          if (v[k]) atomicAdd(&ctr[(id[k] >> 1) * 32 + lane], (id[k] & 1u) ? 0x10000u : 1u);
      }
      __syncwarp();
      // ---- scan: lane l owns rows l and l + 32 (ids 2l, 2l+1 and 2l+64, 2l+65: u16 halves, added
      // at once -- no carry crosses them).  A row is read as eight 16-byte pieces in the rotated
      // order rho, rho+1, .., rho-1 (rho = l & 7: a quarter-warp's lanes hit eight distinct bank
      // groups); pass A: the row total and E0 = the sum of pieces before rho
      const uint32_t rho = lane & 7u;
      uint32_t rs[2] = {0, 0}, e0[2] = {0, 0};
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const uint32_t row = lane + 32 * q;
        if (row < nrows) {
          const uint8_t* a0 = reinterpret_cast<const uint8_t*>(ctr + row * 32) + 16 * rho;
          const uint8_t* a1 = a0 - 128;
          uint32_t run = 0, pre = 0;
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            const bool wrap = static_cast<uint32_t>(k) >= 8u - rho;
            const uint4 v = *reinterpret_cast<const uint4*>((wrap ? a1 : a0) + 16 * k);
            const uint32_t cs = v.x + v.y + v.z + v.w;
            if (wrap) pre += cs;
            run += cs;
          }
          rs[q] = run;
          e0[q] = pre;
        }
      }
      // run bases of the ids inside the warp's staging (exclusive over ids 0, 1, ..): rows of
      // q = 0 hold ids 0..63 in lane order, rows of q = 1 ids 64..127
      uint32_t rb[2];
      {
        const uint32_t t0 = (rs[0] & 0xFFFFu) + (rs[0] >> 16), t1 = (rs[1] & 0xFFFFu) + (rs[1] >> 16);
        uint32_t x0 = t0, x1 = t1;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const uint32_t y0 = __shfl_up_sync(0xffffffffu, x0, o), y1 = __shfl_up_sync(0xffffffffu, x1, o);
          if (lane >= static_cast<uint32_t>(o)) {
            x0 += y0;
            x1 += y1;
          }
        }
        const uint32_t all0 = __shfl_sync(0xffffffffu, x0, 31);
        rb[0] = x0 - t0;                                  // base of id 2l
        rb[1] = all0 + x1 - t1;                           // base of id 2l + 64
      }
      // pass B: every word := its lane's exclusive prefix in the row + the run base (both halves).
      // Piece c = (rho + k) & 7 starts at E_c = R_k + E0 (no wrap) or R_k + E0 - S (wrapped),
      // R_k = the sum of the pieces visited before it
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const uint32_t row = lane + 32 * q;
        if (row < nrows) {
          uint8_t* a0 = reinterpret_cast<uint8_t*>(ctr + row * 32) + 16 * rho;
          uint8_t* a1 = a0 - 128;
          const uint32_t bases = rb[q] | ((rb[q] + (rs[q] & 0xFFFFu)) << 16);
          const uint32_t eb = e0[q] + bases;
          uint32_t rk = 0;
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            const bool wrap = static_cast<uint32_t>(k) >= 8u - rho;
            uint4* p = reinterpret_cast<uint4*>((wrap ? a1 : a0) + 16 * k);
            const uint4 v = *p;
            const uint32_t w0 = wrap ? rk + eb - rs[q] : rk + eb;
            const uint32_t w1 = w0 + v.x, w2 = w1 + v.y, w3 = w2 + v.z;
            *p = make_uint4(w0, w1, w2, w3);
            rk += v.x + v.y + v.z + v.w;
          }
          // the slice's count of both ids, for the other warps
          S.tot[hf][2 * row][cw] = static_cast<uint16_t>(rs[q] & 0xFFFFu);
          S.tot[hf][2 * row + 1][cw] = static_cast<uint16_t>(rs[q] >> 16);
        }
      }
      __syncwarp();
      // ---- walk 2: every match to its staging slot (pattern run + rank in text order: a lane's
      // atomics on one counter take effect in program order, i.e. in text order); four per step
      for (uint64_t mm = mall; mm;) {
        uint32_t sk[4], id[4], slot[4];
        bool v[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          v[k] = mm != 0;
          sk[k] = static_cast<uint32_t>(__ffsll(static_cast<long long>(mm)) - 1);
          mm &= mm - 1;
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) id[k] = v[k] ? idl[sk[k]] : 0u;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const uint32_t sh = (id[k] & 1u) << 4;
          slot[k] = v[k] ? (atomicAdd(&ctr[(id[k] >> 1) * 32 + lane], 1u << sh) >> sh) & 0xFFFFu : 0u;
        }
#pragma unroll
        for (int k = 0; k < 4; ++k)
          if (v[k]) {
            stg[slot[k]] = static_cast<uint16_t>(seg + sk[k]);
            sid[slot[k]] = static_cast<uint8_t>(id[k]);
          }
      }
      bar_cg(kWrWarps);                                   // (every warp's totals of this half)
      // ---- where the warp's runs go: the chunk's first slot of the pattern + the earlier slices
      // of the chunk (this half's warps before cw; in half 1 all of half 0) - the run base
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const uint32_t row = lane + 32 * q;
        if (row < nrows) {
#pragma unroll
          for (int k = 0; k < 2; ++k) {
            const uint32_t d = 2 * row + k;
            const uint4 a = *reinterpret_cast<const uint4*>(&S.tot[hf][d][0]);
            const uint32_t v[4] = {a.x, a.y, a.z, a.w};
            uint32_t before = 0;
#pragma unroll
            for (int w = 0; w < kWrWarps; ++w) {
              const uint32_t x = (v[w >> 1] >> (16 * (w & 1))) & 0xFFFFu;
              if (static_cast<uint32_t>(w) < cw) before += x;
            }
            if (hf == 1) {
              const uint4 b = *reinterpret_cast<const uint4*>(&S.tot[0][d][0]);
              before += (b.x & 0xFFFFu) + (b.x >> 16) + (b.y & 0xFFFFu) + (b.y >> 16) + (b.z & 0xFFFFu) +
                        (b.z >> 16) + (b.w & 0xFFFFu) + (b.w >> 16);
            }
            const uint32_t base = k ? rb[q] + (rs[q] & 0xFFFFu) : rb[q];
            S.wofs[cw][d] = static_cast<int32_t>(before) - static_cast<int32_t>(base);
          }
        }
      }
      // ---- zero the counters for the next half (rotated 16-byte pieces: conflict-free)
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const uint32_t row = lane + 32 * q;
        if (row < nrows) {
          uint4* rp = reinterpret_cast<uint4*>(ctr + row * 32);
#pragma unroll
          for (int i = 0; i < 8; ++i) rp[(lane + i) & 7u] = make_uint4(0u, 0u, 0u, 0u);
        }
      }
      __syncwarp();
      // ---- flush: staging entry e -> output slot cdst[id] + wofs[id] + e (runs are contiguous:
      // consecutive lanes store to consecutive slots)
      const uint32_t T = __shfl_sync(0xffffffffu, (lane == 31) ? rb[1] + (rs[1] & 0xFFFFu) + (rs[1] >> 16) : 0u, 31);
      for (uint32_t e = lane; e < T; e += 32) {
        const uint32_t id = sid[e];
        uint64_t* dst = S.cdst[par][id] + (S.wofs[cw][id] + static_cast<int32_t>(e));
        if (dst < S.oend[id]) st_stream_u64(dst, cbase + stg[e]);
      }
      __syncwarp();
    }
    par ^= 1u;
    if (++stage == kWrStages) {
      stage = 0;
      phase ^= 1u;
    }
  }
}

}  // namespace cg
}  // namespace epsm
