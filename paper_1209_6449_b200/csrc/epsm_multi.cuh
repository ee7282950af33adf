// epsm_multi.cuh -- sm_100a kernels of the single-pass GROUP search: many patterns of one
// length m over one text, the paper's own workload (100 / 1000 patterns "randomly extracted"
// from each text, Sec. 4), with the text streamed once for the whole group.
//
// Every search of a group still returns exactly its own Occ(p_j, t): the
// group only shares the work.  Three observations make that cheap on a GPU:
//   * identical patterns have identical results: the group keeps its D distinct patterns and,
//     per distinct pattern, the searches that asked for it;
//   * all patterns have the same length m, so at a start s at most ONE distinct pattern
//     matches -- a start carries one id (0..D-1) or none;
//   * EPSMc's block fingerprints (Fig. 1 lines 1-12) generalise to many
//     patterns: sample one q-gram every SK text bytes (SK + q - 1 <= m, so every window holds
//     exactly one sample at an offset i < SK), and look the sample up in ONE table holding
//     the q-grams p_d[i .. i+q) of every distinct pattern d and offset i (EPSMc's L[v], there
//     per pattern).  A hit names candidate (s = x - i, d); the naive check
//     of the window against p_d decides.  For q = m (m <= 16) a hit is the whole pattern.
//
// Passes of a group search (host: epsm_multi.cu):
//   1. epsm_multi_kernel<SK, QW, false>  streams the text (TMA ring, as the single-pattern
//      scan) and filters it; per chunk (one 32 KiB tile) it writes the count of every
//      distinct pattern and, where the chunk holds at most kListCap occurrences, the list of
//      them as (chunk offset, id) -- so the positions of sparse chunks are never recomputed;
//   2. epsm_multi_scan_kernel            exclusive prefix over the chunks per distinct pattern
//      (where each chunk's positions go in each output), the totals (every search's occ),
//      and the list of chunks that hold occurrences at all;
//   3. epsm_multi_kernel<SK, QW, true>   visits only those chunks: a chunk with a list is
//      rebuilt from it (no text read), a dense chunk is streamed and filtered again; then the
//      positions of each distinct pattern are ranked in text order and written to every
//      search that asked for that pattern (Fig. 1 line 11: i*alpha + {r}).
// DRAM traffic of a group: the text once (plus dense chunks once more -- those are the
// chunks whose output is many bytes per text byte anyway) + the positions.
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

#include "epsm_ptx.cuh"

namespace epsm {
namespace mp {

constexpr int kTile = 32768;                      // bytes per chunk (one TMA stage)
constexpr int kHalo = 32;                         // >= m - 1 (m <= 32)
constexpr int kStageBytes = kTile + 128;          // tile + halo + unaligned-read slack
#ifndef EPSM_MULTI_ROT
#define EPSM_MULTI_ROT 1                             // lane-rotated piece loads of one-word grams
#endif
#ifndef EPSM_BLOOM_PRED
#define EPSM_BLOOM_PRED 1                            // second Bloom probe only where the first hit
#endif
#ifndef EPSM_MULTI_HALO_LDS
#define EPSM_MULTI_HALO_LDS 1                        // lane's bytes 64..79 loaded, not shuffled
#endif
constexpr int kStages = 4;
constexpr int kConsumerWarps = 16;
constexpr int kThreads = 32 + 32 * kConsumerWarps;   // producer warp + consumers
constexpr int kSegBytes = 64;                     // starts per lane
constexpr int kSliceBytes = 32 * kSegBytes;       // starts per warp and tile (2048)
constexpr int kBatches = kSliceBytes / 32;        // 32-start batches per slice (64)
constexpr int kMaxD = 255;                        // distinct patterns per group (u8 ids)
constexpr uint8_t kNoId = 0xFF;
constexpr int kBitmapLog = 16;                    // sample filter: 2^16 bits
constexpr int kBucketLog = 12;                    // table buckets: 2^12
constexpr int kMaxEntries = 4096;                 // (d, i) pairs: D * SK
constexpr int kMaxJobs = 1024;                    // searches per group
constexpr int kListCap = 256;                     // (offset, id) entries kept per chunk
constexpr int kMaxPW = 8;                         // pattern words (m <= 32)
constexpr int kCodeKeyBits = 14;                  // code mode: m * (bits per symbol) <= 14 (table)
constexpr int kWideKeyBits = 16;                  // ... <= 16 (bitmap + buckets: the wide code mode)
constexpr int kIdsLane = kSegBytes + 4;           // ids of one lane (padded: bank-conflict-free)
constexpr int kIdsWarp = 32 * kIdsLane;
__host__ __device__ constexpr uint32_t id_slot(uint32_t so) {   // slice offset -> ids index
  return (so / kSegBytes) * kIdsLane + so % kSegBytes;
}
static_assert(kSegBytes * 32 * kConsumerWarps == kTile, "lanes tile the chunk");

// The group's preprocessing (built on the host, copied into shared memory once per CTA).
struct __align__(16) GroupDesc {
  uint32_t bitmap[(1 << kBitmapLog) / 32];        // bit h >> 16 set <=> some gram hashes there
  uint16_t boff[(1 << kBucketLog) + 8];           // CSR offsets of bucket h >> 20 into ent
  uint16_t ent[kMaxEntries];                      // d << 8 | i << 4 | (h >> 16) & 15
  uint32_t pat[kMaxD + 1][kMaxPW];                // distinct patterns, zero padded, LE words
  uint32_t pmask[kMaxPW];                         // byte masks of the words (m bytes)
  uint16_t dup_off[kMaxD + 2];                    // searches of pattern d: dup_list[off[d] .. off[d+1])
  uint16_t dup_list[kMaxJobs];
  uint16_t job_d[kMaxJobs];                       // distinct pattern of (local) search j
  uint16_t job_g[kMaxJobs];                       // its index in the caller's batch (occ slot)
  uint8_t cmap[256];                              // code mode: byte -> symbol code, 0x80 = not a
                                                  // pattern byte (the key table overlays bitmap
                                                  // and boff: 2^14 bytes, key -> pattern or 0xFF)
};
static_assert(offsetof(GroupDesc, boff) == offsetof(GroupDesc, bitmap) + 8192 &&
                  sizeof(GroupDesc::bitmap) + sizeof(GroupDesc::boff) >= (1u << kCodeKeyBits),
              "code-mode key table overlays bitmap + boff");

struct JobOut {                 // where search j's positions go
  uint64_t* pos;
  uint64_t cap;
};

struct MParams {
  const uint8_t* text;          // 16-byte aligned virtual base
  uint64_t nbytes;              // readable bytes from text
  uint64_t s_lo, s_hi;          // valid virtual starts [s_lo, s_hi)
  uint64_t pos_bias;            // reported = virtual start + pos_bias
  uint32_t nchunks;             // tiles covering [0, s_hi)
  uint32_t it_lo, it_hi;        // interior tiles: every start in [s_lo, s_hi)
  uint32_t m, mw, D, k;         // pattern length, words, distinct patterns, searches
  uint32_t qmask;               // byte mask of the last key word
  uint32_t bloom2;              // second bitmap probe on (q > 2: hashed keys)
  uint32_t cb;                  // code mode: bits per symbol code
  uint32_t kmask;               // code mode: 2^(m * cb) - 1
  uint32_t mmask;               // code mode: 2^m - 1
  uint32_t spare;               // code mode: bytes outside the alphabet map to a spare code
  uint32_t ident;               // code mode: every pattern byte < 2^cb is its own code; a byte
                                // with a bit in identmask (at or above cb) is outside the alphabet
  uint32_t identmask;
  uint32_t direct;              // code mode, pass 1: count in the scan, no lists (dense groups: the
                                // chunks overflow their lists anyway and pass 3 re-filters them)
  uint32_t hmul[4];             // key word multipliers of the sample hash
  uint32_t desc_bytes;
  const GroupDesc* desc;
  uint16_t* counts;             // [nchunks][D]: pass 1 out
  uint32_t* listlen;            // [nchunks]: occurrences per chunk (pass 1 out)
  uint32_t* lists;              // [nchunks][kListCap]: offset | id << 16 (pass 1 out)
  const unsigned long long* prefix;   // [nchunks][D]: pass 3 in (scan out)
  uint32_t* work;               // [0] chunks with occurrences, [1 ..] their ids (scan out)
  const JobOut* jobs;           // pass 3: output of (local) search j (device memory)
};

struct ScanParams {
  const uint16_t* counts;
  const uint32_t* listlen;
  unsigned long long* prefix;   // NULL: totals only (count)
  uint32_t* work;
  unsigned long long* occ;      // the batch's occ array (slot job_g[j] for local search j)
  const GroupDesc* desc;        // job_d, job_g
  uint32_t nchunks, D, k;
};

#ifdef EPSM_MULTI_DEBUG
#include <cstdio>
#define MP_CHECK(cond, tag, a, b)                                                              \
  do {                                                                                         \
    if (!(cond)) {                                                                             \
      printf("MP_CHECK %s failed: %s a=%llu b=%llu blk=%d tid=%d\n", #cond, tag,               \
             (unsigned long long)(a), (unsigned long long)(b), (int)blockIdx.x, (int)threadIdx.x); \
      __trap();                                                                                \
    }                                                                                          \
  } while (0)
#else
#define MP_CHECK(cond, tag, a, b) do { } while (0)
#endif

template <int SK>
struct Geo {   // sample offsets 0, SK, .. (SK = 0: the code mode, every start keyed)
  static constexpr int kSamples = SK > 0 ? kSegBytes / (SK > 0 ? SK : 1) + (SK > 1 ? 1 : 0) : 0;
};

__device__ __forceinline__ void bar_consumers() {   // named barrier over the 16 consumer warps
  asm volatile("bar.sync 1, %0;" ::"n"(32 * kConsumerWarps) : "memory");
}

// bits 0..15 of x to the even bit positions 0, 2, .., 30
__device__ __forceinline__ uint32_t spread16(uint32_t x) {
  x = (x | (x << 8)) & 0x00FF00FFu;
  x = (x | (x << 4)) & 0x0F0F0F0Fu;
  x = (x | (x << 2)) & 0x33333333u;
  x = (x | (x << 1)) & 0x55555555u;
  return x;
}

// 4 bytes at an arbitrary shared-memory byte offset (4-byte aligned base)
__device__ __forceinline__ uint32_t lds_u32_any(const uint8_t* base, uint32_t off) {
  const uint32_t* w = reinterpret_cast<const uint32_t*>(base + (off & ~3u));
  return __funnelshift_r(w[0], w[1], 8 * (off & 3u));
}

// the second probe of the sample bitmap: a remix of the gram hash (host and device alike)
__host__ __device__ __forceinline__ uint32_t bloom2(uint32_t h) { return (h ^ (h >> 15)) * 0x2C1B3C6Du; }

// a shared-memory word loaded only by the lanes with pred != 0 (0 elsewhere): the inactive
// lanes of the LDS take no bank cycles
__device__ __forceinline__ uint32_t lds_pred(const uint32_t* p, uint32_t pred) {
  uint32_t v = 0;
  const uint32_t a = static_cast<uint32_t>(__cvta_generic_to_shared(p));
  asm("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\t@q ld.shared.u32 %0, [%1];\n\t}"
      : "+r"(v) : "r"(a), "r"(pred));
  return v;
}

// The sample filter's bit for gram hash h: two-probe (Bloom) test, both bits set for every
// table gram (false positives D*SK/2^16 -> (that)^2: one warp in ~3 instead of every warp walks
// a bucket per chunk); q <= 2 (bloom2 off): the key itself, one exact probe.  The second probe
// is loaded only by the lanes whose first probe hit (a few per warp: the random first probes
// cost ~4 bank cycles per warp, the second ~1).
// (plain shifts, not the volatile shf asm of __funnelshift_r: the samples' chains interleave)
__device__ __forceinline__ uint32_t sample_bit(uint32_t h, const GroupDesc& G, const MParams& P);

template <int QW>
__device__ __forceinline__ uint32_t hash_words(const uint32_t (&k)[4], const MParams& P) {
  uint32_t h = k[0] * P.hmul[0];
#pragma unroll
  for (int r = 1; r < QW; ++r) h += k[r] * P.hmul[r];
  return h;
}

// Shared-memory layout of the group kernel.
template <bool WRITE>
struct __align__(128) MSmemT {
  static constexpr int kS = WRITE ? kStages - 1 : kStages;   // pass 3 gives a stage to lbuf
  uint8_t ring[kS][kStageBytes];
  GroupDesc g;
  uint8_t ids[kConsumerWarps][kIdsWarp];             // id of the pattern at each start, kNoId
                                                     // (lane l's 64 starts at l * 68: a lane stride of
                                                     // 17 words keeps the lanes' stores conflict-free)
  uint16_t hist[kConsumerWarps][kMaxD + 1];          // per-slice counts -> exclusive offsets
  uint64_t* cptr[kMaxD + 1];                         // pass 3: the chunk's first slot of each pattern
                                                     // (its first output + the chunk's prefix)
  uint32_t ccnt[kS][kMaxD + 1];                 // pass 1: chunk counts (by stage)
  uint32_t lcur[kS];                            // pass 1: list cursor (by stage)
  uint32_t done[kS];                            // pass 1: warps finished with the stage
  unsigned long long lm[kConsumerWarps][32];         // lane match masks of a slice (list path)
  uint32_t rbuf[kConsumerWarps][32];                 // pass 3: a round of 32 matches (offset | id << 16)
  uint16_t lbuf[WRITE ? kConsumerWarps : 1][WRITE ? kSliceBytes / 2 : 1];   // pass 3: a half slice's
                                                     // matches (slice offsets), text order
  uint64_t* opos[kMaxD + 1];                         // pass 3: the first output of each pattern ...
  uint64_t* oend[kMaxD + 1];                         // ... and its end (first + capacity)
  alignas(8) uint64_t full[kS];
  uint64_t empty[kS];
  uint64_t gfull;
  uint32_t info[kS];                            // chunk | kInfoList, or kEnd
  uint32_t ilen[kS];                            // list length (list stages)
};
static_assert(sizeof(MSmemT<false>) <= 232448 && sizeof(MSmemT<true>) <= 232448,
              "group kernel fits 227 KB of shared memory");
constexpr uint32_t kEnd = 0xFFFFFFFFu;
constexpr uint32_t kInfoList = 0x80000000u;

__device__ __forceinline__ uint32_t sample_bit(uint32_t h, const GroupDesc& G, const MParams& P) {
  uint32_t bit = G.bitmap[h >> (32 - kBitmapLog + 5)] >> ((h >> (32 - kBitmapLog)) & 31u);
  if (P.bloom2) {
    const uint32_t h2 = bloom2(h);
#if EPSM_BLOOM_PRED
    const uint32_t bw2 = lds_pred(&G.bitmap[h2 >> (32 - kBitmapLog + 5)], bit & 1u);
#else
    const uint32_t bw2 = G.bitmap[h2 >> (32 - kBitmapLog + 5)];
#endif
    bit &= bw2 >> ((h2 >> (32 - kBitmapLog)) & 31u);
  }
  return bit & 1u;
}

// Naive check of the window at stage offset st against distinct pattern d.
__device__ __forceinline__ bool verify_window(const uint8_t* ts, uint32_t st, const GroupDesc& G, uint32_t d,
                                              uint32_t mw) {
  const uint32_t* w = reinterpret_cast<const uint32_t*>(ts + (st & ~3u));
  const uint32_t sh = 8 * (st & 3u);
  uint32_t lo = w[0];
  for (uint32_t r = 0; r < mw; ++r) {
    const uint32_t hi = w[r + 1];
    if ((__funnelshift_r(lo, hi, sh) ^ G.pat[d][r]) & G.pmask[r]) return false;
    lo = hi;
  }
  return true;
}

// Code mode: the lane's 80 bytes (64 starts + halo) keyed through the patterns' symbol codes.
// Byte t maps to its code (cmap); the rolling key over t holds the codes of bytes t-m+1 .. t
// (byte t in the low bits), i.e. the window of start t-m+1, and the key table names the pattern
// with exactly those m bytes (or 0xFF) -- EPSMa's per-position compare for all
// patterns at once, exact, so no naive check.  Returns the lane's match mask (bit s: start s).
// DIRECT: count each match into cc[pattern] (shared atomics); else store every start's id
// (0xFF: none) into idb[0..63].
// WIDE (keys of 15-16 bits): the key's bit in the bitmap (exact membership), and on a hit (rare:
// the mode is chosen for sparse groups) the pattern from the key's bucket (key >> 4) whose entry
// holds the key's low 4 bits -- the bucket and the fingerprint together are the whole key.
template <bool WIDE>
__device__ __forceinline__ uint32_t code_lookup(const GroupDesc& G, uint32_t key) {
  if constexpr (!WIDE) {
    return reinterpret_cast<const uint8_t*>(G.bitmap)[key];
  } else {
    if (((G.bitmap[key >> 5] >> (key & 31u)) & 1u) == 0) return 0xFFu;
    const uint32_t bk = key >> 4, e1 = G.boff[bk + 1];
    for (uint32_t e = G.boff[bk]; e < e1; ++e) {
      const uint32_t v = G.ent[e];
      if ((v & 15u) == (key & 15u)) return v >> 8;
    }
    return 0xFFu;
  }
}

template <bool DIRECT, bool WIDE, bool SPARE, bool IDENT>
__device__ __forceinline__ uint64_t code_scan_t(const uint32_t (&W)[20], const GroupDesc& G, const MParams& P,
                                                uint8_t* idb, uint32_t* cc) {
  const uint32_t m1 = P.m - 1, cb = P.cb, kmask = P.kmask;
  uint32_t key = 0, e0 = 0, e1 = 0, e2 = 0, any = 0;
  int last_inv = -64;                            // last byte outside the patterns' alphabet
  uint8_t* const ids0 = idb - m1;                // id slot of the start closed by byte t: ids0[t]
#pragma unroll
  for (int t = 0; t < 80; ++t) {
    const uint32_t by = (W[t >> 2] >> (8 * (t & 3))) & 0xFFu;
    const uint32_t cm = IDENT ? by : G.cmap[by];   // (IDENT: the byte is its own code, no load)
    key = ((key << cb) | cm) & kmask;
    uint32_t d;
    if constexpr (SPARE) {
      // bytes outside the alphabet have the spare code: no pattern key holds it (table: 0xFF)
      d = code_lookup<WIDE>(G, key);
    } else {
      if (cm & (IDENT ? P.identmask : 0x80u)) last_inv = t;   // (its high bits leave the key within m bytes)
      d = (t - last_inv > static_cast<int>(m1)) ? code_lookup<WIDE>(G, key) : 0xFFu;
    }
    const uint32_t s0 = static_cast<uint32_t>(t) - m1;
    const bool mine = s0 < static_cast<uint32_t>(kSegBytes);
    if constexpr (DIRECT) {
      if (mine && d != 0xFFu) {
        atomicAdd(&cc[d], 1u);
        any = 1u;
      }
    } else {
      if (mine) ids0[t] = static_cast<uint8_t>(d);
      const uint32_t hit = d != 0xFFu ? 1u : 0u;
      if (t < 32) e0 |= hit << t;
      else if (t < 64) e1 |= hit << (t - 32);
      else e2 |= hit << (t - 64);
    }
  }
  if constexpr (DIRECT) return any;              // (pass 1 counts directly: only "any match")
  // starts = window ends - m1 (m1 <= 13): the lane's 64 starts out of the 80 ends
  const uint64_t lo = (static_cast<uint64_t>(e1) << 32) | e0;
  return m1 ? ((lo >> m1) | (static_cast<uint64_t>(e2) << (64 - m1))) : lo;
}

template <bool DIRECT, bool WIDE>
__device__ __forceinline__ uint64_t code_scan(const uint32_t (&W)[20], const GroupDesc& G, const MParams& P,
                                              uint8_t* idb, uint32_t* cc) {
  if (P.ident) return code_scan_t<DIRECT, WIDE, false, true>(W, G, P, idb, cc);
  return P.spare ? code_scan_t<DIRECT, WIDE, true, false>(W, G, P, idb, cc)
                 : code_scan_t<DIRECT, WIDE, false, false>(W, G, P, idb, cc);
}

template <int SK, int QW, bool WRITE>
__global__ void __launch_bounds__(kThreads, 1) epsm_multi_kernel(const __grid_constant__ MParams P) {
  extern __shared__ __align__(128) uint8_t smem_raw[];
  using MSmem = MSmemT<WRITE>;
  constexpr int kStages = MSmem::kS;
  MSmem& S = *reinterpret_cast<MSmem*>(smem_raw);
  const uint32_t tid = threadIdx.x;
  const uint32_t lane = tid & 31u;
  const uint32_t warp = tid >> 5;

  if (tid < static_cast<uint32_t>(kStages)) {
    mbar_init(&S.full[tid], 1);
    mbar_init(&S.empty[tid], kConsumerWarps);
    S.lcur[tid] = 0;
    S.done[tid] = 0;
    fence_mbar_init();
  } else if (tid == 32) {
    mbar_init(&S.gfull, 1);
    fence_mbar_init();
  }
  // ids start empty; chunk counters zero
  for (uint32_t i = tid; i < kConsumerWarps * kIdsWarp / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(&S.ids[0][0])[i] = make_uint4(~0u, ~0u, ~0u, ~0u);   // (kIdsWarp % 16 == 0)
  for (uint32_t i = tid; i < kStages * (kMaxD + 1); i += blockDim.x) (&S.ccnt[0][0])[i] = 0;
  for (uint32_t i = tid; i < kConsumerWarps * (kMaxD + 1); i += blockDim.x) (&S.hist[0][0])[i] = 0;
  if (!WRITE && blockIdx.x == 0 && tid == 0) P.work[0] = 0;   // (the scan appends; runs after)
  __syncthreads();

  if (warp == 0) {
    // ================================================================ producer
    if (lane == 0) {
      mbar_arrive_expect_tx(&S.gfull, P.desc_bytes);
      // (in pieces of at most 8 KiB)
      for (uint32_t a = 0; a < P.desc_bytes; a += 8192u) {
        const uint32_t b = P.desc_bytes - a < 8192u ? P.desc_bytes - a : 8192u;
        bulk_g2s_plain(reinterpret_cast<uint8_t*>(&S.g) + a, reinterpret_cast<const uint8_t*>(P.desc) + a, b,
                       &S.gfull);
      }
    }
    const uint64_t policy = policy_evict_first();
    uint32_t stage = 0, phase = 0;
    // (the work count is read through its own pointer: a ternary between a volatile load and a
    // __grid_constant__ member once compiled into a volatile load from the parameter's address)
    uint32_t nwork = P.nchunks;
    if constexpr (WRITE) nwork = *reinterpret_cast<volatile const uint32_t*>(P.work);
    for (uint32_t w = blockIdx.x; w < nwork; w += gridDim.x) {
      const uint32_t c = WRITE ? P.work[1 + w] : w;
      uint32_t len = 0;
      if (WRITE) len = P.listlen[c];
      mbar_wait_sleep(&S.empty[stage], phase ^ 1u, 256);
      if (WRITE && len <= static_cast<uint32_t>(kListCap)) {
        // a sparse chunk: its occurrences were listed by pass 1; the text is not needed
        if (lane == 0) {
          S.info[stage] = c | kInfoList;
          S.ilen[stage] = len;
          const uint32_t bytes = (len * 4u + 15u) & ~15u;
          mbar_arrive_expect_tx(&S.full[stage], bytes);
          bulk_g2s_plain(S.ring[stage], P.lists + static_cast<uint64_t>(c) * kListCap, bytes, &S.full[stage]);
        }
      } else {
        const uint64_t base = static_cast<uint64_t>(c) * kTile;
        const uint64_t want_end = base + kTile + kHalo;
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
      }
      if (++stage == kStages) {
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

  // ================================================================== consumers
  const uint32_t cw = warp - 1;
  const uint32_t seg = cw * kSliceBytes + lane * kSegBytes;    // the lane's 64 starts in a tile
  const uint32_t lt = (1u << lane) - 1u;
  mbar_wait(&S.gfull, 0);
  if constexpr (WRITE) {
    // the first output of every pattern, out of the job table (global) into shared memory: the
    // store of a match then needs no dependent global load
    for (uint32_t d = tid - 32; d < P.D; d += 32 * kConsumerWarps) {
      const JobOut J = P.jobs[S.g.dup_list[S.g.dup_off[d]]];
      S.opos[d] = J.pos;
      S.oend[d] = J.pos ? J.pos + J.cap : J.pos;
    }
    bar_consumers();
  }
  const GroupDesc& G = S.g;
  uint32_t stage = 0, phase = 0;
  uint8_t* const ids = S.ids[cw];
  while (true) {
    mbar_wait(&S.full[stage], phase);
    const uint32_t info = S.info[stage];
    if (info == kEnd) break;
    const uint32_t c = info & ~kInfoList;
    const uint8_t* ts = S.ring[stage];
    uint64_t M = 0;                     // this lane's matched starts (bit i: slice offset 64 lane + i)
    bool direct = false;                // pass 1, code mode: counted in the scan, no ids
    if (WRITE && (info & kInfoList)) {
      // ---- rebuild the chunk's ids from its list (pass 1 kept it: no text)
      S.lm[cw][lane] = 0;
      bar_consumers();
      const uint32_t len = S.ilen[stage];
      const uint32_t* L = reinterpret_cast<const uint32_t*>(ts);
      for (uint32_t e = tid - 32; e < len; e += 32 * kConsumerWarps) {
        const uint32_t v = L[e];
        const uint32_t off = v & 0xFFFFu, d = v >> 16;
        S.ids[off / kSliceBytes][id_slot(off % kSliceBytes)] = static_cast<uint8_t>(d);
        atomicOr(&S.lm[off / kSliceBytes][(off % kSliceBytes) / kSegBytes], 1ull << (off % kSegBytes));
      }
      bar_consumers();
      M = S.lm[cw][lane];
    } else {
      // ---- filter the warp's slice: one sample every SK bytes (EPSMc)
      uint32_t W[20];
      {
        const uint4* src = reinterpret_cast<const uint4*>(ts + seg);
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          const uint4 v = src[r];
          W[4 * r] = v.x;
          W[4 * r + 1] = v.y;
          W[4 * r + 2] = v.z;
          W[4 * r + 3] = v.w;
        }
        // bytes 64..79: the next lane's first 16 (lane 31: the next slice / the tile halo)
#if EPSM_MULTI_HALO_LDS
        {                                   // (one more independent load: no shuffle waiting on
          const uint4 v = src[4];           // the first load on every sample chain)
          W[16] = v.x;
          W[17] = v.y;
          W[18] = v.z;
          W[19] = v.w;
        }
#else
#pragma unroll
        for (int r = 0; r < 4; ++r) W[16 + r] = __shfl_down_sync(0xffffffffu, W[r], 1);
        if (lane == 31) {
          const uint4 v = src[4];
          W[16] = v.x;
          W[17] = v.y;
          W[18] = v.z;
          W[19] = v.w;
        }
#endif
      }
      if constexpr (SK <= 0) {
        // ---- code mode (dense groups, small pattern alphabets): every start keyed exactly.
        // Byte t of the lane's window maps to its symbol code; the rolling key over t holds the
        // codes of bytes t-m+1 .. t (byte t in the low bits), i.e. the window of start t-m+1;
        // the key table names the pattern with exactly those m bytes (or none) -- EPSMa's
        // per-position compare for all patterns at once, without a naive check.
        // Every start of the lane gets its id (0xFF: none) -- no stale ids -- and bit t of
        // E marks the window ENDING at byte t (compile-time bit positions).
        uint8_t* const idb = ids + lane * kIdsLane;
        if (!WRITE && P.direct && c >= P.it_lo && c < P.it_hi) {
          // pass 1 over an interior chunk: count straight into the chunk's counters (no ids,
          // no list: the chunk is re-filtered by pass 3)
          M = code_scan<true, (SK < 0)>(W, G, P, idb, S.ccnt[stage]);
          direct = true;
        } else {
          M = code_scan<false, (SK < 0)>(W, G, P, idb, nullptr);
        }
        if (!(c >= P.it_lo && c < P.it_hi)) {
          // a chunk at the text's ends: starts outside [s_lo, s_hi) do not count (their ids are
          // cleared again below with the others)
          const uint64_t ub = static_cast<uint64_t>(c) * kTile + seg;
          uint64_t keep = ~0ull;
          if (ub + 64 > P.s_hi) keep = P.s_hi <= ub ? 0ull : (~0ull >> (64 - (P.s_hi - ub)));
          if (ub < P.s_lo) keep &= P.s_lo >= ub + 64 ? 0ull : (~0ull << (P.s_lo - ub));
          uint64_t drop = M & ~keep;
          M &= keep;
          while (drop) {
            idb[__ffsll(static_cast<long long>(drop)) - 1] = kNoId;
            drop &= drop - 1;
          }
        }
      }
      constexpr int NS = Geo<SK>::kSamples;
      uint64_t hits = 0;
      uint32_t hit64 = 0;                         // the sample at offset 64 (SK > 1)
      // one-word grams at whole-word strides (q <= 4, SK = 4, 8, 16): the lane reads its four
      // 16-byte pieces in a lane-rotated order (piece (r + lane/2) mod 4 at step r), so a
      // quarter-warp's loads hit distinct bank groups instead of one (64-byte lane stride:
      // 16-way conflicted 32-bit loads); the sample at byte 64 is the next lane's sample 0
      constexpr bool kRot = EPSM_MULTI_ROT && QW == 1 && SK >= 4 && SK <= 16;
      if constexpr (kRot) {
        constexpr int PER = 16 / (kRot ? SK : 16);   // samples per 16-byte piece
        const uint32_t rot = (lane >> 1) & 3u;
        const uint8_t* lp = ts + seg;
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          const uint32_t pc = (static_cast<uint32_t>(r) + rot) & 3u;
          const uint4 v = *reinterpret_cast<const uint4*>(lp + 16u * pc);
          const uint32_t vw[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
          for (int u = 0; u < PER; ++u) {
            const uint32_t key = vw[u * (SK / 4)] & P.qmask;
            hits |= static_cast<uint64_t>(sample_bit(key * P.hmul[0], G, P)) << (pc * PER + u);
          }
        }
        // the sample at byte 64: the next lane's sample 0 (lane 31: the next slice / the halo)
        uint32_t b64 = __shfl_down_sync(0xffffffffu, static_cast<uint32_t>(hits & 1u), 1);
        if (lane == 31) b64 = sample_bit((*reinterpret_cast<const uint32_t*>(lp + 64) & P.qmask) * P.hmul[0], G, P);
        hits |= static_cast<uint64_t>(b64) << (4 * PER);
      }
#pragma unroll
      for (int j = 0; j < (kRot ? 0 : NS); ++j) {
        // key words r < QW at the compile-time byte offset j * SK + 4r of the lane's registers
        uint32_t k[4];
#pragma unroll
        for (int r = 0; r < QW; ++r) {
          const int b = j * SK + 4 * r;
          const int wi = b >> 2, sh = b & 3;
          k[r] = sh == 0 ? W[wi] : ((W[wi] >> (8 * sh)) | (W[wi + 1] << (32 - 8 * sh)));
        }
        k[QW - 1] &= P.qmask;
        const uint32_t h = hash_words<QW>(k, P);
        MP_CHECK((h >> (32 - kBitmapLog + 5)) < 2048u, "bitmap", h, j);
        // two-probe (Bloom) test: both bits set for every table gram (false positives
        // D*SK/2^16 -> (that)^2: one warp in ~3 instead of every warp walks a bucket per chunk)
        // (plain shifts, not the volatile shf asm of __funnelshift_r: the samples' chains interleave)
        const uint32_t bit = sample_bit(h, G, P);
        if (j < 64) hits |= static_cast<uint64_t>(bit) << j;
        else hit64 = bit;
      }
      if (SK > 0 && __any_sync(0xffffffffu, (hits | hit64) != 0)) {
        const uint64_t tbase = static_cast<uint64_t>(c) * kTile;
        const bool interior = c >= P.it_lo && c < P.it_hi;
        // candidates: every table entry (d, i) of the sample's bucket with
        // the sample's fingerprint bits names the start x - i of pattern d; naive check
        uint64_t hm = hits;
        uint32_t h64 = hit64;
        while (hm | h64) {
          uint32_t o;
          if (hm) {
            o = (__ffsll(static_cast<long long>(hm)) - 1) * SK;
            hm &= hm - 1;
          } else {
            o = 64;
            h64 = 0;
          }
          const uint32_t xt = seg + o;               // the sample's stage offset
          uint32_t k[4];
#pragma unroll
          for (int r = 0; r < QW; ++r) k[r] = lds_u32_any(ts, xt + 4 * r);
          k[QW - 1] &= P.qmask;
          const uint32_t h = hash_words<QW>(k, P);
          const uint32_t bk = h >> (32 - kBucketLog);
          const uint32_t fp = (h >> (32 - kBitmapLog)) & 15u;
          const uint32_t e1 = G.boff[bk + 1];
          MP_CHECK(e1 <= 4096u && G.boff[bk] <= e1, "boff", bk, e1);
          for (uint32_t e = G.boff[bk]; e < e1; ++e) {
            const uint32_t v = G.ent[e];
            MP_CHECK((v >> 8) < P.D, "ent", v, e);
            if ((v & 15u) != fp) continue;
            const uint32_t i = (v >> 4) & 15u, d = v >> 8;
            if (i > o || o - i >= static_cast<uint32_t>(kSegBytes)) continue;   // not the lane's start
            const uint32_t st = xt - i;                   // start, stage offset
            if (!interior) {
              const uint64_t vs = tbase + st;
              if (vs < P.s_lo || vs >= P.s_hi) continue;
            }
            MP_CHECK(st < static_cast<uint32_t>(kTile + 64), "st", st, o);
            if (verify_window(ts, st, G, d, P.mw)) {
              ids[lane * kIdsLane + (o - i)] = static_cast<uint8_t>(d);
              M |= 1ull << (o - i);
            }
          }
        }
      }
      __syncwarp();
    }
    // this lane's matches: count and exclusive offset among the warp slice's (text order)
    const uint32_t cl = static_cast<uint32_t>(__popcll(static_cast<long long>(M)));
    uint32_t incl = cl, T = 0;
    if (__any_sync(0xffffffffu, cl != 0)) {                       // (most slices of a sparse group:
#pragma unroll                                                    // none -- no scan chain)
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= static_cast<uint32_t>(o)) incl += y;
      }
      T = __shfl_sync(0xffffffffu, incl, 31);                     // matches of the slice
    }
    uint8_t* const idl = ids + lane * kIdsLane;

    if constexpr (!WRITE) {
      // ---- pass 1: counts per distinct pattern (per-match shared atomics), and the chunk's
      // list while it is short (order irrelevant here: one warp-aggregated slot reservation)
      uint32_t* const cc = S.ccnt[stage];
      if (direct) {
        // (counted already; a chunk with matches is marked dense: pass 3 re-filters it)
        if (T && lane == 0) atomicAdd(&S.lcur[stage], T + kListCap + 1);
      } else if (T) {
        uint32_t base = 0;
        if (lane == 0) base = atomicAdd(&S.lcur[stage], T);
        uint32_t r = __shfl_sync(0xffffffffu, base, 0) + incl - cl;
        uint64_t mm = M;
        while (mm) {
          const uint32_t bit = __ffsll(static_cast<long long>(mm)) - 1;
          mm &= mm - 1;
          const uint32_t id = idl[bit];
          idl[bit] = kNoId;
          MP_CHECK(id < P.D, "id", id, bit);
          atomicAdd(&cc[id], 1u);
          if (r < static_cast<uint32_t>(kListCap))
            P.lists[static_cast<uint64_t>(c) * kListCap + r] = (cw * kSliceBytes + lane * kSegBytes + bit) | (id << 16);
          ++r;
        }
      }
      __syncwarp();
      uint32_t prev = 0;
      if (lane == 0) {
        __threadfence_block();
        prev = atomicAdd(&S.done[stage], 1u);
      }
      prev = __shfl_sync(0xffffffffu, prev, 0);
      if (prev == kConsumerWarps - 1) {
        // the last warp of the chunk publishes its counts and resets the stage's counters
        __threadfence_block();
        for (uint32_t d = lane; d < P.D; d += 32) {
          P.counts[static_cast<uint64_t>(d) * P.nchunks + c] = static_cast<uint16_t>(cc[d]);
          cc[d] = 0;
        }
        if (lane == 0) {
          P.listlen[c] = S.lcur[stage];
          S.lcur[stage] = 0;
          S.done[stage] = 0;
        }
        __syncwarp();
      }
      if (lane == 0) mbar_arrive(&S.empty[stage]);
    } else {
      // ---- pass 3: rank every occurrence among its pattern's in text order, then write it to
      // each search that asked for that pattern at prefix + rank
      uint16_t* const hw = S.hist[cw];
      {
        // the slice's count of every pattern (u16 counters, two per 32-bit word); with more than
        // one round, the first half slice's matches also go to lbuf (see below) on the way
        uint32_t* const hw32 = reinterpret_cast<uint32_t*>(hw);
        uint16_t* const lb = S.lbuf[cw];
        const bool fill = T > 32 && lane < 16;
        uint32_t k = incl - cl;
        uint64_t mm = M;
        while (mm) {
          const uint32_t bit = __ffsll(static_cast<long long>(mm)) - 1;
          mm &= mm - 1;
          const uint32_t id = idl[bit];
          atomicAdd(&hw32[id >> 1], 1u << (16 * (id & 1u)));
          if (fill) lb[k++] = static_cast<uint16_t>(lane * kSegBytes + bit);
        }
        __syncwarp();
      }
      if (lane == 0) mbar_arrive(&S.empty[stage]);   // (lists and text both consumed)
      bar_consumers();
      // exclusive offsets of every slice inside the chunk, per pattern; the chunk's prefix
      for (uint32_t d = tid - 32; d < P.D; d += 32 * kConsumerWarps) {
        uint32_t run = 0;
#pragma unroll 4
        for (int w = 0; w < kConsumerWarps; ++w) {
          const uint32_t v = S.hist[w][d];
          S.hist[w][d] = static_cast<uint16_t>(run);
          run += v;
        }
        S.cptr[d] = S.opos[d] + P.prefix[static_cast<uint64_t>(d) * P.nchunks + c];
      }
      bar_consumers();
      const uint64_t cbase = static_cast<uint64_t>(c) * kTile + P.pos_bias + cw * kSliceBytes;
      // the slice's matches in text order, 32 per round: every lane emits its own (in bit order)
      // into the round buffer, then lane i takes match R + i -- ranks by match_any on the ids
      uint32_t* const rb = S.rbuf[cw];
      uint64_t mm = M;
      uint32_t idx = incl - cl;
      if (T > 32) {
        // more than one round: each half slice's matches (lanes 16h .. 16h + 15) are compacted into
        // lbuf in text order (every lane writes its own run at its exclusive offset), then ranked 32
        // per round -- a round costs one match_any however the matches spread over the lanes
        uint16_t* const lb = S.lbuf[cw];
        const uint32_t t15 = __shfl_sync(0xffffffffu, incl, 15);
#pragma unroll 1
        for (uint32_t h = 0; h < 2; ++h) {
          const uint32_t hb = h ? t15 : 0u, th = h ? T - t15 : t15;
          if (th == 0) continue;
          if (h == 1 && (lane >> 4) == 1) {              // (half 0: filled with the counts)
            uint32_t k = incl - cl - hb;
            while (mm) {
              const uint32_t bit = __ffsll(static_cast<long long>(mm)) - 1;
              mm &= mm - 1;
              lb[k++] = static_cast<uint16_t>(lane * kSegBytes + bit);
            }
          }
          __syncwarp();
#pragma unroll 1
          for (uint32_t R = 0; R < th; R += 32) {
            const bool act = R + lane < th;
            const uint32_t off = act ? lb[R + lane] : 0u;
            uint32_t id = kNoId;
            if (act) {                                 // (the id slot is reset as it is read)
              uint8_t* const ip = ids + id_slot(off);
              id = *ip;
              *ip = kNoId;
            }
            const uint32_t peers = __match_any_sync(0xffffffffu, id);
            uint64_t* dst = nullptr;
            if (act) dst = S.cptr[id] + hw[id] + __popc(peers & lt);
            __syncwarp();
            if (act && (peers & lt) == 0) hw[id] = static_cast<uint16_t>(hw[id] + __popc(peers));
            if (act && dst < S.oend[id]) st_stream_u64(dst, cbase + off);   // (duplicates: copied after)
            __syncwarp();                              // (the next round reads hw)
          }
          __syncwarp();                                // (lbuf is refilled by the next half)
        }
        idx = T;                                      // (the round loop below has nothing left)
      }
      for (uint32_t R = T > 32 ? T : 0; R < T; R += 32) {
        while (mm && idx < R + 32) {
          const uint32_t bit = __ffsll(static_cast<long long>(mm)) - 1;
          mm &= mm - 1;
          const uint32_t id = idl[bit];
          idl[bit] = kNoId;
          rb[idx - R] = (lane * kSegBytes + bit) | (id << 16);
          ++idx;
        }
        __syncwarp();
        const bool act = R + lane < T;
        const uint32_t e = act ? rb[lane] : 0u;
        const uint32_t id = act ? (e >> 16) : static_cast<uint32_t>(kNoId);
        const uint32_t peers = __match_any_sync(0xffffffffu, id);
        uint64_t* dst = nullptr;
        if (act) dst = S.cptr[id] + hw[id] + __popc(peers & lt);
        __syncwarp();
        if (act && (peers & lt) == 0) hw[id] = static_cast<uint16_t>(hw[id] + __popc(peers));
        if (act) {
          const uint64_t pos = cbase + (e & 0xFFFFu);
          if (dst < S.oend[id]) st_stream_u64(dst, pos);   // (duplicates: copied after)
        }
        __syncwarp();                                  // (the round buffer is refilled next)
      }
      __syncwarp();
      // the warp's offsets are spent: zero its row for the next chunk (no other warp reads it
      // before the next chunk's first barrier)
      for (uint32_t d = lane; d < P.D; d += 32) hw[d] = 0;
      __syncwarp();
    }
    if (++stage == kStages) {
      stage = 0;
      phase ^= 1u;
    }
  }
}

// Pass 2: per distinct pattern, the exclusive prefix of its chunk counts (where each chunk's
// positions start in every output of that pattern) and its total (the occ of every search of
// that pattern); plus the list of chunks with occurrences.  Block d < D scans
// pattern d's row of counts ([D][nchunks], contiguous) 1024 chunks at a time (coalesced loads,
// warp + block scans, a running carry); block D builds the work list.
constexpr int kScanThreads = 1024;
__global__ void __launch_bounds__(kScanThreads) epsm_multi_scan_kernel(const __grid_constant__ ScanParams P) {
  __shared__ unsigned long long wsum[kScanThreads / 32];
  __shared__ unsigned long long carry_s;
  const uint32_t lane = threadIdx.x & 31u, w = threadIdx.x >> 5;
  const uint32_t d = blockIdx.x;
  if (d < P.D) {
    const uint16_t* row = P.counts + static_cast<uint64_t>(d) * P.nchunks;
    unsigned long long* prow = P.prefix ? P.prefix + static_cast<uint64_t>(d) * P.nchunks : nullptr;
    unsigned long long carry = 0;
    for (uint32_t c0 = 0; c0 < P.nchunks; c0 += kScanThreads) {
      const uint32_t c = c0 + threadIdx.x;
      const uint32_t v = c < P.nchunks ? row[c] : 0u;
      uint32_t x = v;                                            // warp inclusive scan
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= static_cast<uint32_t>(o)) x += y;
      }
      if (lane == 31) wsum[w] = x;
      __syncthreads();
      if (w == 0) {                                              // scan of the warp sums
        unsigned long long s = wsum[lane], t = s;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const unsigned long long y = __shfl_up_sync(0xffffffffu, t, o);
          if (lane >= static_cast<uint32_t>(o)) t += y;
        }
        wsum[lane] = t - s;                                      // exclusive
        if (lane == 31) carry_s = t;                             // tile total
      }
      __syncthreads();
      if (prow && c < P.nchunks) prow[c] = carry + wsum[w] + (x - v);
      carry += carry_s;
      __syncthreads();
    }
    if (threadIdx.x == 0) {
      // every search of pattern d gets its total
      for (uint32_t q = P.desc->dup_off[d]; q < P.desc->dup_off[d + 1]; ++q)
        P.occ[P.desc->job_g[P.desc->dup_list[q]]] = carry;
    }
    return;
  }
  // block D: chunks with occurrences (order irrelevant: each is handled on its own)
  if (!P.prefix) return;
  for (uint32_t c0b = 0; c0b < P.nchunks; c0b += blockDim.x) {
    const uint32_t cc = c0b + threadIdx.x;
    const bool ne = cc < P.nchunks && P.listlen[cc] > 0;
    const uint32_t bal = __ballot_sync(0xffffffffu, ne);
    uint32_t base = 0;
    if (lane == 0 && bal) base = atomicAdd(P.work, static_cast<uint32_t>(__popc(bal)));
    base = __shfl_sync(0xffffffffu, base, 0);
    if (ne) P.work[1 + base + __popc(bal & ((1u << lane) - 1u))] = cc;
  }
}

}  // namespace mp
}  // namespace epsm
