// epsm_kernels.cuh -- sm_100a kernels of the exact packed string matcher.
//
// One persistent CTA per SM, warp-specialised:
//
//   warp 0      producer   fetches CHUNK ids (4 consecutive 32 KiB tiles = 128 KiB; the
//                          first one is static, the rest come from a global counter) and
//                          streams every tile plus a 32-byte halo (>= m-1 for m <= 32)
//                          into a shared-memory ring with ONE TMA bulk copy per tile
//                          (cp.async.bulk ... mbarrier::complete_tx); the chunk ids are
//                          drawn two ahead so the atomic never stalls the issue.  The
//                          halo is the GPU analogue of EPSMb's wsblend, which only exists
//                          to avoid unaligned loads: shared memory is
//                          byte addressable, so every alignment is read directly.
//   warps 2-17  consumers  each lane owns 64 contiguous text bytes of a tile (4 units of
//                          alpha = 16 candidate starts), a warp a 2 KiB
//                          slice.  The 16 consumer warps never wait for each other (no block
//                          barrier): per-chunk bookkeeping is one shared-memory atomic, and
//                          each warp writes out its own slices:
//       filter   m <= 8: EPSMa's shift-AND (Fig. 1 lines 5-9), packed:
//                Z_k = OR_{i<F} ( S_i[k] XOR B_i ), S_i = the text shifted by i bytes,
//                B_i = p_i * 0x01010101.  A zero byte j of Z_k
//                <=> t[u+4k+j+i] = p_i for all i < F = min(m, 4).  Pair stage first,
//                extended to F bytes only where the pair has candidates.
//                m >= 9: EPSMc's block fingerprints: one gram every SK
//                bytes, looked up in a shared-memory table of the pattern's grams.
//       verify   the "naive check" of each candidate against the
//                zero-padded pattern blocks P_i, last word masked.
//       count    popcount of the 64-bit lane match mask.
//       masks    tiles with matches park their lane masks (8 bytes per 64 text bytes) in a
//                small per-CTA global scratch that stays in L2 (8 chunks, round robin), so
//                a chunk's positions are written once its global offset is known, without
//                re-reading the text.
//   warp 1      look-back  per chunk: walk the predecessors' status words 256 at a time
//                          until an inclusive prefix is found (decoupled look-back over
//                          64-bit launch-tagged words), publish the inclusive prefix.  It
//                          runs concurrently with the consumers through a 16-deep slot
//                          queue; the consumers published the chunk's aggregate already.
//   report       eight chunks later each consumer warp turns ITS 4 slices of the parked
//                chunk into positions slice_base + lane*64 + {r} (PAPER.md:431-441,
//                Fig. 1 line 11), directly or staged in its shared-memory buffer and
//                stored coalesced (16-byte stores) at pos[prefix + slice offset].
//
// Launches use programmatic dependent launch: a grid starts scanning while the previous one
// on the stream drains.  The workspace (counters, status words, parked masks) is double
// buffered by launch parity: launch L waits, through a CTA exit counter, only for launch
// L-2; griddepcontrol.wait precedes only the writes of outputs (positions, occ).
#pragma once
#include <cstdint>
#include <type_traits>
#include <cuda_runtime.h>

#include "epsm_ptx.cuh"

namespace epsm {

constexpr int kUnitBytes = 16;                                   // alpha
constexpr int kTile = 32768;                                     // bytes per TMA stage
constexpr int kHalo = 32;                                        // >= m-1, multiple of 16
constexpr int kStageBytes = kTile + 128;                         // tile + halo + verify slack
// Equality-mask index (planes): plane v of a text holds bit i of word w = [t[64w + i] == v].
// A stage then holds, per plane of the search, the tile's 512 words + the next word (the halo
// of windows crossing the tile), copied as 4112 bytes (16-byte multiple).
constexpr int kPlaneWordsPerTile = kTile / 64;                   // 512
constexpr int kPlaneStride = kTile / 8 + 16;                     // bytes per plane in a stage
constexpr int kMaxPlaneSlots = 8;                                // planes per search (distinct bytes)
static_assert(kMaxPlaneSlots * kPlaneStride <= kStageBytes, "planes of a stage");
// searches of few planes: one stage holds several tiles of every plane (a whole chunk of 4
// tiles for <= 2 planes, 2 tiles for <= 4), so the ring's round trip (copy, consumers,
// release) is paid once per 4 or 2 tiles
static_assert(2 * (4 * (kTile / 8) + 16) <= kStageBytes, "a chunk of 2 planes per stage");
static_assert(4 * (2 * (kTile / 8) + 16) <= kStageBytes, "2 tiles of 4 planes per stage");
constexpr int kStagesSearch = 5;
constexpr int kStagesCount = 6;
constexpr int kChunkTiles = 4;                                   // 128 KiB look-back granularity
constexpr int kChunkBytes = kChunkTiles * kTile;
constexpr int kConsumerWarps = 16;
constexpr int kConsumers = kConsumerWarps * 32;                  // 512
constexpr int kThreads = kConsumers + 64;                        // + producer + look-back warps
constexpr int kUnitsPerTile = kTile / kUnitBytes;                // 2048
constexpr int kUnitsPerThread = kUnitsPerTile / kConsumers;      // 4
constexpr int kSegBytes = kUnitsPerThread * kUnitBytes;          // 64 contiguous text bytes per lane
constexpr int kWarpBytes = 32 * kSegBytes;                       // 2 KiB per consumer warp and tile
// A slice = the 2 KiB of text (128 units, 64 starts per lane) one warp filters in one tile:
// lane l of warp w covers tile bytes [w*2048 + l*64, +64).  Text order of slices is (tile, warp).
constexpr int kSlices = kChunkTiles * kConsumerWarps;            // 64 per chunk
constexpr int kParked = 8;                                       // chunks parked awaiting their prefix
constexpr int kSlots = 16;                                       // look-back queue depth
constexpr int kWarpStage = 1024;                                 // positions per warp round
constexpr int kWarpStagePad = kWarpStage + kWarpStage / 16 + 4;  // slots + 2 pad per 32 + lead
constexpr int kLookbackWindow = 256;                             // statuses per look-back round
// parked masks in global scratch: one u64 (64 starts) per (chunk slot, tile, warp, lane)
constexpr int kScratchPerCta = kParked * kChunkTiles * kConsumerWarps * 32;   // u64 words
static_assert(kSlots % kParked == 0 && kSlots >= 2 * kParked, "slot / parking rotation");
static_assert(kParked * kChunkTiles <= 32, "slow-tile bits of all parked chunks fit one u32");
static_assert(kSlices <= 128 && kChunkTiles <= 8 && kUnitsPerThread == 4, "hand-off scan / mask packing layout");
constexpr uint32_t kTileBitsMask = (1u << kChunkTiles) - 1u;      // slow-tile bits of one parked chunk
static_assert(kChunkTiles == 4, "tiles-per-stage index variants (4 = a chunk, 2 = half)");

constexpr uint32_t kInfoEnd = 0xFFFFFFFFu;

// Sampled (EPSMc-style) filter: fingerprint table of the pattern's q-grams.
// Entry = candidate-offset mask (bits 0..15) | wildcard (bit 16) | 15-bit fingerprint (17..31).
constexpr int kGramBits = 11;
constexpr int kGramTab = 1 << kGramBits;                          // 2048 entries, 8 KiB
__host__ __device__ constexpr uint32_t gram_mul(int r) {   // odd multipliers of the gram hash
  return r == 0 ? 0x9E3779B1u : r == 1 ? 0x85EBCA77u : r == 2 ? 0xC2B2AE3Du : 0x27D4EB2Fu;
}

// Chunk status word: [63:40] epoch, [39:38] flag, [37:0] value.
constexpr int kEpochShift = 40;
constexpr unsigned long long kFlagAgg = 1ull << 38;
constexpr unsigned long long kFlagInc = 2ull << 38;
constexpr unsigned long long kFlagMask = 3ull << 38;
constexpr unsigned long long kValueMask = (1ull << 38) - 1;
constexpr unsigned long long kEpochMask = ~((1ull << kEpochShift) - 1);

// Per-pattern preprocessing, built on the host at plan time and
// kept in device memory; the producer copies it into a shared-memory slot (one TMA bulk copy)
// whenever its CTA starts a chunk of a new search.  The gram table is only copied for the
// sampled variants (kJobHeader bytes otherwise).
struct __align__(16) JobDesc {
  uint32_t bcast[4];            // B_i = p_i * 0x01010101
  uint32_t bcast2[4];           // B_{4+i}: the second filter word (pattern bytes 4..7)
  uint32_t pat[12];             // first 48 pattern bytes, little-endian u32 words, zero padded
  uint32_t pmask[12];           // per-word byte masks (partial last word)
  // EPSMa's shift-AND over exact equality masks, the variant for patterns of
  // 5 <= m <= 11 with at most 2 distinct bytes: value v broadcast, pattern positions holding it
  uint32_t eqv[2];              // value_v * 0x01010101
  uint32_t eqsel[2];            // bit i: p_i == value_v
  uint32_t eqd;                 // number of distinct bytes (1 or 2)
  uint32_t eqpad[3];
  // the same shift-AND over a text's equality-mask index (planes built once per text, shared
  // by every search of a batch): the pattern's distinct bytes (m <= 32, at most 8) in order
  // of first occurrence, and for each the positions i holding it as shift amounts, four per
  // word (byte b of plist[pw0[k] + q]), each plane's list padded to a multiple of four by
  // repeating its first position (AND is idempotent)
  uint32_t plist[16];
  uint8_t pw0[kMaxPlaneSlots];  // first word of plane k's list
  uint8_t pwn[kMaxPlaneSlots];  // words of plane k's list
  uint8_t pval[kMaxPlaneSlots]; // the byte value of plane k
  uint32_t np;                  // distinct bytes (0: more than kMaxPlaneSlots or m > 32)
  uint32_t ppad[5];
  uint8_t pslot[32];            // plane of p_i (short patterns read the planes position by position)
  uint32_t gram_tab[kGramTab];  // sampled filter: q-gram fingerprints -> candidate offsets
};
constexpr uint32_t kJobHeader = 304;                              // bytes before gram_tab
constexpr int kEqMode = -1;                                       // SK value of the equality variant
constexpr int kPlaneMode = -2;                                    // SK of the index variant (<= 8 planes)
constexpr int kPlaneModeC = -4;                                   // ... <= 2 planes: a chunk per stage
constexpr int kPlaneModeC2 = -5;                                  // ... <= 4 planes: 2 tiles per stage
constexpr int kPlaneModeC8 = -6;                                  // ... <= 8 planes: 2 tiles, 2 big stages
__host__ __device__ constexpr bool is_plane(int sk) {
  return sk == kPlaneMode || sk == kPlaneModeC || sk == kPlaneModeC2 || sk == kPlaneModeC8;
}
// tiles per ring stage and bytes per plane in a stage (tiles' words + the halo word)
__host__ __device__ constexpr uint32_t plane_tps(int sk) {
  return sk == kPlaneModeC ? 4u : (sk == kPlaneModeC2 || sk == kPlaneModeC8) ? 2u : 1u;
}
__host__ __device__ constexpr uint32_t plane_stride(int sk) { return plane_tps(sk) * (kTile / 8) + 16; }
static_assert(sizeof(JobDesc) == kJobHeader + 4 * kGramTab, "JobDesc layout");

// One search of a launch: its preprocessing and its outputs.
struct JobRef {
  const JobDesc* desc;          // device copy of the plan's preprocessing
  const uint32_t* dpat;         // m > 32: zero-padded pattern words in device memory
  uint64_t* pos;                // output positions (search)
  uint64_t cap;                 // capacity of pos
  unsigned long long* occ;      // device occ
  uint8_t pid[kMaxPlaneSlots];  // index variant: plane of the search's k-th distinct byte
  uint32_t np;                  // index variant: planes streamed per tile
  uint32_t pad;
};
constexpr int kMaxJobs = 40;                                      // searches per launch

struct KParams {
  const uint8_t* text;          // 16-byte aligned virtual base
  uint64_t nbytes;              // readable bytes from text
  uint64_t s_lo, s_hi;          // valid virtual starts [s_lo, s_hi)
  uint64_t pos_bias;            // reported = virtual start + pos_bias (mod 2^64)
  unsigned long long* status;   // one word per chunk of the launch (search)
  unsigned long long* ctr;      // [0] chunk-id counter (monotonic across launches),
                                // [2] CTA ticket (re-armed to 0), [8 + j] count of search j
  uint64_t* scratch;            // parked masks, kScratchPerCta u64 per CTA (search)
  unsigned long long ctr_base;  // value of ctr[0] when this launch starts
  unsigned long long tag;       // launch number << 40
  uint32_t ntiles;              // tiles covering [0, s_hi)
  uint32_t it_lo, it_hi;        // interior tiles [it_lo, it_hi): every start in [s_lo, s_hi)
  uint32_t nchunks;             // chunks per search (C); chunk g of the launch = search g / C
  uint32_t gchunks;             // chunks of the launch = njobs * C
  uint32_t njobs;               // searches in this launch (same text, same m)
  uint32_t m;                   // pattern length (all searches)
  uint32_t mul8;                // 1 << 24: byte shift by 1 through one IMAD.WIDE
  uint32_t mul24;               // 1 << 8 : byte shift by 3 through one IMAD.WIDE
  uint32_t movemask_mul;        // 0x00204081
  uint32_t desc_bytes;          // bytes of JobDesc the producer copies (header [+ gram table])
  uint32_t flags;               // EPSM_FLAGS (A/B timing): bit 1 = L2 prefetch of the next chunk
                                // (off by default: measured no gain, and under dense position
                                // writes the prefetched lines are evicted and read twice);
                                // bit 2 = slow the look-back warp down (test hook: consumers
                                // then run up to the parking slots' limit)
  unsigned long long* trace;    // diagnostics (epsm_debug_trace): 8 stamps per CTA, or NULL
  unsigned long long* exit_ctr; // CTAs of all launches on this workspace parity that have exited
  unsigned long long exit_expect;   // value meaning "launch L-2 (same parity) has retired"
  const uint64_t* planes;       // index variant: plane v at planes + v * pstride (u64 words)
  uint64_t pstride;
  JobRef jobs[kMaxJobs];
};

// Filter constants of the current search, held in registers by a consumer warp.
struct FParams {
  uint32_t bcast[4];
  const KParams& K;             // launch constants (byte-shift multipliers) stay in the constant bank
};

// %globaltimer stamps for the optional per-CTA timeline (EPSM_TRACE)
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define EPSM_TRACE(P, i) \
  do { if ((P).trace) (P).trace[blockIdx.x * 8 + (i)] = gtimer(); } while (0)

struct ChunkSlot {              // consumers -> look-back warp
  uint32_t chunk;               // chunk id, or kInfoEnd
  uint32_t total;               // occurrences in the chunk
  uint32_t park;                // parking slot holding the chunk
  uint32_t pad;
};

struct __align__(16) ParkedChunk {   // per parking slot
  uint32_t cnt[kSlices];        // per-slice counts, index tile*16 + warp (valid where slow)
  uint32_t off[kSlices];        // exclusive slice offsets inside the chunk, text order (hand-off)
  unsigned long long prefix;    // exclusive prefix (look-back warp)
  uint32_t chunk;               // chunk id
  uint32_t total;               // occurrences (hand-off warp)
  uint32_t ntiles;              // tiles in the chunk (last chunk may be short)
  uint32_t done;                // consumer warps finished with the chunk (smem atomic)
  uint32_t job;                 // search of the chunk, chunk / nchunks  (look-back warp)
  uint32_t scanned;             // 1 + sequence number of the last chunk whose counts were scanned
                                // (or that had none: marked at hand-off); only grows
  uint32_t cidx;                // chunk index inside its search, chunk % nchunks
  uint8_t slow[kConsumerWarps]; // bit t: the warp parked masks for tile t (else all zero)
};

template <int STAGES, bool SEARCH, int STAGE_BYTES = kStageBytes>
struct __align__(128) SmemLayoutT {
  static constexpr int kStages = STAGES;
  static constexpr int kPark = SEARCH ? kParked : 1;
  uint8_t ring[STAGES][STAGE_BYTES];
  uint16_t wstage[SEARCH ? kConsumerWarps : 1][SEARCH ? kWarpStagePad : 2];   // slice-relative
  ParkedChunk park[kPark];
  alignas(8) uint64_t full[STAGES];
  uint64_t empty[STAGES];
  uint64_t lb_full[kSlots];
  uint64_t lb_done[kSlots];
  ChunkSlot slot[kSlots];
  JobDesc job[2];               // preprocessing of the searches in flight (alternating slots)
  uint64_t job_full[2];         // slot loaded (TMA complete_tx)
  uint64_t job_free[2];         // every consumer warp has left the slot's search
  uint32_t info[STAGES];        // tile index in its search | (last-of-chunk << 31), or kInfoEnd
  uint32_t info2[STAGES];       // chunk id of the launch | (job slot << 31)
  uint32_t fin;                 // consumer warps that reached the end
  uint32_t ws_ok;               // the workspace parity is free (launch L-2 retired)
};
using SearchSmem = SmemLayoutT<kStagesSearch, true>;
using CountSmem = SmemLayoutT<kStagesCount, false>;
template <bool SEARCH>
using SmemFor = typename std::conditional<SEARCH, SearchSmem, CountSmem>::type;
// index variant for 5..8 planes: 2 stages of 2 tiles of 8 planes each
template <bool SEARCH>
using Index8Smem = SmemLayoutT<2, SEARCH, kMaxPlaneSlots * (2 * (kTile / 8) + 16)>;
static_assert(sizeof(Index8Smem<true>) <= 232448, "index-8 layout fits 227 KB of shared memory");
template <bool SEARCH, int SK>
using SmemForK = typename std::conditional<SK == kPlaneModeC8, Index8Smem<SEARCH>, SmemFor<SEARCH>>::type;

// ------------------------------------------------------------------ packed filter

// Filter words of one unit, in two stages (EPSMa's shift-AND):
//   stage 1 (pair):   Z[k] = (S_0[k] ^ B_0) | (S_1[k] ^ B_1)
//   stage 2 (extend): Z[k] |= (S_2[k] ^ B_2) | (S_3[k] ^ B_3)      (F > 2, F > 3)
// so that byte j of Z[k] is zero iff t[u+4k+j+i] = p_i for all i < F.  S_i is the text
// shifted by i bytes.  The shifts by 8 and 24 bits come from one 32x32->64 IMAD.WIDE per
// word (FMA pipe): w*2^(32-s) holds w >> s in its high half and w << (32-s) in its low
// half, so S_i[k] = hi(w_k * 2^(32-8i)) | lo(w_{k+1} * 2^(32-8i)); the two halves have
// disjoint bits, so the OR is folded into the 3-input XOR with B_i.
template <int F>
__device__ __forceinline__ void filter_pair(const uint32_t (&w)[5], const FParams& P, uint32_t (&Z)[4]) {
  if (F == 1) {
#pragma unroll
    for (int k = 0; k < 4; ++k) Z[k] = w[k] ^ P.bcast[0];
    return;
  }
  uint64_t p8[5];
#pragma unroll
  for (int k = 0; k < 5; ++k) p8[k] = static_cast<uint64_t>(w[k]) * P.K.mul8;
#pragma unroll
  for (int k = 0; k < 4; ++k)
    Z[k] = (w[k] ^ P.bcast[0]) |
           (static_cast<uint32_t>(p8[k] >> 32) ^ static_cast<uint32_t>(p8[k + 1]) ^ P.bcast[1]);
}

template <int F>
__device__ __forceinline__ void filter_extend(const uint32_t (&w)[5], const FParams& P, uint32_t (&Z)[4]) {
  if (F > 2) {
#pragma unroll
    for (int k = 0; k < 4; ++k) Z[k] |= __funnelshift_r(w[k], w[k + 1], 16) ^ P.bcast[2];
  }
  if (F > 3) {
    uint64_t p24[5];
#pragma unroll
    for (int k = 0; k < 5; ++k) p24[k] = static_cast<uint64_t>(w[k]) * P.K.mul24;
#pragma unroll
    for (int k = 0; k < 4; ++k)
      Z[k] |= static_cast<uint32_t>(p24[k] >> 32) ^ static_cast<uint32_t>(p24[k + 1]) ^ P.bcast[3];
  }
}

// Second filter word (pattern bytes 4 .. 3+F2) for the 16 starts of a unit, evaluated on the
// words w[1..5]: byte j of Y[k] is zero iff t[u+4k+j+4+i] = p_{4+i} for all i < F2.
template <int F2>
__device__ __forceinline__ void filter_second(const uint32_t (&v)[6], const FParams& P, const JobDesc& J,
                                              uint32_t (&Y)[4]) {
  uint64_t p8[5];
#pragma unroll
  for (int k = 0; k < 5; ++k) p8[k] = static_cast<uint64_t>(v[k + 1]) * P.K.mul8;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    uint32_t y = v[k + 1] ^ J.bcast2[0];
    if (F2 > 1) y |= static_cast<uint32_t>(p8[k] >> 32) ^ static_cast<uint32_t>(p8[k + 1]) ^ J.bcast2[1];
    if (F2 > 2) y |= __funnelshift_r(v[k + 1], v[k + 2], 16) ^ J.bcast2[2];
    Y[k] = y;
  }
  if (F2 > 3) {
    uint64_t p24[5];
#pragma unroll
    for (int k = 0; k < 5; ++k) p24[k] = static_cast<uint64_t>(v[k + 1]) * P.K.mul24;
#pragma unroll
    for (int k = 0; k < 4; ++k)
      Y[k] |= static_cast<uint32_t>(p24[k] >> 32) ^ static_cast<uint32_t>(p24[k + 1]) ^ J.bcast2[3];
  }
}

// Nonzero (bit 8j+7 set) iff some byte of some Z[k] is zero (has-zero test, exact as a boolean).
__device__ __forceinline__ uint32_t any_zero_byte(const uint32_t (&Z)[4]) {
  uint32_t h = 0;
#pragma unroll
  for (int k = 0; k < 4; ++k) h |= (Z[k] - 0x01010101u) & ~Z[k];
  return h & 0x80808080u;
}

// Exact 16-bit mask: bit 4k+j set iff byte j of Z[k] is zero.
__device__ __forceinline__ uint32_t zero_byte_mask16(const uint32_t (&Z)[4], uint32_t mm) {
  uint32_t t[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const uint32_t f = ~(((Z[k] & 0x7F7F7F7Fu) + 0x7F7F7F7Fu) | Z[k]) & 0x80808080u;   // flags at 8j+7
    t[k] = f * mm;                                                                      // gathered at 28..31
  }
  return (t[0] >> 28) | ((t[1] >> 24) & 0xF0u) | ((t[2] >> 20) & 0xF00u) | ((t[3] >> 16) & 0xF000u);
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

// Naive check of every candidate bit of r: words qstart..MW-1 of the
// window starting at shared byte offset o+b against the zero-padded pattern (the words
// before qstart were already checked exactly by the packed filter).
template <int MW>
__device__ __forceinline__ uint32_t verify_candidates(uint32_t r, const uint8_t* tile, uint32_t o,
                                                      const JobDesc& J, int qstart) {
  uint32_t keep = r;
  while (r) {
    const int b = __ffs(r) - 1;
    r &= r - 1;
    const uint32_t so = o + b;
    const uint32_t* wp = reinterpret_cast<const uint32_t*>(tile + (so & ~3u));
    const uint32_t sh = (so & 3u) * 8u;
    uint32_t lo = wp[qstart];
#pragma unroll
    for (int q = 1; q < MW; ++q) {
      if (q < qstart) continue;
      const uint32_t hi = wp[q + 1];
      const uint32_t win = __funnelshift_r(lo, hi, sh);
      if ((win ^ J.pat[q]) & J.pmask[q]) {
        keep &= ~(1u << b);
        break;
      }
      lo = hi;
    }
  }
  return keep;
}

// ------------------------------------------------------------------ sampled filter (EPSMc)

// EPSMc's fingerprint h (wscrc there, a multiply-add hash over the gram's
// little-endian words here).  Bits [31:21] index the table, bits [20:6] are the fingerprint.
template <int NW>
__device__ __forceinline__ uint32_t gram_hash(const uint32_t (&w)[NW]) {
  uint32_t h = w[0] * gram_mul(0);
#pragma unroll
  for (int r = 1; r < NW; ++r) h += w[r] * gram_mul(r);
  return h;
}

// SQ bytes of text at a shared-memory address aligned to min(SK, SQ, 16).
template <int SK, int SQ>
__device__ __forceinline__ void load_sample(const uint8_t* p, uint32_t (&w)[SQ / 4]) {
  // the sample address is aligned to min(SK, 16) bytes: widest loads that alignment allows
  if constexpr (SK >= 16 && SQ == 16) {
    const uint4 v = *reinterpret_cast<const uint4*>(p);
    w[0] = v.x;
    w[1] = v.y;
    w[2] = v.z;
    w[3] = v.w;
  } else if constexpr (SK >= 8 && SQ % 8 == 0) {
#pragma unroll
    for (int i = 0; i < SQ / 8; ++i) {
      const uint2 v = *reinterpret_cast<const uint2*>(p + 8 * i);
      w[2 * i] = v.x;
      w[2 * i + 1] = v.y;
    }
  } else {
#pragma unroll
    for (int i = 0; i < SQ / 4; ++i) w[i] = *reinterpret_cast<const uint32_t*>(p + 4 * i);
  }
}

// Naive check (Fig. 1 line 12) of every candidate bit of r against all MW
// zero-padded pattern words (the sampled filter proves nothing about any single word).
template <int MW>
__device__ __forceinline__ uint32_t verify_full(uint32_t r, const uint8_t* tile, uint32_t o, const JobDesc& J) {
  uint32_t keep = r;
  while (r) {
    const int b = __ffs(r) - 1;
    r &= r - 1;
    const uint32_t so = o + b;
    const uint32_t* wp = reinterpret_cast<const uint32_t*>(tile + (so & ~3u));
    const uint32_t sh = (so & 3u) * 8u;
    uint32_t lo = wp[0];
#pragma unroll
    for (int q = 0; q < MW; ++q) {
      const uint32_t hi = wp[q + 1];
      const uint32_t win = __funnelshift_r(lo, hi, sh);
      if ((win ^ J.pat[q]) & J.pmask[q]) {
        keep &= ~(1u << b);
        break;
      }
      lo = hi;
    }
  }
  return keep;
}

// Wait until the producer has seen this launch's workspace parity free (launch L-2 retired).
template <class Smem>
__device__ __forceinline__ void wait_ws(Smem& S) {
  while (*reinterpret_cast<volatile uint32_t*>(&S.ws_ok) == 0u) __nanosleep(64);
  __threadfence_block();
}

// Naive check for long patterns (m > 32, MW = 0 variants): the window runs past the tile
// halo, so it is compared against the text in global memory (L2: the tile was just
// streamed) and the pattern words in device memory.  Reads stay inside the words that hold
// text bytes (the last one lies in the 16-byte block of the text's last byte).
__device__ __forceinline__ uint32_t verify_long(uint32_t r, uint64_t us, const KParams& P, const uint32_t* dpat) {
  const uint32_t* t32 = reinterpret_cast<const uint32_t*>(P.text);
  const uint64_t last_word = (P.nbytes - 1) >> 2;
  const uint32_t nw = (P.m + 3) >> 2;
  const uint32_t tail_mask = (P.m & 3u) ? (0xFFFFFFFFu >> (8u * (4u - (P.m & 3u)))) : 0xFFFFFFFFu;
  uint32_t keep = r;
  while (r) {
    const int b = __ffs(r) - 1;
    r &= r - 1;
    const uint64_t st = us + b;
    const uint64_t w0 = st >> 2;
    const uint32_t sh = static_cast<uint32_t>(st & 3u) * 8u;
    uint32_t lo = __ldg(t32 + w0);
    for (uint32_t q = 0; q < nw; ++q) {
      const uint64_t wi = w0 + q + 1;
      const uint32_t hi = wi <= last_word ? __ldg(t32 + wi) : 0u;
      const uint32_t win = __funnelshift_r(lo, hi, sh);
      const uint32_t pm = q + 1 == nw ? tail_mask : 0xFFFFFFFFu;
      if ((win ^ __ldg(dpat + q)) & pm) {
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

__device__ __forceinline__ uint32_t warp_inclusive_scan(uint32_t x, uint32_t lane) {
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, d);
    if (lane >= static_cast<uint32_t>(d)) x += y;
  }
  return x;
}

// Decoupled look-back over chunk status words (single pass).  One full warp;
// window: kLookbackWindow statuses per round (kLookbackWindow / 32 loads per lane in flight).
// returns the exclusive prefix of `chunk` and publishes its inclusive prefix (its
// aggregate was published by the consumers).  Window: kLookbackWindow predecessors per round,
// lane l / slot i reads predecessor pred - (32 i + l), nearest first.
// With `fin` non-NULL the look-back gives up (returns kAborted, publishes nothing) once all
// consumer warps of the CTA have finished: nobody needs this chunk's prefix any more.
constexpr unsigned long long kAborted = ~0ull;
__device__ __forceinline__ unsigned long long lookback(const KParams& P, uint32_t chunk, uint32_t total,
                                                       uint32_t lane, const volatile uint32_t* fin) {
  const unsigned long long tag = P.tag;
  const long long jbase = static_cast<long long>(chunk / P.nchunks) * P.nchunks;   // its search's chunk 0
  if (chunk == jbase) {
    if (lane == 0) st_relaxed(P.status + chunk, tag | kFlagInc | total);
    return 0;
  }
  // (the chunk's aggregate was already published by the consumers when they finished it)
  unsigned long long prefix = 0;
  long long pred = static_cast<long long>(chunk) - 1;
  uint32_t spins = 0;
  constexpr int kPer = kLookbackWindow / 32;
  while (true) {
    unsigned long long s[kPer];
    while (true) {
      bool valid = true;
#pragma unroll
      for (int i = 0; i < kPer; ++i) {
        const long long idx = pred - (32 * i + static_cast<long long>(lane));
        s[i] = idx >= jbase ? ld_relaxed(P.status + idx) : (tag | kFlagInc);
        valid &= ((s[i] & kEpochMask) == tag) && (s[i] & kFlagMask);
      }
      if (__all_sync(0xffffffffu, valid)) break;
      if (fin && *fin == static_cast<uint32_t>(kConsumerWarps)) return kAborted;
      __nanosleep(32);
      if (++spins > (1u << 24)) __trap();   // a predecessor never published: fail loudly, never hang
    }
    // nearest inclusive predecessor: smallest distance d = 32 i + lane with flag INC
    uint32_t dmin = 0xFFFFFFFFu;
#pragma unroll
    for (int i = kPer - 1; i >= 0; --i)
      if ((s[i] & kFlagMask) == kFlagInc) dmin = 32u * i + lane;
    dmin = __reduce_min_sync(0xffffffffu, dmin);
    unsigned long long v = 0;
#pragma unroll
    for (int i = 0; i < kPer; ++i)
      if (32u * i + lane <= dmin) v += s[i] & kValueMask;
    prefix += warp_sum_u64(v);
    if (dmin != 0xFFFFFFFFu) break;
    pred -= kLookbackWindow;
  }
  if (lane == 0) st_relaxed(P.status + chunk, tag | kFlagInc | (prefix + total));
  return prefix;
}

// Stage the positions of one slice in the warp's shared buffer and store them coalesced at
// dst[0 .. min(tg, room)), kWarpStage per round.  Positions are staged as 16-bit offsets from
// the slice base sbase (lane*64 + bit < 2048), so one round holds half a slice's 2048 starts
// and the 64-bit adds happen only in the coalesced copy-out.  Lane: 64-start mask M,
// exclusive offset `off` inside the slice; tg = slice total.  Every lane walks its bits once
// across the rounds (two per step), stopping at each round's end.
// Stage slot of round entry i is i + lead (lead = 8-byte misalignment of the round's output),
// so slots (2k, 2k+1) are one 16-byte output pair; slot s lives at u16 index s + 2*(s >> 5)
// (a pad every 32 spreads the lanes' scattered writes over the banks and keeps each pair in
// one aligned 32-bit word).
__device__ __forceinline__ uint32_t stage_idx(uint32_t s) { return s + 2u * (s >> 5); }

__device__ __forceinline__ void write_slice(uint16_t* stage, uint64_t* dst, uint64_t room, uint64_t M,
                                            uint32_t off, uint32_t tg, uint64_t sbase, uint32_t lane) {
  uint32_t lo = static_cast<uint32_t>(M), hi = static_cast<uint32_t>(M >> 32);
  const uint32_t lbase = lane * kSegBytes;
  const uint32_t base_lo = static_cast<uint32_t>(sbase), base_hi = static_cast<uint32_t>(sbase >> 32);
  const bool no_carry = base_lo <= 0xFFFFFFFFu - 2048u;         // warp-uniform; 32-bit adds suffice
  uint32_t idx = off;
  for (uint32_t R = 0; R < tg; R += kWarpStage) {
    const uint32_t lim = R + kWarpStage;
    uint64_t* d = dst + R;
    const uint32_t lead = static_cast<uint32_t>((reinterpret_cast<uintptr_t>(d) >> 3) & 1u);
    const uint32_t sh = lead - R;                                  // slot = idx + sh
    while (idx + 1 < lim && (lo & (lo - 1u))) {                    // two bits of lo per step
      const uint32_t b0 = __ffs(lo) - 1;
      lo &= lo - 1;
      const uint32_t b1 = __ffs(lo) - 1;
      lo &= lo - 1;
      const uint32_t s0 = idx + sh;
      stage[stage_idx(s0)] = static_cast<uint16_t>(lbase + b0);
      stage[stage_idx(s0 + 1)] = static_cast<uint16_t>(lbase + b1);
      idx += 2;
    }
    if (lo && idx < lim) {
      const uint32_t b0 = __ffs(lo) - 1;
      lo &= lo - 1;
      stage[stage_idx(idx + sh)] = static_cast<uint16_t>(lbase + b0);
      ++idx;
    }
    while (idx + 1 < lim && (hi & (hi - 1u))) {
      const uint32_t b0 = __ffs(hi) + 31;
      hi &= hi - 1;
      const uint32_t b1 = __ffs(hi) + 31;
      hi &= hi - 1;
      const uint32_t s0 = idx + sh;
      stage[stage_idx(s0)] = static_cast<uint16_t>(lbase + b0);
      stage[stage_idx(s0 + 1)] = static_cast<uint16_t>(lbase + b1);
      idx += 2;
    }
    if (hi && idx < lim) {
      const uint32_t b0 = __ffs(hi) + 31;
      hi &= hi - 1;
      stage[stage_idx(idx + sh)] = static_cast<uint16_t>(lbase + b0);
      ++idx;
    }
    __syncwarp();
    uint32_t n = tg - R < kWarpStage ? tg - R : kWarpStage;
    if (room <= R) n = 0;
    else if (room - R < n) n = static_cast<uint32_t>(room - R);
    if (n) {
      uint64_t* dp = d - lead;                                     // 16-byte aligned
      const uint32_t nslots = n + lead;
      const uint32_t npairs = nslots >> 1;
      for (uint32_t k = lane; k < npairs; k += 32) {
        const uint32_t v = *reinterpret_cast<const uint32_t*>(stage + stage_idx(2 * k));
        if (k == 0 && lead) {
          st_stream_u64(dp + 1, sbase + (v >> 16));
        } else if (no_carry) {
          st_stream_u32x4(dp + 2 * k, base_lo + (v & 0xFFFFu), base_hi, base_lo + (v >> 16), base_hi);
        } else {
          st_stream_u64x2(dp + 2 * k, sbase + (v & 0xFFFFu), sbase + (v >> 16));
        }
      }
      if ((nslots & 1u) && lane == 0) {
        const uint32_t sl = nslots - 1;
        st_stream_u64(dp + sl, sbase + stage[stage_idx(sl)]);
      }
    }
    __syncwarp();
  }
}

// A slice where every start matches (e.g. 'a'^n): positions sbase + 0..2047, written
// arithmetically with 16-byte stores.  Out of line: inlined into the flush loop it costs the
// common sparse flushes registers and ~10%.
__device__ __noinline__ void write_full_slice(uint64_t* d, uint64_t room, uint64_t sbase, uint32_t lane) {
  const uint32_t n = room < static_cast<uint64_t>(kWarpBytes) ? static_cast<uint32_t>(room) : kWarpBytes;
  const uint32_t lead = static_cast<uint32_t>((reinterpret_cast<uintptr_t>(d) >> 3) & 1u);
  if (lead && lane == 0) st_stream_u64(d, sbase);
  const uint32_t npairs = (n - lead) >> 1;
  for (uint32_t k = lane; k < npairs; k += 32) {
    const uint32_t e = lead + 2 * k;
    st_stream_u64x2(d + e, sbase + e, sbase + e + 1);
  }
  if (((n - lead) & 1u) && lane == 0) st_stream_u64(d + n - 1, sbase + n - 1);
}

__device__ __forceinline__ uint32_t popc64(uint64_t v) {
  return __popc(static_cast<uint32_t>(v)) + __popc(static_cast<uint32_t>(v >> 32));
}

// Write this warp's slices of the chunk parked in slot b (its masks in the global
// scratch, the slice offsets computed at hand-off, the prefix from the look-back warp)
// at pos[...] -- the occurrences at i*alpha + {r} of PAPER.md:470 / Fig. 1 line 11, in
// text order.  `slow` bit t: this warp parked masks for tile t (else all zero).
template <class Smem>
__device__ __forceinline__ void flush_slices(const KParams& P, Smem& S, const uint64_t* scratch_cta,
                                             uint32_t b, uint32_t slow, uint32_t cw, uint32_t lane,
                                             uint64_t keep_pol, bool& out_ok) {
  const ParkedChunk& pk = S.park[b];
  if (pk.total == 0 || slow == 0) return;                      // warp-uniform
  const unsigned long long prefix = pk.prefix;
  const JobRef& J = P.jobs[pk.job];
  if (prefix >= J.cap) return;
  if (!out_ok) {                      // the previous grid on the stream may write the same output
    griddep_wait();
    out_ok = true;
  }
  uint64_t* const pos = J.pos;
  const uint64_t cap = J.cap;
  const uint64_t cbase = static_cast<uint64_t>(pk.cidx) * kChunkBytes + P.pos_bias;
  uint16_t* stage = S.wstage[cw];
  const uint32_t nt = pk.ntiles;
  uint64_t mk4[kChunkTiles];
#pragma unroll
  for (int t = 0; t < kChunkTiles; ++t)   // all loads first (L2 latency overlaps)
    mk4[t] = (t < static_cast<int>(nt) && ((slow >> t) & 1u))
                 ? ld_keep_u64(scratch_cta + ((b * kChunkTiles + t) * kConsumerWarps + cw) * 32 + lane, keep_pol)
                 : 0ull;
  const uint32_t lt = (1u << lane) - 1u;
#pragma unroll
  for (int t = 0; t < kChunkTiles; ++t) {
    if (!((slow >> t) & 1u) || t >= static_cast<int>(nt)) continue;
    const uint64_t M = mk4[t];
    const uint32_t c = popc64(M);
    const uint32_t any = __ballot_sync(0xffffffffu, c != 0);
    if (any == 0) continue;
    const uint64_t gidx = prefix + pk.off[t * kConsumerWarps + cw];
    if (gidx >= cap) return;                                // later slices are even further out
    const uint64_t room = cap - gidx;
    const uint64_t sb = cbase + static_cast<uint64_t>(t) * kTile + cw * kWarpBytes + lane * kSegBytes;
    if (__ballot_sync(0xffffffffu, c > 1) == 0) {
      // sparse slice (<= 1 position per lane): lanes store straight to consecutive slots,
      // which one warp store coalesces -- no staging, no scan
      const uint32_t off = __popc(any & lt);
      if (c && off < room) st_stream_u64(pos + gidx + off, sb + static_cast<uint64_t>(__ffsll(M) - 1));
      continue;
    }
    // exclusive offsets from bit-sliced ballots (c <= 64): independent ops, no shuffle chain;
    // as many as the largest lane count has bits (2 for the common sparse slices, not 7)
    const uint32_t nbits = 32u - __clz(__reduce_max_sync(0xffffffffu, c));
    uint32_t off = 0, tg = 0;
#pragma unroll
    for (int bb = 0; bb < 7; ++bb) {
      if (bb >= static_cast<int>(nbits)) break;              // warp-uniform
      const uint32_t bal = __ballot_sync(0xffffffffu, (c >> bb) & 1u);
      off += __popc(bal & lt) << bb;
      tg += __popc(bal) << bb;
    }
    if (tg <= 96) {
      // moderately sparse: direct stores, lane by lane in bit order
      uint32_t lo = static_cast<uint32_t>(M), hi = static_cast<uint32_t>(M >> 32);
      uint32_t i = off;
      while (lo) {
        const uint32_t bit = __ffs(lo) - 1;
        lo &= lo - 1;
        if (i < room) st_stream_u64(pos + gidx + i, sb + bit);
        ++i;
      }
      while (hi) {
        const uint32_t bit = __ffs(hi) + 31;
        hi &= hi - 1;
        if (i < room) st_stream_u64(pos + gidx + i, sb + bit);
        ++i;
      }
      continue;
    }
    if (tg == static_cast<uint32_t>(kWarpBytes)) {   // every start matches (periodic texts)
      write_full_slice(pos + gidx, room, sb - lane * kSegBytes, lane);
      continue;
    }
    write_slice(stage, pos + gidx, room, M, off, tg, sb - lane * kSegBytes, lane);
  }
}

// ------------------------------------------------------------------ lane segments

// The lane's 64-byte segment (4 units) in rotated order: R[r] = unit (r + rot) & 3 with
// rot = (lane >> 1) & 3, so the 8 lanes of every LDS.128 wavefront hit 8 different 16-byte
// bank groups (a plain 64-byte lane stride would be 4-way conflicted).
__device__ __forceinline__ void load_segment(const uint8_t* seg, uint32_t rot, uint4 (&R)[4]) {
#pragma unroll
  for (int r = 0; r < 4; ++r) R[r] = *reinterpret_cast<const uint4*>(seg + 16u * ((r + rot) & 3u));
}

// ------------------------------------------------------------------ the scan kernel

// F  = filter bytes of the first word (min(m, 4)); F2 = filter bytes of the second word
// (min(m, 8) - 4, 0 if m <= 4); MW = ceil(m/4) pattern words (MW <= 1: no verify; MW = 0:
// long pattern, m > 32, verified against device memory);
// SK, SQ = sampled filter (SK > 0: one SQ-byte gram every SK bytes, SK + SQ <= m; replaces
// the packed filter); SEARCH = report positions (else count only).
template <int F, int F2, int MW, int SK, int SQ, bool SEARCH>
__global__ void __launch_bounds__(kThreads, 1) epsm_scan_kernel(const __grid_constant__ KParams P) {
  extern __shared__ __align__(128) uint8_t smem_raw[];
  using Smem = SmemForK<SEARCH, SK>;
  constexpr int kStages = Smem::kStages;
  Smem& S = *reinterpret_cast<Smem*>(smem_raw);
  const uint32_t tid = threadIdx.x;
  const uint32_t lane = tid & 31u;
  const uint32_t warp = tid >> 5;

  if (tid == 0) EPSM_TRACE(P, 0);
  // barrier set-up spread over the threads of warps 0-1 (one mbarrier init each: a serial
  // init of all of them costs ~1 us on the start-up path)
  if (tid < static_cast<uint32_t>(kStages)) {
    mbar_init(&S.full[tid], 1);
    mbar_init(&S.empty[tid], kConsumerWarps);
    fence_mbar_init();
  } else if (tid >= 32 && tid < 32 + static_cast<uint32_t>(kSlots)) {
    mbar_init(&S.lb_full[tid - 32], 1);
    mbar_init(&S.lb_done[tid - 32], 1);
    fence_mbar_init();
  } else if (tid >= 64 && tid < 64 + static_cast<uint32_t>(Smem::kPark)) {
    S.park[tid - 64].done = 0;
    S.park[tid - 64].scanned = 0;
  } else if (tid >= 96 && tid < 98) {
    mbar_init(&S.job_full[tid - 96], 1);
    mbar_init(&S.job_free[tid - 96], kConsumerWarps);
    fence_mbar_init();
  }
  if (tid == 0) {
    S.fin = 0;
    S.ws_ok = 0;
    griddep_launch_dependents();   // the next grid may start its prologue as our CTAs retire
  }
  __syncthreads();

  if (warp == 0) {
    // ================================================================ producer
    const uint64_t policy = policy_evict_first();
    uint32_t stage = 0, phase = 0;
    // chunk ids: the first one is static (blockIdx.x: no atomic on the start-up path), the
    // rest come from a monotonic counter: gridDim.x + (atomicAdd(ctr) - ctr_base).  Every CTA
    // draws until it gets an id >= nchunks, so a launch advances the counter by nchunks.
    // chunk ids: the first one is static (blockIdx.x: no atomic on the start-up path), the
    // rest come from a monotonic counter: gridDim.x + (atomicAdd(ctr) - ctr_base).  Every CTA
    // draws until it gets an id >= nchunks, so a launch advances the counter by nchunks.
    // Two ids are kept ahead: `after` (already known, pulled into L2 one chunk early) and a
    // draw in flight whose result is only consumed when the current chunk has been issued,
    // so the atomic's latency never stalls the TMA issue.
    auto draw = [&]() -> unsigned long long { return gridDim.x + (atomicAdd(P.ctr, 1ull) - P.ctr_base); };
    auto prefetch_l2 = [&](unsigned long long g) {
      if (lane == 0 && g < P.gchunks) {
        const uint64_t pb = (g % P.nchunks) * static_cast<unsigned long long>(kChunkBytes);
        const uint64_t pe_want = pb + kChunkBytes + kHalo;
        const uint64_t pe = (pe_want < P.nbytes ? pe_want : P.nbytes) & ~15ull;
        for (uint64_t a = pb; a < pe; a += kTile) {
          const uint64_t e = a + kTile < pe ? a + kTile : pe;
          bulk_prefetch_l2(P.text + a, static_cast<uint32_t>(e - a));
        }
      }
    };
    // chunk g of the launch belongs to search g / C (C = P.nchunks chunks per search, all
    // searches over the same text); a CTA that starts a chunk of a new search first copies
    // that search's preprocessing into the other job slot (after every consumer warp left
    // the search the slot held before)
    unsigned long long cur = blockIdx.x, after = 0, pend = 0;
    bool first = true;
    bool ws_seen = false;                      // (lane 0) workspace parity seen free
    uint32_t pjob = 0xFFFFFFFFu, jslot = 1, nswitch = 0;
    while (true) {
      if (cur >= P.gchunks) {
        mbar_wait(&S.empty[stage], phase ^ 1u);
        if (lane == 0) {
          S.info[stage] = kInfoEnd;
          mbar_arrive(&S.full[stage]);
          EPSM_TRACE(P, 3);
        }
        break;
      }
      const uint32_t job = static_cast<uint32_t>(cur / P.nchunks);
      if (job != pjob) {
        jslot ^= 1u;
        if (nswitch >= 2) mbar_wait(&S.job_free[jslot], ((nswitch - 2) >> 1) & 1u);
        if (lane == 0) {
          mbar_arrive_expect_tx(&S.job_full[jslot], P.desc_bytes);
          bulk_g2s_plain(&S.job[jslot], P.jobs[job].desc, P.desc_bytes, &S.job_full[jslot]);
        }
        pjob = job;
        ++nswitch;
      }
      const uint32_t t0 = static_cast<uint32_t>(cur % P.nchunks) * kChunkTiles;
      const uint32_t t1 = min(t0 + kChunkTiles, P.ntiles);
      constexpr uint32_t tstep = plane_tps(SK);                          // tiles per stage
      for (uint32_t t = t0; t < t1; t += tstep) {
        mbar_wait(&S.empty[stage], phase ^ 1u);
        const uint64_t base = static_cast<uint64_t>(t) * kTile;
        const uint64_t want_end = base + kTile + kHalo;
        const uint64_t end = want_end < P.nbytes ? want_end : P.nbytes;
        const uint32_t bulk = static_cast<uint32_t>((end & ~15ull) - base);
        const uint32_t tail = static_cast<uint32_t>(end - base) - bulk;   // < 16 bytes
        if constexpr (!is_plane(SK)) {
          if (lane < tail) S.ring[stage][bulk + lane] = P.text[base + bulk + lane];
        }
        __syncwarp();
        if (lane == 0) {
          if constexpr (tstep > 1) {
            // first tile, tile count - 1 in [30:29], last-of-chunk
            const uint32_t ntc = min(tstep, t1 - t);
            S.info[stage] = t | ((ntc - 1) << 29) | (t + ntc == t1 ? 0x80000000u : 0u);
          } else {
            S.info[stage] = t | ((t + 1 == t1) ? 0x80000000u : 0u);
          }
          S.info2[stage] = static_cast<uint32_t>(cur) | (jslot << 31);
          if constexpr (tstep > 1) {
            // the stage's tiles of the search's planes + the halo word, per plane
            const JobRef& J = P.jobs[job];
            const uint32_t bytes = min(tstep, t1 - t) * (kTile / 8) + 16;
            mbar_arrive_expect_tx(&S.full[stage], J.np * bytes);
            for (uint32_t k = 0; k < J.np; ++k)
              bulk_g2s_plain(S.ring[stage] + k * plane_stride(SK),
                             P.planes + J.pid[k] * P.pstride + static_cast<uint64_t>(t) * kPlaneWordsPerTile,
                             bytes, &S.full[stage]);
          } else if constexpr (is_plane(SK)) {
            // the tile's words of the search's planes (padded: always whole)
            const JobRef& J = P.jobs[job];
            mbar_arrive_expect_tx(&S.full[stage], J.np * kPlaneStride);
            // (no evict-first hint: the next searches of the batch read the same planes)
            for (uint32_t k = 0; k < J.np; ++k)
              bulk_g2s_plain(S.ring[stage] + k * kPlaneStride,
                             P.planes + J.pid[k] * P.pstride + static_cast<uint64_t>(t) * kPlaneWordsPerTile,
                             kPlaneStride, &S.full[stage]);
          } else if (bulk) {
            mbar_arrive_expect_tx(&S.full[stage], bulk);
            bulk_g2s(S.ring[stage], P.text + base, bulk, &S.full[stage], policy);
          } else {
            mbar_arrive(&S.full[stage]);
          }
          if (first && t == t0) EPSM_TRACE(P, 1);
          if (t == t0 && !first) pend = draw();   // consumed after this chunk
          if (first && !ws_seen && (t + tstep >= t1 || t + 1 - t0 == static_cast<uint32_t>(kStages))) {
            // the first loads (text only) are in flight; before anything touches the workspace
            // (chunk counter, status words, parked masks) launch L-2, the previous user of
            // this parity, must have retired -- normally long done, so one load.  (Done by the
            // time the ring is full: consumers may wait for it before releasing a stage.)
            while (ld_acquire(P.exit_ctr) < P.exit_expect) __nanosleep(100);
            __threadfence_block();
            *reinterpret_cast<volatile uint32_t*>(&S.ws_ok) = 1u;
            ws_seen = true;
          }
        }
        if (++stage == kStages) {
          stage = 0;
          phase ^= 1u;
        }
      }
      if (first) {
        if (lane == 0) {
          after = draw();
          pend = draw();
        }
        first = false;
      }
      unsigned long long nxt = 0;
      if (lane == 0) {
        nxt = after;
        after = pend;
      }
      cur = __shfl_sync(0xffffffffu, nxt, 0);
      after = __shfl_sync(0xffffffffu, after, 0);
      if (!is_plane(SK) && (P.flags & 2u)) prefetch_l2(after);
    }
  } else if (warp == 1) {
    // ================================================================ look-back
    if constexpr (SEARCH) {
      // (chunks reach this queue only after the consumers saw the workspace free)
      uint32_t q = 0, par = 0, lbk = 0;                   // lbk: sequence number of the chunk
      while (true) {
        mbar_wait_suspend(&S.lb_full[q], par);
        if (P.flags & 4u) {                     // test hook: a lagging look-back warp
          for (int i = 0; i < 16; ++i) __nanosleep(1000);
        }
        const ChunkSlot sl = S.slot[q];
        if (sl.chunk == kInfoEnd) break;
        {
          // exclusive prefix over the chunk's 64 slice counts in text order (tile, warp), for
          // the consumers' write-out (they wait for lb_done before reading it)
          ParkedChunk& pk = S.park[sl.park];
          const uint32_t ntiles = pk.ntiles;
          constexpr int kPerLane = (kSlices + 31) / 32;
          uint32_t v[kPerLane], sum = 0;
#pragma unroll
          for (int i = 0; i < kPerLane; ++i) {
            const uint32_t si = lane * kPerLane + i;
            const uint32_t t = si / kConsumerWarps;
            const uint32_t w = si % kConsumerWarps;
            v[i] = (si < static_cast<uint32_t>(kSlices) && t < ntiles && ((pk.slow[w] >> t) & 1u)) ? pk.cnt[si] : 0u;
            sum += v[i];
          }
          const uint32_t incl = warp_inclusive_scan(sum, lane);
          uint32_t run = incl - sum;
#pragma unroll
          for (int i = 0; i < kPerLane; ++i) {
            if (lane * kPerLane + i < static_cast<uint32_t>(kSlices)) pk.off[lane * kPerLane + i] = run;
            run += v[i];
          }
          __syncwarp();
          __threadfence_block();
          if (lane == 0) atomicMax(&pk.scanned, lbk + 1);
          ++lbk;
        }
        // a chunk without occurrences needs no prefix of its own; its look-back only helps
        // successors (an inclusive status shortens their walks), so it is dropped once every
        // consumer warp of this CTA is done and the CTA could otherwise exit
        const uint32_t cidx = sl.chunk % P.nchunks;
        const bool last = cidx + 1 == P.nchunks;                  // its prefix gives occ
        if (lane == 0) {                                          // (no divisions in the write-out)
          S.park[sl.park].job = sl.chunk / P.nchunks;
          S.park[sl.park].cidx = cidx;
        }
        const volatile uint32_t* fin = (sl.total == 0 && !last) ? &S.fin : nullptr;
        const bool skip = fin && *fin == static_cast<uint32_t>(kConsumerWarps);
        const unsigned long long pre = skip ? kAborted : lookback(P, sl.chunk, sl.total, lane, fin);
        if (lane == 0) {
          if (pre != kAborted) S.park[sl.park].prefix = pre;
          if (last) {
            griddep_wait();                    // the previous grid may write the same occ
            *P.jobs[sl.chunk / P.nchunks].occ = pre + sl.total;
          }
          mbar_arrive(&S.lb_done[q]);
        }
        __syncwarp();
        if (++q == kSlots) {
          q = 0;
          par ^= 1u;
        }
      }
    }
  } else {
    // ================================================================ consumers
    const uint32_t cw = warp - 2;
    const uint32_t seg_off = cw * kWarpBytes + lane * kSegBytes;   // this lane's 64 bytes in a tile
    const uint32_t rot = (lane >> 1) & 3u;                           // load rotation (bank groups)
    uint32_t stage = 0, phase = 0;
    uint32_t seq = 0;                          // chunks this warp has started (same for all warps)
    uint32_t tpos = 0;                         // tile index inside the current chunk
    uint32_t slowbits = 0;                     // bit 4b+t: masks parked for tile t of slot b
    uint32_t acc = 0;                          // count mode: this thread's occurrences
    bool try_pair = true;                      // test the pair stage on its own (adaptive)
    uint32_t pair_streak = 0;                  // consecutive pair tests that found candidates
    uint32_t tiles_seen = 0;
    bool waited = false;                       // workspace parity seen free (S.ws_ok)
    bool out_ok = false;                       // griddepcontrol.wait done (outputs writable)
    uint64_t* scratch_cta = SEARCH ? P.scratch + static_cast<uint64_t>(blockIdx.x) * kScratchPerCta : nullptr;
    const uint64_t keep_pol = policy_evict_last();

    // lb_done[q] completes once per chunk routed through slot q: chunk #k uses slot k % kSlots
    // and phase parity (k / kSlots) & 1.
    auto wait_done = [&](uint32_t k) {
      mbar_wait(&S.lb_done[k % kSlots], (k / kSlots) & 1u);
    };
    // write out chunk #k's slices (parked in slot k % kParked) once its prefix is known
    // (a warp that parked no masks for the chunk has nothing to write and needs no prefix)
    // (with nothing to write the warp still waits until the look-back warp has scanned chunk
    // #k's slice counts: it is about to park chunk #k + kParked in the same slot)
    auto flush_chunk_seq = [&](uint32_t k) {
      const uint32_t b = k % kParked;
      const uint32_t sb = (slowbits >> (kChunkTiles * b)) & kTileBitsMask;
      if (sb) {
        wait_done(k);
        flush_slices(P, S, scratch_cta, b, sb, cw, lane, keep_pol, out_ok);
      } else {
        while (*reinterpret_cast<volatile const uint32_t*>(&S.park[b].scanned) <= k) __nanosleep(32);
      }
      slowbits &= ~(kTileBitsMask << (kChunkTiles * b));
    };

    // the search of the current tile: its job slot, its filter constants (registers)
    uint32_t cur_slot = 2, cur_job = 0, slot_uses = 0;   // slot_uses: [15:0] slot 0, [31:16] slot 1
    const JobDesc* JD = &S.job[0];
    FParams FP{{0u, 0u, 0u, 0u}, P};
    // count mode: this warp's occurrences of the current search go to the workspace counter
    auto flush_count = [&]() {
      if constexpr (!SEARCH) {
        const uint32_t wsum = __reduce_add_sync(0xffffffffu, acc);
        if (wsum) {
          if (!waited) {
            wait_ws(S);
            waited = true;
          }
          if (lane == 0) atomicAdd(P.ctr + 8 + cur_job, static_cast<unsigned long long>(wsum));
        }
        acc = 0;
      }
    };
    bool first_tile = true;
    // chunk-per-stage index variant: sub-tile of the stage's chunk, its first tile and size
    uint32_t sub = 0, c_t0 = 0, c_ntc = 1, gch = 0;
    bool c_last = false;
    while (true) {
      if (plane_tps(SK) == 1 || sub == 0) {
      mbar_wait(&S.full[stage], phase);
      if (first_tile && cw == 0 && lane == 0) EPSM_TRACE(P, 2);
      first_tile = false;
      const uint32_t info = S.info[stage];
      if (info == kInfoEnd) {
        if (cw == 0 && lane == 0) EPSM_TRACE(P, 4);
        break;
      }
      c_t0 = info & (plane_tps(SK) > 1 ? 0x1FFFFFFFu : 0x7FFFFFFFu);   // (first) tile in its search
      c_ntc = plane_tps(SK) > 1 ? ((info >> 29) & 3u) + 1u : 1u;
      c_last = info >> 31;
      const uint32_t info2 = S.info2[stage];
      gch = info2 & 0x7FFFFFFFu;                             // chunk id of the launch
      const uint32_t js = info2 >> 31;                       // job slot of its search
      if (js != cur_slot) {
        // a new search: leave the old slot (the producer may refill it), wait for the new one
        if (cur_slot < 2) {
          flush_count();
          __syncwarp();
          if (lane == 0) mbar_arrive(&S.job_free[cur_slot]);
        }
        const uint32_t k = js ? (slot_uses >> 16) : (slot_uses & 0xFFFFu);
        mbar_wait(&S.job_full[js], k & 1u);
        slot_uses += js ? 0x10000u : 1u;
        cur_slot = js;
        cur_job = gch / P.nchunks;
        JD = &S.job[js];
        const uint4 b0 = *reinterpret_cast<const uint4*>(JD->bcast);
        FP.bcast[0] = b0.x;
        FP.bcast[1] = b0.y;
        FP.bcast[2] = b0.z;
        FP.bcast[3] = b0.w;
      }
      }
      const uint32_t tile = c_t0 + sub;
      const bool last_in_chunk = c_last;   // (the index variants take a stage's tiles at once)
      const uint32_t b = seq % kParked;
      if (SEARCH && tpos == 0 && seq >= kParked) flush_chunk_seq(seq - kParked);   // free slot b
      const uint8_t* ts = S.ring[stage];
      const uint8_t* seg = ts + seg_off;
      const uint64_t tbase = static_cast<uint64_t>(tile) * kTile;
      const bool interior = tile >= P.it_lo && tile < P.it_hi;          // warp-uniform

      // slot r holds unit u = (r + rot) & 3 of the segment: text bytes [seg_off + 16u, +16)
      uint32_t mask[4];                        // 16-bit match mask of the unit in slot r
      uint64_t Meq = 0;                        // equality variant: the lane mask directly
      bool slow;
      if constexpr (SK == kEqMode) {
        // ---- EPSMa (Fig. 1 lines 5-9) for a pattern with <= 2 distinct
        // bytes: exact equality masks E_v of the lane's 64 bytes (+ the next 16, the halo of
        // windows crossing the segment), then r = AND_i (E_{v(p_i)} >> i) -- the shift-AND
        // gives the exact match mask of all 64 starts, no candidates, no check
        uint4 R[4];
        load_segment(seg, rot, R);
        const uint32_t r0 = (4u - rot) & 3u;                // slot holding unit 0
        uint32_t rl = 0xFFFFFFFFu, rh = 0xFFFFFFFFu;       // result, starts 0-31 / 32-63
#pragma unroll
        for (int v = 0; v < 2; ++v) {
          if (v == 1 && JD->eqd < 2) break;                  // warp-uniform
          const uint32_t vb = JD->eqv[v];
          uint32_t e16[4];
#pragma unroll
          for (int r = 0; r < 4; ++r) {
            const uint32_t Zv[4] = {R[r].x ^ vb, R[r].y ^ vb, R[r].z ^ vb, R[r].w ^ vb};
            e16[r] = zero_byte_mask16(Zv, P.movemask_mul);
          }
          uint32_t lo = 0, hi = 0;                          // E_v of starts 0-31, 32-63
#pragma unroll
          for (int r = 0; r < 4; ++r) {
            const uint32_t u = (r + rot) & 3u;
            const uint32_t sh = (u & 1u) * 16u;
            if (u < 2) lo |= e16[r] << sh;
            else hi |= e16[r] << sh;
          }
          // positions 64..79: the next lane's unit 0 (lane 31: the next slice / the halo)
          const uint32_t own0 = r0 == 0 ? e16[0] : r0 == 1 ? e16[1] : r0 == 2 ? e16[2] : e16[3];
          uint32_t halo = __shfl_down_sync(0xffffffffu, own0, 1);
          if (lane == 31) {
            const uint4 h = *reinterpret_cast<const uint4*>(seg + kSegBytes);
            const uint32_t Zh[4] = {h.x ^ vb, h.y ^ vb, h.z ^ vb, h.w ^ vb};
            halo = zero_byte_mask16(Zh, P.movemask_mul);
          }
          const uint32_t sel = JD->eqsel[v];
#pragma unroll
          for (int i = 0; i < 12; ++i) {
            if ((sel >> i) & 1u) {                           // p_i == value_v: AND E_v >> i
              rl &= __funnelshift_r(lo, hi, i);
              rh &= __funnelshift_r(hi, halo, i);
            }
          }
        }
        Meq = (static_cast<uint64_t>(rh) << 32) | rl;
        if (!interior) {
          uint64_t rm = 0;
#pragma unroll
          for (int u = 0; u < 4; ++u)
            rm |= static_cast<uint64_t>(range_mask(tbase + seg_off + 16u * u, P.s_lo, P.s_hi)) << (16 * u);
          Meq &= rm;
        }
        slow = __any_sync(0xffffffffu, Meq != 0ull);
      } else if constexpr (is_plane(SK)) {
        // ---- EPSMa's shift-AND over the text's equality-mask index: the
        // masks E_v of the lane's 64 starts (+ the next 64) are read, not computed --
        // r = AND_i (E_{p_i} >> i), exact, no candidates, no check
        const uint32_t wi = cw * 32u + lane;                 // the lane's word in each plane tile
        constexpr uint32_t kPS = plane_stride(SK);
        constexpr uint32_t kTPS = plane_tps(SK);             // tiles of this stage (<= c_ntc used)
        constexpr uint32_t kPosMax = 8;                      // position by position up to this m
                                                             // (16 measured slower at d = 8)
        uint64_t Mu[kTPS];
        if (P.m <= kPosMax) {
          // short patterns: position by position, each reading the words of its own plane
          // (compile-time shifts, no list); the stage's tiles side by side (independent chains)
          uint32_t rl[kTPS], rh[kTPS];
#pragma unroll
          for (uint32_t u = 0; u < kTPS; ++u) rl[u] = rh[u] = 0xFFFFFFFFu;
#pragma unroll
          for (int i = 0; i < static_cast<int>(kPosMax); ++i) {
            if (i >= static_cast<int>(P.m)) break;
            const uint8_t* pp = ts + JD->pslot[i] * kPS;
#pragma unroll
            for (uint32_t u = 0; u < kTPS; ++u) {
              const uint2* pl = reinterpret_cast<const uint2*>(pp + u * (kTile / 8));
              const uint2 e = pl[wi];
              if (i == 0) {
                rl[u] &= e.x;
                rh[u] &= e.y;
              } else {
                const uint32_t h = pl[wi + 1].x;
                rl[u] &= __funnelshift_r(e.x, e.y, i);
                rh[u] &= __funnelshift_r(e.y, h, i);
              }
            }
          }
#pragma unroll
          for (uint32_t u = 0; u < kTPS; ++u) Mu[u] = (static_cast<uint64_t>(rh[u]) << 32) | rl[u];
        } else {
#pragma unroll
          for (uint32_t u = 0; u < kTPS; ++u) {
            if (u >= c_ntc) {
              Mu[u] = 0;
              continue;
            }
            const uint8_t* pb = ts + u * (kTile / 8);
            uint32_t rl = 0xFFFFFFFFu, rh = 0xFFFFFFFFu;
            const uint32_t np = JD->np;
#pragma unroll
            for (int k = 0; k < kMaxPlaneSlots; ++k) {
              if (k >= static_cast<int>(np)) break;              // warp-uniform
              const uint2* pl = reinterpret_cast<const uint2*>(pb + k * kPS);
              const uint2 e = pl[wi], h = pl[wi + 1];            // starts 0..63, 64..127
              const uint32_t w0 = JD->pw0[k], wn = JD->pwn[k];
              bool live = true;
              for (uint32_t q = 0; q < wn; ++q) {
                // four positions i with p_i == value of plane k (shift amounts: the funnel
                // shift uses the low 5 bits, so the packed word is shifted, not masked)
                const uint32_t sw = JD->plist[w0 + q];
                rl &= __funnelshift_r(e.x, e.y, sw) & __funnelshift_r(e.x, e.y, sw >> 8) &
                      __funnelshift_r(e.x, e.y, sw >> 16) & __funnelshift_r(e.x, e.y, sw >> 24);
                rh &= __funnelshift_r(e.y, h.x, sw) & __funnelshift_r(e.y, h.x, sw >> 8) &
                      __funnelshift_r(e.y, h.x, sw >> 16) & __funnelshift_r(e.y, h.x, sw >> 24);
                // no start of the warp's slice survives: the rest of the AND cannot revive one
                live = __any_sync(0xffffffffu, (rl | rh) != 0u);
                if (!live) break;
              }
              if (!live) break;
            }
            Mu[u] = (static_cast<uint64_t>(rh) << 32) | rl;
          }
        }
#pragma unroll
        for (uint32_t u = 0; u < kTPS; ++u) {
          const uint32_t tl = c_t0 + u;
          if (!(tl >= P.it_lo && tl < P.it_hi)) {              // (warp-uniform) a tile at an end
            const uint64_t tb = static_cast<uint64_t>(tl) * kTile;
            uint64_t rm = 0;
#pragma unroll
            for (int v = 0; v < 4; ++v)
              rm |= static_cast<uint64_t>(range_mask(tb + seg_off + 16u * v, P.s_lo, P.s_hi)) << (16 * v);
            Mu[u] &= rm;
          }
        }
        if constexpr (kTPS > 1) {
          // all but the stage's last tile are parked here; the last goes through the common path
#pragma unroll
          for (uint32_t u = 0; u + 1 < kTPS; ++u) {
            if (u + 1 >= c_ntc) break;                           // warp-uniform
            if (!__any_sync(0xffffffffu, Mu[u] != 0ull)) continue;
            const uint32_t c = popc64(Mu[u]);
            acc += c;
            if constexpr (SEARCH) {
              if (!waited) {
                wait_ws(S);
                waited = true;
              }
              st_keep_u64(scratch_cta + ((b * kChunkTiles + tpos + u) * kConsumerWarps + cw) * 32 + lane, Mu[u],
                          keep_pol);
              const uint32_t sc = __reduce_add_sync(0xffffffffu, c);
              if (lane == 0) S.park[b].cnt[(tpos + u) * kConsumerWarps + cw] = sc;
              slowbits |= 1u << (kChunkTiles * b + tpos + u);
            }
          }
          Meq = c_ntc == 1 ? Mu[0] : c_ntc == 2 ? Mu[1] : kTPS > 2 && c_ntc == 3 ? Mu[kTPS > 2 ? 2 : 0]
                                                                         : Mu[kTPS - 1];
          tpos += c_ntc - 1;
          sub = c_ntc - 1;
        } else {
          Meq = Mu[0];
        }
        slow = __any_sync(0xffffffffu, Meq != 0ull);
      } else if constexpr (SK > 0) {
        // ---- sampled filter (EPSMc, Fig. 1 lines 7-12): the q-gram at unit
        // offset SK*(g+1) is fingerprinted and looked up in the pattern's gram table, which
        // yields the starts of group g whose window holds that gram at the right offset.
        uint32_t anyc = 0;
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          const uint8_t* up = seg + 16u * ((r + rot) & 3u);
          uint32_t c = 0;
#pragma unroll
          for (int g = 0; g < 16 / SK; ++g) {
            constexpr int kw = SQ / 4;
            uint32_t sw[kw];
            load_sample<SK, SQ>(up + SK * (g + 1), sw);
            const uint32_t H = gram_hash<kw>(sw);
            const uint32_t e = JD->gram_tab[H >> (32 - kGramBits)];
            const bool ok = (((e ^ (H << kGramBits)) & 0xFFFE0000u) == 0u) || (e & 0x10000u);
            c |= (ok ? (e & 0xFFFFu) : 0u) << (SK * g);
          }
          mask[r] = c;
          anyc |= c;
        }
        slow = __any_sync(0xffffffffu, anyc != 0u);
        if (slow) {
          uint32_t left = 0;
#pragma unroll
          for (int r = 0; r < 4; ++r) {
            const uint32_t o = seg_off + 16u * ((r + rot) & 3u);
            if (!interior) {
              const uint64_t us = tbase + o;
              if (us < P.s_lo || us + 16 > P.s_hi) mask[r] &= range_mask(us, P.s_lo, P.s_hi);
            }
            if (__any_sync(0xffffffffu, mask[r])) {
              if constexpr (MW == 0) mask[r] = verify_long(mask[r], tbase + o, P, P.jobs[cur_job].dpat);
              else mask[r] = verify_full<MW>(mask[r], ts, o, *JD);
            }
            left |= mask[r];
          }
          slow = __any_sync(0xffffffffu, left != 0u);
        }
      } else {
        // ---- packed filter (EPSMa/b): all units first (independent chains), then one warp
        // vote per stage.  The pair stage is tested on its own only while it pays off (large
        // alphabets: almost never a candidate); otherwise the words are extended to F bytes
        // straight away.  Both paths give the same Z, so the adaptation never changes the result.
        uint4 R[4];
        load_segment(seg, rot, R);
        uint32_t W[4][5];
        uint32_t Z[4][4];
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          W[r][0] = R[r].x;
          W[r][1] = R[r].y;
          W[r][2] = R[r].z;
          W[r][3] = R[r].w;
          W[r][4] = *reinterpret_cast<const uint32_t*>(seg + 16u * ((r + rot) & 3u) + 16u);
          filter_pair<F>(W[r], FP, Z[r]);
        }
        if constexpr (F > 2) {
          bool need_extend = true;
          if (try_pair) {
            uint32_t hz = 0;
#pragma unroll
            for (int r = 0; r < 4; ++r) hz |= any_zero_byte(Z[r]);
            need_extend = __any_sync(0xffffffffu, hz);
            // hysteresis: stop testing the pair stage alone after two hits in a row (small
            // alphabets), retry every 16th tile
            pair_streak = need_extend ? pair_streak + 1 : 0u;
          }
          try_pair = pair_streak < 2 || ((++tiles_seen & 15u) == 0);
          slow = false;
          if (need_extend) {
            uint32_t hz = 0;
#pragma unroll
            for (int r = 0; r < 4; ++r) {
              filter_extend<F>(W[r], FP, Z[r]);
              hz |= any_zero_byte(Z[r]);
            }
            slow = __any_sync(0xffffffffu, hz);
          }
        } else {
          uint32_t hz = 0;
#pragma unroll
          for (int r = 0; r < 4; ++r) hz |= any_zero_byte(Z[r]);
          slow = __any_sync(0xffffffffu, hz);
        }
        if (slow) {
#pragma unroll
          for (int r = 0; r < 4; ++r) {
            mask[r] = zero_byte_mask16(Z[r], P.movemask_mul);
            if (!interior) {
              const uint64_t us = tbase + seg_off + 16u * ((r + rot) & 3u);
              if (us < P.s_lo || us + 16 > P.s_hi) mask[r] &= range_mask(us, P.s_lo, P.s_hi);
            }
          }
          int qstart = 1;
          if constexpr (F2 > 0) {
            // many candidates (small alphabets): check pattern bytes 4..7 for all 16 alignments
            // in packed form before any scalar check
            const uint32_t c4 = __reduce_add_sync(0xffffffffu, __popc(mask[0]) + __popc(mask[1]) +
                                                                  __popc(mask[2]) + __popc(mask[3]));
            if (c4 > 64) {
#pragma unroll
              for (int r = 0; r < 4; ++r) {
                // (words reloaded from the stage: keeping W alive through the slow path would
                // spill registers)
                const uint32_t o = seg_off + 16u * ((r + rot) & 3u);
                const uint4 a = *reinterpret_cast<const uint4*>(ts + o);
                const uint2 c = *reinterpret_cast<const uint2*>(ts + o + 16);
                const uint32_t v[6] = {a.x, a.y, a.z, a.w, c.x, c.y};
                uint32_t Y[4];
                filter_second<F2>(v, FP, *JD, Y);
                mask[r] &= zero_byte_mask16(Y, P.movemask_mul);
              }
              qstart = 2;
            }
          }
          uint32_t left = 0;
#pragma unroll
          for (int r = 0; r < 4; ++r) {
            const uint32_t o = seg_off + 16u * ((r + rot) & 3u);
            if (MW > qstart && __any_sync(0xffffffffu, mask[r])) mask[r] = verify_candidates<MW>(mask[r], ts, o, *JD, qstart);
            left |= mask[r];
          }
          slow = __any_sync(0xffffffffu, left != 0u);
        }
      }
      if (slow) {
        // the lane's 64 starts as one mask: bit 16u + j = start seg_off + 16u + j
        uint64_t M = 0;
        if constexpr (SK == kEqMode || is_plane(SK)) {
          M = Meq;
        } else {
#pragma unroll
          for (int r = 0; r < 4; ++r) M |= static_cast<uint64_t>(mask[r]) << (16u * ((r + rot) & 3u));
        }
        const uint32_t c = popc64(M);
        acc += c;
        if constexpr (SEARCH) {
          if (!waited) {                       // the scratch may still be read by launch L-2
            wait_ws(S);
            waited = true;
          }
          st_keep_u64(scratch_cta + ((b * kChunkTiles + tpos) * kConsumerWarps + cw) * 32 + lane, M, keep_pol);
          const uint32_t sc = __reduce_add_sync(0xffffffffu, c);
          if (lane == 0) S.park[b].cnt[tpos * kConsumerWarps + cw] = sc;
          slowbits |= 1u << (kChunkTiles * b + tpos);
        }
      }
      __syncwarp();
      if (plane_tps(SK) == 1 || sub + 1 == c_ntc) {
        if (lane == 0) mbar_arrive(&S.empty[stage]);   // the text of this stage is no longer needed
        if (++stage == kStages) {
          stage = 0;
          phase ^= 1u;
        }
        sub = 0;
      } else {
        ++sub;                                         // the next tile of the stage's chunk
      }
      if constexpr (!SEARCH) continue;
      ++tpos;
      if (!last_in_chunk) continue;

      // ---- this warp is done with chunk #seq; the last warp to finish hands it off
      if (!waited) {                           // status words may still belong to launch L-2
        wait_ws(S);
        waited = true;
      }
      const uint32_t chunk = gch;
      const uint32_t ntiles = tpos;
      if (lane == 0) S.park[b].slow[cw] = static_cast<uint8_t>((slowbits >> (kChunkTiles * b)) & kTileBitsMask);
      __syncwarp();
      uint32_t prev = 0;
      if (lane == 0) {
        __threadfence_block();
        prev = atomicAdd(&S.park[b].done, 1u);
      }
      prev = __shfl_sync(0xffffffffu, prev, 0);
      if (prev == kConsumerWarps - 1) {
        __threadfence_block();
        // the chunk's total over the 64 slice counts (slices of warps that parked nothing for
        // a tile count zero); the exclusive slice offsets are left to the look-back warp
        constexpr int kPerLane = (kSlices + 31) / 32;
        uint32_t sum = 0;
#pragma unroll
        for (int i = 0; i < kPerLane; ++i) {
          const uint32_t sl = lane * kPerLane + i;              // text order (>= kSlices: none)
          const uint32_t t = sl / kConsumerWarps;
          const uint32_t w = sl % kConsumerWarps;
          sum += (sl < static_cast<uint32_t>(kSlices) && t < ntiles && ((S.park[b].slow[w] >> t) & 1u))
                     ? S.park[b].cnt[sl] : 0u;
        }
        const uint32_t total = __reduce_add_sync(0xffffffffu, sum);
        // a chunk without occurrences has no offsets to scan: its slot may be reused at once
        if (total == 0 && lane == 0) atomicMax(&S.park[b].scanned, seq + 1);
        if (seq >= kSlots) wait_done(seq - kSlots);          // slot seq % kSlots is free again
        if (lane == 0) {
          S.park[b].done = 0;
          S.park[b].chunk = chunk;
          S.park[b].total = total;
          S.park[b].ntiles = ntiles;
          // publish the aggregate at once so successors' look-backs never wait for our queue
          st_relaxed(P.status + chunk, P.tag | (chunk % P.nchunks == 0 ? kFlagInc : kFlagAgg) | total);
          const uint32_t q = seq % kSlots;
          S.slot[q].chunk = chunk;
          S.slot[q].total = total;
          S.slot[q].park = b;
          mbar_arrive(&S.lb_full[q]);
        }
        __syncwarp();
      }
      ++seq;
      tpos = 0;
    }

    if constexpr (!SEARCH) {
      // count: per-warp partials into the per-search workspace counters; the CTA's last warp
      // takes a ticket, and the last CTA publishes every search's occ and re-arms the counters
      // (no memset per call)
      if (cur_slot < 2) flush_count();
      if (!waited) {
        wait_ws(S);
        waited = true;
      }
      if (lane == 0) {
        __threadfence();
        const uint32_t prev = atomicAdd(&S.fin, 1u);
        if (prev == kConsumerWarps - 1) {
          EPSM_TRACE(P, 6);
          const unsigned long long ticket = atomicAdd(P.ctr + 2, 1ull);
          if (ticket == gridDim.x - 1) {
            __threadfence();
            griddep_wait();                    // the previous grid may write the same occ
            for (uint32_t j = 0; j < P.njobs; ++j) *P.jobs[j].occ = atomicExch(P.ctr + 8 + j, 0ull);
            P.ctr[2] = 0;
          }
        }
      }
    } else {
      // ---- drain: write out the chunks still parked, then (last warp) stop the look-back warp
      for (uint32_t k = seq > kParked ? seq - kParked : 0; k < seq; ++k) flush_chunk_seq(k);
      if (cw == 0 && lane == 0) {
        EPSM_TRACE(P, 5);
        if (P.trace) P.trace[blockIdx.x * 8 + 7] = seq;
      }
      uint32_t prev = 0;
      if (lane == 0) {
        __threadfence_block();
        prev = atomicAdd(&S.fin, 1u);
      }
      prev = __shfl_sync(0xffffffffu, prev, 0);
      if (prev == kConsumerWarps - 1 && lane == 0) {
        EPSM_TRACE(P, 6);
        if (seq >= kSlots) mbar_wait(&S.lb_done[(seq - kSlots) % kSlots], ((seq - kSlots) / kSlots) & 1u);
        const uint32_t q = seq % kSlots;
        S.slot[q].chunk = kInfoEnd;
        mbar_arrive(&S.lb_full[q]);
      }
    }
  }
  // retire: this CTA no longer touches the workspace parity (counter, status, parked masks)
  __syncthreads();
  if (tid == 0) red_release_add(P.exit_ctr, 1ull);
}

// ------------------------------------------------------------------ equality-mask index

// EPSMa's equality masks (wscmp of a text block against a broadcast pattern
// byte) computed once per text for a set of byte values and kept in HBM, so that every search
// of a batch over that text reads the masks of its own distinct bytes instead of recomputing
// them from the text: plane k, word w, bit i = [t[64w + i] == vals[k]]; zero past n and in the
// padding words up to pstride (the search kernel streams whole tiles + one halo word).
// Fan-out of one search's result (identical patterns have identical Occ): occ
// and the first min(occ, cap_o) positions of src to every output o.  The source streams
// through shared memory in 32 KiB chunks (TMA bulk loads, a 3-stage ring per CTA) and each
// chunk leaves as ONE TMA bulk store per output (cp.async.bulk.global.shared::cta): long
// contiguous writes, no register traffic -- a store of 8-byte words from registers to many
// interleaved destinations reached only ~3.3 TB/s.  Outputs of another 16-byte phase than
// the source (never produced by the library's own callers) take 8-byte stores from shared
// memory.
#ifndef EPSM_REP_CHUNK
#define EPSM_REP_CHUNK 32768
#endif
#ifndef EPSM_REP_STAGES
#define EPSM_REP_STAGES 3
#endif
#ifndef EPSM_REP_MAXOUT
#define EPSM_REP_MAXOUT 1024
#endif
constexpr uint32_t kRepChunk = EPSM_REP_CHUNK;                     // bytes per chunk
constexpr int kRepStages = EPSM_REP_STAGES;
constexpr uint32_t kRepMaxOut = EPSM_REP_MAXOUT;
constexpr int kRepThreads = 128;
struct RepSmem {
  uint64_t buf[kRepStages][kRepChunk / 8];
  uint64_t* pos[kRepMaxOut];
  uint64_t cnt[kRepMaxOut];
  alignas(8) uint64_t full[kRepStages];
  uint32_t odd_phase;                                              // some output has the other phase
};

__global__ void __launch_bounds__(kRepThreads) epsm_replicate_kernel(const uint64_t* __restrict__ src,
                                                                     const unsigned long long* __restrict__ src_occ,
                                                                     uint64_t src_cap, const XOut* __restrict__ x,
                                                                     uint32_t nx) {
  extern __shared__ __align__(128) uint8_t rep_raw[];
  RepSmem& S = *reinterpret_cast<RepSmem*>(rep_raw);
  const unsigned long long occ = *src_occ;
  if (nx > kRepMaxOut) nx = kRepMaxOut;                            // (the host splits larger fan-outs)
  if (blockIdx.x == 0)
    for (uint32_t o = threadIdx.x; o < nx; o += blockDim.x) *x[o].occ = occ;
  const uint64_t have = occ < src_cap ? occ : src_cap;
  if (!src || have == 0) return;
  const uint64_t lead = (reinterpret_cast<uintptr_t>(src) >> 3) & 1u;   // src + lead: 16-byte aligned
  if (threadIdx.x == 0) S.odd_phase = 0;
  __syncthreads();
  for (uint32_t o = threadIdx.x; o < nx; o += blockDim.x) {
    S.pos[o] = x[o].pos;
    S.cnt[o] = x[o].pos ? (x[o].cap < have ? x[o].cap : have) : 0;
    if (x[o].pos && S.cnt[o] > lead && (((reinterpret_cast<uintptr_t>(x[o].pos) >> 3) & 1u) != lead))
      S.odd_phase = 1;
    if (lead && blockIdx.x == 0 && S.cnt[o]) x[o].pos[0] = src[0];      // the element before the body
  }
  if (threadIdx.x < kRepStages) mbar_init(&S.full[threadIdx.x], 1);
  fence_mbar_init();
  __syncthreads();
  const bool odd = S.odd_phase != 0;
  const uint64_t body = have - lead;                               // elements from src + lead
  const uint64_t per = kRepChunk / 8;
  const uint64_t nchunk = (body + per - 1) / per;
  auto issue = [&](uint64_t c, int st) {                           // thread 0: chunk c -> stage st
    const uint64_t e0 = lead + c * per;
    const uint64_t ne = have - e0 < per ? have - e0 : per;
    const uint32_t bytes = static_cast<uint32_t>((ne * 8) & ~15ull);
    mbar_arrive_expect_tx(&S.full[st], bytes);
    if (bytes) bulk_g2s_plain(S.buf[st], src + e0, bytes, &S.full[st]);
  };
  if (threadIdx.x == 0)
    for (int st = 0; st < kRepStages; ++st) {
      const uint64_t c = blockIdx.x + static_cast<uint64_t>(st) * gridDim.x;
      if (c < nchunk) issue(c, st);
    }
  uint32_t phase = 0;
  int st = 0;
  for (uint64_t c = blockIdx.x; c < nchunk; c += gridDim.x) {
    mbar_wait(&S.full[st], phase);
    const uint64_t e0 = lead + c * per;
    const uint64_t ne = have - e0 < per ? have - e0 : per;
    if (threadIdx.x == 0) {
      const uint64_t last = (ne & 1u) ? src[e0 + ne - 1] : 0;      // (not in the 16-byte bulk part)
      for (uint32_t o = 0; o < nx; ++o) {
        const uint64_t cnt = S.cnt[o];
        if (cnt <= e0) continue;
        uint64_t* d = S.pos[o] + e0;
        if ((reinterpret_cast<uintptr_t>(d) & 15u) != 0) continue;  // other phase: below
        const uint64_t n = cnt - e0 < ne ? cnt - e0 : ne;
        const uint32_t bytes = static_cast<uint32_t>((n * 8) & ~15ull);
        if (bytes) bulk_s2g(d, S.buf[st], bytes);
        if (n & 1u) d[n - 1] = (n == ne) ? last : S.buf[st][n - 1];
      }
      bulk_commit();
    }
    if (odd) {                                                     // 8-byte stores from shared memory
      for (uint32_t o = 0; o < nx; ++o) {
        const uint64_t cnt = S.cnt[o];
        uint64_t* d = S.pos[o] + e0;
        if (cnt <= e0 || (reinterpret_cast<uintptr_t>(d) & 15u) == 0) continue;
        const uint64_t n = cnt - e0 < ne ? cnt - e0 : ne;
        const uint64_t nb = n & ~1ull;                             // the bulk part of the stage
        for (uint64_t i = threadIdx.x; i < nb; i += blockDim.x) d[i] = S.buf[st][i];
        if ((n & 1u) && threadIdx.x == 0) d[n - 1] = src[e0 + n - 1];
      }
    }
    __syncthreads();                                               // shared-memory reads done
    if (threadIdx.x == 0) {
      bulk_wait_read0();                                           // ... and the bulk stores' reads
      const uint64_t cn = c + static_cast<uint64_t>(kRepStages) * gridDim.x;
      if (cn < nchunk) issue(cn, st);
    }
    if (++st == kRepStages) {
      st = 0;
      phase ^= 1u;
    }
  }
  if (threadIdx.x == 0) bulk_wait0();
}

// The fan-outs of many searches in ONE launch (a group's duplicate patterns: dozens of copies of
// a few MB each, which one launch per source spends on ramp and tail): the sources' chunks are
// numbered one after another (job j's chunks start at cfirst[j], from its occ on the device) and
// the CTAs stride over that list; the outputs of the job of the current chunk sit in shared
// memory (reloaded when the job changes).  Only sources and outputs in the 16-byte phase (the
// library's own buffers; the host routes the rest to epsm_replicate_kernel).
constexpr int kRepMaxJobs = 256;
constexpr uint32_t kRepMultiOut = 256;
struct RepJobD {
  const uint64_t* src;
  const unsigned long long* occ;
  uint64_t cap;
  uint32_t x0, nx;              // outputs x[x0 .. x0 + nx)
};
struct RepMultiSmem {
  uint64_t buf[kRepStages][kRepChunk / 8];
  uint64_t* pos[kRepMultiOut];
  uint64_t cnt[kRepMultiOut];
  uint64_t cfirst[kRepMaxJobs + 1];
  uint64_t have[kRepMaxJobs];
  alignas(8) uint64_t full[kRepStages];
};

__global__ void __launch_bounds__(kRepThreads) epsm_replicate_multi_kernel(const RepJobD* __restrict__ J, uint32_t nj,
                                                                           const XOut* __restrict__ x) {
  extern __shared__ __align__(128) uint8_t rep_raw[];
  RepMultiSmem& S = *reinterpret_cast<RepMultiSmem*>(rep_raw);
  for (uint32_t j = threadIdx.x; j < nj; j += blockDim.x) {
    const unsigned long long occ = *J[j].occ;
    S.have[j] = J[j].src ? (occ < J[j].cap ? occ : J[j].cap) : 0;
    if (blockIdx.x == 0)
      for (uint32_t o = 0; o < J[j].nx; ++o) *x[J[j].x0 + o].occ = occ;
  }
  if (threadIdx.x < kRepStages) mbar_init(&S.full[threadIdx.x], 1);
  fence_mbar_init();
  __syncthreads();
  const uint64_t per = kRepChunk / 8;
  if (threadIdx.x == 0) {
    uint64_t c = 0;
    for (uint32_t j = 0; j < nj; ++j) {
      S.cfirst[j] = c;
      c += (S.have[j] + per - 1) / per;
    }
    S.cfirst[nj] = c;
  }
  __syncthreads();
  const uint64_t total = S.cfirst[nj];
  uint32_t jf = 0;                                                 // job of the next chunk to fetch
  auto issue = [&](uint64_t c, int st) {                           // thread 0: chunk c -> stage st
    while (S.cfirst[jf + 1] <= c) ++jf;
    const uint64_t e0 = (c - S.cfirst[jf]) * per;
    const uint64_t ne = S.have[jf] - e0 < per ? S.have[jf] - e0 : per;
    const uint32_t bytes = static_cast<uint32_t>((ne * 8) & ~15ull);
    mbar_arrive_expect_tx(&S.full[st], bytes);
    if (bytes) bulk_g2s_plain(S.buf[st], J[jf].src + e0, bytes, &S.full[st]);
  };
  if (threadIdx.x == 0)
    for (int st = 0; st < kRepStages; ++st) {
      const uint64_t c = blockIdx.x + static_cast<uint64_t>(st) * gridDim.x;
      if (c < total) issue(c, st);
    }
  uint32_t phase = 0, jc = 0, cur = 0xFFFFFFFFu;
  int st = 0;
  for (uint64_t c = blockIdx.x; c < total; c += gridDim.x) {
    while (S.cfirst[jc + 1] <= c) ++jc;                             // (uniform: every thread alike)
    if (jc != cur) {                                               // the outputs of job jc
      const uint64_t have = S.have[jc];
      for (uint32_t o = threadIdx.x; o < J[jc].nx; o += blockDim.x) {
        const XOut X = x[J[jc].x0 + o];
        S.pos[o] = X.pos;
        S.cnt[o] = X.pos ? (X.cap < have ? X.cap : have) : 0;
      }
      __syncthreads();
      cur = jc;
    }
    mbar_wait(&S.full[st], phase);
    const uint64_t e0 = (c - S.cfirst[jc]) * per;
    const uint64_t ne = S.have[jc] - e0 < per ? S.have[jc] - e0 : per;
    if (threadIdx.x == 0) {
      const uint64_t last = (ne & 1u) ? J[jc].src[e0 + ne - 1] : 0;   // (not in the 16-byte bulk part)
      const uint32_t nx = J[jc].nx;
      for (uint32_t o = 0; o < nx; ++o) {
        const uint64_t cnt = S.cnt[o];
        if (cnt <= e0) continue;
        uint64_t* d = S.pos[o] + e0;
        const uint64_t n = cnt - e0 < ne ? cnt - e0 : ne;
        const uint32_t bytes = static_cast<uint32_t>((n * 8) & ~15ull);
        if (bytes) bulk_s2g(d, S.buf[st], bytes);
        if (n & 1u) d[n - 1] = (n == ne) ? last : S.buf[st][n - 1];
      }
      bulk_commit();
    }
    __syncthreads();                                               // shared-memory reads done
    if (threadIdx.x == 0) {
      bulk_wait_read0();                                           // ... and the bulk stores' reads
      const uint64_t cn = c + static_cast<uint64_t>(kRepStages) * gridDim.x;
      if (cn < total) issue(cn, st);
    }
    if (++st == kRepStages) {
      st = 0;
      phase ^= 1u;
    }
  }
  if (threadIdx.x == 0) bulk_wait0();
}

constexpr int kMaxPlanes = 256;
struct IdxParams {
  const uint8_t* text;          // 16-byte aligned
  uint64_t n;
  uint64_t* planes;             // nv planes of pstride words
  uint64_t pstride;
  uint32_t nv;
  uint8_t vals[kMaxPlanes];     // the byte value of plane k
};

// The 64 bytes of text word w (bytes past n read as 0; `valid` masks their starts).
__device__ __forceinline__ void idx_load_word(const IdxParams& P, uint64_t w, uint32_t (&W)[16], uint64_t& valid) {
  const uint64_t b0 = w * 64;
  valid = ~0ull;
  if (b0 + 64 <= P.n) {
    const uint4* src = reinterpret_cast<const uint4*>(P.text + b0);
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const uint4 v = __ldg(src + r);
      W[4 * r] = v.x;
      W[4 * r + 1] = v.y;
      W[4 * r + 2] = v.z;
      W[4 * r + 3] = v.w;
    }
  } else {
#pragma unroll
    for (int q = 0; q < 16; ++q) W[q] = 0;
    const uint32_t have = b0 < P.n ? static_cast<uint32_t>(P.n - b0) : 0u;
    for (uint32_t i = 0; i < have; ++i) W[i >> 2] |= static_cast<uint32_t>(P.text[b0 + i]) << (8 * (i & 3));
    valid = have ? (1ull << have) - 1ull : 0ull;
  }
}

// Many values: bit-slice the 64 bytes once (8 masks: bit b of every byte), then every value's
// plane word is an AND of 8 masks or their complements -- ~16 logic ops per value instead of
// ~110 for comparing the bytes again.
__global__ void __launch_bounds__(256) epsm_eqidx_bits_kernel(const __grid_constant__ IdxParams P) {
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t w = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; w < P.pstride; w += stride) {
    uint32_t W[16];
    uint64_t valid;
    idx_load_word(P, w, W, valid);
    uint32_t lo[8], hi[8];                                  // bit b of the bytes at 0-31, 32-63
#pragma unroll
    for (int b = 0; b < 8; ++b) {
      uint32_t l = 0, h = 0;
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        l |= ((((W[k] >> b) & 0x01010101u) * 0x01020408u) >> 24) << (4 * k);
        h |= ((((W[k + 8] >> b) & 0x01010101u) * 0x01020408u) >> 24) << (4 * k);
      }
      lo[b] = l;
      hi[b] = h;
    }
    const uint32_t vl = static_cast<uint32_t>(valid), vh = static_cast<uint32_t>(valid >> 32);
    for (uint32_t q = 0; q < P.nv; ++q) {
      const uint32_t v = P.vals[q];
      uint32_t rl = vl, rh = vh;
#pragma unroll
      for (int b = 0; b < 8; ++b) {
        const uint32_t flip = ((v >> b) & 1u) - 1u;          // 0: bit set, ~0: bit clear
        rl &= lo[b] ^ flip;
        rh &= hi[b] ^ flip;
      }
      P.planes[q * P.pstride + w] = (static_cast<uint64_t>(rh) << 32) | rl;
    }
  }
}

__global__ void __launch_bounds__(256) epsm_eqidx_kernel(const __grid_constant__ IdxParams P) {
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t w = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; w < P.pstride; w += stride) {
    const uint64_t b0 = w * 64;
    uint4 R[4];
    uint64_t valid = ~0ull;
    if (b0 + 64 <= P.n) {
      const uint4* src = reinterpret_cast<const uint4*>(P.text + b0);
#pragma unroll
      for (int r = 0; r < 4; ++r) R[r] = __ldg(src + r);
    } else {
      // the text's last partial word (or padding): bytes past n read as 0 and masked out
      uint32_t wd[16];
#pragma unroll
      for (int q = 0; q < 16; ++q) wd[q] = 0;
      const uint32_t have = b0 < P.n ? static_cast<uint32_t>(P.n - b0) : 0u;
      for (uint32_t i = 0; i < have; ++i) wd[i >> 2] |= static_cast<uint32_t>(P.text[b0 + i]) << (8 * (i & 3));
#pragma unroll
      for (int r = 0; r < 4; ++r) R[r] = make_uint4(wd[4 * r], wd[4 * r + 1], wd[4 * r + 2], wd[4 * r + 3]);
      valid = have ? (1ull << have) - 1ull : 0ull;
    }
    for (uint32_t k = 0; k < P.nv; ++k) {
      const uint32_t vb = 0x01010101u * P.vals[k];
      uint64_t M = 0;
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const uint32_t Z[4] = {R[r].x ^ vb, R[r].y ^ vb, R[r].z ^ vb, R[r].w ^ vb};
        M |= static_cast<uint64_t>(zero_byte_mask16(Z, 0x00204081u)) << (16 * r);
      }
      P.planes[k * P.pstride + w] = M & valid;
    }
  }
}

}  // namespace epsm
