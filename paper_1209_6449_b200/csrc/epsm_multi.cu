// epsm_multi.cu -- host side of the group search (many patterns of one length over one text
// in one pass): group construction (deduplication, the shared EPSMc-style
// gram table, the choice of gram length and sampling stride), workspace and the three launches.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <map>
#include <mutex>
#include <new>
#include <string>
#include <vector>

#include "epsm.h"
#include "epsm_internal.h"
#include "epsm_multi.cuh"
#include "epsm_code.cuh"
#include "epsm_mask.cuh"

namespace mp = epsm::mp;
namespace cg = epsm::cg;

namespace {

// One pass over the text serves at most kMaxD distinct patterns (u8 ids in shared memory);
// a group of more is split into subgroups (one pass each).
struct RepJob {                        // a pattern with duplicate searches: its first output ...
  uint64_t* pos;
  uint64_t cap;
  unsigned long long* occ;
  uint32_t nx;                         // ... and the number of further outputs (rep_x, in order)
};

struct Subgroup {
  uint32_t D = 0, k = 0;               // distinct patterns, searches
  int q = 1, sk = 1, qw = 1;           // sk = 0: code mode (every start keyed, exact)
  uint32_t cb = 0;                     // code mode: bits per symbol code
  bool spare = false;                  // code mode: a spare code marks bytes outside the alphabet
  bool ident = false;                  // code mode: every pattern byte < 2^cb is its own code
  uint32_t qmask = 0xFFu, hmul[4] = {0, 0, 0, 0};
  std::vector<uint32_t> jobs;          // the caller's search index of local search j
  mp::GroupDesc* h_desc = nullptr;
  mp::GroupDesc* d_desc = nullptr;
  double cost = 0;                     // model estimate (instructions per 64 text bytes)
  std::vector<RepJob> rep_jobs;        // per call: duplicate searches to copy after pass 3
  std::vector<epsm::XOut> rep_x;
};

constexpr uint32_t kMul[4] = {0x9E3779B1u, 0x85EBCA77u, 0xC2B2AE3Du, 0x27D4EB2Fu};

uint32_t hash_key(const uint8_t* g, int q, const Subgroup& S) {
  uint32_t h = 0;
  for (int r = 0; r < S.qw; ++r) {
    uint32_t w = 0;
    for (int b = 0; b < 4 && 4 * r + b < q; ++b) w |= static_cast<uint32_t>(g[4 * r + b]) << (8 * b);
    h += w * S.hmul[r];
  }
  return h;
}

// Sampling geometry (q-gram length, stride SK) for D distinct patterns of length m whose bytes
// have collision probability p2 (a pair of random text bytes is equal with probability ~p2 if
// the text looks like the patterns -- they are extracted from it).  Cost model in
// lane instructions per 64 text bytes: samples (key extraction, hash, bitmap test), bitmap
// hits (bucket walk), candidates (naive check).  Speed only: every geometry is exact.
void choose_geometry(uint32_t m, uint32_t D, double p2, Subgroup& S) {
  double best = 1e300;
  const int mw = static_cast<int>((m + 3) / 4);
  for (int q = 1; q <= static_cast<int>(std::min<uint32_t>(m, 16)); ++q) {
    const int qw = (q + 3) / 4;
    const double pq = std::pow(p2, q);                       // a sample equals a given gram
    for (int sk = 1; sk <= 16; sk *= 2) {
      if (sk > static_cast<int>(m) - q + 1 || static_cast<uint64_t>(sk) * D > mp::kMaxEntries) continue;
      const double nsamp = 64.0 / sk + (sk > 1 ? 1 : 0);
      const double entries = static_cast<double>(sk) * D;
      const double p_true = std::min(1.0, entries * pq);
      const double fill = 1.0 - std::exp(-2.0 * entries / 65536.0);   // two probes per gram
      const double p_false = q <= 2 ? 0.0 : fill * fill;
      const double p_hit = std::min(1.0, p_true + p_false);
      const double c_sample = 14 + 2 * qw;
      const double c_hit = 14 + 3 * qw + 3 * (entries / 4096.0);
      const double cand_per_start = std::min(64.0, D * pq);  // true gram matches per start
      const double c_verify = 10 + 4 * mw;
      // a bucket walk is divergent: a warp pays it when ANY of its 32 lanes hits, for as many
      // rounds as its busiest lane has hits
      const double lane_hits = nsamp * p_hit;
      const double p_warp = 1.0 - std::pow(1.0 - std::min(1.0, lane_hits), 32.0);
      const double cost = nsamp * c_sample + p_warp * c_hit * std::max(1.0, 2.0 * lane_hits) +
                          64.0 * cand_per_start * c_verify;
      if (cost < best * 0.999 || (cost <= best * 1.001 && q > S.q)) {
        best = std::min(best, cost);
        S.q = q;
        S.sk = sk;
        S.qw = qw;
      }
    }
  }
  S.cost = best;
  S.qmask = (S.q % 4 == 0) ? 0xFFFFFFFFu : ((1u << (8 * (S.q % 4))) - 1u);
  if (S.q <= 2) {
    S.hmul[0] = 1u << 16;                                    // the key itself: an exact bitmap
  } else {
    for (int r = 0; r < 4; ++r) S.hmul[r] = kMul[r];
  }
}

using MKernel = void (*)(mp::MParams);

template <int SK, int QW>
MKernel pick_mk(bool write) {
  return write ? &mp::epsm_multi_kernel<SK, QW, true> : &mp::epsm_multi_kernel<SK, QW, false>;
}

template <int SK>
MKernel pick_qw(int qw, bool write) {
  switch (qw) {
    case 1: return pick_mk<SK, 1>(write);
    case 2: return pick_mk<SK, 2>(write);
    case 3: return pick_mk<SK, 3>(write);
    default: return pick_mk<SK, 4>(write);
  }
}

MKernel multi_kernel_for(int sk, int qw, bool write) {
  switch (sk) {
    case -1: return pick_mk<-1, 1>(write);
    case 0: return pick_mk<0, 1>(write);
    case 1: return pick_qw<1>(qw, write);
    case 2: return pick_qw<2>(qw, write);
    case 4: return pick_qw<4>(qw, write);
    case 8: return pick_qw<8>(qw, write);
    default: return pick_qw<16>(qw, write);
  }
}

// EPSM_MULTI_GEOM="q:sk" forces the geometry of every subgroup (A/B timing; must satisfy
// sk + q - 1 <= m and D * sk <= 4096, else ignored).
void geometry_override(uint32_t m, uint32_t D, Subgroup& S) {
  static const char* e = getenv("EPSM_MULTI_GEOM");
  if (!e || !e[0]) return;
  int q = 0, sk = 0;
  if (sscanf(e, "%d:%d", &q, &sk) != 2) return;
  if (q < 1 || q > 16 || (sk & (sk - 1)) || sk < 1 || sk > 16 || sk + q - 1 > static_cast<int>(m) ||
      static_cast<uint64_t>(sk) * D > mp::kMaxEntries)
    return;
  S.q = q;
  S.sk = sk;
  S.qw = (q + 3) / 4;
  S.qmask = (q % 4 == 0) ? 0xFFFFFFFFu : ((1u << (8 * (q % 4))) - 1u);
  if (q <= 2) {
    S.hmul[0] = 1u << 16;
    S.hmul[1] = S.hmul[2] = S.hmul[3] = 0;
  } else {
    for (int r = 0; r < 4; ++r) S.hmul[r] = kMul[r];
  }
}

}  // namespace

struct epsm_group_s {
  uint32_t m = 0, k = 0, D = 0;
  int device = -1;
  std::vector<Subgroup> subs;
  std::vector<std::string> pats;                  // distinct patterns
  std::vector<std::vector<uint32_t>> dups;        // searches per distinct pattern
  // dense distinct patterns (estimated >= 2^-dense_log2 occurrences per text byte): searched
  // one by one through the single-pattern kernels (their positions, >= 4 bytes of output per
  // 1000 text bytes, dominate; the shared pass gains little there); the rest share the passes
  std::vector<uint32_t> sparse, dense;            // distinct pattern indices
  double sparse_rate = 0;                         // estimated matches per text byte of the sparse ones
  bool forced_geom = false;                       // epsm_group_set_geometry (tests, A/B)
  std::vector<epsm_plan_t*> dplans;               // plan of dense[i] (one scan, fanned out to its
                                                  // searches: they have the same positions)
};

// EPSM_MULTI_CODE=0 disables the code mode (A/B timing; every mode is exact)
static bool code_disabled() {
  static const bool v = [] {
    const char* e = getenv("EPSM_MULTI_CODE");
    return e && e[0] == '0';
  }();
  return v;
}
// EPSM_CODE_IDENT=0: code mode always codes the pattern bytes by rank (A/B; both exact)
static bool ident_disabled() {
  static const bool v = [] {
    const char* e = getenv("EPSM_CODE_IDENT");
    return e && e[0] == '0';
  }();
  return v;
}

// the code mode's cost in the cost model's units (lane instructions per 64 text bytes): 80 key
// steps of ~10 instructions
constexpr double kCodeCost = 850.0;

static int build_subgroup(const std::vector<std::string>& pats, uint32_t m, Subgroup& S,
                          const std::vector<std::vector<uint32_t>>& dups, int force_q = 0, int force_sk = 0) {
  const uint32_t D = static_cast<uint32_t>(pats.size());
  // collision probability of the patterns' bytes (unbiased: pairs of distinct positions)
  uint64_t cnt[256] = {};
  uint64_t N = 0;
  for (const auto& p : pats)
    for (unsigned char ch : p) ++cnt[ch], ++N;
  double p2 = 1.0;
  if (N > 1) {
    double num = 0;
    for (int c = 0; c < 256; ++c) num += static_cast<double>(cnt[c]) * (cnt[c] ? cnt[c] - 1 : 0);
    p2 = std::max(num / (static_cast<double>(N) * (N - 1)), 1.0 / 256.0);
  }
  S.D = D;
  choose_geometry(m, D, p2, S);
  geometry_override(m, D, S);
  // code mode: the patterns' distinct bytes coded in cb bits, m * cb <= 14 bits of key; it
  // costs ~10 instructions per start whatever the density, so it wins where the sampled filter
  // meets many candidates (dense groups over small alphabets)
  uint32_t sigp = 0;
  for (int c = 0; c < 256; ++c) sigp += cnt[c] ? 1u : 0u;
  uint32_t cb = 1;
  while ((1u << cb) < sigp) ++cb;
  // (the wide mode -- keys of 15-16 bits in a bitmap + buckets -- only when forced: its ~1.3 ms
  // per 256 MiB never beat the sampled filter in the measured cases, sigma=4 m=8 1.32 vs 0.39 ms,
  // sigma=256 m=2 1.44 vs 0.36 ms; the table mode does where the sampled filter meets many
  // candidates: sigma=64 m=2 0.96 vs 2.3 ms)
  const bool code_ok = m * cb <= static_cast<uint32_t>(mp::kWideKeyBits) && !code_disabled();
  const bool wide = m * cb > static_cast<uint32_t>(mp::kCodeKeyBits);   // bitmap + buckets, no table
  const bool force_code = force_q && force_sk == 0;
  if (force_code && !code_ok) return EPSM_EINVAL;
  if ((code_ok && !wide && !force_q && S.cost > kCodeCost) || force_code) {
    S.sk = wide ? -1 : 0;
    S.q = static_cast<int>(m);
    S.qw = 1;
    S.cb = cb;
    // a spare code (one more bit if the key still fits the table) spares the kernel the
    // tracking of bytes outside the alphabet
    S.spare = (1u << cb) > sigp;
    if (!S.spare && !wide && m * (cb + 1) <= static_cast<uint32_t>(mp::kCodeKeyBits)) {
      S.cb = cb + 1;
      S.spare = true;
    }
    // identity codes where every pattern byte is below 2^cb' and the key still fits the table
    // (the code-mode kernels then skip the byte -> code load per start); no spare code needed:
    // a non-pattern byte below 2^cb' is its own code (no pattern key holds it), one above is
    // invalid
    uint32_t maxb = 0;
    for (int c = 0; c < 256; ++c)
      if (cnt[c]) maxb = static_cast<uint32_t>(c);
    uint32_t cbi = 1;
    while ((1u << cbi) <= maxb) ++cbi;
    if (!wide && m * cbi <= static_cast<uint32_t>(mp::kCodeKeyBits) && !ident_disabled()) {
      S.cb = cbi;
      S.spare = false;
      S.ident = true;
    }
  } else if (force_q) {
    S.q = force_q;
    S.sk = force_sk;
    S.qw = (force_q + 3) / 4;
    S.qmask = (force_q % 4 == 0) ? 0xFFFFFFFFu : ((1u << (8 * (force_q % 4))) - 1u);
    for (int r = 0; r < 4; ++r) S.hmul[r] = force_q <= 2 ? (r == 0 ? 1u << 16 : 0u) : kMul[r];
  }
  if (!S.h_desc) S.h_desc = new (std::nothrow) mp::GroupDesc();
  if (!S.h_desc) return EPSM_ENOMEM;
  mp::GroupDesc& G = *S.h_desc;
  std::memset(&G, 0, sizeof(G));
  // patterns, zero padded, and the byte masks of their words
  for (uint32_t d = 0; d < D; ++d)
    for (uint32_t b = 0; b < m; ++b)
      G.pat[d][b / 4] |= static_cast<uint32_t>(static_cast<unsigned char>(pats[d][b])) << (8 * (b % 4));
  for (uint32_t b = 0; b < m; ++b) G.pmask[b / 4] |= 0xFFu << (8 * (b % 4));
  std::vector<std::vector<uint16_t>> wide_buckets;
  if (S.sk <= 0) {
    // code mode: byte -> code (pattern bytes in order of value), key table (the codes of a
    // window, its LAST byte in the low bits -- the kernel's rolling key) -> pattern; the wide
    // mode (keys of 15-16 bits) keeps an exact 2^16-bit bitmap of the keys and buckets by key >> 4
    // whose entries hold the pattern and the key's low 4 bits
    uint32_t code = 0;
    for (int c = 0; c < 256; ++c) code += cnt[c] ? 1u : 0u;
    std::memset(G.cmap, S.spare ? static_cast<int>(code) : 0x80, sizeof(G.cmap));   // (spare code = sigma')
    code = 0;
    if (S.ident) {
      for (int c = 0; c < (1 << S.cb); ++c) G.cmap[c] = static_cast<uint8_t>(c);
    } else {
      for (int c = 0; c < 256; ++c)
        if (cnt[c]) G.cmap[c] = static_cast<uint8_t>(code++);
    }
    uint8_t* lut = reinterpret_cast<uint8_t*>(G.bitmap);
    if (S.sk == 0) std::memset(lut, 0xFF, 1u << mp::kCodeKeyBits);
    else wide_buckets.assign(1u << mp::kBucketLog, {});
    for (uint32_t d = 0; d < D; ++d) {
      uint32_t key = 0;
      for (uint32_t j = 0; j < m; ++j)
        key = (key << S.cb) | G.cmap[static_cast<unsigned char>(pats[d][j])];
      if (S.sk == 0) {
        lut[key] = static_cast<uint8_t>(d);
      } else {
        G.bitmap[key >> 5] |= 1u << (key & 31u);
        wide_buckets[key >> 4].push_back(static_cast<uint16_t>((d << 8) | (key & 15u)));
      }
    }
  }
  // the table (EPSMc's L, for every pattern at once): gram p_d[i .. i+q) of
  // every distinct pattern d and offset i < SK, bucketed by the top 12 bits of its hash
  std::vector<std::vector<uint16_t>> buckets(1u << mp::kBucketLog);
  for (uint32_t d = 0; d < D && S.sk > 0; ++d) {
    for (int i = 0; i < S.sk; ++i) {
      const uint32_t h = hash_key(reinterpret_cast<const uint8_t*>(pats[d].data()) + i, S.q, S);
      G.bitmap[h >> (32 - mp::kBitmapLog + 5)] |= 1u << ((h >> (32 - mp::kBitmapLog)) & 31u);
      if (S.q > 2) {
        const uint32_t h2 = mp::bloom2(h);
        G.bitmap[h2 >> (32 - mp::kBitmapLog + 5)] |= 1u << ((h2 >> (32 - mp::kBitmapLog)) & 31u);
      }
      buckets[h >> (32 - mp::kBucketLog)].push_back(
          static_cast<uint16_t>((d << 8) | (static_cast<uint32_t>(i) << 4) | ((h >> (32 - mp::kBitmapLog)) & 15u)));
    }
  }
  uint32_t e = 0;
  if (S.sk != 0) {
    const auto& bks = S.sk > 0 ? buckets : wide_buckets;
    for (uint32_t b = 0; b < (1u << mp::kBucketLog); ++b) {
      G.boff[b] = static_cast<uint16_t>(e);
      for (uint16_t v : bks[b]) G.ent[e++] = v;
    }
    for (uint32_t b = (1u << mp::kBucketLog); b < (1u << mp::kBucketLog) + 8; ++b)
      G.boff[b] = static_cast<uint16_t>(e);
  }
  // searches per distinct pattern
  uint32_t q = 0;
  S.jobs.clear();
  for (uint32_t d = 0; d < D; ++d) {
    G.dup_off[d] = static_cast<uint16_t>(q);
    for (uint32_t j : dups[d]) {
      G.dup_list[q] = static_cast<uint16_t>(S.jobs.size());
      G.job_d[S.jobs.size()] = static_cast<uint16_t>(d);
      G.job_g[S.jobs.size()] = static_cast<uint16_t>(j);
      S.jobs.push_back(j);
      ++q;
    }
  }
  G.dup_off[D] = static_cast<uint16_t>(q);
  G.dup_off[D + 1] = static_cast<uint16_t>(q);
  S.k = q;
  return EPSM_OK;
}

static void group_release(epsm_group_t* g) {
  if (!g) return;
  for (epsm_plan_t* p : g->dplans) epsm_plan_free(p);
  bool synced = false;
  for (auto& S : g->subs) {
    if (S.d_desc) {
      if (!synced && g->device >= 0) {
        cudaSetDevice(g->device);
        cudaDeviceSynchronize();
        synced = true;
      }
      cudaFree(S.d_desc);
    }
    delete S.h_desc;
  }
  delete g;
}

// Make the workspace of stream s hold the group buffers for `chunks` chunks of D patterns.
static int ensure_multi_ws(epsm_workspace* ws, uint64_t chunks, uint32_t D, cudaStream_t s) {
  auto grow = [&](void** p, uint64_t& cap, uint64_t want, const char* what) -> int {
    if (want <= cap) return EPSM_OK;
    if (*p) {
      cudaStreamSynchronize(s);
      cudaFree(*p);
      *p = nullptr;
      cap = 0;
    }
    const uint64_t bytes = std::max<uint64_t>(want, 4096);
    cudaError_t e = cudaMalloc(p, bytes);
    if (e != cudaSuccess) {
      cudaGetLastError();
      *p = nullptr;
      epsm_set_error("cudaMalloc(%s, %llu bytes): %s", what, (unsigned long long)bytes, cudaGetErrorString(e));
      return EPSM_ENOMEM;
    }
    cap = bytes;
    return EPSM_OK;
  };
  int rc = grow(reinterpret_cast<void**>(&ws->m_counts), ws->m_counts_cap, chunks * D * sizeof(uint16_t), "counts");
  if (!rc) rc = grow(reinterpret_cast<void**>(&ws->m_prefix), ws->m_prefix_cap, chunks * D * 8, "prefix");
  if (!rc) rc = grow(reinterpret_cast<void**>(&ws->m_listlen), ws->m_listlen_cap, chunks * 4, "list lengths");
  if (!rc)
    rc = grow(reinterpret_cast<void**>(&ws->m_lists), ws->m_lists_cap, chunks * mp::kListCap * 4ull, "chunk lists");
  if (!rc) rc = grow(reinterpret_cast<void**>(&ws->m_work), ws->m_work_cap, (chunks + 1) * 4, "work list");
  if (!rc)
    rc = grow(reinterpret_cast<void**>(&ws->m_jobs), ws->m_jobs_cap, mp::kMaxJobs * sizeof(mp::JobOut), "job table");
  return rc;
}

static int multi_smem_bytes(bool write) {
  return static_cast<int>(write ? sizeof(mp::MSmemT<true>) : sizeof(mp::MSmemT<false>));
}

static int set_multi_smem(MKernel fn, bool write) {
  // (the attribute is per device: remember (kernel, device) pairs)
  int dev = 0;
  cudaGetDevice(&dev);
  static std::vector<std::pair<MKernel, int>> done;
  static std::mutex mu;
  std::lock_guard<std::mutex> lk(mu);
  if (std::find(done.begin(), done.end(), std::make_pair(fn, dev)) != done.end()) return EPSM_OK;
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       multi_smem_bytes(write));
  if (e != cudaSuccess) return epsm_cuda_fail(e, "cudaFuncSetAttribute(group kernel smem)");
  done.emplace_back(fn, dev);
  return EPSM_OK;
}

// EPSM_CODE_CG=0: code-mode groups keep the general group kernels (A/B timing; both exact)
static bool cg_disabled() {
  static const bool v = [] {
    const char* e = getenv("EPSM_CODE_CG");
    return e && e[0] == '0';
  }();
  return v;
}

using CKernel = void (*)(cg::CParams);

template <int M>
CKernel pick_cg(bool write, bool ident) {
  if (ident) return write ? &cg::cg_write_kernel<M, true> : &cg::cg_count_kernel<M, true>;
  return write ? &cg::cg_write_kernel<M, false> : &cg::cg_count_kernel<M, false>;
}

static CKernel cg_kernel_for(uint32_t m, bool write, bool ident) {
  switch (m) {
    case 1: return pick_cg<1>(write, ident);
    case 2: return pick_cg<2>(write, ident);
    case 3: return pick_cg<3>(write, ident);
    case 4: return pick_cg<4>(write, ident);
    case 5: return pick_cg<5>(write, ident);
    case 6: return pick_cg<6>(write, ident);
    case 7: return pick_cg<7>(write, ident);
    default: return pick_cg<8>(write, ident);
  }
}

static int set_cg_smem(CKernel fn, bool write) {
  int dev = 0;
  cudaGetDevice(&dev);
  static std::vector<std::pair<CKernel, int>> done;
  static std::mutex mu;
  std::lock_guard<std::mutex> lk(mu);
  if (std::find(done.begin(), done.end(), std::make_pair(fn, dev)) != done.end()) return EPSM_OK;
  const int bytes = static_cast<int>(write ? sizeof(cg::WrSmem) : sizeof(cg::CntSmem));
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e != cudaSuccess) return epsm_cuda_fail(e, "cudaFuncSetAttribute(code-mode kernel smem)");
  done.emplace_back(fn, dev);
  return EPSM_OK;
}

// The three launches of one subgroup over d_text[0..nbytes): starts [0, nstarts) reported as
// start + base.  pos/caps/occ are the caller's batch arrays (indexed by the caller's search).
static int subgroup_launch(epsm_group_t* g, Subgroup& S, const uint8_t* d_text, uint64_t nbytes, uint64_t nstarts,
                           uint64_t base, uint64_t* const* d_pos, const uint64_t* caps, uint64_t* d_occ, bool search,
                           cudaStream_t s) {
  if (!S.d_desc) {
    cudaError_t e = cudaMalloc(&S.d_desc, sizeof(mp::GroupDesc));
    if (e != cudaSuccess) {
      S.d_desc = nullptr;
      epsm_set_error("cudaMalloc(group descriptor): %s", cudaGetErrorString(e));
      return EPSM_ENOMEM;
    }
    e = cudaMemcpy(S.d_desc, S.h_desc, sizeof(mp::GroupDesc), cudaMemcpyHostToDevice);
    if (e != cudaSuccess) return epsm_cuda_fail(e, "cudaMemcpy(group descriptor)");
  }
  if (nstarts == 0) {
    for (uint32_t j : S.jobs) {
      cudaError_t e = cudaMemsetAsync(d_occ + j, 0, 8, s);
      if (e != cudaSuccess) return epsm_cuda_fail(e, "cudaMemsetAsync(occ)");
    }
    return EPSM_OK;
  }
  const uint64_t mis = reinterpret_cast<uintptr_t>(d_text) & 15u;
  mp::MParams P;
  std::memset(&P, 0, sizeof(P));
  P.text = d_text - mis;
  P.nbytes = nbytes + mis;
  P.s_lo = mis;
  P.s_hi = mis + nstarts;
  P.pos_bias = base - mis;
  const uint64_t chunks = (P.s_hi + mp::kTile - 1) / mp::kTile;
  if (chunks > 0x7FFFFFFFull) {
    epsm_set_error("text too large for a group search");
    return EPSM_EINVAL;
  }
  P.nchunks = static_cast<uint32_t>(chunks);
  P.it_lo = mis ? 1u : 0u;
  P.it_hi = static_cast<uint32_t>(P.s_hi / mp::kTile);
  P.m = g->m;
  P.mw = (g->m + 3) / 4;
  P.D = S.D;
  P.k = S.k;
  P.qmask = S.qmask;
  P.bloom2 = (S.sk > 0 && S.q > 2) ? 1u : 0u;
  P.cb = S.cb;
  P.kmask = S.sk <= 0 ? (1u << (g->m * S.cb)) - 1u : 0u;
  P.mmask = S.sk <= 0 ? (1u << g->m) - 1u : 0u;
  P.spare = S.sk <= 0 && S.spare ? 1u : 0u;
  P.ident = S.sk == 0 && S.ident ? 1u : 0u;
  P.identmask = 0xFFu & ~((1u << S.cb) - 1u);
  // direct counting in pass 1 only where the chunks would overflow their lists anyway (> 256
  // expected matches per 32 KiB chunk); sparser groups keep the lists (pass 3 without the text)
  P.direct = (S.sk <= 0 && g->sparse_rate * mp::kTile > static_cast<double>(mp::kListCap)) ? 1u : 0u;
  for (int r = 0; r < 4; ++r) P.hmul[r] = S.hmul[r];
  P.desc = S.d_desc;
  P.desc_bytes = sizeof(mp::GroupDesc);
  epsm_workspace* ws = epsm_get_workspace(g->device, s);
  if (!ws) return EPSM_ENOMEM;
  if (ws->num_sms <= 0) {
    cudaError_t e = cudaDeviceGetAttribute(&ws->num_sms, cudaDevAttrMultiProcessorCount, g->device);
    if (e != cudaSuccess) return epsm_cuda_fail(e, "cudaDeviceGetAttribute(SM count)");
  }
  int rc = ensure_multi_ws(ws, chunks, S.D, s);
  if (rc) return rc;
  P.counts = ws->m_counts;
  P.listlen = ws->m_listlen;
  P.lists = ws->m_lists;
  P.prefix = ws->m_prefix;
  P.work = ws->m_work;
  if (search) {
    // the searches' outputs, in stream order into the workspace's job table (a pageable copy
    // is staged before cudaMemcpyAsync returns, so the host vector may go)
    std::vector<mp::JobOut> jt(S.k);
    for (uint32_t j = 0; j < S.k; ++j) {
      const uint32_t gj = S.jobs[j];
      jt[j].pos = d_pos ? d_pos[gj] : nullptr;
      jt[j].cap = (d_pos && d_pos[gj] && caps) ? caps[gj] : 0;
    }
    // pass 3 writes each pattern's FIRST output only (the largest capacity: the outputs are
    // swapped among the pattern's searches -- their occ is the same); the others are copied from
    // it afterwards by the replicate kernel (fan-out, like the dense patterns' searches)
    const mp::GroupDesc& Gh = *S.h_desc;
    std::vector<epsm::XOut> xo;
    std::vector<std::pair<uint32_t, uint32_t>> rep;   // (first local job, number of further outputs)
    for (uint32_t d = 0; d < S.D; ++d) {
      const uint32_t a = Gh.dup_off[d], b = Gh.dup_off[d + 1];
      if (b - a < 2) continue;
      uint32_t best = a;
      for (uint32_t q = a + 1; q < b; ++q)
        if (jt[Gh.dup_list[q]].cap > jt[Gh.dup_list[best]].cap) best = q;
      std::swap(jt[Gh.dup_list[a]], jt[Gh.dup_list[best]]);
      rep.emplace_back(Gh.dup_list[a], b - a - 1);
      for (uint32_t q = a + 1; q < b; ++q) {
        const mp::JobOut& J = jt[Gh.dup_list[q]];
        xo.push_back(epsm::XOut{J.cap ? J.pos : nullptr, J.cap,
                                reinterpret_cast<unsigned long long*>(d_occ + Gh.job_g[Gh.dup_list[q]])});
      }
    }
    S.rep_jobs.clear();
    for (const auto& r : rep) {
      const mp::JobOut& J = jt[r.first];
      S.rep_jobs.push_back(RepJob{J.pos, J.cap, reinterpret_cast<unsigned long long*>(d_occ + Gh.job_g[r.first]),
                                  r.second});
    }
    S.rep_x = xo;
    cudaError_t e = cudaMemcpyAsync(ws->m_jobs, jt.data(), S.k * sizeof(mp::JobOut), cudaMemcpyHostToDevice, s);
    if (e != cudaSuccess) return epsm_cuda_fail(e, "cudaMemcpyAsync(group job table)");
    P.jobs = ws->m_jobs;
  }
  const int smem = multi_smem_bytes(false), smem3 = multi_smem_bytes(true);
  // code-mode groups of <= 127 distinct patterns of length <= 8: the dedicated kernels
  // (epsm_code.cuh: per-lane counters + staged coalesced write-out instead of match_any rounds)
  // -- where the chunks overflow the general pass 1's occurrence lists anyway (the lists spare
  // sparser groups a second read of the text), or where the code mode was forced
  const bool use_cg = S.sk == 0 && S.D <= static_cast<uint32_t>(cg::kMaxD) && g->m <= static_cast<uint32_t>(cg::kMaxM) &&
                      !cg_disabled() && (P.direct || g->forced_geom);
  cg::CParams C;
  std::memset(&C, 0, sizeof(C));
  C.text = P.text;
  C.nbytes = P.nbytes;
  C.s_lo = P.s_lo;
  C.s_hi = P.s_hi;
  C.pos_bias = P.pos_bias;
  C.nchunks = P.nchunks;
  C.it_lo = P.it_lo;
  C.it_hi = P.it_hi;
  C.cb = P.cb;
  C.kmask = P.kmask;
  C.D = P.D;
  C.invmask = S.ident ? (0xFFu & ~((1u << S.cb) - 1u)) : 0x80u;
  C.desc = P.desc;
  C.counts = P.counts;
  C.listlen = P.listlen;
  C.prefix = P.prefix;
  C.work = P.work;
  C.jobs = P.jobs;
  const unsigned grid = static_cast<unsigned>(std::min<uint64_t>(chunks, static_cast<uint64_t>(ws->num_sms)));
  if (use_cg) {
    // pass 1: counts per (chunk, distinct pattern)
    CKernel c1 = cg_kernel_for(g->m, false, S.ident);
    rc = set_cg_smem(c1, false);
    if (rc) return rc;
    c1<<<grid, cg::kCntThreads, sizeof(cg::CntSmem), s>>>(C);
  } else {
    // pass 1: counts per (chunk, distinct pattern), lists of sparse chunks
    MKernel k1 = multi_kernel_for(S.sk, S.qw, false);
    rc = set_multi_smem(k1, false);
    if (rc) return rc;
    k1<<<grid, mp::kThreads, smem, s>>>(P);
  }
  epsm_count_launch();
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return epsm_cuda_fail(e, "epsm_multi_kernel (pass 1) launch");
  // pass 2: prefixes, totals (occ), chunks with occurrences
  mp::ScanParams Q;
  Q.counts = ws->m_counts;
  Q.listlen = ws->m_listlen;
  Q.prefix = search ? ws->m_prefix : nullptr;
  Q.work = ws->m_work;
  Q.occ = reinterpret_cast<unsigned long long*>(d_occ);
  Q.desc = S.d_desc;
  Q.nchunks = P.nchunks;
  Q.D = S.D;
  Q.k = S.k;
  mp::epsm_multi_scan_kernel<<<S.D + 1, mp::kScanThreads, 0, s>>>(Q);
  epsm_count_launch();
  e = cudaGetLastError();
  if (e != cudaSuccess) return epsm_cuda_fail(e, "epsm_multi_scan_kernel launch");
  if (!search) return EPSM_OK;
  // pass 3: positions of the chunks with occurrences
  if (use_cg) {
    CKernel c3 = cg_kernel_for(g->m, true, S.ident);
    rc = set_cg_smem(c3, true);
    if (rc) return rc;
    c3<<<ws->num_sms, cg::kWrThreads, sizeof(cg::WrSmem), s>>>(C);
  } else {
    MKernel k3 = multi_kernel_for(S.sk, S.qw, true);
    rc = set_multi_smem(k3, true);
    if (rc) return rc;
    k3<<<ws->num_sms, mp::kThreads, smem3, s>>>(P);
  }
  epsm_count_launch();
  e = cudaGetLastError();
  if (e != cudaSuccess) return epsm_cuda_fail(e, "epsm_multi_kernel (pass 3) launch");
  if (!S.rep_x.empty()) {
    // duplicate searches: copies of their pattern's first output (one replicate per pattern)
    if (S.rep_x.size() > ws->xout_cap) {
      if (ws->d_xout) {
        cudaStreamSynchronize(s);
        cudaFree(ws->d_xout);
        ws->d_xout = nullptr;
        ws->xout_cap = 0;
      }
      e = cudaMalloc(&ws->d_xout, S.rep_x.size() * sizeof(epsm::XOut));
      if (e != cudaSuccess) {
        epsm_set_error("cudaMalloc(fan-out table): %s", cudaGetErrorString(e));
        return EPSM_ENOMEM;
      }
      ws->xout_cap = S.rep_x.size();
    }
    e = cudaMemcpyAsync(ws->d_xout, S.rep_x.data(), S.rep_x.size() * sizeof(epsm::XOut), cudaMemcpyHostToDevice, s);
    if (e != cudaSuccess) return epsm_cuda_fail(e, "cudaMemcpyAsync(fan-out table)");
    // every duplicated pattern's further outputs in one fan-out launch
    std::vector<epsm_rep_req> rq;
    uint32_t off = 0;
    for (const RepJob& r : S.rep_jobs) {
      rq.push_back(epsm_rep_req{r.pos, r.cap, r.occ, off, r.nx});
      off += r.nx;
    }
    rc = epsm_replicate_many(rq.data(), static_cast<uint32_t>(rq.size()), ws->d_xout, S.rep_x.data(), true, s, ws);
    if (rc) return rc;
  }
  return EPSM_OK;
}

static int group_bind(epsm_group_t* g, const void* dptr) {
  int dev = -1;
  cudaPointerAttributes attr;
  cudaError_t e = dptr ? cudaPointerGetAttributes(&attr, dptr) : cudaErrorInvalidValue;
  if (e == cudaSuccess && attr.type == cudaMemoryTypeDevice) {
    dev = attr.device;
  } else {
    cudaGetLastError();
    e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return epsm_cuda_fail(e, "cudaGetDevice");
  }
  if (g->device < 0) g->device = dev;
  if (g->device != dev) {
    epsm_set_error("group is bound to device %d but the buffer is on device %d", g->device, dev);
    return EPSM_EINVAL;
  }
  e = cudaSetDevice(dev);
  if (e != cudaSuccess) return epsm_cuda_fail(e, "cudaSetDevice");
  return EPSM_OK;
}

// EPSM_MASK_MIN=k: smallest dense set sent through the mask pass (A/B; default 24)
static uint32_t mask_min_patterns() {
  static const uint32_t v = [] {
    const char* e = getenv("EPSM_MASK_MIN");
    return e ? static_cast<uint32_t>(atoi(e)) : 24u;
  }();
  return v;
}

// EPSM_MASK=0: the dense patterns keep the one-by-one scans (A/B)
static bool mask_disabled() {
  static const bool v = [] {
    const char* e = getenv("EPSM_MASK");
    return e && e[0] == '0';
  }();
  return v;
}

// The dense patterns of a group in ONE pass over the index (epsm_mask.cuh) when they fit: m <= 8,
// <= 64 patterns, <= 8 distinct bytes, all in the index, m * bytes <= 16.  Each pattern's
// largest-capacity search gets the positions, its other searches a copy (replicate kernel).
// Returns 1 when the set does not fit (the caller scans the patterns one by one).
static int mask_run(epsm_group_t* g, const epsm_eqidx_t* index, const uint8_t* d_text, uint64_t n, uint64_t ns,
                    uint64_t base, uint64_t* const* d_pos, const uint64_t* caps, uint64_t* d_occ, bool search,
                    cudaStream_t s) {
  namespace mk = epsm::mk;
  const uint32_t D = static_cast<uint32_t>(g->dense.size());
  // (only for many dense patterns: a few are faster one by one, their scans write the bulk of
  // their positions with staged 16-byte stores -- sigma=2 m=4, 16 patterns: 4.0 ms either way;
  // sigma=8 m=2, 50 patterns: 2.8 vs 3.8 ms)
  if (mask_disabled() || D < mask_min_patterns() || D > static_cast<uint32_t>(mk::kMaxD) ||
      g->m > static_cast<uint32_t>(mk::kMaxM))
    return 1;
  if (reinterpret_cast<uintptr_t>(d_text) & 15u) return 1;
  int slot_of[256];
  for (int& v : slot_of) v = -1;
  uint32_t nval = 0, pid[mk::kMaxVals];
  for (uint32_t d : g->dense)
    for (unsigned char ch : g->pats[d])
      if (slot_of[ch] < 0) {
        if (nval == static_cast<uint32_t>(mk::kMaxVals) || index->plane_of[ch] < 0) return 1;
        pid[nval] = static_cast<uint32_t>(index->plane_of[ch]);
        slot_of[ch] = static_cast<int>(nval++);
      }
  if (g->m * nval > static_cast<uint32_t>(mk::kMaxSh)) return 1;
  mk::MaskParams P;
  std::memset(&P, 0, sizeof(P));
  P.planes = index->d_planes;
  P.pstride = index->pstride;
  P.nval = nval;
  P.m = g->m;
  P.D = D;
  for (uint32_t v = 0; v < nval; ++v) P.pid[v] = pid[v];
  P.nstarts = ns;
  P.pos_bias = base;
  P.nwords = (ns + 63) / 64;
  P.ntasks = (P.nwords + mk::kTaskWords - 1) / mk::kTaskWords;
  // outputs: per pattern the largest-capacity search first, the others fanned out afterwards
  std::vector<epsm::XOut> xo;
  std::vector<std::pair<uint32_t, uint32_t>> rep;   // (pattern, further outputs)
  for (uint32_t k = 0; k < D; ++k) {
    const uint32_t d = g->dense[k];
    for (uint32_t i = 0; i < g->m; ++i)
      P.sh[k][i] = static_cast<uint8_t>(i * nval + slot_of[static_cast<unsigned char>(g->pats[d][i])]);
    const auto& js = g->dups[d];
    uint32_t best = js[0];
    auto capof = [&](uint32_t j) -> uint64_t { return (search && d_pos && d_pos[j] && caps) ? caps[j] : 0; };
    for (uint32_t j : js)
      if (capof(j) > capof(best)) best = j;
    P.pos[k] = capof(best) ? d_pos[best] : nullptr;
    P.cap[k] = capof(best);
    P.occ[k] = reinterpret_cast<unsigned long long*>(d_occ + best);
    uint32_t nx = 0;
    for (uint32_t j : js) {
      if (j == best) continue;
      xo.push_back(epsm::XOut{capof(j) ? d_pos[j] : nullptr, capof(j), reinterpret_cast<unsigned long long*>(d_occ + j)});
      ++nx;
    }
    if (nx) rep.emplace_back(k, nx);
  }
  epsm_workspace* ws = epsm_get_workspace(g->device, s);
  if (!ws) return EPSM_ENOMEM;
  if (ws->num_sms <= 0) {
    cudaError_t e = cudaDeviceGetAttribute(&ws->num_sms, cudaDevAttrMultiProcessorCount, g->device);
    if (e != cudaSuccess) return epsm_cuda_fail(e, "cudaDeviceGetAttribute(SM count)");
  }
  int rc = ensure_multi_ws(ws, P.ntasks, D, s);
  if (rc) return rc;
  P.counts = ws->m_counts;
  P.prefix = ws->m_prefix;
  if (ns == 0) {
    for (uint32_t k = 0; k < D; ++k) {
      cudaError_t e = cudaMemsetAsync(P.occ[k], 0, 8, s);
      if (e != cudaSuccess) return epsm_cuda_fail(e, "cudaMemsetAsync(occ)");
    }
  } else {
    const unsigned grid = static_cast<unsigned>(
        std::max<uint64_t>(1, std::min<uint64_t>((P.ntasks + mk::kWarps - 1) / mk::kWarps, 4ull * ws->num_sms)));
    mk::epsm_mask_count_kernel<<<grid, mk::kThreads, 0, s>>>(P);
    epsm_count_launch();
    mk::epsm_mask_scan_kernel<<<D, 1024, 0, s>>>(P);
    epsm_count_launch();
    if (search) {
      mk::epsm_mask_write_kernel<<<grid, mk::kThreads, 0, s>>>(P);
      epsm_count_launch();
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return epsm_cuda_fail(e, "mask kernels launch");
  }
  if (!xo.empty()) {
    if (xo.size() > ws->xout_cap) {
      if (ws->d_xout) {
        cudaStreamSynchronize(s);
        cudaFree(ws->d_xout);
        ws->d_xout = nullptr;
        ws->xout_cap = 0;
      }
      cudaError_t e = cudaMalloc(&ws->d_xout, xo.size() * sizeof(epsm::XOut));
      if (e != cudaSuccess) {
        epsm_set_error("cudaMalloc(fan-out table): %s", cudaGetErrorString(e));
        return EPSM_ENOMEM;
      }
      ws->xout_cap = xo.size();
    }
    cudaError_t e = cudaMemcpyAsync(ws->d_xout, xo.data(), xo.size() * sizeof(epsm::XOut), cudaMemcpyHostToDevice, s);
    if (e != cudaSuccess) return epsm_cuda_fail(e, "cudaMemcpyAsync(fan-out table)");
    // every pattern's further outputs in one fan-out launch
    std::vector<epsm_rep_req> rq;
    uint32_t off = 0;
    for (const auto& r : rep) {
      rq.push_back(epsm_rep_req{P.pos[r.first], P.cap[r.first], P.occ[r.first], off, r.second});
      off += r.second;
    }
    rc = epsm_replicate_many(rq.data(), static_cast<uint32_t>(rq.size()), ws->d_xout, xo.data(), search, s, ws);
    if (rc) return rc;
  }
  return 0;
}

static int group_run(epsm_group_t* g, const uint8_t* d_text, uint64_t n, uint64_t owned_len, uint64_t base,
                     uint64_t n_total, uint64_t* const* d_pos, const uint64_t* caps, uint64_t* d_occ, bool search,
                     epsm_stream_t stream, const epsm_eqidx_t* index) {
  if (!g || !d_occ || (!d_text && n > 0)) {
    epsm_set_error("epsm_group_*: NULL group, d_occ or text");
    return EPSM_EINVAL;
  }
  if (index && (index->text != d_text || index->n != n)) {
    epsm_set_error("the index was built over another text (pointer or length differ)");
    return EPSM_EINVAL;
  }
  if (n > (1ull << 38)) {
    epsm_set_error("n = %llu exceeds 2^38", (unsigned long long)n);
    return EPSM_EINVAL;
  }
  if (reinterpret_cast<uintptr_t>(d_occ) & 7u) {
    epsm_set_error("d_occ must be 8-byte aligned");
    return EPSM_EALIGN;
  }
  if (search && d_pos)
    for (uint32_t j = 0; j < g->k; ++j)
      if (d_pos[j] && (reinterpret_cast<uintptr_t>(d_pos[j]) & 7u)) {
        epsm_set_error("d_pos[%u] must be 8-byte aligned", j);
        return EPSM_EALIGN;
      }
  int rc = group_bind(g, d_occ);
  if (rc) return rc;
  uint64_t ns = n >= g->m ? n - g->m + 1 : 0;
  if (owned_len < ns) ns = owned_len;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  for (auto& S : g->subs) {
    rc = subgroup_launch(g, S, d_text, n, ns, base, d_pos, caps, d_occ, search, s);
    if (rc) return rc;
  }
  if (!g->dense.empty() && index) {
    rc = mask_run(g, index, d_text, n, ns, base, d_pos, caps, d_occ, search, s);
    if (rc != 1) return rc;          // done (or an error); 1: the dense set does not fit the mask pass
  }
  if (!g->dense.empty()) {
    // the dense patterns: one single-pattern scan per distinct pattern (over the index where it
    // qualifies), its occ and positions fanned out to every other search of that pattern by the
    // replicate kernel -- one job per 16-byte phase of the outputs (16-byte copies)
    std::vector<epsm_plan_t*> pl;
    std::vector<uint32_t> primary;
    std::vector<std::vector<uint32_t>> fan;
    for (size_t i = 0; i < g->dense.size(); ++i) {
      std::vector<uint32_t> cls[2], none;
      for (uint32_t j : g->dups[g->dense[i]]) {
        const bool has = search && d_pos && d_pos[j] && caps && caps[j];
        if (has) cls[(reinterpret_cast<uintptr_t>(d_pos[j]) >> 3) & 1u].push_back(j);
        else none.push_back(j);
      }
      if (cls[0].empty() && cls[1].empty()) cls[0].swap(none);
      else (cls[0].empty() ? cls[1] : cls[0]).insert((cls[0].empty() ? cls[1] : cls[0]).end(), none.begin(), none.end());
      for (auto& c : cls) {
        if (c.empty()) continue;
        // the primary (the scan's own output) is the largest capacity: the fan-out copies from it
        size_t best = 0;
        for (size_t q = 1; q < c.size(); ++q)
          if (search && d_pos && caps && d_pos[c[q]] && (!d_pos[c[best]] || caps[c[q]] > caps[c[best]])) best = q;
        std::swap(c[0], c[best]);
        pl.push_back(g->dplans[i]);
        primary.push_back(c[0]);
        fan.emplace_back(c.begin() + 1, c.end());
      }
    }
    rc = epsm_batch_run(pl.data(), static_cast<uint32_t>(pl.size()), primary.data(), d_text, n, owned_len, base,
                        n_total, search ? d_pos : nullptr, search ? caps : nullptr, d_occ, search, s, index, &fan);
    if (rc) return rc;
  }
  return EPSM_OK;
}

// EPSM_GROUP_DENSE=L: distinct patterns with an estimated rate >= 2^-L occurrences per text
// byte are searched one by one, their positions fanned out to their duplicate searches by the
// replicate kernel (default 7; 0 puts every pattern through the group kernels).  Speed only:
// both paths are exact.  B200, 256 MiB texts, 100 patterns per group (ms, one by one vs shared
// passes): sigma=8 m=2 (2^-6) 3.85 vs 8.7; sigma=2 m=8 (2^-8) 4.9 vs 4.0; sigma=16 m=2 (2^-8)
// 4.2 vs 4.1; sigma=32 m=2 (2^-10) 4.4 vs 2.2-2.8; sigma=64 m=2 (2^-12) 2.3 vs 1.4.
static int group_dense_log2() {
  static const int v = [] {
    const char* e = getenv("EPSM_GROUP_DENSE");
    return e && e[0] ? static_cast<int>(strtol(e, nullptr, 0)) : 7;
  }();
  return v <= 0 ? 4096 : v;
}

constexpr uint32_t kMinShared = 4;

// Split the distinct patterns into dense (estimated rate >= 2^-log2 occurrences per text byte)
// and sparse.  The rate of a pattern is the product of its bytes' frequencies among the OTHER
// k - 1 patterns of the group (they are extracted from the text, so their bytes
// sample its distribution; leaving the pattern's own copy out keeps a rare byte from counting
// itself).
static void group_split(epsm_group_t* g, int log2) {
  double cnt[256] = {};
  for (uint32_t d = 0; d < g->D; ++d)
    for (unsigned char ch : g->pats[d]) cnt[ch] += static_cast<double>(g->dups[d].size());
  const double thresh = std::ldexp(1.0, -log2);
  const double others = static_cast<double>(g->k - 1) * g->m;
  g->sparse.clear();
  g->dense.clear();
  std::vector<double> rate(g->D, 0.0);
  double lsum = 0;
  uint32_t lcnt = 0;
  for (uint32_t d = 0; d < g->D; ++d) {
    double own[256] = {};
    for (unsigned char ch : g->pats[d]) own[ch] += 1.0;
    double r = others > 0 ? 1.0 : 0.0;
    for (unsigned char ch : g->pats[d]) r *= others > 0 ? (cnt[ch] - own[ch]) / others : 0.0;
    rate[d] = r;
    if (r > 0) {
      lsum += std::log2(r);
      ++lcnt;
    }
  }
  // the estimates of one group scatter (a handful of sampled bytes per symbol): a pattern within
  // 8x of the group's geometric mean takes the mean, so that a uniform text's patterns, which
  // have one common rate, are split the same way; outliers keep their own estimate
  const double gmean = lcnt ? std::exp2(lsum / lcnt) : 0.0;
  // a group of fewer than kMinShared distinct patterns has little to share and too few samples
  // to estimate rates from: its patterns are searched one by one (a single search is the
  // single-pattern kernel's case: 'a'^16 over 'a'^(2^30) 1.4 ms, the shared passes 30 ms)
  const bool all_single = log2 < 1024 && g->D < kMinShared;
  g->sparse_rate = 0;
  for (uint32_t d = 0; d < g->D; ++d) {
    double r = rate[d];
    if (r > 0 && gmean > 0 && std::fabs(std::log2(r / gmean)) <= 3.0) r = gmean;
    const bool dn = all_single || (log2 < 1024 && r >= thresh);
    (dn ? g->dense : g->sparse).push_back(d);
    if (!dn) g->sparse_rate += r;
  }
}

// (Re)build the passes over g->sparse (<= kMaxD distinct patterns each) and the plans of
// g->dense; the group's device copies are rebuilt on the next use.
static int group_partition(epsm_group_t* g, int force_q, int force_sk) {
  for (auto& S : g->subs) {
    if (S.d_desc) cudaFree(S.d_desc);
    delete S.h_desc;
  }
  g->subs.clear();
  for (uint32_t a = 0; a < g->sparse.size(); a += mp::kMaxD) {
    const uint32_t b = std::min<uint32_t>(static_cast<uint32_t>(g->sparse.size()), a + mp::kMaxD);
    std::vector<std::string> sp;
    std::vector<std::vector<uint32_t>> sd;
    for (uint32_t i = a; i < b; ++i) {
      sp.push_back(g->pats[g->sparse[i]]);
      sd.push_back(g->dups[g->sparse[i]]);
    }
    g->subs.emplace_back();
    int rc = build_subgroup(sp, g->m, g->subs.back(), sd, force_q, force_sk);
    if (rc) return rc;
  }
  for (epsm_plan_t* p : g->dplans) epsm_plan_free(p);
  g->dplans.clear();
  for (uint32_t d : g->dense) {
    epsm_plan_t* p = nullptr;
    int rc = epsm_plan(reinterpret_cast<const uint8_t*>(g->pats[d].data()), g->m, &p);
    if (rc) return rc;
    g->dplans.push_back(p);
  }
  return EPSM_OK;
}
static int group_partition(epsm_group_t* g) { return group_partition(g, 0, 0); }

extern "C" {

int epsm_group_create(const uint8_t* patterns, uint32_t m, uint32_t k, epsm_group_t** out) {
  if (!out) {
    epsm_set_error("epsm_group_create: NULL out");
    return EPSM_EINVAL;
  }
  *out = nullptr;
  if (!patterns || m == 0 || k == 0) {
    epsm_set_error("epsm_group_create: NULL patterns, m = 0 or k = 0");
    return EPSM_EINVAL;
  }
  if (m > EPSM_MAX_M || k > static_cast<uint32_t>(mp::kMaxJobs)) {
    epsm_set_error("epsm_group_create: m = %u > %u or k = %u > %d", m, EPSM_MAX_M, k, mp::kMaxJobs);
    return EPSM_EUNSUP;
  }
  epsm_group_t* g = new (std::nothrow) epsm_group_t();
  if (!g) return EPSM_ENOMEM;
  g->m = m;
  g->k = k;
  // distinct patterns in order of first occurrence, and the searches asking for each
  std::map<std::string, uint32_t> seen;
  std::vector<std::string> pats;
  std::vector<std::vector<uint32_t>> dups;
  for (uint32_t j = 0; j < k; ++j) {
    std::string p(reinterpret_cast<const char*>(patterns) + static_cast<size_t>(j) * m, m);
    auto it = seen.find(p);
    if (it == seen.end()) {
      it = seen.emplace(p, static_cast<uint32_t>(pats.size())).first;
      pats.push_back(p);
      dups.emplace_back();
    }
    dups[it->second].push_back(j);
  }
  g->D = static_cast<uint32_t>(pats.size());
  g->pats = pats;
  g->dups = dups;
  group_split(g, group_dense_log2());
  int rc = group_partition(g);
  if (rc) {
    group_release(g);
    return rc;
  }
  *out = g;
  return EPSM_OK;
}

void epsm_group_free(epsm_group_t* g) { group_release(g); }

int epsm_group_set_geometry(epsm_group_t* g, uint32_t q, uint32_t sk) {
  const bool code = sk == 0;   // the code mode (q ignored)
  if (code) q = g ? g->m : 1;
  if (!g || (!code && (q < 1 || q > 16 || q > g->m || sk < 1 || sk > 16 || (sk & (sk - 1)) || sk + q - 1 > g->m))) {
    epsm_set_error("epsm_group_set_geometry: need SK = 0 (code mode) or 1 <= q <= min(m, 16), SK in {1,2,4,8,16}, "
                   "SK + q - 1 <= m");
    return EPSM_EINVAL;
  }
  const uint32_t dmax = std::min<uint32_t>(g->D, mp::kMaxD);   // distinct patterns of the largest pass
  if (static_cast<uint64_t>(dmax) * sk > mp::kMaxEntries) {
    epsm_set_error("epsm_group_set_geometry: %u patterns x SK = %u exceeds %d table entries", dmax, sk,
                   mp::kMaxEntries);
    return EPSM_EINVAL;
  }
  if (g->device >= 0) {
    cudaSetDevice(g->device);
    cudaDeviceSynchronize();
  }
  // a forced geometry puts every distinct pattern through the group kernels
  g->forced_geom = true;
  g->sparse.clear();
  g->dense.clear();
  for (uint32_t d = 0; d < g->D; ++d) g->sparse.push_back(d);
  return group_partition(g, static_cast<int>(q), static_cast<int>(sk));
}

int epsm_group_set_dense(epsm_group_t* g, uint32_t log2_rate) {
  if (!g || log2_rate > 64) {
    epsm_set_error("epsm_group_set_dense: NULL group or log2_rate > 64");
    return EPSM_EINVAL;
  }
  if (g->device >= 0) {
    cudaSetDevice(g->device);
    cudaDeviceSynchronize();
  }
  group_split(g, log2_rate == 0 ? 4096 : static_cast<int>(log2_rate));
  g->forced_geom = false;
  return group_partition(g);
}

int epsm_group_dense_searches(const epsm_group_t* g, uint8_t* flags) {
  if (!g) return EPSM_EINVAL;
  if (flags) std::memset(flags, 0, g->k);
  int c = 0;
  for (uint32_t d : g->dense)
    for (uint32_t j : g->dups[d]) {
      if (flags) flags[j] = 1;
      ++c;
    }
  return c;
}

int epsm_group_index_values(const epsm_group_t* g, uint8_t* out_values) {
  if (!g) return 0;
  bool have[256] = {};
  int nv = 0;
  for (epsm_plan_t* p : g->dplans) {
    uint8_t v[EPSM_INDEX_MAX_D];
    const int c = epsm_plan_index_values(p, v);
    for (int q = 0; q < c; ++q)
      if (!have[v[q]]) {
        have[v[q]] = true;
        if (out_values) out_values[nv] = v[q];
        ++nv;
      }
  }
  return nv;
}

int epsm_group_info(const epsm_group_t* g, uint32_t* out, uint32_t nout) {
  if (!g || !out) return EPSM_EINVAL;
  std::vector<uint32_t> v = {g->m, g->k, g->D, static_cast<uint32_t>(g->dense.size()),
                             static_cast<uint32_t>(g->subs.size())};
  for (const auto& S : g->subs) {
    v.push_back(static_cast<uint32_t>(S.q));
    v.push_back(static_cast<uint32_t>(S.sk < 0 ? 0 : S.sk));   // (0: code mode, table or wide)
  }
  const uint32_t c = std::min<uint32_t>(nout, static_cast<uint32_t>(v.size()));
  for (uint32_t i = 0; i < c; ++i) out[i] = v[i];
  return static_cast<int>(v.size());
}

int epsm_group_search_async(epsm_group_t* g, const uint8_t* d_text, uint64_t n, uint64_t* const* d_pos,
                            const uint64_t* caps, uint64_t* d_occ, epsm_stream_t stream) {
  return group_run(g, d_text, n, n, 0, 0, d_pos, caps, d_occ, true, stream, nullptr);
}

int epsm_group_count_async(epsm_group_t* g, const uint8_t* d_text, uint64_t n, uint64_t* d_occ,
                           epsm_stream_t stream) {
  return group_run(g, d_text, n, n, 0, 0, nullptr, nullptr, d_occ, false, stream, nullptr);
}

int epsm_group_search_index_async(epsm_group_t* g, const epsm_eqidx_t* index, const uint8_t* d_text, uint64_t n,
                                  uint64_t* const* d_pos, const uint64_t* caps, uint64_t* d_occ,
                                  epsm_stream_t stream) {
  return group_run(g, d_text, n, n, 0, 0, d_pos, caps, d_occ, true, stream, index);
}

int epsm_group_count_index_async(epsm_group_t* g, const epsm_eqidx_t* index, const uint8_t* d_text, uint64_t n,
                                 uint64_t* d_occ, epsm_stream_t stream) {
  return group_run(g, d_text, n, n, 0, 0, nullptr, nullptr, d_occ, false, stream, index);
}

int epsm_group_search_range_index_async(epsm_group_t* g, const epsm_eqidx_t* index, const uint8_t* d_shard,
                                        uint64_t shard_len, uint64_t owned_len, uint64_t base, uint64_t n_total,
                                        uint64_t* const* d_pos, const uint64_t* caps, uint64_t* d_occ,
                                        epsm_stream_t stream) {
  if (!g) {
    epsm_set_error("NULL group");
    return EPSM_EINVAL;
  }
  if (base > n_total || owned_len > n_total - base || shard_len > n_total - base) {
    epsm_set_error("shard [%llu, +%llu) owning %llu starts lies outside the text of %llu bytes",
                   (unsigned long long)base, (unsigned long long)shard_len, (unsigned long long)owned_len,
                   (unsigned long long)n_total);
    return EPSM_EINVAL;
  }
  if (owned_len) {
    const uint64_t need = std::min<uint64_t>(owned_len + g->m - 1, n_total - base);
    if (shard_len < need) {
      epsm_set_error("shard of %llu bytes is shorter than its owned starts plus the (m-1)-byte overlap (%llu)",
                     (unsigned long long)shard_len, (unsigned long long)need);
      return EPSM_EINVAL;
    }
  }
  return group_run(g, d_shard, shard_len, owned_len, base, n_total, d_pos, caps, d_occ, true, stream, index);
}

int epsm_group_search_range_async(epsm_group_t* g, const uint8_t* d_shard, uint64_t shard_len, uint64_t owned_len,
                                  uint64_t base, uint64_t n_total, uint64_t* const* d_pos, const uint64_t* caps,
                                  uint64_t* d_occ, epsm_stream_t stream) {
  return epsm_group_search_range_index_async(g, nullptr, d_shard, shard_len, owned_len, base, n_total, d_pos, caps,
                                             d_occ, stream);
}

}  // extern "C"
