// epsm.cu -- host side of the C ABI declared in include/epsm.h.
//
// Plan construction (preprocessing, PAPER.md:453-457 / 492, dispatch by m
// PAPER.md:150-152), workspace management, kernel dispatch and the host-buffer
// convenience call.  The sharded (NCCL) call lives in epsm_sharded.cu.
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <algorithm>
#include <atomic>
#include <mutex>
#include <new>
#include <vector>

#include "epsm.h"
#include "epsm_internal.h"
#include "epsm_kernels.cuh"

namespace {

thread_local char g_last_error[512] = "";
std::atomic<uint64_t> g_launches{0};

// Diagnostics: EPSM_TRACE=<slots> makes every launch record a per-CTA timeline
// (8 x u64 per CTA, slot = launch index mod slots); epsm_debug_trace copies it out.
constexpr uint64_t kTraceWordsPerLaunch = 8 * 1024;
unsigned long long* g_trace = nullptr;
uint64_t g_trace_slots = 0;
int g_trace_device = -1;

unsigned long long* trace_slot(int device) {
  static const uint64_t slots = [] {
    const char* v = getenv("EPSM_TRACE");
    return v && v[0] ? static_cast<uint64_t>(atoll(v)) : 0ull;
  }();
  if (slots == 0) return nullptr;
  if (!g_trace) {
    if (cudaMalloc(&g_trace, slots * kTraceWordsPerLaunch * sizeof(unsigned long long)) != cudaSuccess) {
      g_trace = nullptr;
      return nullptr;
    }
    cudaMemset(g_trace, 0, slots * kTraceWordsPerLaunch * sizeof(unsigned long long));
    g_trace_slots = slots;
    g_trace_device = device;
  }
  if (device != g_trace_device) return nullptr;
  return g_trace + (g_launches.load() % g_trace_slots) * kTraceWordsPerLaunch;
}

// Diagnostics for benchmarks (epsm_ktimer_enable / epsm_ktimer_read): while on, every launch of
// the fan-out kernel is bracketed by a pair of CUDA events on its own stream, and the launch's
// jobs are kept so that its algorithmic bytes (source positions read once, every output's
// positions written) can be summed from the device occ values once the launches are done.
struct KtJob {
  const unsigned long long* occ;
  uint64_t cap;
  std::vector<uint64_t> out_caps;              // 0: no output buffer
};
struct KtRec {
  cudaEvent_t ev[2];
  std::vector<KtJob> jobs;
};
std::mutex g_kt_mu;
std::atomic<bool> g_kt_on{false};
std::vector<KtRec> g_kt_recs;

using KernelFn = void (*)(epsm::KParams);

template <int F, int F2, int MW, int SK = 0, int SQ = 0>
constexpr KernelFn pick(bool search) {
  return search ? &epsm::epsm_scan_kernel<F, F2, MW, SK, SQ, true>
                : &epsm::epsm_scan_kernel<F, F2, MW, SK, SQ, false>;
}

// Smallest m that takes the sampled (EPSMc-style) filter; EPSM_SAMPLE_MIN_M overrides
// (A/B timing).  Below it the packed filter (EPSMa/b) runs.
uint32_t sample_min_m() {
  static const uint32_t v = [] {
    const char* e = getenv("EPSM_SAMPLE_MIN_M");
    return e && e[0] ? static_cast<uint32_t>(atoi(e)) : 9u;
  }();
  return v;
}

// EPSM_NO_EQ=1 disables the equality-mask variant (A/B timing).
static bool eq_disabled() {
  static const bool off = [] {
    const char* v = getenv("EPSM_NO_EQ");
    return v && v[0] && v[0] != '0';
  }();
  return off;
}

// Sampled-filter geometry of a pattern: one SQ-byte gram every SK bytes (SK + SQ <= m), (0, 0)
// for the packed filter.  Must agree with kernel_for.  m = 8..11 sits at the crossover: the
// packed filter wins on binary texts and on large alphabets, the sampled 4-byte grams on
// 4..8-letter alphabets (B200, m = 8: sigma=4 107 -> 89 us, sigma=8 74 -> 68 us per 256 MiB;
// m = 10: sigma=4 108 -> 88 us, sigma=256 58 -> 47 us packed), so the choice follows the
// pattern's number of distinct bytes d (an extracted pattern's d tracks the text's
// alphabet): sampled for 3 <= d <= 5.  EPSM_SAMPLE_MIN_M <= 8 forces the sampled filter.
// Speed only: both filters are exact.
void sampled_geometry(uint32_t m, const uint8_t* pattern, int* sk, int* sq) {
  *sk = *sq = 0;
  uint32_t seen[8] = {0, 0, 0, 0, 0, 0, 0, 0}, d = 0;   // distinct bytes of the pattern
  for (uint32_t i = 0; i < m && i < EPSM_MAX_M; ++i) {
    const uint32_t b = pattern[i];
    if (!((seen[b >> 5] >> (b & 31)) & 1u)) {
      seen[b >> 5] |= 1u << (b & 31);
      ++d;
    }
  }
  // m = 8..11: (4,4) grams on 4..8-letter alphabets, the packed filter otherwise
  const bool mid = m >= 8 && m <= 11;
  const bool take_mid = mid && d >= 3 && d <= 5;
  if (m > EPSM_MAX_M) {
    *sk = 16, *sq = 16;
  } else if (m >= 5 && m <= 11 && d <= 2 && !eq_disabled()) {
    *sk = epsm::kEqMode;                 // EPSMa's equality masks + shift-AND (binary alphabets)
  } else if (m >= 8 && (mid ? (take_mid || sample_min_m() <= 8) : m >= sample_min_m())) {
    if (m <= 11) *sk = 4, *sq = 4;
    else if (m <= 15) *sk = 8, *sq = 4;
    else if (m <= 19) *sk = 8, *sq = 8;
    // one gram per 16-byte unit (SK + SQ <= m) where the pattern's bytes carry enough entropy
    // for a short gram; binary patterns keep two longer grams per unit
    else if (m <= 23) *sk = d <= 2 ? 8 : 16, *sq = d <= 2 ? 8 : 4;
    else if (m <= 27) *sk = d <= 2 ? 8 : 16, *sq = d <= 2 ? 16 : 8;
    else if (m <= 31) *sk = d <= 2 ? 8 : 16, *sq = d <= 2 ? 16 : 12;
    else *sk = 16, *sq = 16;
    // small alphabets (few distinct bytes): longer grams at a 4-byte stride -- four lookups
    // per unit, but far fewer candidates to check (genome-like m = 12: 300 -> ~240 us/GiB)
    if (m >= 12 && m <= 15 && d <= 5) *sk = 4, *sq = 8;
    else if (m >= 16 && m <= 23 && d <= 2) *sk = 4, *sq = 12;
  }
  // EPSM_GEOM="m:sk:sq" overrides the geometry of one pattern length (A/B timing; the kernel
  // must exist for it -- see kernel_for)
  static const int g_m = [] {
    const char* e = getenv("EPSM_GEOM");
    return e && e[0] ? atoi(e) : 0;
  }();
  if (g_m > 0 && static_cast<uint32_t>(g_m) == m) {
    const char* e = getenv("EPSM_GEOM");
    int a = 0, b = 0, c = 0;
    if (sscanf(e, "%d:%d:%d", &a, &b, &c) == 3 && b + c <= static_cast<int>(m)) *sk = b, *sq = c;
  }
}

// EPSMc preprocessing (Fig. 1 lines 1-5): the fingerprint of every gram
// p[i .. i+SQ-1], i = 1..SK, enters the table; the entry's mask bit SK-i marks the start
// (sample offset - i) as a candidate.  Fingerprint = the kernel's gram_hash (a multiply-add
// over little-endian words); bits [31:21] index the table, bits [20:6] are kept in the entry
// so that a sample with another fingerprint is rejected.  Grams of different fingerprints
// that share a bucket make it a wildcard (no fingerprint check).
void build_gram_table(const uint8_t* pattern, int sk, int sq, uint32_t* tab) {
  std::memset(tab, 0, sizeof(uint32_t) * epsm::kGramTab);
  uint32_t H[16];
  for (int i = 1; i <= sk; ++i) {
    uint32_t h = 0;
    for (int r = 0; r < sq / 4; ++r) {
      const uint8_t* b = pattern + i + 4 * r;
      const uint32_t w = b[0] | (b[1] << 8) | (b[2] << 16) | (static_cast<uint32_t>(b[3]) << 24);
      h += w * epsm::gram_mul(r);
    }
    H[i - 1] = h;
  }
  constexpr int shift = 32 - epsm::kGramBits;
  for (int i = 1; i <= sk; ++i) {
    const uint32_t h = H[i - 1];
    uint32_t mask = 0, wild = 0;
    for (int l = 1; l <= sk; ++l) {
      const uint32_t hl = H[l - 1];
      if ((hl >> shift) == (h >> shift)) {
        mask |= 1u << (sk - l);
        if (((hl ^ h) << epsm::kGramBits) & 0xFFFE0000u) wild = 1u;
      }
    }
    tab[h >> shift] = mask | (wild << 16) | ((h << epsm::kGramBits) & 0xFFFE0000u);
  }
}

// Kernel variant for a pattern of length m (dispatch by m).
//   packed:  F = min(m, 4) bytes in the first filter word, F2 = min(m, 8) - 4 in the second
//            (used where candidates are dense), MW = ceil(m/4) words;
//   sampled: one SQ-byte gram every SK bytes (SK + SQ <= m), MW words verified.
KernelFn kernel_for(uint32_t m, int sk, int sq, bool search) {
  if (m > EPSM_MAX_M) return pick<4, 4, 0, 16, 16>(search);     // long: EPSMc + device-memory check
  if (sk == epsm::kEqMode) return pick<4, 4, 1, epsm::kEqMode, 0>(search);   // EPSMa, <= 2 values
  if (sk == epsm::kPlaneMode) return pick<4, 4, 1, epsm::kPlaneMode, 0>(search);   // EPSMa, index
  if (sk == epsm::kPlaneModeC) return pick<4, 4, 1, epsm::kPlaneModeC, 0>(search);
  if (sk == epsm::kPlaneModeC2) return pick<4, 4, 1, epsm::kPlaneModeC2, 0>(search);
  if (sk == epsm::kPlaneModeC8) return pick<4, 4, 1, epsm::kPlaneModeC8, 0>(search);
  if (sk == 4 && sq == 8) return m == 12 ? pick<4, 4, 3, 4, 8>(search) : pick<4, 4, 4, 4, 8>(search);
  if (sk == 4 && sq == 12) {
    if (m == 16) return pick<4, 4, 4, 4, 12>(search);
    if (m <= 20) return pick<4, 4, 5, 4, 12>(search);
    return pick<4, 4, 6, 4, 12>(search);
  }
  if (sk == 16 && sq == 4) return m <= 20 ? pick<4, 4, 5, 16, 4>(search) : pick<4, 4, 6, 16, 4>(search);
  if (sk == 8 && sq == 4 && m == 16) return pick<4, 4, 4, 8, 4>(search);
  if (sk == 16 && sq == 8) return m <= 24 ? pick<4, 4, 6, 16, 8>(search) : pick<4, 4, 7, 16, 8>(search);
  if (sk == 16 && sq == 12) return pick<4, 4, 8, 16, 12>(search);
  if (sk > 0) {
    switch (m) {
      case 8: return pick<4, 4, 2, 4, 4>(search);
      case 9: case 10: case 11: return pick<4, 4, 3, 4, 4>(search);
      case 12: return pick<4, 4, 3, 8, 4>(search);
      case 13: case 14: case 15: return pick<4, 4, 4, 8, 4>(search);
      case 16: return pick<4, 4, 4, 8, 8>(search);
      case 17: case 18: case 19: case 20: return pick<4, 4, 5, 8, 8>(search);
      case 21: case 22: case 23: return pick<4, 4, 6, 8, 8>(search);
      case 24: return pick<4, 4, 6, 8, 16>(search);
      case 25: case 26: case 27: case 28: return pick<4, 4, 7, 8, 16>(search);
      case 29: case 30: case 31: return pick<4, 4, 8, 8, 16>(search);
      default: return pick<4, 4, 8, 16, 16>(search);
    }
  }
  switch (m) {
    case 1: return pick<1, 0, 1>(search);
    case 2: return pick<2, 0, 1>(search);
    case 3: return pick<3, 0, 1>(search);
    case 4: return pick<4, 0, 1>(search);
    case 5: return pick<4, 1, 2>(search);
    case 6: return pick<4, 2, 2>(search);
    case 7: return pick<4, 3, 2>(search);
    case 8: return pick<4, 4, 2>(search);
    default: break;
  }
  switch ((m + 3) / 4) {
    case 3: return pick<4, 4, 3>(search);
    case 4: return pick<4, 4, 4>(search);
    case 5: return pick<4, 4, 5>(search);
    case 6: return pick<4, 4, 6>(search);
    case 7: return pick<4, 4, 7>(search);
    default: return pick<4, 4, 8>(search);
  }
}

}  // namespace

void epsm_set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_last_error, sizeof(g_last_error), fmt, ap);
  va_end(ap);
}

int epsm_cuda_fail(cudaError_t e, const char* what) {
  epsm_set_error("%s: %s", what, cudaGetErrorString(e));
  return EPSM_ECUDA;
}

void epsm_count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

// Bind the calling thread to the device that owns ptr (torch and this library each
// carry their own CUDA runtime; the pointer is the unambiguous source of truth).
int epsm_bind_device(epsm_plan_t* plan, const void* dptr) {
  int dev = -1;
  cudaPointerAttributes attr;
  cudaError_t e = cudaPointerGetAttributes(&attr, dptr);
  if (e == cudaSuccess && attr.type == cudaMemoryTypeDevice) {
    dev = attr.device;
  } else {
    cudaGetLastError();
    e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return epsm_cuda_fail(e, "cudaGetDevice");
  }
  if (plan->device < 0) plan->device = dev;
  if (plan->device != dev) {
    epsm_set_error("plan is bound to device %d but the buffer is on device %d", plan->device, dev);
    return EPSM_EINVAL;
  }
  e = cudaSetDevice(dev);
  if (e != cudaSuccess) return epsm_cuda_fail(e, "cudaSetDevice");
  return EPSM_OK;
}

// ---- scan workspace pool, one per (device, stream)

constexpr uint64_t kCtrWords = 8 + epsm::kMaxJobs;   // per parity

namespace {
std::mutex g_ws_mu;
std::vector<epsm_workspace*> g_ws;
}  // namespace

epsm_workspace* epsm_get_workspace(int device, cudaStream_t s) {
  std::lock_guard<std::mutex> lk(g_ws_mu);
  for (epsm_workspace* w : g_ws)
    if (w->device == device && w->stream == s) return w;
  epsm_workspace* w = new (std::nothrow) epsm_workspace();
  if (!w) return nullptr;
  w->device = device;
  w->stream = s;
  g_ws.push_back(w);
  return w;
}

// Make the workspace of stream s big enough for a launch of `chunks` chunks on `ctas` CTAs.
// Growing it synchronises the stream first (no grid may still use the old buffers).
static int ensure_workspace(epsm_workspace* ws, uint64_t chunks, uint64_t ctas, bool search, cudaStream_t s) {
  if (!ws->d_ctr) {
    cudaError_t e = cudaMalloc(&ws->d_ctr, 2 * kCtrWords * sizeof(unsigned long long));
    if (e != cudaSuccess) {
      epsm_set_error("cudaMalloc(counters): %s", cudaGetErrorString(e));
      return EPSM_ENOMEM;
    }
    e = cudaMemsetAsync(ws->d_ctr, 0, 2 * kCtrWords * sizeof(unsigned long long), s);
    if (e != cudaSuccess) return epsm_cuda_fail(e, "cudaMemsetAsync(counters)");
  }
  if (!search) return EPSM_OK;
  if (ctas > ws->scratch_ctas) {
    cudaStreamSynchronize(s);
    for (auto& p : ws->d_scratch) {
      if (p) cudaFree(p);
      p = nullptr;
    }
    ws->scratch_ctas = 0;
    const size_t bytes = static_cast<size_t>(ctas) * epsm::kScratchPerCta * sizeof(uint64_t);
    for (auto& p : ws->d_scratch) {
      cudaError_t e = cudaMalloc(&p, bytes);
      if (e != cudaSuccess) {
        epsm_set_error("cudaMalloc(parked masks, %zu bytes): %s", bytes, cudaGetErrorString(e));
        return EPSM_ENOMEM;
      }
    }
    ws->scratch_ctas = ctas;
  }
  if (chunks > ws->status_cap) {
    cudaStreamSynchronize(s);
    for (auto& p : ws->d_status) {
      if (p) cudaFree(p);
      p = nullptr;
    }
    ws->status_cap = 0;
    const uint64_t cap = chunks < 1024 ? 1024 : chunks;
    for (auto& p : ws->d_status) {
      cudaError_t e = cudaMalloc(&p, cap * sizeof(unsigned long long));
      if (e != cudaSuccess) {
        epsm_set_error("cudaMalloc(status, %llu chunks): %s", (unsigned long long)cap, cudaGetErrorString(e));
        return EPSM_ENOMEM;
      }
      e = cudaMemsetAsync(p, 0, cap * sizeof(unsigned long long), s);
      if (e != cudaSuccess) return epsm_cuda_fail(e, "cudaMemsetAsync(status)");
    }
    ws->status_cap = cap;
  }
  return EPSM_OK;
}

int epsm_ensure_occ(epsm_plan_t* plan) {
  if (plan->d_occ) return EPSM_OK;
  cudaError_t e = cudaMalloc(&plan->d_occ, 2 * sizeof(unsigned long long));
  if (e != cudaSuccess) {
    epsm_set_error("cudaMalloc(occ): %s", cudaGetErrorString(e));
    return EPSM_ENOMEM;
  }
  e = cudaMallocHost(&plan->h_occ, 2 * sizeof(unsigned long long));
  if (e != cudaSuccess) {
    epsm_set_error("cudaMallocHost(occ): %s", cudaGetErrorString(e));
    return EPSM_ENOMEM;
  }
  return EPSM_OK;
}

// One-time per (device, kernel variant): opt in to > 48 KiB of dynamic shared memory.
static int set_smem_attr(KernelFn fn, int device, int smem) {
  static std::atomic<KernelFn> done[16][64];
  if (device < 0 || device >= 16) device = 15;
  for (auto& slot : done[device]) {
    KernelFn f = slot.load(std::memory_order_acquire);
    if (f == fn) return EPSM_OK;
    if (f == nullptr) break;
  }
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       smem);
  if (e != cudaSuccess) return epsm_cuda_fail(e, "cudaFuncSetAttribute(max dynamic smem)");
  for (auto& slot : done[device]) {
    KernelFn expected = nullptr;
    if (slot.compare_exchange_strong(expected, fn) || expected == fn) break;
  }
  return EPSM_OK;
}

// PDL on by default; EPSM_NO_PDL=1 turns it off (debugging / A-B timing).
static bool plan_pdl_enabled() {
  static const bool on = [] {
    const char* v = getenv("EPSM_NO_PDL");
    return !(v && v[0] && v[0] != '0');
  }();
  return on;
}

// Upload a plan's preprocessing (and, for m > 32, its pattern words) on first use.
static int ensure_plan_device(epsm_plan_t* plan, cudaStream_t s) {
  if (!plan->d_desc) {
    cudaError_t e = cudaMalloc(&plan->d_desc, sizeof(epsm::JobDesc));
    if (e != cudaSuccess) {
      plan->d_desc = nullptr;
      epsm_set_error("cudaMalloc(plan descriptor): %s", cudaGetErrorString(e));
      return EPSM_ENOMEM;
    }
    e = cudaMemcpyAsync(plan->d_desc, plan->h_desc, sizeof(epsm::JobDesc), cudaMemcpyHostToDevice, s);
    if (e != cudaSuccess) return epsm_cuda_fail(e, "cudaMemcpyAsync(plan descriptor)");
  }
  if (plan->m > EPSM_MAX_M && !plan->d_pat) return epsm_upload_pattern(plan, s);
  return EPSM_OK;
}

// long patterns: the zero-padded pattern words in device memory (the naive check)
int epsm_upload_pattern(epsm_plan_t* plan, cudaStream_t s) {
  const size_t bytes = ((plan->m + 3) / 4 + 1) * sizeof(uint32_t);
  cudaError_t e = cudaMalloc(&plan->d_pat, bytes);
  if (e != cudaSuccess) {
    plan->d_pat = nullptr;
    epsm_set_error("cudaMalloc(pattern, %zu bytes): %s", bytes, cudaGetErrorString(e));
    return EPSM_ENOMEM;
  }
  e = cudaMemcpyAsync(plan->d_pat, plan->pattern, bytes, cudaMemcpyHostToDevice, s);
  if (e != cudaSuccess) return epsm_cuda_fail(e, "cudaMemcpyAsync(pattern)");
  return EPSM_OK;
}

static int launch_fanout(const epsm_job* jobs, uint32_t k, bool search, cudaStream_t s, epsm_workspace* ws);

// Core launcher: k <= kMaxJobs searches of one pattern length over the device text
// d_text[0..nbytes-1]; starts [0, nstarts) are reported (nstarts <= nbytes - m + 1), each
// shifted by `base`.  One persistent grid streams the chunks of all k searches in turn.
int epsm_launch_jobs(const epsm_job* jobs, uint32_t k, const uint8_t* d_text, uint64_t nbytes, uint64_t nstarts,
                     uint64_t base, bool search, cudaStream_t s, const epsm_eqidx_t* index) {
  if (k == 0) return EPSM_OK;
  if (k > static_cast<uint32_t>(epsm::kMaxJobs)) {
    epsm_set_error("%u searches in one launch (max %d)", k, epsm::kMaxJobs);
    return EPSM_EINVAL;
  }
  epsm_plan_t* plan0 = jobs[0].plan;
  if (nstarts == 0) {
    for (uint32_t j = 0; j < k; ++j) {
      cudaError_t e = cudaMemsetAsync(jobs[j].d_occ, 0, sizeof(unsigned long long), s);
      for (uint32_t o = 0; o < jobs[j].nx && e == cudaSuccess; ++o)
        e = cudaMemsetAsync(jobs[j].xh[o].occ, 0, sizeof(unsigned long long), s);
      if (e != cudaSuccess) return epsm_cuda_fail(e, "cudaMemsetAsync(occ)");
    }
    return EPSM_OK;
  }
  if (!index && epsm_long_applies(plan0)) {
    // long patterns at EPSMc's sampling stride: their own kernels, one search at a time
    epsm_workspace* wsl = nullptr;
    for (uint32_t j = 0; j < k; ++j) {
      int rc = epsm_long_launch(jobs[j].plan, d_text, nbytes, nstarts, base, jobs[j].d_pos, jobs[j].cap,
                                jobs[j].d_occ, search, s);
      if (rc) return rc;
    }
    wsl = epsm_get_workspace(plan0->device, s);
    return wsl ? launch_fanout(jobs, k, search, s, wsl) : EPSM_ENOMEM;
  }
  const uint64_t mis = reinterpret_cast<uintptr_t>(d_text) & 15u;
  epsm::KParams P;
  std::memset(&P, 0, sizeof(P));
  P.text = d_text - mis;
  P.nbytes = nbytes + mis;
  P.s_lo = mis;
  P.s_hi = mis + nstarts;
  P.it_lo = mis ? 1u : 0u;                                   // tile 0 holds starts < mis
  P.it_hi = static_cast<uint32_t>(P.s_hi / epsm::kTile);     // tiles wholly below s_hi
  P.pos_bias = base - mis;
  P.mul8 = 1u << 24;
  P.mul24 = 1u << 8;
  P.movemask_mul = 0x00204081u;
  P.m = plan0->m;
  P.njobs = k;
  P.desc_bytes = (plan0->sk > 0 && !index) ? static_cast<uint32_t>(sizeof(epsm::JobDesc)) : epsm::kJobHeader;
  if (index) {
    if (mis != 0 || index->text != d_text || index->n != nbytes) {
      epsm_set_error("index searches need the aligned text the index was built over");
      return EPSM_EINVAL;
    }
    P.planes = index->d_planes;
    P.pstride = index->pstride;
  }
  for (uint32_t j = 0; j < k; ++j) {
    epsm_plan_t* pl = jobs[j].plan;
    if (pl->m != plan0->m || (!index && pl->sk != plan0->sk) || pl->device != plan0->device) {
      epsm_set_error("searches of one launch need the same pattern length, filter and device");
      return EPSM_EINVAL;
    }
    if (index) {
      const epsm::JobDesc& D = *pl->h_desc;
      if (D.np == 0 || pl->m > EPSM_MAX_M) {
        epsm_set_error("pattern does not qualify for the index (m <= 32, <= 8 distinct bytes)");
        return EPSM_EINVAL;
      }
      P.jobs[j].np = D.np;
      for (uint32_t q = 0; q < D.np; ++q) {
        const int pid = index->plane_of[D.pval[q]];
        if (pid < 0) {
          epsm_set_error("byte %u of the pattern is not in the index", static_cast<unsigned>(D.pval[q]));
          return EPSM_EINVAL;
        }
        P.jobs[j].pid[q] = static_cast<uint8_t>(pid);
      }
    }
    int rc = ensure_plan_device(pl, s);
    if (rc) return rc;
    P.jobs[j].desc = pl->d_desc;
    P.jobs[j].dpat = pl->d_pat;
    P.jobs[j].pos = jobs[j].d_pos;
    P.jobs[j].cap = jobs[j].d_pos ? jobs[j].cap : 0;
    P.jobs[j].occ = jobs[j].d_occ;
  }
  const uint64_t tiles = (P.s_hi + epsm::kTile - 1) / epsm::kTile;
  const uint64_t chunks = (tiles + epsm::kChunkTiles - 1) / epsm::kChunkTiles;
  if (tiles > 0x7FFFFFFFull || chunks * k > 0x7FFFFFFFull) {
    epsm_set_error("text too large: %llu tiles x %u searches", (unsigned long long)tiles, k);
    return EPSM_EINVAL;
  }
  const uint64_t gchunks = chunks * k;
  epsm_workspace* ws = epsm_get_workspace(plan0->device, s);
  if (!ws) return EPSM_ENOMEM;
  if (ws->num_sms <= 0) {
    cudaError_t e = cudaDeviceGetAttribute(&ws->num_sms, cudaDevAttrMultiProcessorCount, plan0->device);
    if (e != cudaSuccess) return epsm_cuda_fail(e, "cudaDeviceGetAttribute(SM count)");
  }
  const uint64_t grid = gchunks < static_cast<uint64_t>(ws->num_sms) ? gchunks : ws->num_sms;
  int rc = ensure_workspace(ws, gchunks, grid, search, s);
  if (rc) return rc;
  // launch L uses parity L & 1; its status tag is L mod 2^24.  The first search launch of
  // every epoch (L >> 24) clears both status buffers (in stream order) before it runs, so a
  // word left by an earlier epoch can never carry a live tag -- whatever launch (count or
  // search) happened to take the number at the epoch boundary.  Tag 0 is skipped (a zeroed
  // word must never look like a valid status).
  uint64_t L = ws->launches;
  if (search && ((L >> 24) != ws->status_epoch || (L & 0xFFFFFFull) == 0)) {
    for (auto* p : ws->d_status) {
      cudaError_t e = cudaMemsetAsync(p, 0, ws->status_cap * sizeof(unsigned long long), s);
      if (e != cudaSuccess) return epsm_cuda_fail(e, "cudaMemsetAsync(status)");
    }
    if ((L & 0xFFFFFFull) == 0) ws->launches = ++L;
    ws->status_epoch = L >> 24;
  }
  const int par = static_cast<int>(L & 1u);
  P.ntiles = static_cast<uint32_t>(tiles);
  P.nchunks = static_cast<uint32_t>(chunks);
  P.gchunks = static_cast<uint32_t>(gchunks);
  P.ctr = ws->d_ctr + kCtrWords * par;
  P.ctr_base = ws->ctr_base[par];
  P.exit_ctr = ws->d_ctr + kCtrWords * par + 3;
  P.exit_expect = ws->exit_total[par];      // every CTA of launch L-2 (and before) has exited
  if (search) {
    P.status = ws->d_status[par];
    P.scratch = ws->d_scratch[par];
    P.tag = static_cast<unsigned long long>(L & 0xFFFFFFull) << epsm::kEpochShift;
  }
  P.trace = trace_slot(plan0->device);
  static const uint32_t env_flags = [] {
    const char* v = getenv("EPSM_FLAGS");
    return v && v[0] ? static_cast<uint32_t>(strtoul(v, nullptr, 0)) : 0u;
  }();
  P.flags = env_flags;
  // index searches of at most 2 (4) planes each take the variant with 4 (2) tiles per stage
  uint32_t max_np = 0;
  for (uint32_t j = 0; j < k && index; ++j) max_np = std::max(max_np, P.jobs[j].np);
  static const bool multi_tile = [] {
    const char* v = getenv("EPSM_INDEXC");
    return !(v && v[0] == '0');
  }();
  static const bool index8 = [] {
    const char* v = getenv("EPSM_INDEX8");
    return !(v && v[0] == '0');
  }();
  const int pmode = !multi_tile ? epsm::kPlaneMode
                    : max_np <= 2 ? epsm::kPlaneModeC
                    : max_np <= 4 ? epsm::kPlaneModeC2
                    : index8      ? epsm::kPlaneModeC8 : epsm::kPlaneMode;
  KernelFn fn = index ? kernel_for(plan0->m, pmode, 0, search) : kernel_for(plan0->m, plan0->sk, plan0->sq, search);
  const int smem = (index && pmode == epsm::kPlaneModeC8)
                       ? (search ? static_cast<int>(sizeof(epsm::Index8Smem<true>))
                                 : static_cast<int>(sizeof(epsm::Index8Smem<false>)))
                   : search ? static_cast<int>(sizeof(epsm::SearchSmem)) : static_cast<int>(sizeof(epsm::CountSmem));
  rc = set_smem_attr(fn, plan0->device, smem);
  if (rc) return rc;
  // programmatic dependent launch: the kernel starts while the previous grid on the stream
  // drains; it synchronises with that grid (griddepcontrol.wait) only before writing outputs,
  // and with launch L-2 (same workspace parity) through the CTA exit counter
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(static_cast<unsigned>(grid));
  cfg.blockDim = dim3(epsm::kThreads);
  cfg.dynamicSmemBytes = static_cast<size_t>(smem);
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = plan_pdl_enabled() ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, fn, P);
  epsm_count_launch();
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) return epsm_cuda_fail(e, "epsm_scan_kernel launch");
  // CTAs start on chunks [0, grid) and draw the rest from the counter, two draws ahead of the
  // chunk they stream: (gchunks - grid) useful draws + exactly 2 draws past the end per CTA
  ws->ctr_base[par] += gchunks + grid;
  ws->exit_total[par] += grid;
  ws->launches = L + 1;
  return launch_fanout(jobs, k, search, s, ws);
}

// fan-out: occ and positions of a job to its further outputs (identical patterns)
static int launch_fanout(const epsm_job* jobs, uint32_t k, bool search, cudaStream_t s, epsm_workspace* ws) {
  // the fan-outs of the launch's searches together (one launch where the buffers allow): every
  // job's outputs are a run of the same device / host XOut tables
  int j0 = -1;
  for (uint32_t j = 0; j < k; ++j)
    if (jobs[j].nx && jobs[j].xh && (j0 < 0 || jobs[j].xh < jobs[j0].xh)) j0 = static_cast<int>(j);
  bool tables = j0 >= 0;
  for (uint32_t j = 0; j < k && tables; ++j)
    if (jobs[j].nx && !jobs[j].xh) tables = false;
  if (tables) {
    std::vector<epsm_rep_req> rq;
    for (uint32_t j = 0; j < k; ++j)
      if (jobs[j].nx)
        rq.push_back(epsm_rep_req{jobs[j].d_pos, jobs[j].cap, jobs[j].d_occ,
                                  static_cast<uint32_t>(jobs[j].xh - jobs[j0].xh), jobs[j].nx});
    return epsm_replicate_many(rq.data(), static_cast<uint32_t>(rq.size()), jobs[j0].x, jobs[j0].xh, search, s, ws);
  }
  for (uint32_t j = 0; j < k; ++j) {
    if (jobs[j].nx == 0) continue;
    int rc = epsm_replicate(jobs[j].d_pos, jobs[j].cap, jobs[j].d_occ, jobs[j].x, jobs[j].nx, search, s, ws);
    if (rc) return rc;
  }
  return EPSM_OK;
}

int epsm_replicate(const uint64_t* d_pos, uint64_t cap, const unsigned long long* d_occ, const epsm::XOut* x,
                   uint32_t nx, bool search, cudaStream_t s, epsm_workspace* ws) {
  cudaError_t e = cudaSuccess;
  {
    const uint64_t have = (search && d_pos) ? cap : 0;
    {                                                  // (per device: the attribute is per device)
      static std::mutex mu;
      static std::vector<int> devs;
      std::lock_guard<std::mutex> lk(mu);
      if (std::find(devs.begin(), devs.end(), ws->device) == devs.end()) {
        e = cudaFuncSetAttribute(epsm::epsm_replicate_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(sizeof(epsm::RepSmem)));
        if (e != cudaSuccess) return epsm_cuda_fail(e, "cudaFuncSetAttribute(replicate)");
        devs.push_back(ws->device);
      }
    }
    // (grid sized by the capacity; CTAs past the occ's chunks exit at once)
    const uint64_t chunks = (have + epsm::kRepChunk / 8 - 1) / (epsm::kRepChunk / 8);
#ifndef EPSM_REP_CTAS_PER_SM
#define EPSM_REP_CTAS_PER_SM 2
#endif
    const unsigned blocks = static_cast<unsigned>(
        std::max<uint64_t>(1, std::min<uint64_t>(EPSM_REP_CTAS_PER_SM * static_cast<uint64_t>(ws->num_sms), chunks)));
    for (uint32_t a = 0; a < nx; a += epsm::kRepMaxOut) {
      const uint32_t nxa = std::min<uint32_t>(nx - a, epsm::kRepMaxOut);
      epsm::epsm_replicate_kernel<<<blocks, epsm::kRepThreads, sizeof(epsm::RepSmem), s>>>(
          search ? d_pos : nullptr, d_occ, have, x + a, nxa);
      epsm_count_launch();
    }
    e = cudaGetLastError();
    if (e != cudaSuccess) return epsm_cuda_fail(e, "epsm_replicate_kernel launch");
  }
  return EPSM_OK;
}

int epsm_replicate_many(const epsm_rep_req* r, uint32_t nr, const epsm::XOut* d_x, const epsm::XOut* h_x, bool search,
                        cudaStream_t s, epsm_workspace* ws) {
  auto a16 = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; };
  std::vector<epsm::RepJobD> jobs;
  for (uint32_t i = 0; i < nr; ++i) {
    const epsm_rep_req& q = r[i];
    bool ok = q.nx <= epsm::kRepMultiOut && a16(q.pos);
    for (uint32_t o = 0; ok && o < q.nx; ++o)
      if (h_x[q.x0 + o].pos && !a16(h_x[q.x0 + o].pos)) ok = false;
    if (!ok || !search) {                                          // (the single-source kernel)
      int rc = epsm_replicate(q.pos, q.cap, q.occ, d_x + q.x0, q.nx, search, s, ws);
      if (rc) return rc;
      continue;
    }
    jobs.push_back(epsm::RepJobD{q.pos, q.occ, q.cap, q.x0, q.nx});
  }
  if (jobs.empty()) return EPSM_OK;
  cudaError_t e = cudaSuccess;
  if (ws->num_sms <= 0) {
    e = cudaDeviceGetAttribute(&ws->num_sms, cudaDevAttrMultiProcessorCount, ws->device);
    if (e != cudaSuccess) return epsm_cuda_fail(e, "cudaDeviceGetAttribute(SM count)");
  }
  {                                                                // (per device: the attribute is per device)
    static std::mutex mu;
    static std::vector<int> devs;
    std::lock_guard<std::mutex> lk(mu);
    if (std::find(devs.begin(), devs.end(), ws->device) == devs.end()) {
      e = cudaFuncSetAttribute(epsm::epsm_replicate_multi_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               static_cast<int>(sizeof(epsm::RepMultiSmem)));
      if (e != cudaSuccess) return epsm_cuda_fail(e, "cudaFuncSetAttribute(replicate multi)");
      devs.push_back(ws->device);
    }
  }
  for (size_t a = 0; a < jobs.size(); a += epsm::kRepMaxJobs) {
    const uint32_t nj = static_cast<uint32_t>(std::min<size_t>(jobs.size() - a, epsm::kRepMaxJobs));
    if (ws->repjobs_cap < jobs.size()) {
      if (ws->d_repjobs) {
        cudaStreamSynchronize(s);
        cudaFree(ws->d_repjobs);
        ws->d_repjobs = nullptr;
        ws->repjobs_cap = 0;
      }
      e = cudaMalloc(&ws->d_repjobs, jobs.size() * sizeof(epsm::RepJobD));
      if (e != cudaSuccess) {
        epsm_set_error("cudaMalloc(fan-out job table): %s", cudaGetErrorString(e));
        return EPSM_ENOMEM;
      }
      ws->repjobs_cap = jobs.size();
    }
    epsm::RepJobD* dj = static_cast<epsm::RepJobD*>(ws->d_repjobs) + a;
    // (a pageable source is staged before cudaMemcpyAsync returns: the vector may go)
    e = cudaMemcpyAsync(dj, jobs.data() + a, nj * sizeof(epsm::RepJobD), cudaMemcpyHostToDevice, s);
    if (e != cudaSuccess) return epsm_cuda_fail(e, "cudaMemcpyAsync(fan-out job table)");
    KtRec kt{};
    const bool timed = g_kt_on.load(std::memory_order_relaxed);
    if (timed) {
      for (cudaEvent_t& ev : kt.ev)
        if ((e = cudaEventCreate(&ev)) != cudaSuccess) return epsm_cuda_fail(e, "cudaEventCreate(ktimer)");
      for (uint32_t j = a; j < a + nj; ++j) {
        KtJob kj{jobs[j].occ, jobs[j].src ? jobs[j].cap : 0, {}};
        for (uint32_t o = 0; o < jobs[j].nx; ++o) {
          const epsm::XOut& X = h_x[jobs[j].x0 + o];
          kj.out_caps.push_back(X.pos ? X.cap : 0);
        }
        kt.jobs.push_back(std::move(kj));
      }
      cudaEventRecord(kt.ev[0], s);
    }
    epsm::epsm_replicate_multi_kernel<<<EPSM_REP_CTAS_PER_SM * ws->num_sms, epsm::kRepThreads,
                                        sizeof(epsm::RepMultiSmem), s>>>(dj, nj, d_x);
    epsm_count_launch();
    e = cudaGetLastError();
    if (e != cudaSuccess) return epsm_cuda_fail(e, "epsm_replicate_multi_kernel launch");
    if (timed) {
      cudaEventRecord(kt.ev[1], s);
      std::lock_guard<std::mutex> lk(g_kt_mu);
      g_kt_recs.push_back(std::move(kt));
    }
  }
  return EPSM_OK;
}

int epsm_launch(epsm_plan_t* plan, const uint8_t* d_text, uint64_t nbytes, uint64_t nstarts, uint64_t base,
                uint64_t* d_pos, uint64_t cap, unsigned long long* d_occ, bool search, cudaStream_t s) {
  const epsm_job job{plan, d_pos, cap, d_occ};
  return epsm_launch_jobs(&job, 1, d_text, nbytes, nstarts, base, search, s);
}

static bool aligned8(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 7u) == 0; }

static int check_common(epsm_plan_t* plan, const uint8_t* d_text, uint64_t n) {
  if (!plan) {
    epsm_set_error("NULL plan");
    return EPSM_EINVAL;
  }
  if (!d_text && n > 0) {
    epsm_set_error("NULL text with n > 0");
    return EPSM_EINVAL;
  }
  if (n > (1ull << 38)) {
    epsm_set_error("n = %llu exceeds 2^38", (unsigned long long)n);
    return EPSM_EINVAL;
  }
  return EPSM_OK;
}

static uint64_t n_starts(uint32_t m, uint64_t n) { return n >= m ? n - m + 1 : 0; }

extern "C" {

int epsm_plan(const uint8_t* pattern, uint32_t m, epsm_plan_t** out) {
  if (!out) {
    epsm_set_error("NULL out");
    return EPSM_EINVAL;
  }
  *out = nullptr;
  if (!pattern || m == 0) {
    epsm_set_error("pattern must be non-NULL with m >= 1");
    return EPSM_EINVAL;
  }
  if (m > EPSM_MAX_M_LONG) {
    epsm_set_error("m = %u > %u is not supported", m, EPSM_MAX_M_LONG);
    return EPSM_EUNSUP;
  }
  epsm_plan_t* p = new (std::nothrow) epsm_plan_t();
  if (!p) return EPSM_ENOMEM;
  p->m = m;
  std::memcpy(p->pattern, pattern, m);
  // B[i] = (p_i)^alpha restricted to one 32-bit lane, i < min(m, 4)
  for (uint32_t i = 0; i < 4; ++i) p->bcast[i] = i < m ? 0x01010101u * pattern[i] : 0u;
  for (uint32_t i = 0; i < 4; ++i) p->bcast2[i] = 4 + i < m ? 0x01010101u * pattern[4 + i] : 0u;
  // P_i blocks, zero padded, as little-endian words + byte masks
  for (uint32_t q = 0; q < 9; ++q) {
    uint32_t w = 0, mk = 0;
    for (uint32_t b = 0; b < 4; ++b) {
      const uint32_t idx = 4 * q + b;
      if (idx < m) {
        w |= static_cast<uint32_t>(pattern[idx]) << (8 * b);
        mk |= 0xFFu << (8 * b);
      }
    }
    p->pat[q] = w;
    p->pmask[q] = mk;
  }
  // the kernels' per-search descriptor: filter words, P_i blocks (first 48 bytes) and, for the
  // sampled variants, EPSMc's table L of gram fingerprints
  p->h_desc = new (std::nothrow) epsm::JobDesc();
  if (!p->h_desc) {
    delete p;
    return EPSM_ENOMEM;
  }
  epsm::JobDesc& D = *p->h_desc;
  std::memset(&D, 0, sizeof(D));
  std::memcpy(D.bcast, p->bcast, sizeof(D.bcast));
  std::memcpy(D.bcast2, p->bcast2, sizeof(D.bcast2));
  for (uint32_t q = 0; q < 12; ++q) {
    uint32_t w = 0, mk = 0;
    for (uint32_t b = 0; b < 4; ++b) {
      const uint32_t idx = 4 * q + b;
      if (idx < m) {
        w |= static_cast<uint32_t>(pattern[idx]) << (8 * b);
        mk |= 0xFFu << (8 * b);
      }
    }
    D.pat[q] = w;
    D.pmask[q] = mk;
  }
  // EPSMa's equality masks: the pattern's distinct bytes (if at most 2)
  // and the positions holding each
  {
    uint32_t d = 0;
    uint8_t vals[2] = {0, 0};
    for (uint32_t i = 0; i < m && i < 12 && d <= 2; ++i) {
      uint32_t v = 0;
      while (v < d && vals[v] != pattern[i]) ++v;
      if (v == d) {
        if (d < 2) vals[d] = pattern[i];
        ++d;
      }
      if (v < 2) D.eqsel[v] |= 1u << i;
    }
    if (d <= 2 && m <= 11) {
      D.eqd = d;
      for (uint32_t v = 0; v < d; ++v) D.eqv[v] = 0x01010101u * vals[v];
    } else {
      D.eqd = 0;
      D.eqsel[0] = D.eqsel[1] = 0;
    }
  }
  // the same shift-AND over an equality-mask index: up to kMaxPlaneSlots distinct bytes in
  // order of first occurrence, and the positions holding each (m <= 32) as packed shift lists
  if (m <= EPSM_MAX_M) {
    constexpr uint32_t kSlots = static_cast<uint32_t>(epsm::kMaxPlaneSlots);
    uint32_t d = 0, sel[kSlots] = {};
    for (uint32_t i = 0; i < m && d <= kSlots; ++i) {
      uint32_t v = 0;
      while (v < d && D.pval[v] != pattern[i]) ++v;
      if (v == d) {
        if (d < kSlots) D.pval[d] = pattern[i];
        ++d;
      }
      if (v < kSlots) sel[v] |= 1u << i;
    }
    if (d <= kSlots) {
      D.np = d;
      uint32_t w = 0;
      for (uint32_t v = 0; v < d; ++v) {
        uint8_t list[32 + 3];
        uint32_t c = 0;
        for (uint32_t i = 0; i < m; ++i)
          if ((sel[v] >> i) & 1u) list[c++] = static_cast<uint8_t>(i);
        while (c % 4) list[c] = list[0], ++c;            // pad: repeat the first position
        for (uint32_t i = 0; i < m; ++i)
          if ((sel[v] >> i) & 1u) D.pslot[i] = static_cast<uint8_t>(v);
        D.pw0[v] = static_cast<uint8_t>(w);
        D.pwn[v] = static_cast<uint8_t>(c / 4);
        for (uint32_t q = 0; q < c / 4; ++q, ++w)
          D.plist[w] = list[4 * q] | (list[4 * q + 1] << 8) | (list[4 * q + 2] << 16) |
                       (static_cast<uint32_t>(list[4 * q + 3]) << 24);
      }
    }
  }
  if (D.np == 0) {
    std::memset(D.plist, 0, sizeof(D.plist));
    std::memset(D.pw0, 0, sizeof(D.pw0));
    std::memset(D.pwn, 0, sizeof(D.pwn));
    std::memset(D.pval, 0, sizeof(D.pval));
  }
  sampled_geometry(m, p->pattern, &p->sk, &p->sq);
  if (p->sk > 0) build_gram_table(p->pattern, p->sk, p->sq, D.gram_tab);
  p->device = -1;
  *out = p;
  return EPSM_OK;
}

void epsm_plan_free(epsm_plan_t* plan) {
  if (!plan) return;
  if (plan->device >= 0) {
    cudaSetDevice(plan->device);
    cudaDeviceSynchronize();
  }
  if (plan->d_occ) cudaFree(plan->d_occ);
  if (plan->d_desc) cudaFree(plan->d_desc);
  delete plan->h_desc;
  if (plan->d_pat) cudaFree(plan->d_pat);
  if (plan->d_long) cudaFree(plan->d_long);
  epsm_long_free(plan);
  if (plan->h_occ) cudaFreeHost(plan->h_occ);
  if (plan->d_text_buf) cudaFree(plan->d_text_buf);
  if (plan->d_pos_buf) cudaFree(plan->d_pos_buf);
  if (plan->d_scratch) cudaFree(plan->d_scratch);
  if (plan->d_counts) cudaFree(plan->d_counts);
  if (plan->h_counts) cudaFreeHost(plan->h_counts);
  delete plan;
}

uint32_t epsm_plan_m(const epsm_plan_t* plan) { return plan ? plan->m : 0; }

int epsm_count_async(epsm_plan_t* plan, const uint8_t* d_text, uint64_t n, uint64_t* d_occ, epsm_stream_t stream) {
  int rc = check_common(plan, d_text, n);
  if (rc) return rc;
  if (!d_occ || !aligned8(d_occ)) {
    epsm_set_error("d_occ must be a non-NULL 8-byte aligned device pointer");
    return d_occ ? EPSM_EALIGN : EPSM_EINVAL;
  }
  rc = epsm_bind_device(plan, d_occ);
  if (rc) return rc;
  return epsm_launch(plan, d_text, n, n_starts(plan->m, n), 0, nullptr, 0,
                     reinterpret_cast<unsigned long long*>(d_occ), false, static_cast<cudaStream_t>(stream));
}

int64_t epsm_count(epsm_plan_t* plan, const uint8_t* d_text, uint64_t n, epsm_stream_t stream) {
  int rc = check_common(plan, d_text, n);
  if (rc) return rc;
  rc = epsm_bind_device(plan, d_text ? (const void*)d_text : nullptr);
  if (rc) return rc;
  rc = epsm_ensure_occ(plan);
  if (rc) return rc;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  rc = epsm_launch(plan, d_text, n, n_starts(plan->m, n), 0, nullptr, 0, plan->d_occ, false, s);
  if (rc) return rc;
  cudaError_t e = cudaMemcpyAsync(plan->h_occ, plan->d_occ, 8, cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return epsm_cuda_fail(e, "epsm_count");
  return static_cast<int64_t>(plan->h_occ[0]);
}

int epsm_search_async(epsm_plan_t* plan, const uint8_t* d_text, uint64_t n, uint64_t* d_pos, uint64_t cap,
                      uint64_t* d_occ, epsm_stream_t stream) {
  int rc = check_common(plan, d_text, n);
  if (rc) return rc;
  if (!d_occ || (cap > 0 && !d_pos)) {
    epsm_set_error("d_occ required; d_pos required when cap > 0");
    return EPSM_EINVAL;
  }
  if (!aligned8(d_occ) || (d_pos && !aligned8(d_pos))) {
    epsm_set_error("d_pos and d_occ must be 8-byte aligned");
    return EPSM_EALIGN;
  }
  rc = epsm_bind_device(plan, d_occ);
  if (rc) return rc;
  return epsm_launch(plan, d_text, n, n_starts(plan->m, n), 0, cap ? d_pos : nullptr, cap,
                     reinterpret_cast<unsigned long long*>(d_occ), true, static_cast<cudaStream_t>(stream));
}

// Largest number of distinct pattern bytes a search runs over an index with (EPSM_INDEX_MAX_D
// overrides, 0 disables; A/B timing).  Speed only: both paths are exact.
static uint32_t index_max_d() {
  static const uint32_t v = [] {
    const char* e = getenv("EPSM_INDEX_MAX_D");
    return e && e[0] ? static_cast<uint32_t>(strtoul(e, nullptr, 0)) : static_cast<uint32_t>(EPSM_INDEX_MAX_D);
  }();
  return v;
}

// Does plans' search run over the index?  Its distinct bytes must all be in the index.  Speed
// rule (B200, 256 MiB texts, us per search text -> index): the shift-AND over planes wins for
// m <= 8 at every alphabet the index covers (sigma=2 m=8 137 -> 59, sigma=16 m=4 63 -> 27,
// sigma=32 m=8 61 -> 51) and for m <= 31 with <= 4 distinct bytes (sigma=2 m=16 68 -> 43,
// sigma=2 m=24 48 -> 40, sigma=4 m=24 38 -> 36); at m = 32 the text kernels are at the HBM
// roofline already (38 us) and the per-position shifts cost as much (binary texts: 38 -> 39);
// m 9..31 with 5..8 distinct bytes loses to the sampled filter.
static bool index_worthwhile(const epsm_plan_t* pl) {
  static const uint32_t max_m = [] {   // EPSM_INDEX_MAX_M: longest pattern with <= 4 bytes (A/B)
    const char* e = getenv("EPSM_INDEX_MAX_M");
    return e && e[0] ? static_cast<uint32_t>(strtoul(e, nullptr, 0)) : 31u;
  }();
  const epsm::JobDesc& D = *pl->h_desc;
  if (pl->m > EPSM_MAX_M || D.np == 0 || D.np > index_max_d()) return false;
  static const uint32_t any_d_m = [] {   // EPSM_INDEX_ANYD_M: longest pattern with any d <= 8 (A/B)
    const char* e = getenv("EPSM_INDEX_ANYD_M");
    return e && e[0] ? static_cast<uint32_t>(strtoul(e, nullptr, 0)) : 8u;
  }();
  return pl->m <= any_d_m || (pl->m <= max_m && D.np <= 4);
}

static bool use_index(const epsm_plan_t* pl, const epsm_eqidx_t* ix) {
  if (!ix || !index_worthwhile(pl) || (pl->device >= 0 && pl->device != ix->device)) return false;
  const epsm::JobDesc& D = *pl->h_desc;
  for (uint32_t q = 0; q < D.np; ++q)
    if (ix->plane_of[D.pval[q]] < 0) return false;
  return true;
}

int epsm_plan_index_values(const epsm_plan_t* plan, uint8_t* out_values) {
  if (!plan || !index_worthwhile(plan)) return 0;
  const epsm::JobDesc& D = *plan->h_desc;
  if (out_values) std::memcpy(out_values, D.pval, D.np);
  return static_cast<int>(D.np);
}

// A shard [base, base + n) of a text of n_total bytes that owns the starts [base, base +
// owned_len) must hold every owned window: n >= min(owned_len + m - 1, n_total - base).
static int check_overlap(uint64_t n, uint64_t owned_len, uint64_t base, uint64_t n_total, uint32_t m) {
  if (base > n_total || owned_len > n_total - base || n > n_total - base) {
    epsm_set_error("shard [%llu, +%llu) owning %llu starts lies outside the text of %llu bytes",
                   (unsigned long long)base, (unsigned long long)n, (unsigned long long)owned_len,
                   (unsigned long long)n_total);
    return EPSM_EINVAL;
  }
  if (owned_len == 0) return EPSM_OK;
  const uint64_t need = owned_len + m - 1 < n_total - base ? owned_len + m - 1 : n_total - base;
  if (n < need) {
    epsm_set_error("shard of %llu bytes is shorter than its owned starts plus the (m-1)-byte overlap "
                   "(%llu bytes for m = %u)", (unsigned long long)n, (unsigned long long)need, m);
    return EPSM_EINVAL;
  }
  return EPSM_OK;
}

static int batch_common(epsm_plan_t* const* plans, uint32_t k, const uint8_t* d_text, uint64_t n, uint64_t owned_len,
                        uint64_t base, uint64_t* const* d_pos, const uint64_t* caps, uint64_t* d_occ, bool search,
                        epsm_stream_t stream, const epsm_eqidx_t* index = nullptr, uint64_t n_total = 0,
                        const uint32_t* slot = nullptr, const std::vector<std::vector<uint32_t>>* fan = nullptr) {
  if (k == 0) return EPSM_OK;
  if (index && (index->text != d_text || index->n != n)) {
    epsm_set_error("the index was built over another text (pointer or length differ)");
    return EPSM_EINVAL;
  }
  if (!plans || !d_occ || (!d_text && n > 0)) {
    epsm_set_error("epsm_search_(range_)batch_async: NULL plans, d_occ or text");
    return EPSM_EINVAL;
  }
  if (n > (1ull << 38)) {
    epsm_set_error("n = %llu exceeds 2^38", (unsigned long long)n);
    return EPSM_EINVAL;
  }
  if (!aligned8(d_occ)) {
    epsm_set_error("d_occ must be 8-byte aligned");
    return EPSM_EALIGN;
  }
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  std::vector<epsm_job> jobs(k);
  for (uint32_t j = 0; j < k; ++j) {
    if (!plans[j]) {
      epsm_set_error("epsm_search_batch_async: plans[%u] is NULL", j);
      return EPSM_EINVAL;
    }
    if (n_total) {                     // a shard: every plan's window must fit its overlap
      int rc = check_overlap(n, owned_len, base, n_total, plans[j]->m);
      if (rc) return rc;
    }
    const uint32_t sj = slot ? slot[j] : j;   // the caller's arrays are indexed by slot[j]
    uint64_t* pos = d_pos ? d_pos[sj] : nullptr;
    const uint64_t cap = (pos && caps) ? caps[sj] : 0;
    if (pos && !aligned8(pos)) {
      epsm_set_error("d_pos[%u] must be 8-byte aligned", j);
      return EPSM_EALIGN;
    }
    int rc = epsm_bind_device(plans[j], d_occ);
    if (rc) return rc;
    jobs[j] = epsm_job{plans[j], cap ? pos : nullptr, cap, reinterpret_cast<unsigned long long*>(d_occ + sj)};
  }
  // fan-out outputs: host table, then one upload into the stream's workspace (stream order
  // keeps an earlier call's launches reading their table before this copy lands)
  std::vector<epsm::XOut> xh;
  std::vector<uint64_t> xoff(k, 0);
  if (fan) {
    for (uint32_t j = 0; j < k; ++j) {
      xoff[j] = xh.size();
      for (uint32_t q : (*fan)[j]) {
        uint64_t* pos = d_pos ? d_pos[q] : nullptr;
        const uint64_t cap = (pos && caps) ? caps[q] : 0;
        if (pos && !aligned8(pos)) {
          epsm_set_error("d_pos[%u] must be 8-byte aligned", q);
          return EPSM_EALIGN;
        }
        xh.push_back(epsm::XOut{cap ? pos : nullptr, cap, reinterpret_cast<unsigned long long*>(d_occ + q)});
      }
    }
  }
  if (!xh.empty()) {
    epsm_workspace* ws = epsm_get_workspace(plans[0]->device, s);
    if (!ws) return EPSM_ENOMEM;
    if (xh.size() > ws->xout_cap) {
      if (ws->d_xout) {
        cudaStreamSynchronize(s);
        cudaFree(ws->d_xout);
        ws->d_xout = nullptr;
        ws->xout_cap = 0;
      }
      cudaError_t e = cudaMalloc(&ws->d_xout, xh.size() * sizeof(epsm::XOut));
      if (e != cudaSuccess) {
        epsm_set_error("cudaMalloc(fan-out table): %s", cudaGetErrorString(e));
        return EPSM_ENOMEM;
      }
      ws->xout_cap = xh.size();
    }
    cudaError_t e = cudaMemcpyAsync(ws->d_xout, xh.data(), xh.size() * sizeof(epsm::XOut), cudaMemcpyHostToDevice, s);
    if (e != cudaSuccess) return epsm_cuda_fail(e, "cudaMemcpyAsync(fan-out table)");
    for (uint32_t j = 0; j < k; ++j) {
      jobs[j].nx = static_cast<uint32_t>((*fan)[j].size());
      if (jobs[j].nx) {
        jobs[j].x = ws->d_xout + xoff[j];
        jobs[j].xh = xh.data() + xoff[j];
      }
    }
  }
  // searches are independent: group them by kernel variant (m, filter or index), keeping
  // their order within a group, and launch each group in runs of at most kMaxJobs
  std::vector<int> variant(k);
  for (uint32_t j = 0; j < k; ++j)
    variant[j] = !use_index(plans[j], index) ? plans[j]->sk
                 : plans[j]->h_desc->np <= 2 ? epsm::kPlaneModeC
                 : plans[j]->h_desc->np <= 4 ? epsm::kPlaneModeC2 : epsm::kPlaneModeC8;
  std::vector<uint32_t> order(k);
  for (uint32_t j = 0; j < k; ++j) order[j] = j;
  std::stable_sort(order.begin(), order.end(), [&](uint32_t x, uint32_t y) {
    if (plans[x]->m != plans[y]->m) return plans[x]->m < plans[y]->m;
    return variant[x] < variant[y];
  });
  std::vector<epsm_job> run;
  uint32_t a = 0;
  while (a < k) {
    uint32_t b = a + 1;
    const epsm_plan_t* pa = plans[order[a]];
    const int va = variant[order[a]];
    while (b < k && b - a < static_cast<uint32_t>(epsm::kMaxJobs) && plans[order[b]]->m == pa->m &&
           variant[order[b]] == va)
      ++b;
    run.clear();
    for (uint32_t i = a; i < b; ++i) run.push_back(jobs[order[i]]);
    const uint32_t m = pa->m;
    uint64_t ns = n >= m ? n - m + 1 : 0;
    if (owned_len < ns) ns = owned_len;
    int rc = epsm_launch_jobs(run.data(), b - a, d_text, n, ns, base, search, s,
                              epsm::is_plane(va) ? index : nullptr);
    if (rc) return rc;
    a = b;
  }
  return EPSM_OK;
}

}  // extern "C"

int epsm_batch_run(epsm_plan_t* const* plans, uint32_t k, const uint32_t* slot, const uint8_t* d_text, uint64_t n,
                   uint64_t owned_len, uint64_t base, uint64_t n_total, uint64_t* const* d_pos, const uint64_t* caps,
                   uint64_t* d_occ, bool search, cudaStream_t s, const epsm_eqidx_t* index,
                   const std::vector<std::vector<uint32_t>>* fan) {
  return batch_common(plans, k, d_text, n, owned_len, base, d_pos, caps, d_occ, search, s, index, n_total, slot, fan);
}

extern "C" {

int epsm_search_range_batch_async(epsm_plan_t* const* plans, uint32_t k, const uint8_t* d_text, uint64_t n,
                                  uint64_t owned_len, uint64_t base, uint64_t n_total, uint64_t* const* d_pos,
                                  const uint64_t* caps, uint64_t* d_occ, epsm_stream_t stream) {
  if (n_total == 0 && (n > 0 || owned_len > 0)) {
    epsm_set_error("epsm_search_range_batch_async: n_total = 0");
    return EPSM_EINVAL;
  }
  return batch_common(plans, k, d_text, n, owned_len, base, d_pos, caps, d_occ, true, stream, nullptr, n_total);
}

int epsm_search_batch_async(epsm_plan_t* const* plans, uint32_t k, const uint8_t* d_text, uint64_t n,
                            uint64_t* const* d_pos, const uint64_t* caps, uint64_t* d_occ, epsm_stream_t stream) {
  return batch_common(plans, k, d_text, n, n, 0, d_pos, caps, d_occ, true, stream);
}

int epsm_count_batch_async(epsm_plan_t* const* plans, uint32_t k, const uint8_t* d_text, uint64_t n,
                           uint64_t* d_occ, epsm_stream_t stream) {
  return batch_common(plans, k, d_text, n, n, 0, nullptr, nullptr, d_occ, false, stream);
}

int epsm_search_range_batch_index_async(epsm_plan_t* const* plans, uint32_t k, const epsm_eqidx_t* index,
                                        const uint8_t* d_text, uint64_t n, uint64_t owned_len, uint64_t base,
                                        uint64_t n_total, uint64_t* const* d_pos, const uint64_t* caps,
                                        uint64_t* d_occ, epsm_stream_t stream) {
  if (n_total == 0 && (n > 0 || owned_len > 0)) {
    epsm_set_error("epsm_search_range_batch_index_async: n_total = 0");
    return EPSM_EINVAL;
  }
  return batch_common(plans, k, d_text, n, owned_len, base, d_pos, caps, d_occ, true, stream, index, n_total);
}

int epsm_count_batch_index_async(epsm_plan_t* const* plans, uint32_t k, const epsm_eqidx_t* index,
                                 const uint8_t* d_text, uint64_t n, uint64_t* d_occ, epsm_stream_t stream) {
  return batch_common(plans, k, d_text, n, n, 0, nullptr, nullptr, d_occ, false, stream, index);
}

int epsm_search_batch_index_async(epsm_plan_t* const* plans, uint32_t k, const epsm_eqidx_t* index,
                                  const uint8_t* d_text, uint64_t n, uint64_t* const* d_pos, const uint64_t* caps,
                                  uint64_t* d_occ, epsm_stream_t stream) {
  return batch_common(plans, k, d_text, n, n, 0, d_pos, caps, d_occ, true, stream, index);
}

// ---- equality-mask index (EPSMa's wscmp masks of a whole text)

int epsm_eqidx_create(epsm_eqidx_t** out) {
  if (!out) {
    epsm_set_error("epsm_eqidx_create: NULL out");
    return EPSM_EINVAL;
  }
  epsm_eqidx_t* ix = new (std::nothrow) epsm_eqidx_t();
  if (!ix) return EPSM_ENOMEM;
  for (int v = 0; v < 256; ++v) ix->plane_of[v] = -1;
  *out = ix;
  return EPSM_OK;
}

void epsm_eqidx_free(epsm_eqidx_t* ix) {
  if (!ix) return;
  if (ix->d_planes) {
    cudaSetDevice(ix->device);
    cudaDeviceSynchronize();
    cudaFree(ix->d_planes);
  }
  delete ix;
}

int epsm_eqidx_values(const epsm_eqidx_t* ix, uint8_t* out_values) {
  if (!ix) return 0;
  if (out_values) std::memcpy(out_values, ix->vals, ix->nv);
  return static_cast<int>(ix->nv);
}

int epsm_eqidx_build_async(epsm_eqidx_t* ix, const uint8_t* d_text, uint64_t n, const uint8_t* values, uint32_t nv,
                           epsm_stream_t stream) {
  if (!ix || !values || (!d_text && n > 0) || nv == 0 || nv > EPSM_MAX_PLANES) {
    epsm_set_error("epsm_eqidx_build_async: NULL argument or nv = %u not in [1, %u]", nv, EPSM_MAX_PLANES);
    return EPSM_EINVAL;
  }
  if (n > (1ull << 38)) {
    epsm_set_error("n = %llu exceeds 2^38", (unsigned long long)n);
    return EPSM_EINVAL;
  }
  if (reinterpret_cast<uintptr_t>(d_text) & 15u) {
    epsm_set_error("epsm_eqidx_build_async: d_text must be 16-byte aligned");
    return EPSM_EALIGN;
  }
  bool seen[256] = {};
  for (uint32_t q = 0; q < nv; ++q) {
    if (seen[values[q]]) {
      epsm_set_error("epsm_eqidx_build_async: value %u listed twice", static_cast<unsigned>(values[q]));
      return EPSM_EINVAL;
    }
    seen[values[q]] = true;
  }
  int dev = -1;
  cudaPointerAttributes attr;
  cudaError_t e = d_text ? cudaPointerGetAttributes(&attr, d_text) : cudaErrorInvalidValue;
  if (e == cudaSuccess && attr.type == cudaMemoryTypeDevice) {
    dev = attr.device;
  } else {
    cudaGetLastError();
    e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return epsm_cuda_fail(e, "cudaGetDevice");
  }
  e = cudaSetDevice(dev);
  if (e != cudaSuccess) return epsm_cuda_fail(e, "cudaSetDevice");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const uint64_t tiles = (n + epsm::kTile - 1) / epsm::kTile;
  const uint64_t pstride = tiles * epsm::kPlaneWordsPerTile + 2;   // + the last tile's halo word
  const uint64_t words = pstride * nv;
  if (ix->d_planes && (ix->device != dev || words > ix->cap_words)) {
    cudaStreamSynchronize(s);
    cudaSetDevice(ix->device);
    cudaDeviceSynchronize();
    cudaFree(ix->d_planes);
    cudaSetDevice(dev);
    ix->d_planes = nullptr;
    ix->cap_words = 0;
  }
  if (!ix->d_planes) {
    e = cudaMalloc(&ix->d_planes, words * sizeof(uint64_t));
    if (e != cudaSuccess) {
      cudaGetLastError();
      ix->d_planes = nullptr;
      epsm_set_error("cudaMalloc(%llu bytes) for the index planes failed", (unsigned long long)(words * 8));
      return EPSM_ENOMEM;
    }
    ix->cap_words = words;
  }
  ix->device = dev;
  ix->text = d_text;
  ix->n = n;
  ix->nv = nv;
  ix->pstride = pstride;
  for (int v = 0; v < 256; ++v) ix->plane_of[v] = -1;
  epsm::IdxParams P;
  std::memset(&P, 0, sizeof(P));
  P.text = d_text;
  P.n = n;
  P.planes = ix->d_planes;
  P.pstride = pstride;
  P.nv = nv;
  for (uint32_t q = 0; q < nv; ++q) {
    ix->vals[q] = values[q];
    ix->plane_of[values[q]] = static_cast<int16_t>(q);
    P.vals[q] = values[q];
  }
  int sms = 0;
  e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (e != cudaSuccess) return epsm_cuda_fail(e, "cudaDeviceGetAttribute(SM count)");
  const uint64_t want = (pstride + 255) / 256;
  const uint64_t cap = static_cast<uint64_t>(sms) * 64;   // (enough loads in flight)
  const unsigned grid = static_cast<unsigned>(want < cap ? want : cap);
  // few values: compare the bytes per value; many: bit-slice once, then 16 logic ops per value
  if (nv >= 8)
    epsm::epsm_eqidx_bits_kernel<<<grid, 256, 0, s>>>(P);
  else
    epsm::epsm_eqidx_kernel<<<grid, 256, 0, s>>>(P);
  epsm_count_launch();
  e = cudaGetLastError();
  if (e != cudaSuccess) return epsm_cuda_fail(e, "epsm_eqidx_kernel launch");
  return EPSM_OK;
}

int epsm_search_range_async(epsm_plan_t* plan, const uint8_t* d_shard, uint64_t shard_len, uint64_t owned_len,
                            uint64_t base, uint64_t n_total, uint64_t* d_pos, uint64_t cap, uint64_t* d_occ,
                            epsm_stream_t stream) {
  int rc = check_common(plan, d_shard, shard_len);
  if (rc) return rc;
  rc = check_overlap(shard_len, owned_len, base, n_total, plan->m);
  if (rc) return rc;
  if (!d_occ || (cap > 0 && !d_pos)) {
    epsm_set_error("d_occ required; d_pos required when cap > 0");
    return EPSM_EINVAL;
  }
  if (!aligned8(d_occ) || (d_pos && !aligned8(d_pos))) {
    epsm_set_error("d_pos and d_occ must be 8-byte aligned");
    return EPSM_EALIGN;
  }
  rc = epsm_bind_device(plan, d_occ);
  if (rc) return rc;
  uint64_t ns = n_starts(plan->m, shard_len);
  if (owned_len < ns) ns = owned_len;
  return epsm_launch(plan, d_shard, shard_len, ns, base, cap ? d_pos : nullptr, cap,
                     reinterpret_cast<unsigned long long*>(d_occ), true, static_cast<cudaStream_t>(stream));
}

int64_t epsm_search(epsm_plan_t* plan, const uint8_t* d_text, uint64_t n, uint64_t* d_pos, uint64_t cap,
                    epsm_stream_t stream) {
  int rc = check_common(plan, d_text, n);
  if (rc) return rc;
  if (cap > 0 && !d_pos) {
    epsm_set_error("d_pos required when cap > 0");
    return EPSM_EINVAL;
  }
  if (d_pos && !aligned8(d_pos)) {
    epsm_set_error("d_pos must be 8-byte aligned");
    return EPSM_EALIGN;
  }
  rc = epsm_bind_device(plan, d_text ? (const void*)d_text : (const void*)d_pos);
  if (rc) return rc;
  rc = epsm_ensure_occ(plan);
  if (rc) return rc;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  rc = epsm_launch(plan, d_text, n, n_starts(plan->m, n), 0, cap ? d_pos : nullptr, cap, plan->d_occ, true, s);
  if (rc) return rc;
  cudaError_t e = cudaMemcpyAsync(plan->h_occ, plan->d_occ, 8, cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return epsm_cuda_fail(e, "epsm_search");
  return static_cast<int64_t>(plan->h_occ[0]);
}

int64_t epsm_search_host(epsm_plan_t* plan, const uint8_t* h_text, uint64_t n, uint64_t* h_pos, uint64_t cap,
                         epsm_stream_t stream) {
  int rc = check_common(plan, h_text, n);
  if (rc) return rc;
  if (cap > 0 && !h_pos) {
    epsm_set_error("h_pos required when cap > 0");
    return EPSM_EINVAL;
  }
  if (plan->device < 0) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return epsm_cuda_fail(e, "cudaGetDevice");
    plan->device = dev;
  }
  cudaError_t e = cudaSetDevice(plan->device);
  if (e != cudaSuccess) return epsm_cuda_fail(e, "cudaSetDevice");
  rc = epsm_ensure_occ(plan);
  if (rc) return rc;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (n > plan->text_cap) {
    if (plan->d_text_buf) {
      cudaStreamSynchronize(s);
      cudaFree(plan->d_text_buf);
      plan->d_text_buf = nullptr;
      plan->text_cap = 0;
    }
    e = cudaMalloc(&plan->d_text_buf, n);
    if (e != cudaSuccess) {
      epsm_set_error("cudaMalloc(text, %llu): %s", (unsigned long long)n, cudaGetErrorString(e));
      return EPSM_ENOMEM;
    }
    plan->text_cap = n;
  }
  if (cap > plan->pos_cap) {
    if (plan->d_pos_buf) {
      cudaStreamSynchronize(s);
      cudaFree(plan->d_pos_buf);
      plan->d_pos_buf = nullptr;
      plan->pos_cap = 0;
    }
    e = cudaMalloc(&plan->d_pos_buf, cap * sizeof(uint64_t));
    if (e != cudaSuccess) {
      epsm_set_error("cudaMalloc(pos, %llu): %s", (unsigned long long)cap, cudaGetErrorString(e));
      return EPSM_ENOMEM;
    }
    plan->pos_cap = cap;
  }
  if (n) {
    e = cudaMemcpyAsync(plan->d_text_buf, h_text, n, cudaMemcpyHostToDevice, s);
    if (e != cudaSuccess) return epsm_cuda_fail(e, "cudaMemcpyAsync(H2D text)");
  }
  rc = epsm_launch(plan, plan->d_text_buf, n, n_starts(plan->m, n), 0, cap ? plan->d_pos_buf : nullptr, cap,
                   plan->d_occ, true, s);
  if (rc) return rc;
  e = cudaMemcpyAsync(plan->h_occ, plan->d_occ, 8, cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return epsm_cuda_fail(e, "epsm_search_host");
  const uint64_t occ = plan->h_occ[0];
  const uint64_t k = occ < cap ? occ : cap;
  if (k) {
    e = cudaMemcpyAsync(h_pos, plan->d_pos_buf, k * sizeof(uint64_t), cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return epsm_cuda_fail(e, "cudaMemcpyAsync(D2H positions)");
  }
  return static_cast<int64_t>(occ);
}

const char* epsm_strerror(int64_t code) {
  switch (code) {
    case EPSM_OK: return "EPSM_OK: success";
    case EPSM_EINVAL: return "EPSM_EINVAL: invalid argument";
    case EPSM_EUNSUP: return "EPSM_EUNSUP: unsupported pattern length (m > 4096)";
    case EPSM_EALIGN: return "EPSM_EALIGN: misaligned output pointer (needs 8-byte alignment)";
    case EPSM_ECUDA: return "EPSM_ECUDA: CUDA error";
    case EPSM_ENCCL: return "EPSM_ENCCL: NCCL error";
    case EPSM_ENOMEM: return "EPSM_ENOMEM: out of memory";
    default: return code > 0 ? "success (count)" : "unknown error";
  }
}

const char* epsm_last_error(void) { return g_last_error; }

uint64_t epsm_launch_count(void) { return g_launches.load(std::memory_order_relaxed); }

int epsm_version(void) { return 200; }

int epsm_ktimer_enable(int on) {
  g_kt_on.store(on != 0);
  return EPSM_OK;
}

int epsm_ktimer_read(uint64_t* launches, double* ms, double* bytes) {
  std::vector<KtRec> recs;
  {
    std::lock_guard<std::mutex> lk(g_kt_mu);
    recs.swap(g_kt_recs);
  }
  double t = 0.0, b = 0.0;
  int rc = EPSM_OK;
  for (KtRec& r : recs) {
    if (rc == EPSM_OK) {
      float f = 0.f;
      cudaError_t e = cudaEventSynchronize(r.ev[1]);
      if (e == cudaSuccess) e = cudaEventElapsedTime(&f, r.ev[0], r.ev[1]);
      for (size_t j = 0; e == cudaSuccess && j < r.jobs.size(); ++j) {
        unsigned long long occ = 0;
        e = cudaMemcpy(&occ, r.jobs[j].occ, sizeof(occ), cudaMemcpyDeviceToHost);
        const uint64_t have = occ < r.jobs[j].cap ? occ : r.jobs[j].cap;
        b += 8.0 * static_cast<double>(have);                       // source read once
        for (uint64_t oc : r.jobs[j].out_caps) b += 8.0 * static_cast<double>(oc < have ? oc : have);
      }
      if (e != cudaSuccess) rc = epsm_cuda_fail(e, "epsm_ktimer_read");
      t += f;
    }
    cudaEventDestroy(r.ev[0]);
    cudaEventDestroy(r.ev[1]);
  }
  if (launches) *launches = recs.size();
  if (ms) *ms = t;
  if (bytes) *bytes = b;
  return rc;
}

int64_t epsm_debug_trace(uint64_t* h_out, uint64_t max_words) {
  if (!g_trace) return 0;
  const uint64_t words = g_trace_slots * kTraceWordsPerLaunch;
  const uint64_t k = words < max_words ? words : max_words;
  cudaSetDevice(g_trace_device);
  cudaError_t e = cudaDeviceSynchronize();
  if (e == cudaSuccess) e = cudaMemcpy(h_out, g_trace, k * sizeof(uint64_t), cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) return epsm_cuda_fail(e, "epsm_debug_trace");
  return static_cast<int64_t>(k);
}

}  // extern "C"
