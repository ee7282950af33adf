// epsm_long.cu -- host side of the long-pattern path at EPSMc's sampling stride (SURVEY NEXT-1,
// PAPER.md:576-603): the table of the pattern's 16-byte substrings, the workspace and the three
// launches of one search (epsm_long.cuh).
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <new>
#include <vector>

#include "epsm.h"
#include "epsm_internal.h"
#include "epsm_long.cuh"

namespace lg = epsm::lg;

uint32_t epsm_long_stride(uint32_t m) { return m >= 32 ? 16u * (m / 16u - 1u) : 0u; }

void epsm_long_free(epsm_plan_t* plan) {
  delete plan->h_long;
  plan->h_long = nullptr;
}

bool epsm_long_applies(const epsm_plan_t* plan) {
  // EPSM_LONG_STRIDE=0 keeps every long pattern on the full-text sampled kernel (A/B)
  static const bool off = [] {
    const char* e = getenv("EPSM_LONG_STRIDE");
    return e && e[0] == '0';
  }();
  return !off && plan->m >= kLongStrideMinM && plan->m <= EPSM_MAX_M_LONG;
}

// The table L: the pattern's 16-byte substrings p[j .. j+16) for j < L (the
// offsets a start can have from its first sampled block), by the hash of their four words.
static int build_long_desc(epsm_plan_t* plan) {
  if (plan->h_long) return EPSM_OK;
  lg::LongDesc* D = new (std::nothrow) lg::LongDesc();
  if (!D) return EPSM_ENOMEM;
  std::memset(D, 0, sizeof(*D));
  const uint32_t L = epsm_long_stride(plan->m);
  std::vector<std::vector<uint16_t>> buckets(1u << lg::kBucketLog);
  for (uint32_t j = 0; j < L; ++j) {
    uint32_t w[4];
    std::memcpy(w, plan->pattern + j, 16);
    const uint32_t h = lg::long_hash(w[0], w[1], w[2], w[3]);
    const uint32_t h2 = lg::long_bloom2(h);
    D->bitmap[h >> 21] |= 1u << ((h >> 16) & 31u);
    D->bitmap[h2 >> 21] |= 1u << ((h2 >> 16) & 31u);
    buckets[h >> (32 - lg::kBucketLog)].push_back(static_cast<uint16_t>((j << 4) | ((h >> 16) & 15u)));
  }
  uint32_t e = 0;
  for (uint32_t b = 0; b < (1u << lg::kBucketLog); ++b) {
    D->boff[b] = static_cast<uint16_t>(e);
    auto& v = buckets[b];
    std::sort(v.begin(), v.end(), [](uint16_t a, uint16_t c) { return (a >> 4) > (c >> 4); });   // descending j
    for (uint16_t x : v) D->ent[e++] = x;
  }
  for (uint32_t b = (1u << lg::kBucketLog); b < (1u << lg::kBucketLog) + 8; ++b) D->boff[b] = static_cast<uint16_t>(e);
  plan->h_long = D;
  return EPSM_OK;
}

static int grow(void** p, uint64_t& cap, uint64_t want, cudaStream_t s, const char* what) {
  if (want <= cap) return EPSM_OK;
  if (*p) {
    cudaStreamSynchronize(s);
    cudaFree(*p);
    *p = nullptr;
    cap = 0;
  }
  cudaError_t e = cudaMalloc(p, std::max<uint64_t>(want, 256));
  if (e != cudaSuccess) {
    cudaGetLastError();
    *p = nullptr;
    epsm_set_error("cudaMalloc(%s, %llu bytes): %s", what, (unsigned long long)want, cudaGetErrorString(e));
    return EPSM_ENOMEM;
  }
  cap = want;
  return EPSM_OK;
}

int epsm_long_launch(epsm_plan_t* plan, const uint8_t* d_text, uint64_t nbytes, uint64_t nstarts, uint64_t base,
                     uint64_t* d_pos, uint64_t cap, unsigned long long* d_occ, bool search, cudaStream_t s) {
  if (nstarts == 0) {
    cudaError_t e = cudaMemsetAsync(d_occ, 0, sizeof(unsigned long long), s);
    return e == cudaSuccess ? EPSM_OK : epsm_cuda_fail(e, "cudaMemsetAsync(occ)");
  }
  int rc = build_long_desc(plan);
  if (rc) return rc;
  if (!plan->d_long) {
    cudaError_t e = cudaMalloc(&plan->d_long, sizeof(lg::LongDesc));
    if (e != cudaSuccess) {
      plan->d_long = nullptr;
      epsm_set_error("cudaMalloc(long-pattern table): %s", cudaGetErrorString(e));
      return EPSM_ENOMEM;
    }
    e = cudaMemcpyAsync(plan->d_long, plan->h_long, sizeof(lg::LongDesc), cudaMemcpyHostToDevice, s);
    if (e != cudaSuccess) return epsm_cuda_fail(e, "cudaMemcpyAsync(long-pattern table)");
  }
  if (!plan->d_pat) {
    rc = epsm_upload_pattern(plan, s);
    if (rc) return rc;
  }
  const uint64_t mis = reinterpret_cast<uintptr_t>(d_text) & 15u;
  lg::LParams P;
  std::memset(&P, 0, sizeof(P));
  P.text = d_text - mis;
  P.nbytes = nbytes + mis;
  P.s_lo = mis;
  P.s_hi = mis + nstarts;
  P.pos_bias = base - mis;
  P.L = epsm_long_stride(plan->m);
  P.m = plan->m;
  P.nsamples = (P.s_hi - 1 + P.L - 1) / P.L + 1;
  P.nchunks = (P.nsamples + lg::kChunk - 1) / lg::kChunk;
  P.desc = plan->d_long;
  P.dpat = plan->d_pat;
  P.occ = d_occ;
  P.pos = search ? d_pos : nullptr;
  P.cap = (search && d_pos) ? cap : 0;
  epsm_workspace* ws = epsm_get_workspace(plan->device, s);
  if (!ws) return EPSM_ENOMEM;
  if (ws->num_sms <= 0) {
    cudaError_t e = cudaDeviceGetAttribute(&ws->num_sms, cudaDevAttrMultiProcessorCount, plan->device);
    if (e != cudaSuccess) return epsm_cuda_fail(e, "cudaDeviceGetAttribute(SM count)");
  }
  rc = grow(reinterpret_cast<void**>(&ws->l_counts), ws->l_counts_cap, P.nchunks * 4, s, "long-pattern counts");
  if (!rc) rc = grow(reinterpret_cast<void**>(&ws->l_prefix), ws->l_prefix_cap, P.nchunks * 8, s, "long-pattern prefix");
  if (rc) return rc;
  P.counts = ws->l_counts;
  P.prefix = ws->l_prefix;
  const unsigned grid = static_cast<unsigned>(std::min<uint64_t>(P.nchunks, 4ull * ws->num_sms));
  lg::epsm_long_count_kernel<<<grid, lg::kThreads, 0, s>>>(P);
  epsm_count_launch();
  lg::epsm_long_scan_kernel<<<1, 1024, 0, s>>>(P);
  epsm_count_launch();
  if (search && P.cap) {
    lg::epsm_long_write_kernel<<<grid, lg::kThreads, 0, s>>>(P);
    epsm_count_launch();
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return epsm_cuda_fail(e, "long-pattern kernels launch");
  return EPSM_OK;
}
