// epsm_host.cu -- the end-to-end call with HOST buffers for the paper's whole protocol on one
// text: every pattern of every length searched over it (Sec. 4: sets of
// patterns of each length m, "randomly extracted" from the text, timings "including any
// preprocessing").  One call copies the text in, builds the equality-mask index its dense
// searches need (EPSMa's masks), counts, searches every group (one pass per
// group, PAPER.md:18-20 per search) and copies every search's positions back out, the copies of
// group i overlapped with the search of group i + 1 on an internal copy stream.
#include <algorithm>
#include <cstring>
#include <mutex>
#include <new>
#include <vector>

#include "epsm.h"
#include "epsm_internal.h"

namespace {

// Device buffers of the host call, per (device, stream) -- reused across calls, grown on demand.
struct HostSession {
  int device = -1;
  cudaStream_t stream = nullptr;
  cudaStream_t copy = nullptr;
  cudaEvent_t searched[2] = {nullptr, nullptr};   // group's positions complete (compute stream)
  cudaEvent_t drained[2] = {nullptr, nullptr};    // arena copied out (copy stream)
  uint8_t* d_text = nullptr;
  uint64_t text_cap = 0;
  epsm_eqidx_t* index = nullptr;
  uint64_t* arena[2] = {nullptr, nullptr};        // positions of one group (alternating)
  uint64_t arena_cap[2] = {0, 0};                 // words
  uint64_t* d_occ = nullptr;                      // occ of every search of the call
  uint64_t* h_occ = nullptr;                      // pinned copy
  uint64_t occ_cap = 0;
};

std::mutex g_hs_mu;
std::vector<HostSession*> g_hs;

HostSession* get_session(int device, cudaStream_t s) {
  std::lock_guard<std::mutex> lk(g_hs_mu);
  for (HostSession* h : g_hs)
    if (h->device == device && h->stream == s) return h;
  HostSession* h = new (std::nothrow) HostSession();
  if (!h) return nullptr;
  h->device = device;
  h->stream = s;
  g_hs.push_back(h);
  return h;
}

int grow_device(void** p, uint64_t& cap, uint64_t want_bytes, cudaStream_t s, const char* what) {
  if (want_bytes <= cap) return EPSM_OK;
  if (*p) {
    cudaStreamSynchronize(s);
    cudaFree(*p);
    *p = nullptr;
    cap = 0;
  }
  cudaError_t e = cudaMalloc(p, std::max<uint64_t>(want_bytes, 256));
  if (e != cudaSuccess) {
    cudaGetLastError();
    *p = nullptr;
    epsm_set_error("cudaMalloc(%s, %llu bytes): %s", what, (unsigned long long)want_bytes, cudaGetErrorString(e));
    return EPSM_ENOMEM;
  }
  cap = want_bytes;
  return EPSM_OK;
}

}  // namespace

extern "C" {

int epsm_search_text_host(epsm_group_t* const* groups, uint32_t ngroups, const uint8_t* h_text, uint64_t n,
                          uint64_t* const* h_pos, const uint64_t* caps, uint64_t* h_occ, epsm_stream_t stream) {
  if (!groups || ngroups == 0 || !h_occ || (!h_text && n > 0)) {
    epsm_set_error("epsm_search_text_host: NULL groups, h_occ or text, or no group");
    return EPSM_EINVAL;
  }
  if (n > (1ull << 38)) {
    epsm_set_error("n = %llu exceeds 2^38", (unsigned long long)n);
    return EPSM_EINVAL;
  }
  std::vector<uint32_t> first(ngroups + 1, 0);    // search index of each group's first search
  for (uint32_t i = 0; i < ngroups; ++i) {
    if (!groups[i]) {
      epsm_set_error("epsm_search_text_host: groups[%u] is NULL", i);
      return EPSM_EINVAL;
    }
    uint32_t info[5];
    epsm_group_info(groups[i], info, 5);
    first[i + 1] = first[i] + info[1];
  }
  const uint32_t K = first[ngroups];
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return epsm_cuda_fail(e, "cudaGetDevice");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  HostSession* hs = get_session(dev, s);
  if (!hs) return EPSM_ENOMEM;
  if (!hs->copy) {
    e = cudaStreamCreateWithFlags(&hs->copy, cudaStreamNonBlocking);
    for (int a = 0; a < 2 && e == cudaSuccess; ++a) {
      e = cudaEventCreateWithFlags(&hs->searched[a], cudaEventDisableTiming);
      if (e == cudaSuccess) e = cudaEventCreateWithFlags(&hs->drained[a], cudaEventDisableTiming);
    }
    if (e != cudaSuccess) return epsm_cuda_fail(e, "copy stream / events");
  }
  // 1. the text, host -> device
  int rc = grow_device(reinterpret_cast<void**>(&hs->d_text), hs->text_cap, n, s, "text");
  if (rc) return rc;
  if (n) {
    e = cudaMemcpyAsync(hs->d_text, h_text, n, cudaMemcpyHostToDevice, s);
    if (e != cudaSuccess) return epsm_cuda_fail(e, "cudaMemcpyAsync(H2D text)");
  }
  // 2. the equality-mask index over the byte values the groups' dense searches read
  uint8_t vals[256];
  bool have[256] = {};
  uint32_t nv = 0;
  for (uint32_t i = 0; i < ngroups; ++i) {
    uint8_t v[256];
    const int c = epsm_group_index_values(groups[i], v);
    for (int q = 0; q < c; ++q)
      if (!have[v[q]]) {
        have[v[q]] = true;
        vals[nv++] = v[q];
      }
  }
  const epsm_eqidx_t* ix = nullptr;
  if (nv && n) {
    if (!hs->index) {
      rc = epsm_eqidx_create(&hs->index);
      if (rc) return rc;
    }
    rc = epsm_eqidx_build_async(hs->index, hs->d_text, n, vals, nv, stream);
    if (rc) return rc;
    ix = hs->index;
  }
  // 3. every search's occ (sizes the device outputs); one readback
  if (K > hs->occ_cap) {
    if (hs->d_occ) {
      cudaStreamSynchronize(s);
      cudaFree(hs->d_occ);
      cudaFreeHost(hs->h_occ);
      hs->d_occ = hs->h_occ = nullptr;
      hs->occ_cap = 0;
    }
    e = cudaMalloc(&hs->d_occ, K * sizeof(uint64_t));
    if (e == cudaSuccess) e = cudaMallocHost(&hs->h_occ, K * sizeof(uint64_t));
    if (e != cudaSuccess) {
      epsm_set_error("occ buffers: %s", cudaGetErrorString(e));
      return EPSM_ENOMEM;
    }
    hs->occ_cap = K;
  }
  for (uint32_t i = 0; i < ngroups; ++i) {
    rc = epsm_group_count_index_async(groups[i], ix, hs->d_text, n, hs->d_occ + first[i], stream);
    if (rc) return rc;
  }
  e = cudaMemcpyAsync(hs->h_occ, hs->d_occ, K * sizeof(uint64_t), cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return epsm_cuda_fail(e, "occ readback");
  // 4. per group: positions into an arena (two, alternating), then copied out on the copy
  //    stream while the next group searches into the other arena
  std::vector<uint64_t> want(K);
  uint64_t most = 0;
  for (uint32_t i = 0; i < ngroups; ++i) {
    uint64_t t = 0;
    for (uint32_t j = first[i]; j < first[i + 1]; ++j) {
      const uint64_t c = (h_pos && h_pos[j] && caps) ? caps[j] : 0;
      want[j] = std::min<uint64_t>(hs->h_occ[j], c);
      t += want[j];
    }
    most = std::max(most, t);
  }
  const int narena = ngroups > 1 ? 2 : 1;
  for (int a = 0; a < narena; ++a) {
    uint64_t capb = hs->arena_cap[a] * 8;
    rc = grow_device(reinterpret_cast<void**>(&hs->arena[a]), capb, most * 8, s, "position arena");
    hs->arena_cap[a] = capb / 8;
    if (rc) return rc;
  }
  std::vector<uint64_t*> dp;
  std::vector<uint64_t> dc;
  for (uint32_t i = 0; i < ngroups; ++i) {
    const int a = narena == 2 ? static_cast<int>(i & 1u) : 0;
    if (i >= static_cast<uint32_t>(narena)) {
      e = cudaStreamWaitEvent(s, hs->drained[a], 0);       // its previous group is copied out
      if (e != cudaSuccess) return epsm_cuda_fail(e, "cudaStreamWaitEvent(drained)");
    }
    const uint32_t k = first[i + 1] - first[i];
    dp.assign(k, nullptr);
    dc.assign(k, 0);
    uint64_t off = 0;
    for (uint32_t j = 0; j < k; ++j) {
      const uint64_t w = want[first[i] + j];
      if (w) {
        dp[j] = hs->arena[a] + off;
        dc[j] = w;
        off += w;
      }
    }
    rc = epsm_group_search_index_async(groups[i], ix, hs->d_text, n, dp.data(), dc.data(), hs->d_occ + first[i],
                                       stream);
    if (rc) return rc;
    e = cudaEventRecord(hs->searched[a], s);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(hs->copy, hs->searched[a], 0);
    for (uint32_t j = 0; j < k && e == cudaSuccess; ++j)
      if (dc[j])
        e = cudaMemcpyAsync(h_pos[first[i] + j], dp[j], dc[j] * 8, cudaMemcpyDeviceToHost, hs->copy);
    if (e == cudaSuccess) e = cudaEventRecord(hs->drained[a], hs->copy);
    if (e != cudaSuccess) return epsm_cuda_fail(e, "position copies");
  }
  e = cudaStreamSynchronize(hs->copy);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return epsm_cuda_fail(e, "epsm_search_text_host");
  std::memcpy(h_occ, hs->h_occ, K * sizeof(uint64_t));
  return EPSM_OK;
}

}  // extern "C"
