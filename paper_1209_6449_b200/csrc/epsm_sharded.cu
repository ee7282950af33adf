// epsm_sharded.cu -- epsm_search_sharded: data parallelism over the text across
// the GPUs of one node (BASELINE.json north_star: "splits the text across the GPUs
// ... with an (m-1)-byte overlap, each GPU scanning its shard, then gathering
// counts and offsets and allgathering the positions over NVLink with NCCL").
//
// The paper is single-core; sharding is this build's reading R11:
// rank r reports only the starts it owns, [base, base + owned_len), and its shard
// carries the m-1 following bytes so every owned window is local.  The one real
// exchange step is the all-gather of positions (grouped ncclBroadcast, one root
// per rank, each writing its slice at the exclusive prefix of the counts).
//
// NCCL is resolved at run time with dlopen("libnccl.so.2"): inside a PyTorch
// process this returns the copy torch already loaded, so the communicator that
// torch's ProcessGroupNCCL created can be used directly.
#include <dlfcn.h>
#include <mutex>
#include <vector>

#include <nccl.h>

#include "epsm.h"
#include "epsm_internal.h"

namespace {

struct NcclApi {
  bool ok = false;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  ncclResult_t (*CommCount)(const ncclComm_t, int*) = nullptr;
  ncclResult_t (*CommUserRank)(const ncclComm_t, int*) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return;
    api.AllGather = reinterpret_cast<decltype(api.AllGather)>(dlsym(h, "ncclAllGather"));
    api.Broadcast = reinterpret_cast<decltype(api.Broadcast)>(dlsym(h, "ncclBroadcast"));
    api.GroupStart = reinterpret_cast<decltype(api.GroupStart)>(dlsym(h, "ncclGroupStart"));
    api.GroupEnd = reinterpret_cast<decltype(api.GroupEnd)>(dlsym(h, "ncclGroupEnd"));
    api.CommCount = reinterpret_cast<decltype(api.CommCount)>(dlsym(h, "ncclCommCount"));
    api.CommUserRank = reinterpret_cast<decltype(api.CommUserRank)>(dlsym(h, "ncclCommUserRank"));
    api.GetErrorString = reinterpret_cast<decltype(api.GetErrorString)>(dlsym(h, "ncclGetErrorString"));
    api.ok = api.AllGather && api.Broadcast && api.GroupStart && api.GroupEnd && api.CommCount &&
             api.CommUserRank && api.GetErrorString;
  });
  return api;
}

int nccl_fail(ncclResult_t r, const char* what) {
  epsm_set_error("%s: %s", what, nccl().GetErrorString ? nccl().GetErrorString(r) : "NCCL error");
  return EPSM_ENCCL;
}

int grow_scratch(epsm_plan_t* plan, uint64_t want, cudaStream_t s) {
  if (want <= plan->scratch_cap) return EPSM_OK;
  if (plan->d_scratch) {
    cudaStreamSynchronize(s);
    cudaFree(plan->d_scratch);
    plan->d_scratch = nullptr;
    plan->scratch_cap = 0;
  }
  cudaError_t e = cudaMalloc(&plan->d_scratch, want * sizeof(uint64_t));
  if (e != cudaSuccess) {
    epsm_set_error("cudaMalloc(scratch, %llu positions): %s", (unsigned long long)want, cudaGetErrorString(e));
    return EPSM_ENOMEM;
  }
  plan->scratch_cap = want;
  return EPSM_OK;
}

}  // namespace

extern "C" int64_t epsm_search_sharded(epsm_plan_t* plan, const uint8_t* d_shard, uint64_t base,
                                       uint64_t owned_len, uint64_t shard_len, uint64_t n_total,
                                       uint64_t* d_pos, uint64_t cap, void* nccl_comm, epsm_stream_t stream) {
  if (!plan || !nccl_comm || (cap > 0 && !d_pos) || (!d_shard && shard_len > 0)) {
    epsm_set_error("epsm_search_sharded: NULL plan/comm/shard, or d_pos NULL with cap > 0");
    return EPSM_EINVAL;
  }
  if (d_pos && (reinterpret_cast<uintptr_t>(d_pos) & 7u)) {
    epsm_set_error("d_pos must be 8-byte aligned");
    return EPSM_EALIGN;
  }
  if (base > n_total || owned_len > n_total - base) {
    epsm_set_error("owned range [%llu, +%llu) outside the text of %llu bytes", (unsigned long long)base,
                   (unsigned long long)owned_len, (unsigned long long)n_total);
    return EPSM_EINVAL;
  }
  const uint64_t m = plan->m;
  const uint64_t need = owned_len == 0 ? 0 : (owned_len + m - 1 < n_total - base ? owned_len + m - 1 : n_total - base);
  if (shard_len < need) {
    epsm_set_error("shard of %llu bytes is shorter than the owned range plus the (m-1)-byte overlap (%llu)",
                   (unsigned long long)shard_len, (unsigned long long)need);
    return EPSM_EINVAL;
  }
  NcclApi& api = nccl();
  if (!api.ok) {
    epsm_set_error("libnccl.so.2 could not be loaded");
    return EPSM_ENCCL;
  }
  ncclComm_t comm = static_cast<ncclComm_t>(nccl_comm);
  int nranks = 0, rank = 0;
  ncclResult_t nr = api.CommCount(comm, &nranks);
  if (nr != ncclSuccess) return nccl_fail(nr, "ncclCommCount");
  nr = api.CommUserRank(comm, &rank);
  if (nr != ncclSuccess) return nccl_fail(nr, "ncclCommUserRank");

  const void* bind_ptr = d_shard ? static_cast<const void*>(d_shard) : static_cast<const void*>(d_pos);
  int rc = epsm_bind_device(plan, bind_ptr);
  if (rc) return rc;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (plan->counts_cap < nranks + 1) {
    if (plan->d_counts) cudaFree(plan->d_counts);
    if (plan->h_counts) cudaFreeHost(plan->h_counts);
    plan->d_counts = nullptr;
    plan->h_counts = nullptr;
    cudaError_t e = cudaMalloc(&plan->d_counts, (nranks + 1) * sizeof(unsigned long long));
    if (e == cudaSuccess) e = cudaMallocHost(&plan->h_counts, (nranks + 1) * sizeof(unsigned long long));
    if (e != cudaSuccess) {
      epsm_set_error("counts buffers: %s", cudaGetErrorString(e));
      return EPSM_ENOMEM;
    }
    plan->counts_cap = nranks + 1;
  }
  unsigned long long* d_local = plan->d_counts + nranks;

  // 1. local scan of the owned starts into scratch (global positions = local + base)
  uint64_t nstarts = shard_len >= m ? shard_len - m + 1 : 0;
  if (owned_len < nstarts) nstarts = owned_len;
  uint64_t want = cap < nstarts ? cap : nstarts;
  if (want > (1ull << 20)) want = 1ull << 20;   // grow on demand below
  rc = grow_scratch(plan, want ? want : 1, s);
  if (rc) return rc;
  uint64_t local_cap = cap < plan->scratch_cap ? cap : plan->scratch_cap;
  rc = epsm_launch(plan, d_shard, shard_len, nstarts, base, local_cap ? plan->d_scratch : nullptr, local_cap,
                   d_local, true, s);
  if (rc) return rc;
  cudaError_t e = cudaMemcpyAsync(plan->h_counts + nranks, d_local, 8, cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return epsm_cuda_fail(e, "sharded local scan");
  const uint64_t occ_local = plan->h_counts[nranks];
  const uint64_t keep = occ_local < cap ? occ_local : cap;
  if (keep > local_cap) {   // dense shard: grow the scratch once and rescan
    rc = grow_scratch(plan, keep, s);
    if (rc) return rc;
    local_cap = keep;
    rc = epsm_launch(plan, d_shard, shard_len, nstarts, base, plan->d_scratch, local_cap, d_local, true, s);
    if (rc) return rc;
  }

  // 2. all-gather the per-rank counts
  nr = api.AllGather(d_local, plan->d_counts, 1, ncclUint64, comm, s);
  if (nr != ncclSuccess) return nccl_fail(nr, "ncclAllGather(counts)");
  e = cudaMemcpyAsync(plan->h_counts, plan->d_counts, nranks * sizeof(unsigned long long), cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return epsm_cuda_fail(e, "counts readback");
  std::vector<uint64_t> counts(plan->h_counts, plan->h_counts + nranks);
  uint64_t total = 0;
  for (uint64_t c : counts) total += c;

  // 3. all-gather(v) the positions: root q broadcasts its first min(occ_q, cap - off_q)
  if (cap > 0) {
    nr = api.GroupStart();
    if (nr != ncclSuccess) return nccl_fail(nr, "ncclGroupStart");
    uint64_t off = 0;
    for (int q = 0; q < nranks; ++q) {
      const uint64_t room = off < cap ? cap - off : 0;
      const uint64_t cnt = counts[q] < room ? counts[q] : room;
      if (cnt) {
        nr = api.Broadcast(q == rank ? plan->d_scratch : nullptr, d_pos + off, cnt, ncclUint64, q, comm, s);
        if (nr != ncclSuccess) {
          api.GroupEnd();
          return nccl_fail(nr, "ncclBroadcast(positions)");
        }
      }
      off += counts[q];
    }
    nr = api.GroupEnd();
    if (nr != ncclSuccess) return nccl_fail(nr, "ncclGroupEnd");
  }
  e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return epsm_cuda_fail(e, "epsm_search_sharded");
  return static_cast<int64_t>(total);
}

// epsm_allgatherv_async -- the positions exchange of a sharded batch (BASELINE.json north_star:
// "gathering counts and offsets and allgathering the positions over NVLink with NCCL"): for
// every search j, rank q's counts[q * k + j] positions d_local[j] (on rank q) are broadcast into
// every rank's d_out[j] at the exclusive prefix of the counts -- k all-gather(v)s as grouped
// ncclBroadcasts, 64 searches per NCCL group call.
extern "C" int epsm_allgatherv_async(uint32_t k, const uint64_t* const* d_local, const uint64_t* counts,
                                     uint64_t* const* d_out, const uint64_t* caps, void* nccl_comm,
                                     epsm_stream_t stream) {
  if (k == 0) return EPSM_OK;
  if (!d_local || !counts || !d_out || !nccl_comm) {
    epsm_set_error("epsm_allgatherv_async: NULL argument");
    return EPSM_EINVAL;
  }
  NcclApi& api = nccl();
  if (!api.ok) {
    epsm_set_error("libnccl.so.2 could not be loaded");
    return EPSM_ENCCL;
  }
  ncclComm_t comm = static_cast<ncclComm_t>(nccl_comm);
  int nranks = 0, rank = 0;
  ncclResult_t nr = api.CommCount(comm, &nranks);
  if (nr != ncclSuccess) return nccl_fail(nr, "ncclCommCount");
  nr = api.CommUserRank(comm, &rank);
  if (nr != ncclSuccess) return nccl_fail(nr, "ncclCommUserRank");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  constexpr uint32_t kPerGroup = 64;
  for (uint32_t a = 0; a < k; a += kPerGroup) {
    const uint32_t b = a + kPerGroup < k ? a + kPerGroup : k;
    nr = api.GroupStart();
    if (nr != ncclSuccess) return nccl_fail(nr, "ncclGroupStart");
    for (uint32_t j = a; j < b; ++j) {
      const uint64_t cap = caps ? caps[j] : ~0ull;
      uint64_t off = 0;
      for (int q = 0; q < nranks; ++q) {
        const uint64_t c = counts[static_cast<uint64_t>(q) * k + j];
        const uint64_t room = off < cap ? cap - off : 0;
        const uint64_t cnt = c < room ? c : room;
        if (cnt && d_out[j]) {
          nr = api.Broadcast(q == rank ? d_local[j] : nullptr, d_out[j] + off, cnt, ncclUint64, q, comm, s);
          if (nr != ncclSuccess) {
            api.GroupEnd();
            return nccl_fail(nr, "ncclBroadcast(positions)");
          }
        }
        off += c;
      }
    }
    nr = api.GroupEnd();
    if (nr != ncclSuccess) return nccl_fail(nr, "ncclGroupEnd");
  }
  return EPSM_OK;
}
