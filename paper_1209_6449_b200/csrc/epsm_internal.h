// epsm_internal.h -- plan layout and helpers shared by the host translation units.
#pragma once
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

#include "epsm.h"

namespace epsm {
struct JobDesc;
struct XOut;
namespace lg { struct LongDesc; }
namespace mp { struct JobOut; }
}  // namespace epsm

struct epsm_plan_s {
  uint32_t m = 0;
  uint8_t pattern[EPSM_MAX_M_LONG] = {};
  uint32_t* d_pat = nullptr;  // m > 32: zero-padded pattern words in device memory
  epsm::lg::LongDesc* h_long = nullptr;   // m >= 64: EPSMc table at the sampling stride (host)
  epsm::lg::LongDesc* d_long = nullptr;   // ... and its device copy
  epsm::JobDesc* h_desc = nullptr;   // preprocessing (filter words, gram table), host copy
  epsm::JobDesc* d_desc = nullptr;   // ... and its device copy (uploaded on first search)
  int sk = 0, sq = 0;                // sampled-filter geometry (0: packed filter)
  uint32_t bcast[4] = {};   // B_i = p_i * 0x01010101
  uint32_t bcast2[4] = {};  // B_{4+i}: second filter word
  uint32_t pat[9] = {};     // zero-padded pattern words
  uint32_t pmask[9] = {};   // byte masks of the words
  int device = -1;          // bound on first device use
  // (the scan workspace -- look-back status words, chunk counters, parked masks -- belongs
  //  to the (device, stream) the search runs on, see epsm_workspace below)
  // occ readback for the synchronous calls
  unsigned long long* d_occ = nullptr;
  unsigned long long* h_occ = nullptr;
  // epsm_search_host buffers
  uint8_t* d_text_buf = nullptr;
  uint64_t text_cap = 0;
  uint64_t* d_pos_buf = nullptr;
  uint64_t pos_cap = 0;
  // epsm_search_sharded scratch
  uint64_t* d_scratch = nullptr;
  uint64_t scratch_cap = 0;
  unsigned long long* d_counts = nullptr;   // [nranks] + [1] local occ
  unsigned long long* h_counts = nullptr;
  int counts_cap = 0;
};

// Scan workspace of one (device, stream), double-buffered by launch parity so that a search
// may start while the previous one on the stream is still draining (programmatic dependent
// launch): launch L uses parity L & 1 and first waits, on the device, until launch L-2 (the
// previous user of that parity) has retired all its CTAs.
struct epsm_workspace {
  int device = -1;
  cudaStream_t stream = nullptr;
  int num_sms = 0;
  uint64_t launches = 0;                      // launch sequence number of the next launch
  uint64_t status_epoch = 0;                  // epoch (launches >> 24) the status words were
                                              // last cleared in (0: zeroed at allocation)
  unsigned long long* d_status[2] = {nullptr, nullptr};   // one status word per chunk
  uint64_t status_cap = 0;
  uint64_t* d_scratch[2] = {nullptr, nullptr};            // parked masks, per CTA
  uint64_t scratch_ctas = 0;
  unsigned long long* d_ctr = nullptr;        // [parity][kCtrWords]: chunk counter, -, count
                                              // ticket, CTA exit counter, -, per-search counts
  unsigned long long ctr_base[2] = {0, 0};    // chunk counter value at the next launch
  // group search (epsm_multi.cu): per-(chunk, distinct pattern) counts and prefixes, per-chunk
  // occurrence lists, the chunks with occurrences (capacities in bytes)
  uint16_t* m_counts = nullptr;
  uint64_t m_counts_cap = 0;
  unsigned long long* m_prefix = nullptr;
  uint64_t m_prefix_cap = 0;
  uint32_t* m_listlen = nullptr;
  uint64_t m_listlen_cap = 0;
  uint32_t* m_lists = nullptr;
  uint64_t m_lists_cap = 0;
  uint32_t* m_work = nullptr;
  uint64_t m_work_cap = 0;
  epsm::mp::JobOut* m_jobs = nullptr;         // outputs of the searches of a pass
  uint64_t m_jobs_cap = 0;
  uint32_t* l_counts = nullptr;               // long patterns: matches per chunk of samples
  uint64_t l_counts_cap = 0;                  // (bytes)
  unsigned long long* l_prefix = nullptr;     // ... and their exclusive prefix
  uint64_t l_prefix_cap = 0;
  epsm::XOut* d_xout = nullptr;               // fan-out outputs of a batch call (device)
  uint64_t xout_cap = 0;                      // entries
  void* d_repjobs = nullptr;                  // job table of the multi-source fan-out (device)
  uint64_t repjobs_cap = 0;                   // entries
  unsigned long long exit_total[2] = {0, 0};  // CTAs launched so far on each parity
};

epsm_workspace* epsm_get_workspace(int device, cudaStream_t s);

void epsm_set_error(const char* fmt, ...);
int epsm_cuda_fail(cudaError_t e, const char* what);
void epsm_count_launch();   // one more kernel launched by this library (epsm_launch_count)
int epsm_bind_device(epsm_plan_t* plan, const void* dptr);
int epsm_ensure_occ(epsm_plan_t* plan);
int epsm_launch(epsm_plan_t* plan, const uint8_t* d_text, uint64_t nbytes, uint64_t nstarts, uint64_t base,
                uint64_t* d_pos, uint64_t cap, unsigned long long* d_occ, bool search, cudaStream_t s);

// One search of a multi-search launch (all over the same text, same m).  Fan-out: nx further
// outputs (identical patterns of a batch) get the same positions -- x is their device array,
// xh the host copy (for the occ of an empty range), capmax the largest capacity of all.
struct epsm_job {
  epsm_plan_t* plan;
  uint64_t* d_pos;
  uint64_t cap;
  unsigned long long* d_occ;
  const epsm::XOut* x = nullptr;
  const epsm::XOut* xh = nullptr;
  uint32_t nx = 0;
};
// index: run the searches over its equality-mask planes (every plan qualifies), else the text
int epsm_launch_jobs(const epsm_job* jobs, uint32_t k, const uint8_t* d_text, uint64_t nbytes, uint64_t nstarts,
                     uint64_t base, bool search, cudaStream_t s, const epsm_eqidx_t* index = nullptr);

// The batch path (epsm_search_(range_)batch(_index)_async) for k searches whose outputs sit at
// the caller's slots slot[j] of d_pos / caps / d_occ (slot NULL: j); n_total 0 = not a shard.
// fan (optional): fan[j] = further slots of the caller's arrays that receive search j's results
// (their d_pos must have the same 16-byte phase as slot[j]'s)
int epsm_batch_run(epsm_plan_t* const* plans, uint32_t k, const uint32_t* slot, const uint8_t* d_text, uint64_t n,
                   uint64_t owned_len, uint64_t base, uint64_t n_total, uint64_t* const* d_pos, const uint64_t* caps,
                   uint64_t* d_occ, bool search, cudaStream_t s, const epsm_eqidx_t* index,
                   const std::vector<std::vector<uint32_t>>* fan = nullptr);

// Long patterns at EPSMc's sampling stride (epsm_long.cu): m >= kLongStrideMinM
// (stride (floor(m/16) - 1) * 16 >= 192 bytes; a sample costs a 128-byte DRAM line, so below
// that the full-text kernel is faster: B200, 1 GiB, us per search m=144 182 vs 158, m=256 112 vs 158).
constexpr uint32_t kLongStrideMinM = 208;
uint32_t epsm_long_stride(uint32_t m);
bool epsm_long_applies(const epsm_plan_t* plan);
void epsm_long_free(epsm_plan_t* plan);   // the host table (its type is complete only in epsm_long.cu)
int epsm_long_launch(epsm_plan_t* plan, const uint8_t* d_text, uint64_t nbytes, uint64_t nstarts, uint64_t base,
                     uint64_t* d_pos, uint64_t cap, unsigned long long* d_occ, bool search, cudaStream_t s);
int epsm_upload_pattern(epsm_plan_t* plan, cudaStream_t s);
// occ and the first min(occ, cap_o) positions of d_pos (capacity cap) to nx further outputs x
// (device XOut table), on stream s
int epsm_replicate(const uint64_t* d_pos, uint64_t cap, const unsigned long long* d_occ, const epsm::XOut* x,
                   uint32_t nx, bool search, cudaStream_t s, epsm_workspace* ws);
// Many fan-outs at once: request r copies source pos[r] (capacity cap[r], occ occ[r]) to the
// outputs d_x[x0 .. x0 + nx) (device table; h_x: the same table on the host, for the alignment
// check).  Sources and outputs in the 16-byte phase go through one launch, the rest one by one.
struct epsm_rep_req {
  const uint64_t* pos;
  uint64_t cap;
  const unsigned long long* occ;
  uint32_t x0, nx;
};
int epsm_replicate_many(const epsm_rep_req* r, uint32_t nr, const epsm::XOut* d_x, const epsm::XOut* h_x, bool search,
                        cudaStream_t s, epsm_workspace* ws);

// Equality-mask index of one text (epsm_eqidx_build_async).
struct epsm_eqidx_s {
  int device = -1;
  const uint8_t* text = nullptr;     // the text the planes were built over
  uint64_t n = 0;
  uint32_t nv = 0;
  uint8_t vals[EPSM_MAX_PLANES] = {};
  int16_t plane_of[256] = {};        // plane of a byte value, -1 if absent
  uint64_t* d_planes = nullptr;      // nv planes of pstride words
  uint64_t pstride = 0;
  uint64_t cap_words = 0;            // allocated words
};
