/*
 * epsm.h -- C ABI of the B200-native exact packed string matcher.
 *
 * Operation (Sec. 1): given a byte text t[0..n-1] and a pattern
 * p[0..m-1] (Sec. 2), report *all* occurrences of p in t:
 *
 *     Occ(p, t) = { s : 0 <= s <= n-m and t[s+j] = p[j] for all 0 <= j < m }
 *
 * as strictly increasing uint64 start offsets, overlapping occurrences included.
 * EPSM's procedures (EPSMa/b, Sec. 3.2-3.3) filter with a packed
 * compare of alpha = 16 alignments per 128-bit word and then "naively check"
 * candidates; every entry point here returns exactly Occ(p, t).
 * Readings where the paper is silent are listed in DESIGN.md (R1-R16).
 *
 * Conventions shared by every call
 * --------------------------------
 *  - Return value: >= 0 is success (an occurrence count where the call returns
 *    one); < 0 is one of the EPSM_E* codes below.  epsm_strerror() names a code,
 *    epsm_last_error() gives the calling thread's last detailed message.
 *  - Device pointers (d_*) are caller-owned CUDA global memory on the current
 *    device; the library never frees them.  d_text may have any alignment; it is
 *    read only in [d_text, d_text + n) (plus, at most, the bytes of the 16-byte
 *    aligned blocks that contain its first and last byte).  d_pos and d_occ
 *    must be 8-byte aligned.
 *  - Positions are written as uint64 in ascending order.  With cap < occ only
 *    the cap smallest positions are written and the full occ is still returned
 *    (snprintf-style), so a caller can resize and retry.  cap = 0 behaves like a
 *    count and d_pos may then be NULL.
 *  - stream is a cudaStream_t (NULL = the legacy default stream).  All device
 *    work is enqueued on it.  The *_async calls return without synchronising;
 *    the others end with one cudaStreamSynchronize(stream).
 *  - A plan holds the preprocessed pattern (a ~8 KiB device descriptor, uploaded
 *    on its first search) and an 8-byte occ slot for the synchronous calls.  The
 *    scan workspace (look-back status words, 8 bytes per 128 KiB chunk of text,
 *    and parked match masks, 128 KiB per SM) belongs to the (device, stream) a
 *    search is enqueued on, double-buffered by launch so that consecutive
 *    searches on a stream overlap; it is allocated on first use and grows (with a
 *    stream synchronisation) when a larger text needs it.  Calls on one stream
 *    must come from one host thread at a time; the synchronous calls of one plan
 *    must not run concurrently.  Plans are bound to the device of their first
 *    search.
 *  - Maximum n: 2^38 bytes (256 GiB) per call.
 */
#ifndef EPSM_H
#define EPSM_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define EPSM_OK       0
#define EPSM_EINVAL  (-1)   /* NULL argument, m = 0, d_pos NULL with cap > 0, n too large */
#define EPSM_EUNSUP  (-2)   /* m > EPSM_MAX_M_LONG                                        */
#define EPSM_EALIGN  (-3)   /* d_pos or d_occ not 8-byte aligned                          */
#define EPSM_ECUDA   (-4)   /* a CUDA runtime call or kernel launch failed                */
#define EPSM_ENCCL   (-5)   /* NCCL missing or an NCCL call failed (sharded search)       */
#define EPSM_ENOMEM  (-6)   /* device or pinned-host allocation failed                    */

#define EPSM_MAX_M   32u     /* short patterns: the packed / sampled filters of Sec. 3.2-3.4   */
#define EPSM_MAX_M_LONG 4096u /* long patterns (EPSMc block fingerprints)  */

typedef struct epsm_plan_s epsm_plan_t;   /* opaque, host-owned */
typedef struct epsm_eqidx_s epsm_eqidx_t; /* opaque, host-owned (equality-mask index) */
#define EPSM_MAX_PLANES 256u /* byte values one equality-mask index holds (all of them)    */
#define EPSM_INDEX_MAX_D 8u  /* distinct pattern bytes a search over an index may have     */
typedef void *epsm_stream_t;              /* a cudaStream_t     */

/*
 * epsm_plan -- preprocessing (Sec. 3.2: B[i] = (p_i)^alpha for
 * i < m' = min(m, 4); Sec. 3.3: the filter prefix p'; dispatch by m,
 * PAPER.md:150-152).  Copies pattern[0..m-1] (1 <= m <= EPSM_MAX_M_LONG) into a
 * new plan, builds the broadcast words and selects the kernel variant for m
 * (m > 32: EPSMc's sampled block fingerprints with the naive check of each
 * candidate against the pattern in device memory, PAPER.md:576-603 -- for
 * m >= 208 at EPSMc's own stride, one 16-byte block every (floor(m/16) - 1) * 16
 * text bytes, so only part of the text is read; the plan
 * uploads the pattern and its block table on its first search).  No device work.  *out receives the
 * plan (caller frees with epsm_plan_free).
 * Returns EPSM_OK, EPSM_EINVAL (NULL pattern/out, m = 0) or EPSM_EUNSUP
 * (m > EPSM_MAX_M_LONG).
 */
int epsm_plan(const uint8_t *pattern, uint32_t m, epsm_plan_t **out);

/* epsm_plan_free -- release a plan and its device memory.  NULL-safe.
 * Synchronises the plan's device before freeing device memory. */
void epsm_plan_free(epsm_plan_t *plan);

/* epsm_plan_m -- the pattern length a plan was built for (0 for NULL). */
uint32_t epsm_plan_m(const epsm_plan_t *plan);

/*
 * epsm_count -- occ = |Occ(p, t)| (the popcount of every match mask,
 * PAPER.md:437-439, Sec. 3.1.5) for the device text d_text[0..n-1].
 * Returns occ >= 0 or a negative error.  Synchronises stream.
 */
int64_t epsm_count(epsm_plan_t *plan, const uint8_t *d_text, uint64_t n,
                   epsm_stream_t stream);

/* epsm_count_async -- as epsm_count, but leaves occ in the device uint64
 * *d_occ and does not synchronise.  Returns EPSM_OK or a negative error. */
int epsm_count_async(epsm_plan_t *plan, const uint8_t *d_text, uint64_t n,
                     uint64_t *d_occ, epsm_stream_t stream);

/*
 * epsm_search -- report Occ(p, t) (the occurrences at i*alpha + {r} of
 * PAPER.md:470 and Fig. 1, in block order) for the device text
 * d_text[0..n-1] into d_pos[0 .. min(occ, cap)), ascending.  One pass over the
 * text; tiles are ordered by a single-pass decoupled look-back scan.
 * Returns occ >= 0 or a negative error.  Synchronises stream.
 */
int64_t epsm_search(epsm_plan_t *plan, const uint8_t *d_text, uint64_t n,
                    uint64_t *d_pos, uint64_t cap, epsm_stream_t stream);

/* epsm_search_async -- as epsm_search, but leaves occ in the device uint64
 * *d_occ (required, 8-byte aligned) and does not synchronise. */
int epsm_search_async(epsm_plan_t *plan, const uint8_t *d_text, uint64_t n,
                      uint64_t *d_pos, uint64_t cap, uint64_t *d_occ,
                      epsm_stream_t stream);

/*
 * epsm_search_batch_async -- k searches over ONE device text d_text[0..n-1] (the
 * paper's protocol: many patterns per text), as epsm_search_async
 * for each j: positions of plans[j] into d_pos[j][0 .. min(occ_j, caps[j])), occ_j
 * into the device uint64 d_occ[j] (d_occ: k contiguous, 8-byte aligned words).
 * d_pos may be NULL (or d_pos[j] NULL / caps NULL) to count only.  The searches
 * are grouped by kernel variant (pattern length and filter) and each group runs
 * as persistent launches of up to 40 searches: the grid streams the text once
 * per search, back to back, without a launch boundary between them.  Returns
 * EPSM_OK or a negative error; does not synchronise.
 */
int epsm_search_batch_async(epsm_plan_t *const *plans, uint32_t k,
                            const uint8_t *d_text, uint64_t n,
                            uint64_t *const *d_pos, const uint64_t *caps,
                            uint64_t *d_occ, epsm_stream_t stream);

/* epsm_count_batch_async -- as epsm_search_batch_async with no positions: the count
 * kernel (popcounts only) for k patterns over one text; occ_j
 * into d_occ[j].  Does not synchronise. */
int epsm_count_batch_async(epsm_plan_t *const *plans, uint32_t k,
                           const uint8_t *d_text, uint64_t n, uint64_t *d_occ,
                           epsm_stream_t stream);

/*
 * Equality-mask index of a text (EPSMa).  EPSMa compares a text
 * block with the broadcast pattern bytes (wscmp) and combines the masks by
 * shift-AND.  For a batch of searches over ONE text (the paper's protocol,
 * PAPER.md:630-632) the masks depend only on (text, byte value), so the index
 * computes them once: plane v holds bit i of word w = [t[64w + i] == v] (bits
 * past n zero), nv planes of (ceil(n / 32768) * 512 + 2) uint64 words in device
 * memory owned by the index.  A search whose distinct pattern bytes are all in
 * the index and that qualifies (epsm_plan_index_values > 0) then streams only
 * its d planes (d/8 bytes per text byte) and runs the shift-AND on them;
 * results are identical to the text path.
 *
 * epsm_eqidx_create -- an empty index (no device memory yet).  Returns EPSM_OK,
 *   EPSM_EINVAL (NULL out) or EPSM_ENOMEM.
 * epsm_eqidx_free -- release the index and its planes (synchronises the device
 *   first).  NULL-safe.
 * epsm_eqidx_build_async -- (re)build the planes of d_text[0..n-1] for the
 *   distinct byte values values[0..nv-1] (1 <= nv <= EPSM_MAX_PLANES) on stream
 *   (ordered before later work on that stream).  d_text must be 16-byte aligned
 *   (EPSM_EALIGN otherwise).  The index remembers (d_text, n): searches name the
 *   same text.  Growing the planes re-allocates (synchronises the stream).
 *   Searches on other streams that read the planes must be ordered before a
 *   rebuild by the caller (events), as for any buffer shared across streams.
 *   Returns EPSM_OK or EPSM_EINVAL (NULL, nv out of range, duplicate values,
 *   n > 2^38), EPSM_EALIGN, EPSM_ENOMEM, EPSM_ECUDA.
 * epsm_eqidx_values -- the values the index holds: writes up to 256 bytes into
 *   out_values and returns nv (0 before the first build).
 */
int epsm_eqidx_create(epsm_eqidx_t **out);
void epsm_eqidx_free(epsm_eqidx_t *index);
int epsm_eqidx_build_async(epsm_eqidx_t *index, const uint8_t *d_text, uint64_t n,
                           const uint8_t *values, uint32_t nv, epsm_stream_t stream);
int epsm_eqidx_values(const epsm_eqidx_t *index, uint8_t *out_values);

/* epsm_plan_index_values -- the byte values a search with this plan would read
 * from an index: writes its d <= EPSM_INDEX_MAX_D distinct pattern bytes (in order
 * of first occurrence) into out_values and returns d, or returns 0 if the plan
 * never runs over an index (m > 31, more than 4 distinct bytes at 9 <= m <= 31,
 * or more than EPSM_INDEX_MAX_D; there the text kernels are faster). */
int epsm_plan_index_values(const epsm_plan_t *plan, uint8_t *out_values);

/*
 * epsm_search_batch_index_async -- as epsm_search_batch_async over d_text[0..n-1]
 * (which must be the text `index` was last built over: same pointer and n,
 * EPSM_EINVAL otherwise), with every search that qualifies (see above) run over
 * the index's planes; the others take the text kernels.  index may be NULL
 * (then identical to epsm_search_batch_async).  Does not synchronise.
 */
int epsm_search_batch_index_async(epsm_plan_t *const *plans, uint32_t k,
                                  const epsm_eqidx_t *index,
                                  const uint8_t *d_text, uint64_t n,
                                  uint64_t *const *d_pos, const uint64_t *caps,
                                  uint64_t *d_occ, epsm_stream_t stream);

/* epsm_search_range_batch_index_async -- the local step of a sharded batch
 * (epsm_search_range_batch_async) with the qualifying searches run over `index`,
 * built over this rank's shard d_text[0..n-1] (same pointer and n). */
int epsm_search_range_batch_index_async(epsm_plan_t *const *plans, uint32_t k,
                                        const epsm_eqidx_t *index,
                                        const uint8_t *d_text, uint64_t n,
                                        uint64_t owned_len, uint64_t base,
                                        uint64_t n_total,
                                        uint64_t *const *d_pos, const uint64_t *caps,
                                        uint64_t *d_occ, epsm_stream_t stream);

/* epsm_count_batch_index_async -- as epsm_count_batch_async (counts only, the
 * count kernel) with the qualifying searches run over the index's planes. */
int epsm_count_batch_index_async(epsm_plan_t *const *plans, uint32_t k,
                                 const epsm_eqidx_t *index,
                                 const uint8_t *d_text, uint64_t n, uint64_t *d_occ,
                                 epsm_stream_t stream);

/*
 * epsm_search_range_batch_async -- the local step of a sharded batch: as
 * epsm_search_batch_async over the shard d_text[0..n-1], reporting only starts
 * s < owned_len, each as s + base (the rank's global offset).  The global text
 * has n_total bytes: base + owned_len <= n_total, and for every plan the shard
 * must hold the (m-1)-byte overlap, n >= min(owned_len + m - 1, n_total - base)
 * (EPSM_EINVAL otherwise: an owned start whose window runs past the shard would
 * be silently dropped).  With the per-rank counts exchanged (every rank learns
 * each search's global occ and its own offset), the union of the ranks' outputs
 * is each search's Occ, in rank order.
 */
int epsm_search_range_batch_async(epsm_plan_t *const *plans, uint32_t k,
                                  const uint8_t *d_text, uint64_t n,
                                  uint64_t owned_len, uint64_t base,
                                  uint64_t n_total,
                                  uint64_t *const *d_pos, const uint64_t *caps,
                                  uint64_t *d_occ, epsm_stream_t stream);

/*
 * epsm_search_host -- end-to-end convenience: h_text[0..n-1] and h_pos are HOST
 * buffers (pinned memory gives full PCIe bandwidth; pageable works).  Copies
 * the text to a plan-owned device buffer, runs epsm_search, and copies the
 * first min(occ, cap) positions back into h_pos.  Returns occ or an error.
 */
int64_t epsm_search_host(epsm_plan_t *plan, const uint8_t *h_text, uint64_t n,
                         uint64_t *h_pos, uint64_t cap, epsm_stream_t stream);

/*
 * epsm_search_sharded -- collective over the NCCL communicator nccl_comm
 * (an ncclComm_t; every rank calls it with a plan for the same pattern).
 * The global text has n_total bytes.  This rank's buffer d_shard holds global
 * bytes [base, base + shard_len) and the rank OWNS the starts
 * [base, base + owned_len); shard_len must be >= min(owned_len + m - 1,
 * n_total - base) so that every owned window is inside the shard (the
 * (m-1)-byte overlap).  Owned ranges of the ranks must partition [0, n_total).
 * Each rank scans only its shard, the per-rank counts are all-gathered, and
 * the positions are all-gathered (grouped ncclBroadcast, one root per rank) so
 * that every rank's d_pos receives the first min(occ, cap) GLOBAL positions,
 * ascending.  Returns the global occ on every rank, or a negative error.
 * NCCL is loaded at run time (libnccl.so.2, the copy PyTorch already loaded).
 * Synchronises stream.
 */
int64_t epsm_search_sharded(epsm_plan_t *plan, const uint8_t *d_shard,
                            uint64_t base, uint64_t owned_len,
                            uint64_t shard_len, uint64_t n_total,
                            uint64_t *d_pos, uint64_t cap, void *nccl_comm,
                            epsm_stream_t stream);

/*
 * epsm_allgatherv_async -- the positions exchange of a sharded batch of k searches
 * (collective over the NCCL communicator nccl_comm; every rank calls it with the same
 * k, counts and caps).  counts is a HOST array [nranks][k]: counts[q*k + j] = rank q's
 * occurrences of search j (from a counts exchange, e.g. the all-gather of the
 * per-rank d_occ of epsm_search_range_batch_async / epsm_group_search_range_async).
 * d_local[j] holds this rank's GLOBAL positions of search j (device); every rank's
 * d_out[j] (device) receives the first min(occ_j, caps[j]) global positions
 * (occ_j = sum over q; caps NULL: no limit), rank 0's first, so ascending.  Grouped
 * ncclBroadcasts, one root per rank and search.  Enqueued on stream; does not
 * synchronise.  Returns EPSM_OK, EPSM_EINVAL or EPSM_ENCCL.
 */
int epsm_allgatherv_async(uint32_t k, const uint64_t *const *d_local,
                          const uint64_t *counts, uint64_t *const *d_out,
                          const uint64_t *caps, void *nccl_comm, epsm_stream_t stream);

/*
 * epsm_search_range_async -- the local step of the sharded search, exposed so
 * that a host runtime (e.g. torch.distributed) can do the exchange itself:
 * scans d_shard[0..shard_len-1], reports only starts s < owned_len, and writes
 * s + base into d_pos (first min(occ_local, cap)); occ_local goes to *d_occ.
 * n_total is the global text length; the shard must hold the overlap,
 * shard_len >= min(owned_len + m - 1, n_total - base), else EPSM_EINVAL.
 */
int epsm_search_range_async(epsm_plan_t *plan, const uint8_t *d_shard,
                            uint64_t shard_len, uint64_t owned_len,
                            uint64_t base, uint64_t n_total,
                            uint64_t *d_pos, uint64_t cap,
                            uint64_t *d_occ, epsm_stream_t stream);

/*
 * Group search: k searches of one pattern length m over one text in ONE pass.
 * The paper's protocol searches sets of 1000 patterns of fixed length m, randomly
 * extracted from each text (Sec. 4); every search of a group
 * returns exactly its own Occ(p_j, t), as if searched alone, but
 * the text is streamed once for the group: identical patterns are searched once,
 * and the distinct ones share one EPSMc-style table of sampled q-grams
 * (Fig. 1 lines 1-12: one table lookup per sample names
 * candidate (start, pattern) pairs, each naively checked).
 */
typedef struct epsm_group_s epsm_group_t;   /* opaque, host-owned */

/*
 * epsm_group_create -- preprocess k patterns of length m (1 <= m <= EPSM_MAX_M,
 * 1 <= k <= 1024) stored back to back in patterns[0 .. k*m).  Search j of the
 * group is pattern j.  Copies the patterns; no device work (the group's tables
 * are uploaded on first use, to the device of that call).  More than 255
 * distinct patterns are split internally into passes of <= 255.
 * Dense patterns -- an expected rate of >= 2^-7 occurrences per text byte, the
 * product of their bytes' frequencies among the k patterns (which are extracted
 * from the text) -- are searched one by one through the
 * single-pattern kernels (and over an index where one is passed and the search
 * qualifies): their positions, not the text, dominate the traffic.  The
 * environment variable EPSM_GROUP_DENSE=L moves the threshold to 2^-L (0: every
 * pattern shares the passes).  Results never depend on the split.
 * Returns EPSM_OK, EPSM_EINVAL (NULL argument, m = 0, k = 0), EPSM_EUNSUP
 * (m > 32 or k > 1024) or EPSM_ENOMEM.
 */
int epsm_group_create(const uint8_t *patterns, uint32_t m, uint32_t k,
                      epsm_group_t **out);

/* epsm_group_free -- release a group (synchronises its device first). NULL-safe. */
void epsm_group_free(epsm_group_t *g);

/* epsm_group_set_dense -- tuning / test hook: re-split the group with the dense
 * threshold 2^-log2_rate occurrences per text byte (0: no pattern is dense, every
 * one shares the passes).  Synchronises the group's device if it was used.
 * Returns EPSM_OK or EPSM_EINVAL (NULL, log2_rate > 64). */
int epsm_group_set_dense(epsm_group_t *g, uint32_t log2_rate);

/* epsm_group_dense_searches -- which searches of the group are searched one by one
 * (dense patterns): flags[j] = 1 for those, 0 for the shared passes (flags: k bytes,
 * may be NULL).  Returns their number, or EPSM_EINVAL for NULL g. */
int epsm_group_dense_searches(const epsm_group_t *g, uint8_t *flags);

/* epsm_group_index_values -- the byte values an equality-mask index needs for the
 * group's dense searches to run over it: writes up to 256 distinct values into
 * out_values (may be NULL) and returns their number (0: none qualifies, or NULL). */
int epsm_group_index_values(const epsm_group_t *g, uint8_t *out_values);

/* epsm_group_info -- diagnostics: writes min(nout, 5 + 2*P) values
 * [m, k, distinct patterns, dense distinct patterns (searched one by one),
 * passes P, then (q, SK) per pass: the sampled gram length and stride] to out
 * and returns 5 + 2*P (EPSM_EINVAL on NULL). */
int epsm_group_info(const epsm_group_t *g, uint32_t *out, uint32_t nout);

/* epsm_group_set_geometry -- tuning / test hook: use sampled q-grams (1 <= q <=
 * min(m, 16)) every SK bytes (SK in {1, 2, 4, 8, 16}, SK + q - 1 <= m, SK times
 * the distinct patterns of a pass <= 4096) instead of the cost model's choice,
 * for EVERY distinct pattern (dense ones included: none is searched one by one
 * afterwards).  Every geometry returns the same results.  Synchronises the group's device if
 * it was used.  Returns EPSM_OK or EPSM_EINVAL. */
int epsm_group_set_geometry(epsm_group_t *g, uint32_t q, uint32_t sk);

/*
 * epsm_group_search_async -- all k searches of the group over d_text[0..n-1]
 * (any alignment): search j writes its first min(occ_j, caps[j]) positions,
 * ascending, to the device array d_pos[j] (d_pos[j] may be NULL, or d_pos
 * itself NULL: counts only) and occ_j to d_occ[j] (device, k entries, 8-byte
 * aligned).  Scratch (per-chunk counts, prefixes and occurrence lists, ~1/30 of
 * n bytes) belongs to the (device, stream) workspace.  Does not synchronise.
 */
int epsm_group_search_async(epsm_group_t *g, const uint8_t *d_text, uint64_t n,
                            uint64_t *const *d_pos, const uint64_t *caps,
                            uint64_t *d_occ, epsm_stream_t stream);

/* epsm_group_count_async -- occ_j of every search into d_occ[j] (no positions). */
int epsm_group_count_async(epsm_group_t *g, const uint8_t *d_text, uint64_t n,
                           uint64_t *d_occ, epsm_stream_t stream);

/* epsm_group_search_index_async / epsm_group_count_index_async -- as the calls
 * above, with the dense patterns' searches run over the equality-mask index
 * `index` where they qualify (epsm_search_batch_index_async); index must have been
 * built over the same d_text and n (EPSM_EINVAL otherwise) and may be NULL. */
int epsm_group_search_index_async(epsm_group_t *g, const epsm_eqidx_t *index,
                                  const uint8_t *d_text, uint64_t n,
                                  uint64_t *const *d_pos, const uint64_t *caps,
                                  uint64_t *d_occ, epsm_stream_t stream);
int epsm_group_count_index_async(epsm_group_t *g, const epsm_eqidx_t *index,
                                 const uint8_t *d_text, uint64_t n,
                                 uint64_t *d_occ, epsm_stream_t stream);

/* epsm_group_search_range_async -- the local step of a sharded group search: as
 * epsm_search_range_batch_async (starts s < owned_len of the shard, reported as
 * s + base; shard_len >= min(owned_len + m - 1, n_total - base), else
 * EPSM_EINVAL) for every search of the group in one pass. */
int epsm_group_search_range_async(epsm_group_t *g, const uint8_t *d_shard,
                                  uint64_t shard_len, uint64_t owned_len,
                                  uint64_t base, uint64_t n_total,
                                  uint64_t *const *d_pos, const uint64_t *caps,
                                  uint64_t *d_occ, epsm_stream_t stream);

/* epsm_group_search_range_index_async -- the same with a shard's index (built over
 * d_shard[0..shard_len-1]) for the dense patterns' searches. */
int epsm_group_search_range_index_async(epsm_group_t *g, const epsm_eqidx_t *index,
                                        const uint8_t *d_shard, uint64_t shard_len,
                                        uint64_t owned_len, uint64_t base,
                                        uint64_t n_total, uint64_t *const *d_pos,
                                        const uint64_t *caps, uint64_t *d_occ,
                                        epsm_stream_t stream);

/*
 * epsm_search_text_host -- end to end over a HOST text, the paper's protocol for one
 * text (sets of patterns of each length, timings including the
 * preprocessing): copies h_text[0..n-1] to the device, builds the equality-mask index
 * the groups' dense searches need (epsm_group_index_values), counts every search,
 * runs every group (epsm_group_search_index_async) and copies each search's first
 * min(occ, caps[j]) positions into the HOST array h_pos[j] (pinned memory gives full
 * PCIe bandwidth; h_pos or h_pos[j] NULL, or caps NULL: count only).  Search j
 * numbers the searches of groups[0], then groups[1], ...; its occ goes to h_occ[j].
 * Device buffers (text, index, two position arenas of the largest group's output,
 * occ) belong to the calling (device, stream) and are reused by later calls; the
 * copies of group i overlap the search of group i + 1 on an internal stream.
 * Synchronises.  Returns EPSM_OK or a negative error.
 */
int epsm_search_text_host(epsm_group_t *const *groups, uint32_t ngroups,
                          const uint8_t *h_text, uint64_t n,
                          uint64_t *const *h_pos, const uint64_t *caps,
                          uint64_t *h_occ, epsm_stream_t stream);

/* epsm_strerror -- static name/description of an EPSM_E* code. */
const char *epsm_strerror(int64_t code);

/* epsm_last_error -- the calling thread's last detailed error message ("" if none). */
const char *epsm_last_error(void);

/* epsm_launch_count -- number of CUDA kernels this library has launched in the
 * process so far (all plans, all threads); used by benchmarks to report how many
 * of the library's kernels ran in a timed region. */
uint64_t epsm_launch_count(void);

/* epsm_ktimer_enable -- benchmark instrumentation of the dominant kernel (the
 * positions fan-out, epsm_replicate_multi_kernel: DESIGN.md section 6).  While on
 * (on != 0), every launch of that kernel is bracketed by two CUDA events recorded on
 * the stream it is launched on, and its jobs (source occ pointer and capacity, the
 * outputs' capacities) are kept on the host.  Off by default; returns EPSM_OK. */
int epsm_ktimer_enable(int on);

/* epsm_ktimer_read -- waits for the recorded launches, then returns (each pointer may
 * be NULL) their number, the sum of their event-timed durations in ms, and their
 * algorithmic bytes: per job 8 * min(occ, cap) read once plus 8 * min(occ, cap_o)
 * written per output o, occ read back from the device occ each job names (so those
 * buffers must still be alive).  Clears the records.  EPSM_ECUDA on a CUDA error. */
int epsm_ktimer_read(uint64_t *launches, double *ms, double *bytes);

/* epsm_version -- ABI version (major * 10000 + minor * 100 + patch). */
int epsm_version(void);

/*
 * epsm_debug_trace -- diagnostics only.  When the process was started with
 * EPSM_TRACE=<slots>, every kernel launch records a per-CTA timeline of
 * %globaltimer stamps (8 uint64 per CTA: start, first TMA issued, first tile
 * ready, producer done, consumers done, drain done, CTA done, chunks) into slot
 * (launch index mod slots) of a device buffer of 8192 words per slot.  Copies
 * min(max_words, slots * 8192) words into the HOST buffer h_out (synchronises
 * the device) and returns the count; 0 when tracing is off.
 */
int64_t epsm_debug_trace(uint64_t *h_out, uint64_t max_words);

#ifdef __cplusplus
}
#endif
#endif /* EPSM_H */
