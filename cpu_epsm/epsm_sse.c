/*
 * epsm_sse.c -- the paper's own method on the host CPU: EPSM with SSE4.2.
 *
 * A second HOST BASELINE beside the brute-force oracle, not the oracle and not the product:
 * it puts the paper's x86 design on the GPU box's cores.  It shares no code with the CUDA
 * path (paper_1209_6449_b200/) or with the oracle (oracle/); tests compare it with the
 * oracle, bench.py times it.
 *
 * Followed step by step from PAPER.md (Fig. 1):
 *   EPSMa (Fig. 1 top)    m < 4:  B[j] = (p_j)^16 (lines 1-4); per block T_i
 *       s_j = wscmp(T_i, B[j]) = movemask(cmpeq_epi8), r = s_0 & (s_1 >> 1) & ...
 *       (LSB = offset 0, DESIGN R10), report i*16 + {r} (line 11); the m'-1 starts that
 *       cross into T_{i+1} are naively checked (lines 13-14; DESIGN R-c9: the starts
 *       (i+1)*16 - m' + 1 .. (i+1)*16 - 1).
 *   EPSMb (Fig. 1 middle) 4 <= m < 32: r = wsmatch(T_i, p') with the emulation
 *       mpsadbw + compare-with-zero + movemask -- the SAD of the 4-byte prefix at
 *       offsets 0..7; compared per 16-bit lane (the printed cmpeq_epi8 is garbled);
 *       then S = wsblend(T_i, T_{i+1}) = T_i[8..15] T_{i+1}[0..7] (emulated with
 *       blend_epi16 + shuffle_epi32) for offsets 8..15 (lines 9-14);
 *       every candidate is naively checked against the whole pattern (line 8).
 *   EPSMc (Fig. 1 bottom) m >= 32: h(a) = wscrc(a) & (2^11 - 1), with
 *       wscrc = _mm_crc32_u64 over the block's two 64-bit halves, low half first (P:423-428,
 *       SURVEY c14); L[v] = the offsets j of the pattern's 16-byte substrings with h = v
 *       (lines 1-5); the text is inspected one block every sh = (floor(m/16) - 1) * 16 bytes
 *       (line 6) and every listed start x - j is naively checked (lines 8-12).
 *
 * Readings: dispatch m < 4 / 4 <= m < 32 / m >= 32 -- EPSMc needs one
 * whole aligned 16-byte block inside every window, which holds for m >= 31 (P:152's m >= 16
 * gives sh = 0); the table holds offsets j = 0 .. sh - 1 (every start is
 * examined exactly once, through the first inspected block at or after it), so positions
 * are produced in ascending order without duplicates; blocks past the last whole
 * one are handled by the naive check (the paper is silent on n mod 16).
 *
 * Positions: first min(occ, cap) written to pos (may be NULL with cap = 0); returns occ,
 * or -1 for m = 0.  Compile with -O2 -msse4.2 -mpopcnt.
 */
#include <nmmintrin.h>
#include <smmintrin.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
  uint64_t *pos;
  uint64_t cap;
  uint64_t occ;
} sink_t;

static inline void report(sink_t *o, uint64_t s) {
  if (o->occ < o->cap) o->pos[o->occ] = s;
  o->occ++;
}

/* the naive check */
static inline int check(const uint8_t *t, uint64_t n, uint64_t s, const uint8_t *p, uint32_t m) {
  if (s + m > n) return 0;
  for (uint32_t j = 0; j < m; ++j)
    if (t[s + j] != p[j]) return 0;
  return 1;
}

static inline __m128i load16(const uint8_t *t, uint64_t off) {
  return _mm_loadu_si128((const __m128i *)(t + off));
}

/* ---------------------------------------------------------------------------- EPSMa */
static void epsm_a(const uint8_t *p, uint32_t m, const uint8_t *t, uint64_t n, sink_t *o) {
  const uint32_t mp = m < 8 ? m : 8; /* m' = min(m, alpha/2); m < 4 here, so m' = m */
  __m128i B[8];
  for (uint32_t j = 0; j < mp; ++j) B[j] = _mm_set1_epi8((char)p[j]); /* lines 1-4 */
  const uint64_t nb = n / 16;
  for (uint64_t i = 0; i < nb; ++i) {
    const __m128i T = load16(t, 16 * i);
    uint32_t r = 0xFFFFu;                                             /* line 6 */
    for (uint32_t j = 0; j < mp; ++j) {
      const uint32_t s = (uint32_t)_mm_movemask_epi8(_mm_cmpeq_epi8(T, B[j])); /* wscmp */
      r &= s >> j;                                                    /* line 9 */
    }
    r &= 0xFFFFu >> (mp - 1);         /* starts whose prefix lies inside T_i */
    while (r) {                       /* lines 10-12: report / check i*16 + {r} */
      const uint32_t k = (uint32_t)__builtin_ctz(r);
      r &= r - 1;
      const uint64_t s = 16 * i + k;
      if (mp == m ? s + m <= n : check(t, n, s, p, m)) report(o, s);
    }
    for (uint32_t j = mp - 1; j >= 1; --j) { /* lines 13-14: the m'-1 crossing starts */
      const uint64_t s = 16 * (i + 1) - j;
      if (check(t, n, s, p, m)) report(o, s);
    }
  }
  for (uint64_t s = 16 * nb; s + m <= n; ++s) /* the partial last block */
    if (check(t, n, s, p, m)) report(o, s);
}

/* ---------------------------------------------------------------------------- EPSMb */
/* wsmatch(a, p'): bit k (k = 0..7) set iff a[k..k+3] = p'[0..3] (the mpsadbw emulation) */
static inline uint32_t wsmatch(__m128i a, __m128i pp) {
  const __m128i h = _mm_mpsadbw_epu8(a, pp, 0);
  const __m128i l = _mm_cmpeq_epi16(h, _mm_setzero_si128());
  return (uint32_t)_mm_movemask_epi8(_mm_packs_epi16(l, _mm_setzero_si128())) & 0xFFu;
}

static void epsm_b(const uint8_t *p, uint32_t m, const uint8_t *t, uint64_t n, sink_t *o) {
  uint8_t pb[16] = {0};
  memcpy(pb, p, 4);
  const __m128i pp = _mm_loadu_si128((const __m128i *)pb); /* p' (its first 4 bytes filter) */
  /* blocks i with T_{i+1} in the text: both halves by wsmatch (T_i) and wsmatch(wsblend) */
  const uint64_t nb = n / 16;
  uint64_t i = 0;
  for (; i + 1 < nb; ++i) {
    const __m128i Ti = load16(t, 16 * i), Tn = load16(t, 16 * (i + 1));
    uint32_t r = wsmatch(Ti, pp);                                     /* line 4 */
    while (r) {
      const uint32_t k = (uint32_t)__builtin_ctz(r);
      r &= r - 1;
      const uint64_t s = 16 * i + k;
      if (check(t, n, s, p, m)) report(o, s);                        /* lines 6-8 */
    }
    /* S = wsblend(T_i, T_{i+1}) = T_i[8..15] T_{i+1}[0..7]: blend_epi16 + shuffle_epi32 */
    const __m128i S = _mm_shuffle_epi32(_mm_blend_epi16(Ti, Tn, 0x0F), _MM_SHUFFLE(1, 0, 3, 2));
    r = wsmatch(S, pp);                                               /* line 10 */
    while (r) {
      const uint32_t k = (uint32_t)__builtin_ctz(r);
      r &= r - 1;
      const uint64_t s = 16 * i + 8 + k;
      if (check(t, n, s, p, m)) report(o, s);                        /* lines 12-14 */
    }
  }
  for (uint64_t s = 16 * i; s + m <= n; ++s) /* the last block(s): no blend partner */
    if (check(t, n, s, p, m)) report(o, s);
}

/* ---------------------------------------------------------------------------- EPSMc */
#define EPSMC_K 11

static inline uint32_t wscrc(const uint8_t *a) {
  uint64_t lo, hi;
  memcpy(&lo, a, 8);
  memcpy(&hi, a + 8, 8);
  return (uint32_t)_mm_crc32_u64(_mm_crc32_u64(0, lo), hi);
}

static int cmp_desc_u32(const void *a, const void *b) {
  const uint32_t x = *(const uint32_t *)a, y = *(const uint32_t *)b;
  return x < y ? 1 : x > y ? -1 : 0;
}

static void epsm_c(const uint8_t *p, uint32_t m, const uint8_t *t, uint64_t n, sink_t *o) {
  const uint32_t mask = (1u << EPSMC_K) - 1u;                          /* line 1 */
  const uint32_t sh = (m / 16 - 1) * 16;                               /* line 6 */
  /* L[v]: CSR lists of offsets j in [0, sh) (lines 2-5), each list in descending j so that
     the starts x - j of one inspected block come out ascending */
  uint32_t *head = calloc((1u << EPSMC_K) + 1, sizeof(uint32_t));
  uint32_t *js = malloc(sh * sizeof(uint32_t));
  uint32_t *hv = malloc(sh * sizeof(uint32_t));
  for (uint32_t j = 0; j < sh; ++j) {
    hv[j] = wscrc(p + j) & mask;
    head[hv[j] + 1]++;
  }
  for (uint32_t v = 0; v < (1u << EPSMC_K); ++v) head[v + 1] += head[v];
  uint32_t *fill = malloc((1u << EPSMC_K) * sizeof(uint32_t));
  memcpy(fill, head, (1u << EPSMC_K) * sizeof(uint32_t));
  for (uint32_t j = 0; j < sh; ++j) js[fill[hv[j]]++] = j;
  for (uint32_t v = 0; v < (1u << EPSMC_K); ++v)
    if (head[v + 1] - head[v] > 1) qsort(js + head[v], head[v + 1] - head[v], sizeof(uint32_t), cmp_desc_u32);
  /* inspected blocks x = 0, sh, 2 sh, ...: start s is examined through the first block
     x >= s (j = x - s < sh, and x + 16 <= s + m since sh <= m - 16) */
  uint64_t next = 0; /* the first start not yet examined */
  for (uint64_t x = 0; x + 16 <= n; x += sh) {                          /* lines 7, 13 */
    const uint32_t v = wscrc(t + x) & mask;                             /* lines 8-9 */
    for (uint32_t e = head[v]; e < head[v + 1]; ++e) {                  /* line 10 */
      if (js[e] > x) continue;                                          /* line 11: 0 <= x - j */
      const uint64_t s = x - js[e];
      if (check(t, n, s, p, m)) report(o, s);                           /* line 12 */
    }
    next = x + 1;
  }
  /* starts after the last inspected block (their first block would lie past the text) */
  for (uint64_t s = next; s + m <= n; ++s)
    if (check(t, n, s, p, m)) report(o, s);
  free(head);
  free(js);
  free(hv);
  free(fill);
}

int64_t cpu_epsm_search(const uint8_t *p, uint64_t m, const uint8_t *t, uint64_t n, uint64_t *pos,
                        uint64_t cap) {
  if (m == 0 || p == NULL) return -1;
  sink_t o = {pos, pos ? cap : 0, 0};
  if (n < m) return 0;
  if (m < 4)
    epsm_a(p, (uint32_t)m, t, n, &o);
  else if (m < 32)
    epsm_b(p, (uint32_t)m, t, n, &o);
  else
    epsm_c(p, (uint32_t)m, t, n, &o);
  return (int64_t)o.occ;
}

/* which procedure the dispatch picks (0 = a, 1 = b, 2 = c) */
int cpu_epsm_variant(uint64_t m) { return m < 4 ? 0 : m < 32 ? 1 : 2; }
