/*
 * epsm_oracle.c -- CPU oracle for exact string matching (TEST INFRASTRUCTURE).
 *
 * This file is test infrastructure, not product code.  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
 * may load or call it.  It shares no code, header, table or helper with the
 * CUDA path under paper_1209_6449_b200/; neither side includes the other.
 *
 * What it computes (Sec. 1, "the exact string matching
 * problem consists in finding all occurrences of the pattern p in t";
 * notation p[0..m-1] from PAPER.md:114-116, Sec. 2):
 *
 *     Occ(p, t) = { s : 0 <= s <= n-m  and  t[s+j] = p[j] for all 0 <= j < m }
 *
 * emitted in ascending order as uint64.  EPSMa/b/c all end in a "naive check"
 * of every candidate (Sec. 3; Sec. 3.2; PAPER.md:563,
 * Sec. 3.3), so this set is exactly what the method reaches; the oracle is the
 * definition written out as the plain O(nm) brute force (the "naive check" at
 * every start).  Readings taken where the paper is silent (R1-R6):
 *   - overlapping occurrences are all reported (R1: "all occurrences");
 *   - 0-based start offsets, ascending, no duplicates (R2/R3);
 *   - the start n-m is included (R4), n < m gives the empty set, m = 0 is an
 *     error (R5; the paper requires m > 0);
 *   - every byte value 0..255 is a symbol, no terminator (R7; sigma = 256,
 *     PAPER.md:168).
 *
 * Parity pins (tests/test_oracle.py, all run with -m "not gpu"):
 *   the paper's wsmatch worked figure (tests/golden/),
 *   exhaustive binary texts/patterns against CPython's bytes.find,
 *   random inputs against the `re` engine, closed forms for a^m in a^n and
 *   periodic texts.  No function here is "parity unpinned".
 *
 * Plain C loops only: no intrinsics, no memmem/memcmp, no SIMD.  The compiler
 * may auto-vectorise (built with -O2); that is disclosed in DESIGN.md.
 */
#include <stdint.h>

/* Error code shared in meaning (not in code) with the product header. */
#define ORACLE_EINVAL (-1)

/*
 * oracle_search: write the first min(occ, cap) positions of Occ(p, t) in
 * ascending order into out[] (out may be NULL when cap == 0) and return
 * occ = |Occ(p, t)|.  Returns ORACLE_EINVAL for m == 0, a NULL pattern, a NULL
 * text with n > 0, or out == NULL with cap > 0.
 */
int64_t oracle_search(const uint8_t *p, uint64_t m, const uint8_t *t,
                      uint64_t n, uint64_t *out, uint64_t cap)
{
    if (m == 0 || p == 0 || (t == 0 && n > 0) || (out == 0 && cap > 0))
        return ORACLE_EINVAL;
    if (n < m)
        return 0;
    int64_t occ = 0;
    for (uint64_t s = 0; s <= n - m; ++s) {     /* every start, 0 <= s <= n-m */
        uint64_t j = 0;
        while (j < m && t[s + j] == p[j])       /* naive check of window s */
            ++j;
        if (j == m) {
            if ((uint64_t)occ < cap)
                out[occ] = s;
            ++occ;
        }
    }
    return occ;
}

/* oracle_count: |Occ(p, t)|, same argument rules as oracle_search. */
int64_t oracle_count(const uint8_t *p, uint64_t m, const uint8_t *t, uint64_t n)
{
    return oracle_search(p, m, t, n, 0, 0);
}

/*
 * oracle_verify: the "naive check" of one start (Sec. 3):
 * 1 iff 0 <= s <= n-m and t[s..s+m-1] = p, else 0.
 */
int oracle_verify(const uint8_t *p, uint64_t m, const uint8_t *t, uint64_t n,
                  uint64_t s)
{
    if (m == 0 || n < m || s > n - m)
        return 0;
    for (uint64_t j = 0; j < m; ++j)
        if (t[s + j] != p[j])
            return 0;
    return 1;
}
