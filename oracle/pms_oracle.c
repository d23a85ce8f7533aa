/*
 * pms_oracle.c -- CPU ORACLE for Skip-Brute-Force planted (l,d) motif search.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * The product path (paper_1403_1313_b200/, include/pms.h) never links,
 * imports or calls it, and this file includes nothing from the product.
 *
 * It is deliberately plain and slow: l-mers are decoded to characters and
 * compared character by character with the window bytes of the input.  No
 * 2-bit packing, no bit tricks, no blocking.  Each function cites the
 * passage of PAPER.md ("P:<line>", section) or SPEC.md ("S:<line>") it
 * follows; readings of the paper are listed in DESIGN.md section 3.
 *
 * Pins (tests/test_oracle.py): SPEC worked examples, closed forms
 * (Hamming-ball volume, two-string intersection count, d=0 set
 * intersection, d>=l all codes), brute force on tiny inputs (naive BF and
 * the independent Hamming-ball intersection below), planted recovery, per-motif
 * re-verification, metamorphic relations.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>

/* Status codes.  Same meaning and order of checks as include/pms.h (the
 * numbers are restated here, not included, so the two sides share no file). */
enum {
    ORC_OK = 0,
    ORC_E_ARG = -1,
    ORC_E_CHAR = -2,
    ORC_E_TOO_LARGE = -3,
    ORC_E_CUDA = -4,
    ORC_E_TRUNCATED = -5,
    ORC_E_NOMEM = -6
};

#define ORC_MAX_L 31      /* oracle_find64 / verify (u64 codes) */
#define ORC_MAX_L32 16    /* oracle_find / naive / ball (u32 codes, include/pms.h) */

static const char ORC_ALPHABET[4] = {'A', 'C', 'G', 'T'}; /* A0 C1 G2 T3 */

/* Upper-case one byte if it is a/c/g/t; returns 0 for any byte outside
 * ACGTacgt (case-insensitive, 'N' and others rejected). */
static char orc_norm(uint8_t b)
{
    switch (b) {
    case 'A': case 'a': return 'A';
    case 'C': case 'c': return 'C';
    case 'G': case 'g': return 'G';
    case 'T': case 't': return 'T';
    default: return 0;
    }
}

/* S:66-74 decode_lmer: big-endian base-4 expansion of the rank, digit j
 * (j = 0 is the first base) = (rank >> 2(l-1-j)) & 3, mapped through the
 * code->symbol bijection. */
void oracle_decode(uint64_t rank, int32_t l, char *out)
{
    for (int32_t j = 0; j < l; ++j)
        out[j] = ORC_ALPHABET[(rank >> (2 * (l - 1 - j))) & 3u];
    out[l] = '\0';
}

/* S:86-94 hamming_distance: count of positions whose characters differ. */
int32_t oracle_hamming(const char *a, const char *b, int32_t l)
{
    int32_t h = 0;
    for (int32_t j = 0; j < l; ++j)
        if (a[j] != b[j]) ++h;
    return h;
}

/* Argument checks of include/pms.h, in the documented order (ARG, then
 * CHAR).  On success writes the upper-cased copy of seqs into norm. */
static int orc_validate(const uint8_t *seqs, int32_t n, int32_t t, int32_t l,
                        int32_t d, const void *out, uint64_t max_out,
                        const uint64_t *count, char *norm, int32_t max_l)
{
    if (seqs == NULL || count == NULL) return ORC_E_ARG;
    if (out == NULL && max_out > 0) return ORC_E_ARG;
    if (n < 1 || t < 1 || l < 1 || l > max_l) return ORC_E_ARG;
    if (l > t) return ORC_E_ARG;   /* S:80 MotifLongerThanSequence */
    if (d < 0) return ORC_E_ARG;
    for (int64_t p = 0; p < (int64_t)n * t; ++p) {
        char c = orc_norm(seqs[p]);
        if (c == 0) return ORC_E_CHAR;
        if (norm) norm[p] = c;
    }
    return ORC_OK;
}

/* ---------------------------------------------------------------------- */
/* Skip-Brute-Force, P:63 (section III.A) and S:222-240.                   */
/* ---------------------------------------------------------------------- */

typedef struct {
    const char *s;        /* upper-cased sequences, n rows of t chars */
    int32_t n, t, l, d;
    uint64_t lo, hi;      /* this worker's half-open rank range */
    uint64_t *found;      /* ranks of motifs in this range, ascending */
    uint64_t nfound, cap;
    uint64_t c_alg;       /* windows compared, first-match stop */
    int status;
} orc_job;

/* S:222-230 sequence_matches for one candidate m against sequence row s:
 * windows are the t-l+1 substrings starting at k = 0..t-l; a window
 * matches iff the number of mismatching characters is <= d ("less than
 * or equal").  Stops at the first matching window ("may stop") and
 * counts the windows it looked at into *cmp. */
static int orc_sequence_matches(const char *m, const char *s, int32_t t,
                                int32_t l, int32_t d, uint64_t *cmp)
{
    for (int32_t k = 0; k + l <= t; ++k) {
        int32_t mism = 0;
        for (int32_t j = 0; j < l; ++j) {
            if (s[k + j] != m[j] && ++mism > d) break;
        }
        if (mism <= d) {
            *cmp += (uint64_t)k + 1;
            return 1;
        }
    }
    *cmp += (uint64_t)(t - l + 1);
    return 0;
}

static int orc_push(orc_job *jb, uint64_t r)
{
    if (jb->nfound == jb->cap) {
        uint64_t nc = jb->cap ? 2 * jb->cap : 1024;
        uint64_t *p = (uint64_t *)realloc(jb->found, nc * sizeof(uint64_t));
        if (!p) return ORC_E_NOMEM;
        jb->found = p;
        jb->cap = nc;
    }
    jb->found[jb->nfound++] = r;
    return ORC_OK;
}

/* S:232-240 skip_bf_search over [lo,hi): ranks in increasing order; the
 * l-mer is generated from its rank on the fly ("no need of generating
 * all the possible l-mers prior to the search"); sequences are tested in
 * input order and the candidate is abandoned at the first sequence with no
 * matching window -- the skip rule ("skips checking the rest of the
 * sequences and start comparison with the next l-mer"). */
static void *orc_skip_bf_worker(void *arg)
{
    orc_job *jb = (orc_job *)arg;
    char m[ORC_MAX_L + 1];
    for (uint64_t r = jb->lo; r < jb->hi; ++r) {
        oracle_decode(r, jb->l, m);
        int all = 1;
        for (int32_t i = 0; i < jb->n; ++i) {
            if (!orc_sequence_matches(m, jb->s + (int64_t)i * jb->t, jb->t,
                                      jb->l, jb->d, &jb->c_alg)) {
                all = 0;
                break; /* skip rule */
            }
        }
        if (all && (jb->status = orc_push(jb, r)) != ORC_OK) return NULL;
    }
    return NULL;
}

/* S:242-249 naive_bf_search: every candidate against every window of every
 * sequence, full Hamming distance, no skipping of any kind. */
static void *orc_naive_worker(void *arg)
{
    orc_job *jb = (orc_job *)arg;
    char m[ORC_MAX_L + 1];
    for (uint64_t r = jb->lo; r < jb->hi; ++r) {
        oracle_decode(r, jb->l, m);
        int nmatched = 0;
        for (int32_t i = 0; i < jb->n; ++i) {
            const char *s = jb->s + (int64_t)i * jb->t;
            int any = 0;
            for (int32_t k = 0; k + jb->l <= jb->t; ++k) {
                ++jb->c_alg;
                if (oracle_hamming(m, s + k, jb->l) <= jb->d) any = 1;
            }
            nmatched += any;
        }
        if (nmatched == jb->n && (jb->status = orc_push(jb, r)) != ORC_OK)
            return NULL;
    }
    return NULL;
}

/* S:295-303 make_partition: W contiguous ranges of [lo,hi); base size
 * floor(N/W), the first N mod W ranges get one extra ("the number of
 * the first and the last l-mer each thread should generate"). */
void oracle_partition(uint64_t lo, uint64_t hi, int32_t workers,
                      uint64_t *starts /* workers+1 entries */)
{
    uint64_t N = hi - lo, base = N / (uint64_t)workers,
             rem = N % (uint64_t)workers, at = lo;
    for (int32_t w = 0; w < workers; ++w) {
        starts[w] = at;
        at += base + ((uint64_t)w < rem ? 1 : 0);
    }
    starts[workers] = at;
}

/* Fig. 1: windows prepared once, then `threads` workers each search
 * their own contiguous rank range in parallel over the shared
 * read-only input; per-worker outputs concatenated in range order, which is
 * already ascending. */
static int orc_run(void *(*worker)(void *), const uint8_t *seqs, int32_t n,
                   int32_t t, int32_t l, int32_t d, uint64_t lo, uint64_t hi,
                   int32_t threads, void *out, int wide, uint64_t max_out,
                   uint64_t *count, uint64_t *c_alg)
{
    char *norm = (char *)malloc(seqs && n > 0 && t > 0 ? (size_t)n * t : 1);
    if (!norm) return ORC_E_NOMEM;
    int st = orc_validate(seqs, n, t, l, d, out, max_out, count, norm,
                          wide ? ORC_MAX_L : ORC_MAX_L32);
    if (st != ORC_OK) { free(norm); return st; }
    uint64_t total = 1ull << (2 * l);
    if (hi > total) hi = total;
    if (lo > hi) { free(norm); return ORC_E_ARG; }
    if (threads < 1) threads = 1;

    orc_job *jobs = (orc_job *)calloc((size_t)threads, sizeof(orc_job));
    pthread_t *tid = (pthread_t *)calloc((size_t)threads, sizeof(pthread_t));
    uint64_t *starts = (uint64_t *)calloc((size_t)threads + 1, sizeof(uint64_t));
    if (!jobs || !tid || !starts) { free(norm); free(jobs); free(tid); free(starts); return ORC_E_NOMEM; }
    oracle_partition(lo, hi, threads, starts);
    for (int32_t w = 0; w < threads; ++w) {
        jobs[w].s = norm; jobs[w].n = n; jobs[w].t = t; jobs[w].l = l; jobs[w].d = d;
        jobs[w].lo = starts[w]; jobs[w].hi = starts[w + 1];
    }
    int spawned = 0;
    for (int32_t w = 1; w < threads; ++w)
        if (pthread_create(&tid[w], NULL, worker, &jobs[w]) == 0) ++spawned;
        else { jobs[w].status = 1; }
    worker(&jobs[0]);
    for (int32_t w = 1; w < threads; ++w)
        if (jobs[w].status != 1) pthread_join(tid[w], NULL);
    for (int32_t w = 1; w < threads; ++w)   /* a worker that failed to start runs here */
        if (jobs[w].status == 1) { jobs[w].status = 0; worker(&jobs[w]); }

    uint64_t nres = 0, work = 0;
    st = ORC_OK;
    for (int32_t w = 0; w < threads; ++w) {
        if (jobs[w].status != ORC_OK) st = jobs[w].status;
        nres += jobs[w].nfound;
        work += jobs[w].c_alg;
    }
    if (st == ORC_OK) {
        uint64_t at = 0;
        for (int32_t w = 0; w < threads; ++w)
            for (uint64_t k = 0; k < jobs[w].nfound; ++k, ++at)
                if (at < max_out) {
                    if (wide) ((uint64_t *)out)[at] = jobs[w].found[k];
                    else ((uint32_t *)out)[at] = (uint32_t)jobs[w].found[k];
                }
        *count = nres;
        if (c_alg) *c_alg = work;
        if (nres > max_out) st = ORC_E_TRUNCATED;
    }
    for (int32_t w = 0; w < threads; ++w) free(jobs[w].found);
    free(jobs); free(tid); free(starts); free(norm);
    (void)spawned;
    return st;
}

/* Skip-BF over ranks [lo,hi) with `threads` workers.  c_alg (may be NULL)
 * receives the number of windows compared with first-match stopping,
 * sequences in input order (SURVEY 8(d) C_alg). */
int oracle_find(const uint8_t *seqs, int32_t n, int32_t t, int32_t l,
                int32_t d, uint64_t lo, uint64_t hi, int32_t threads,
                uint32_t *out, uint64_t max_out, uint64_t *count,
                uint64_t *c_alg)
{
    return orc_run(orc_skip_bf_worker, seqs, n, t, l, d, lo, hi, threads,
                   out, 0, max_out, count, c_alg);
}

/* The same skip-BF for l <= 31 with 64-bit codes (SPEC.md:117 caps l at 31 so
 * a rank fits 64 bits). */
int oracle_find64(const uint8_t *seqs, int32_t n, int32_t t, int32_t l,
                  int32_t d, uint64_t lo, uint64_t hi, int32_t threads,
                  uint64_t *out, uint64_t max_out, uint64_t *count,
                  uint64_t *c_alg)
{
    return orc_run(orc_skip_bf_worker, seqs, n, t, l, d, lo, hi, threads,
                   out, 1, max_out, count, c_alg);
}

/* Naive BF (no skip rule, no early abort) over [lo,hi); c_alg receives the
 * full n*W windows per candidate. */
int oracle_naive_find(const uint8_t *seqs, int32_t n, int32_t t, int32_t l,
                      int32_t d, uint64_t lo, uint64_t hi, int32_t threads,
                      uint32_t *out, uint64_t max_out, uint64_t *count,
                      uint64_t *c_alg)
{
    return orc_run(orc_naive_worker, seqs, n, t, l, d, lo, hi, threads, out, 0,
                   max_out, count, c_alg);
}

/* ---------------------------------------------------------------------- */
/* Independent cross-check: neighbourhood intersection.                    */
/* result = intersection over i of (union over windows k of Ball(w_ik, d)) */
/* where Ball(x,d) = all l-mers within Hamming distance d of x, enumerated */
/* by choosing <= d positions and a different letter at each.  Shares no   */
/* loop with the candidate-major search above.  Tiny l only (4^l bytes).   */
/* ---------------------------------------------------------------------- */

static void orc_ball_mark(char *x, int32_t l, int32_t pos, int32_t left,
                          uint8_t *mark)
{
    /* x is the current string; positions < pos are fixed; mark the string
     * itself and every variant obtained by changing up to `left` more
     * positions >= pos to a different letter. */
    if (pos == l || left == 0) {
        uint64_t r = 0; /* rank of x: big-endian base 4 */
        for (int32_t j = 0; j < l; ++j) {
            uint64_t c = 0;
            while (ORC_ALPHABET[c] != x[j]) ++c;
            r = r * 4 + c;
        }
        mark[r] = 1;
        if (pos == l) return;
        /* left == 0: no further changes allowed; done */
        return;
    }
    /* leave position pos unchanged */
    orc_ball_mark(x, l, pos + 1, left, mark);
    /* change position pos to each of the 3 other letters */
    char keep = x[pos];
    for (int c = 0; c < 4; ++c) {
        if (ORC_ALPHABET[c] == keep) continue;
        x[pos] = ORC_ALPHABET[c];
        orc_ball_mark(x, l, pos + 1, left - 1, mark);
    }
    x[pos] = keep;
}

int oracle_ball_find(const uint8_t *seqs, int32_t n, int32_t t, int32_t l,
                     int32_t d, uint32_t *out, uint64_t max_out,
                     uint64_t *count)
{
    if (l > 12) return ORC_E_ARG; /* 4^12 = 16 MB bitmaps; tiny inputs only */
    char *norm = (char *)malloc(seqs && n > 0 && t > 0 ? (size_t)n * t : 1);
    if (!norm) return ORC_E_NOMEM;
    int st = orc_validate(seqs, n, t, l, d, out, max_out, count, norm, ORC_MAX_L32);
    if (st != ORC_OK) { free(norm); return st; }
    uint64_t total = 1ull << (2 * l);
    uint8_t *acc = (uint8_t *)malloc(total), *cur = (uint8_t *)malloc(total);
    if (!acc || !cur) { free(acc); free(cur); free(norm); return ORC_E_NOMEM; }
    memset(acc, 1, total);
    char x[ORC_MAX_L + 1];
    int32_t budget = d < l ? d : l;
    for (int32_t i = 0; i < n; ++i) {
        memset(cur, 0, total);
        for (int32_t k = 0; k + l <= t; ++k) {
            memcpy(x, norm + (int64_t)i * t + k, (size_t)l);
            x[l] = '\0';
            orc_ball_mark(x, l, 0, budget, cur);
        }
        for (uint64_t r = 0; r < total; ++r) acc[r] = (uint8_t)(acc[r] & cur[r]);
    }
    uint64_t c = 0;
    for (uint64_t r = 0; r < total; ++r)
        if (acc[r]) { if (c < max_out) out[c] = (uint32_t)r; ++c; }
    *count = c;
    free(acc); free(cur); free(norm);
    return c > max_out ? ORC_E_TRUNCATED : ORC_OK;
}

/* S:251-253 verify_motif: independent re-check that the l-mer of `rank`
 * has a window within Hamming distance d in every sequence, using the
 * plain full Hamming distance (no early abort).  Returns 1/0, or <0 on a
 * bad argument. */
int oracle_verify_motif(const uint8_t *seqs, int32_t n, int32_t t, int32_t l,
                        int32_t d, uint64_t rank)
{
    uint64_t dummy = 0;
    char *norm = (char *)malloc(seqs && n > 0 && t > 0 ? (size_t)n * t : 1);
    if (!norm) return ORC_E_NOMEM;
    int st = orc_validate(seqs, n, t, l, d, NULL, 0, &dummy, norm, ORC_MAX_L);
    if (st != ORC_OK) { free(norm); return st; }
    if (rank >= (1ull << (2 * l))) { free(norm); return ORC_E_ARG; }
    char m[ORC_MAX_L + 1];
    oracle_decode(rank, l, m);
    int ok = 1;
    for (int32_t i = 0; i < n && ok; ++i) {
        int best = l + 1;
        for (int32_t k = 0; k + l <= t; ++k) {
            int h = oracle_hamming(m, norm + (int64_t)i * t + k, l);
            if (h < best) best = h;
        }
        ok = best <= d;
    }
    free(norm);
    return ok;
}
