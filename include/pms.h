/*
 * pms.h -- C ABI of the B200 (sm_100a) Skip-Brute-Force planted (l,d) motif
 * search library, libpms_b200.so.
 *
 * Operation (section I.A problem statement; PAPER.md:63 section
 * III.A skip-brute-force; section IV.A candidates generated from
 * their index): given n DNA sequences s_0..s_{n-1} of length t over
 * {A,C,G,T}, return every l-mer m such that EVERY sequence has a window
 * (length-l substring, t-l+1 of them) at Hamming distance <= d from m.
 * The search enumerates all 4^l candidates and abandons a candidate at the
 * first sequence with no such window (the skip rule).  The result is a
 * set; it does not depend on the skip rule, the scan order or the launch
 * configuration.
 *
 * Codes: A=0 C=1 G=2 T=3; an l-mer's code is big-endian base 4 (first base in
 * the most significant digit), so code order = lexicographic order (SPEC.md:
 * 66-74).  The uint32-code entry points take l <= 16 (PMS_MAX_L); the
 * uint64-code ones (pms_find64*, pms_plan_execute64) take l <= 31
 * (PMS_MAX_L64: "l is capped at 31 so ranks fit a 64-bit
 * integer").
 *
 * Conventions for every entry point:
 *   - sizes are element counts unless stated; all functions are thread-safe
 *     for distinct plans; a plan is used by one host thread at a time;
 *   - the caller owns every buffer it passes; the library keeps no pointer
 *     to caller memory after a call returns (pms_plan_execute: until the work
 *     it enqueued has completed on the given stream);
 *   - all work runs on the CUDA device that is current on the calling thread;
 *   - there is no CPU fallback: with no usable device the status is
 *     PMS_E_CUDA.
 *
 * Error checks happen in this order (the oracle mirrors it): PMS_E_ARG, then
 * PMS_E_CHAR, then device errors (PMS_E_CUDA), then PMS_E_TRUNCATED.
 */
#ifndef PMS_B200_H
#define PMS_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
    PMS_OK = 0,
    PMS_E_ARG = -1,       /* NULL seqs/count, out_codes NULL with max_out>0,
                             n<1, t<1, l<1, l>16 (l>31 for the 64-bit
                             entry points), l>t, d<0, lo>hi,
                             uint32 output from a plan with l>16 */
    PMS_E_CHAR = -2,      /* a byte outside "ACGTacgt" (incl. 'N') */
    PMS_E_TOO_LARGE = -3, /* n*t or the packed table exceeds 2^31 bytes.
                             (SURVEY 8(b) reserved this status for a window
                             table larger than shared memory; here such a
                             table is read through L1/L2 instead -- the same
                             result, pms_stats.table_in_smem = 0 -- so the
                             status only marks sizes the 32-bit indexing
                             cannot address.)                              */
    PMS_E_CUDA = -4,      /* no device, allocation/launch/runtime failure */
    PMS_E_TRUNCATED = -5  /* more motifs than max_out; *count is exact */
};

#define PMS_MAX_L 16    /* uint32 codes */
#define PMS_MAX_L64 31  /* uint64 codes */

/* Launch overrides (all 0 = automatic).  Results never depend on them. */
typedef struct pms_launch {
    int32_t ctas_per_sm;     /* persistent CTAs per SM (grid = SMs * this)   */
    int32_t warps_per_cta;   /* warps per CTA                                */
    int32_t batch;           /* candidates per atomic grab (multiple of 256;
                                0 = auto: one block for the slice family)   */
    int32_t lanes_per_cand;  /* 16 or 32 lanes per candidate, 0 = pick the
                                one with less window padding                 */
    int32_t force_generic;   /* 1 = windows never register-resident          */
    int32_t grid_ctas;       /* total persistent CTAs (overrides ctas_per_sm;
                                the "workers" of the paper's Fig. 3/4 sweep)  */
    int32_t no_skip;         /* 1 = plain brute force (PAPER.md:63 before the
                                "enhanced version"): every candidate (block
                                family: every block) scans all n sequences;
                                same result.  With algo = AUTO this runs the
                                candidate family (n*W compares per candidate)*/
    int32_t algo;            /* PMS_ALGO_*: which kernel family (0 = auto)   */
    int32_t block_digits;    /* block families' suffix digits S (5: 1024-,
                                6: 4096-, 7: 16384-candidate blocks; 7 only
                                in PMS_ALGO_SLICE); 0 = auto (slice: 7 if
                                l >= 13, else 5; block: 6 if l >= 13,
                                else 5)                                      */
    int32_t table_global;    /* 1 = read the packed table from global memory
                                (L1/L2) instead of staging it in smem        */
    int32_t handoff;         /* block family: a block with at most this many
                                live candidates finishes them one by one
                                (0 = auto)                                   */
    int32_t wide_words;      /* 1 = 64-bit window words (two 32-bit bit
                                planes) even for l <= 16; automatic for
                                l > 16.  Same result                         */
    int32_t seq_parallel;    /* PMS_ALGO_SLICE with few blocks: 1 = scan every
                                (block, sequence) pair in parallel and AND
                                the per-sequence masks (no sequential skip
                                rule; a block whose AND is empty is skipped);
                                -1 = never; 0 = auto (when there are fewer
                                than 1/4 as many blocks as resident warps)   */
    int32_t overlap_prepass; /* plan API: 1 = no timing event between the
                                pre-pass and the search kernel, so the search
                                (a programmatic dependent launch) overlaps the
                                pre-pass's tail; pms_stats.pack_ms is then 0
                                and search_ms covers both (pms_find* without
                                stats always run this way)                   */
} pms_launch;

/* Kernel families (pms_launch.algo).  Every family returns the same set.
 *   PMS_ALGO_CANDIDATE: one candidate per 16/32 lanes; each candidate-window
 *     Hamming test is XOR, XOR-OR fold, POPC.
 *   PMS_ALGO_BLOCK: the 4^S candidates sharing their first l-S digits (S = 5
 *     or 6) are tested together (bit-parallel over candidates): one
 *     XOR/fold/POPC of the shared prefix against a window gives the prefix
 *     distance p, and the candidates whose last S digits lie within d-p of the
 *     window's last S digits match that window (a Hamming-ball bitmask).  Each candidate keeps
 *     PAPER.md:63's semantics: it is compared with the windows of sequence
 *     0, 1, ... and dropped at the first sequence with no window within d; the
 *     block is abandoned when no candidate is left (the skip rule on 4^S
 *     candidates at once).  Needs l >= 5 (else the candidate family runs).
 *   PMS_ALGO_SLICE: the block family's computation (same blocks, same
 *     per-candidate skip rule, same set) with the prefix test bit-sliced over
 *     windows (a lane's 32 windows at once: one-hot base planes of the prefix
 *     positions summed by a carry-save adder tree, no per-window POPC) and
 *     the hits resolved in batches through per-warp queues.
 *     Applies to l <= 16, t - l + 1 <= 1024 and d < l - S; elsewhere a
 *     request for it runs PMS_ALGO_BLOCK.
 *   PMS_ALGO_AUTO (0): PMS_ALGO_SLICE where it applies, else PMS_ALGO_BLOCK
 *     when l >= 5, else PMS_ALGO_CANDIDATE. */
enum { PMS_ALGO_AUTO = 0, PMS_ALGO_CANDIDATE = 1, PMS_ALGO_BLOCK = 2, PMS_ALGO_SLICE = 3 };

/* Counters and timings of the last execution of a plan. */
typedef struct pms_stats {
    double pack_ms;            /* device time of the window pre-pass        */
    double search_ms;          /* device time of the search kernel          */
    double total_ms;           /* device time from first to last enqueue    */
    uint64_t candidates;       /* hi - lo                                    */
    uint64_t issued_compares;  /* candidate-window Hamming tests the kernel
                                  issued on real (unpadded) windows          */
    uint64_t motifs;           /* total motifs found (= *count)              */
    int32_t grid, block, lanes_per_cand, windows_per_lane, generic,
            table_in_smem;
    uint32_t smem_bytes;
    int32_t algo;              /* PMS_ALGO_* actually run                    */
    uint64_t block_scans;      /* PMS_ALGO_BLOCK: (block, sequence) scans;
                                  each is W prefix compares serving 4^S
                                  candidates                                 */
    int32_t block_digits;      /* PMS_ALGO_BLOCK suffix digits S (0 if none) */
    int32_t mode_flags;        /* bit 0: the slice family ran sequence-
                                  parallel (pms_launch.seq_parallel);
                                  bit 1: its hand-off checks ran on the
                                  staged tables (few blocks per warp)       */
    uint64_t sparse_steps;     /* PMS_ALGO_SLICE sparse mode: (candidate
                                  list, sequence) steps; each checks the
                                  list's candidates against W windows (the
                                  checks are in issued_compares)           */
} pms_stats;

/* ---------------------------------------------------------------------
 * pms_find -- one complete search from HOST buffers (synchronous).
 *   seqs      host, n*t bytes, row-major (sequence i at seqs + i*t), ASCII
 *             A/C/G/T in any case.  Read only.
 *   out_codes host, capacity max_out codes; may be NULL iff max_out == 0.
 *             On PMS_OK receives *count codes ascending, without duplicates.
 *             On PMS_E_TRUNCATED its contents are unspecified.
 *   count     host, required: receives the exact number of motifs (also on
 *             PMS_E_TRUNCATED, so max_out = 0 works as a size query).
 * An empty result is PMS_OK with *count = 0; d >= l yields all 4^l codes.
 * Steps: validate arguments -> H2D copy -> device pre-pass (byte check +
 * window packing) -> persistent search kernel with in-kernel atomic-append
 * compaction -> one D2H copy of the state, the count and the first
 * min(max_out, 1024) codes (contiguous in the context's result block; the
 * rest only if the set is larger) -> host sort.
 * A call without stats that repeats the previous call's shape, range and
 * capacity (same pooled context) replays the device work as one CUDA graph;
 * set the environment variable PMS_NO_GRAPH to always enqueue it call by call.
 * The search kernel is a programmatic dependent launch of the pre-pass (it
 * waits in-kernel for the pre-pass's writes); without stats no timing event
 * separates the two, so its launch overlaps the pre-pass (PMS_NO_PDL: plain
 * stream order).
 * ------------------------------------------------------------------- */
int pms_find(const uint8_t *seqs, int32_t n, int32_t t, int32_t l, int32_t d,
             uint32_t *out_codes, uint64_t max_out, uint64_t *count);

/* pms_find over the candidate-code range [lo, hi) (hi is clipped to 4^l),
 * with optional launch overrides and stats (each may be NULL).  Range
 * additivity holds: results over [a,b) and [b,c) concatenate to [a,c). */
int pms_find_ex(const uint8_t *seqs, int32_t n, int32_t t, int32_t l,
                int32_t d, uint64_t lo, uint64_t hi, const pms_launch *launch,
                uint32_t *out_codes, uint64_t max_out, uint64_t *count,
                pms_stats *stats);

/* ---------------------------------------------------------------------
 * pms_find64 / pms_find64_ex -- the same operation with uint64 codes for
 * l <= 31.  Arguments, ownership, status
 * order and range semantics are those of pms_find / pms_find_ex, with
 * out_codes a host array of uint64 (capacity max_out) and hi clipped to
 * 4^l <= 2^62.  Every l in [1, 31] is accepted (l <= 16 gives the same set as
 * pms_find, widened).  Windows are packed into 64-bit words (two 32-bit bit
 * planes); the table is n * ceil32(t-l+1) * 8 bytes.  Exhaustive enumeration
 * of 4^l candidates is the caller's budget: use [lo, hi) ranges for large l.
 * ------------------------------------------------------------------- */
int pms_find64(const uint8_t *seqs, int32_t n, int32_t t, int32_t l, int32_t d,
               uint64_t *out_codes, uint64_t max_out, uint64_t *count);

int pms_find64_ex(const uint8_t *seqs, int32_t n, int32_t t, int32_t l,
                  int32_t d, uint64_t lo, uint64_t hi, const pms_launch *launch,
                  uint64_t *out_codes, uint64_t max_out, uint64_t *count,
                  pms_stats *stats);

/* ---------------------------------------------------------------------
 * Plans: device-resident, asynchronous form for callers that own device
 * memory and streams (the Python binding passes torch tensors and
 * torch.cuda.current_stream()).  A plan holds the packed window table, the
 * work/result counters and timing events for one (n, t, l, d) shape.
 * ------------------------------------------------------------------- */
typedef struct pms_plan pms_plan;

/* Allocates device workspace for the shape (1 <= l <= 31; plans with l > 16
 * use 64-bit window words and must be executed with pms_plan_execute64).
 * *plan receives the handle. */
int pms_plan_create(int32_t n, int32_t t, int32_t l, int32_t d,
                    const pms_launch *launch, pms_plan **plan);

/* Enqueues pre-pass + search on `stream` (a cudaStream_t; NULL = legacy
 * default stream).  Does not synchronize.
 *   d_seqs   device, n*t bytes as for pms_find.
 *   d_out    device, capacity `cap` codes (NULL iff cap == 0): receives the
 *            first min(total, cap) motif codes in UNSPECIFIED order.
 *   d_count  device, one uint64: receives the total number of motifs once the
 *            work completes (also when total > cap).
 * Byte errors are detected on the device; query them with pms_plan_wait. */
int pms_plan_execute(pms_plan *plan, const uint8_t *d_seqs, uint64_t lo,
                     uint64_t hi, uint32_t *d_out, uint64_t cap,
                     uint64_t *d_count, void *stream);

/* pms_plan_execute with uint64 result codes (d_out: device, capacity `cap`
 * uint64 codes); valid for every plan (1 <= l <= 31).  pms_plan_execute on a
 * plan with l > 16 returns PMS_E_ARG. */
int pms_plan_execute64(pms_plan *plan, const uint8_t *d_seqs, uint64_t lo,
                       uint64_t hi, uint64_t *d_out, uint64_t cap,
                       uint64_t *d_count, void *stream);

/* Waits for the plan's last execution (its search work, on a private stream
 * ordered after it; later work the caller enqueued on `stream` is not waited
 * for) and reads the plan's device state back; returns PMS_E_CHAR if the
 * pre-pass saw an invalid byte (the search then did no work and *d_count is
 * 0), PMS_E_CUDA on a device error, else PMS_OK.  Fills *stats if non-NULL
 * (stats->motifs is 0 here: the count is in the caller's d_count). */
int pms_plan_wait(pms_plan *plan, pms_stats *stats);

void pms_plan_destroy(pms_plan *plan);

/* ---------------------------------------------------------------------
 * Integer-pipe roofline microbenchmark (SURVEY 8(d) R_mix): runs the search
 * kernel's exact per-compare instruction sequence (XOR; XOR-OR fold with
 * the 16-bit-rotated operands; POPC; 3-way min) on register-resident
 * windows with no early exit, on every SM, for `iters` candidates per warp.
 *   compares_per_s   receives compares / second (CUDA-event timed)
 *   compares_per_clk_sm receives compares / SM-clock / SM, using the SM
 *                    clock rate the driver reports (may be NULL)
 *   ms               receives the kernel time (may be NULL)
 * ------------------------------------------------------------------- */
int pms_roofline(int32_t iters, double *compares_per_s,
                 double *compares_per_clk_sm, double *ms);

/* ---------------------------------------------------------------------
 * Roofline microbenchmark of the slice family:
 * runs the plan's own per-scan code on the tables of its last execution
 * (pms_plan_execute*, completed or not: this call waits for it) with
 * everything dynamic removed -- no work counter, no skip rule, no hand-off,
 * no output; warp g walks consecutive blocks of its own region of the code
 * space and scans each against sequences 0 .. D-1, D = the last execution's
 * (block, sequence) scans per block (the mix the skip rule produced), for
 * scans_per_warp scans, every warp busy throughout.
 *   mode 0: pass 1 only (plane loads + carry-save hit classification): R_pass1
 *   mode 1: pass 1 + hit resolution + end of scan at the instance's own hit
 *           mix: R_scan
 *   mode 2: sparse-mode steps with lists of the last
 *           execution's mean list size: R_sparse
 *   mode 3: dense scans with the last execution's sparse steps per scan
 *           interleaved (its own mix of both units): R_mix
 *   tests_per_s  receives (block, sequence) scans * W / second (required);
 *                mode 2: candidate-sequence checks * W / second; mode 3:
 *                (scans + checks) * W / second
 *   scans_per_s, ms  scans (mode 2: sparse steps) / second and the kernel
 *                time (may be NULL)
 * The tables are placed as the plan's search kernel places them (shared
 * memory, or L1/L2 when they do not fit).  PMS_E_ARG unless the plan runs
 * PMS_ALGO_SLICE and has been executed; CUDA-event timed, best of three
 * after one warm-up, on the plan's private stream.
 * ------------------------------------------------------------------- */
int pms_plan_roofline(pms_plan *plan, int32_t mode, int32_t scans_per_warp,
                      double *tests_per_s, double *scans_per_s, double *ms);

/* Static description of a status code. */
const char *pms_strerror(int status);

/* Where the last PMS_E_CUDA on the calling host thread came from (source
 * line and CUDA error string); "" if none.  Owned by the library. */
const char *pms_last_error(void);

/* Debug builds (libpms_b200_debug.so, -DPMS_DEBUG_CHECKS) count failed
 * device checks -- out-of-range indices and hit-queue / candidate-word protocol
 * violations; the checked access itself still runs, the count
 * is a detector.  Returns the count (reset to 0 if `reset`), -1 in release
 * builds, -2 on a device error. */
int64_t pms_debug_violations(int32_t reset);

/* Number of SMs and the opt-in shared memory per block of the current
 * device (for reporting); PMS_E_CUDA without a device. */
int pms_device_info(int32_t *sms, int32_t *smem_optin_bytes,
                    int32_t *clock_khz);

#ifdef __cplusplus
}
#endif
#endif /* PMS_B200_H */
