// pms_slice.cuh -- PMS_ALGO_SLICE: the block family with a bit-sliced pass 1
// and batched hit resolution (32-bit codes, l <= 16).  DESIGN.md section 6c.
//
// What it computes is exactly what pms_search_block computes (PAPER.md:63
// skip-BF, per candidate, sequences in input order): the 4^S candidates of a
// block share their first LP = l - S digits (the prefix P); for a window w with
// prefix distance p = Hamming(P, w[0..LP)) <= d, the block candidates that
// match w are the suffixes within r = d - p of w's suffix (Hamming distance is
// additive over positions).  Only the mapping onto the machine differs:
//
// pass 1, bit-sliced over windows.  Lane L owns the NWl = ceil(W/32)
//   consecutive windows k = L*NWl + q (bit q of its words).  The pre-pass
//   stores, per (sequence i, prefix position j, base b, lane L), the 32-bit
//   "match plane" whose bit q says window L*NWl+q has base b at position j.
//   A block's prefix digits b_j pick one plane per position, so the lane
//   loads LP words (one conflict-free 128-B row per warp each) and adds the LP
//   match bits of all its windows at once with a carry-save adder tree
//   (2 LOP3 per full adder) into a 5-bit counter preloaded with K = 16 - T,
//   T = LP - d: bit 4 of K + matches is "matches >= T", i.e. p <= d (a hit),
//   and the low four bits are then r = d - p.  No POPC, no per-window work.
//
// pass 2, batched.  The measured cost of a shared-memory atomic is ~4 SM
//   cycles per warp instruction whatever the number of active lanes
//   (tests/tools/ubench_smem.cu), so hits are resolved full-width instead of
//   by divergent per-lane loops:
//   * r = 0 hits (the window's own suffix only) are resolved by the lane
//     that found them: one slot load and one red each;
//   * r = 1 hits (the radius-1 ball, NU = 6 + 3X words) are appended, as
//     precomputed slots (byte offset of the window's suffix word in the
//     block's mask | bit << 11), to a per-warp queue (one shared atomicAdd
//     claims the positions of all hit classes) and resolved hit-major: lane
//     L takes hit b + L and applies its NU updates, word = slot XOR a
//     compile-time constant, bits from the hit's padded R1 row;
//   * r >= 2 hits (rare): broadcast to all lanes, which read their own words'
//     bits from the ball table T[r][e][m] (as pms_search_block).
//   A queue overflow (possible only when hits are dense: small LP, large d)
//   resolves that scan with per-lane atomics instead; results are the same.
//
// The candidate mask words are word-major (word k of lane L at k*32 + L), so
// a lane's words, the ball-table broadcast atomics and the end-of-scan reads
// are bank-conflict-free.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "pms_device.cuh"
#include "pms_kernels.cuh"

namespace pms {

struct SliceArgs {
    const uint32_t* planes;   // [n][LP][4][32] match planes (global)
    const uint32_t* splanes;  // [n][S][4][32] match planes of the suffix positions (sparse mode)
    const uint16_t* slots;    // [n][Wp] r = 0 slot of each window (global; row order: slot_idx)
    const uint32_t* words;    // [n][Wp] packed Bp32 windows (hand-off checks, global)
    const uint32_t* ball;     // slice ball table (kSTWords words, global)
    int n, W, Wp, NWl;        // Wp = 32 * NWl
    uint32_t dp;              // min(d, l)
    uint32_t kmask[4];        // bits of K = 16 - (LP - d) as 0 / ~0 masks
    unsigned long long lo, hi, lo_al, span;
    int batch, skip, handoff;
    int out_wide;
    uint32_t plane_bytes, slot_bytes;  // staged sizes (16-B multiples)
    // sequence-parallel mode (pms_search_slice_sp): per block of the range, its
    // candidate mask (32*KW words, ANDed over sequences) and a counter
    // (completed units | kSpDead once the mask is empty)
    uint32_t* spmask;
    uint32_t* spcnt;
    unsigned long long sp_blocks;
    DevState* st;
    uint32_t epoch;
    unsigned long long* nout;
    void* out;
    unsigned long long cap;
};

using SliceFn = void (*)(SliceArgs);
using SlicePackFn = void (*)(const uint8_t*, int, int, int, int, int, int, uint32_t*, uint16_t*,
                             uint32_t*, DevState*, unsigned long long*, uint32_t, uint32_t*,
                             uint32_t*, int, int);
using SliceRoofFn = void (*)(SliceArgs, int, int, unsigned long long, unsigned long long*);

// Kernel instances, one translation unit each (pms_slice.cu, pms_roof.cu),
// so they compile in parallel with pms.cu and pms64.cu.
struct SliceKernel {
    int S, LP;
    SliceFn fn_smem, fn_global;
};
const SliceKernel* slice_kernels(int* count);              // pms_slice.cu
const SliceKernel* slice_kernels_wide(int* count);         // pms_slice_wide.cu (l = 17..31)
SliceFn slice_seqpar_kernel(int S, int LP);                // pms_slice.cu (staged tables)
SliceFn slice_ht_kernel(int S, int LP);                    // pms_slice_ht.cu (staged tables,
                                                           // hand-off on the tables)
SlicePackFn slice_pack_kernel(int S);                      // pms_slice.cu
SliceRoofFn slice_roofline_kernel(int S, int LP, int mode, bool smem);  // pms_roof.cu
int64_t debug_violations_slice(int reset);
int64_t debug_violations_roof(int reset);
int64_t debug_violations_ht(int reset);
int64_t debug_violations_wide(int reset);

// Slice ball table: T[rho][e][m] (rho = 0..6, as pms_search_block's) then the
// radius-1 rows R1[e][u] (kSR1Stride words per e): u = 0: T[1][e][0]; u = 1..5:
// T[1][e][1 << (u-1)]; u = 6..14: 1 << e (the centre bit, for the words one
// upper position away); 15: 0.
constexpr int kSR1Off = 7 * 1024;
// R1 rows padded to 17 words: the rows of the 5 hits of an r = 1 round then
// start in 5 different banks (a 16-word stride put them all in 2: ~2.8-way
// conflicts on the row loads, ncu source page)
constexpr int kSR1Stride = 17;
constexpr int kSTWords = kSR1Off + 32 * kSR1Stride;  // 30.1 KB
constexpr int kSliceMaxLP = 24;              // l <= 31 (S = 7); LP - d <= 16, d <= 15
#ifndef PMS_SLICE_R0_DIRECT
#define PMS_SLICE_R0_DIRECT 1  // r = 0 hits resolved per lane (no queue); 0: queued
#endif
#ifndef PMS_SLICE_R0_PAIR
#define PMS_SLICE_R0_PAIR 1  // r = 0 loop: two hits per iteration (duplicate reds are idempotent)
#endif
#ifndef PMS_SLICE_EXCH
#define PMS_SLICE_EXCH 1  // end of scan: atom.exch(word, 0) instead of load + store
#endif
#ifndef PMS_SLICE_R1_DIRECT
#define PMS_SLICE_R1_DIRECT 0  // r = 1 hits resolved per lane (NU reds each); 0: queued
#endif
#ifndef PMS_SLICE_CHECK_VOTE
#define PMS_SLICE_CHECK_VOTE 1  // tables hand-off check: hit classes r >= 2, 1, 0 with a vote per step
#endif
#ifndef PMS_SLICE_SLOTS_QMAJOR
// slot rows stored bit-major -- window (lane L, bit q) at q * 32 + L -- so the
// lanes of a hit loop, each at its own q, read 2-byte slots that share banks
// only within a lane pair (window-major rows: L * NWl + q, birthday conflicts,
// ~2 wavefronts per LDS.U16 in the ncu source page)
#define PMS_SLICE_SLOTS_QMAJOR 1
#endif
#ifndef PMS_SLICE_PIN_WQ
#define PMS_SLICE_PIN_WQ 1  // the warp's queue-block address pinned in a register
#endif
constexpr uint32_t kSpDead = 0x80000000u;     // spcnt flag: the block's AND is empty
constexpr uint32_t kPoison16 = 0xFFFFu;      // debug builds: consumed / unwritten queue entry
constexpr uint32_t kPoison32 = 0xFFFFFFFFu;  // (no real entry: slots < 2^14, r < 16)
constexpr int kSlicePackThreads = 256;

// Per block size: S = 5, 6 run 32 warps per SM (64 registers); S = 7 (16
// words per lane) runs 16 warps with 128 registers.
template <int S>
struct SliceCfg {
    static constexpr int X = S - 5;
    static constexpr int KW = 1 << (2 * X);   // mask words per lane
    static constexpr int NU = 6 + 3 * X;      // words of a radius-1 ball
#ifndef PMS_SLICE7_NT
#define PMS_SLICE7_NT 1024
#endif
    static constexpr int NT = S >= 7 ? PMS_SLICE7_NT : 1024;
    static constexpr int NWARP = NT / 32;
    // per-warp queue capacities (a scan whose hits exceed one resolves them
    // per lane instead): r = 0 / r = 1 entries are u16 slots, r >= 2 entries
    // are slot | r << 16
    static constexpr int kCap0 = S >= 7 ? 192 : 256;
    static constexpr int kCap1 = S >= 7 ? 96 : 128;
    static constexpr int kCap2 = S >= 7 ? 32 : 64;
    // dynamic shared memory in front of the staged tables: [ball table]
    // [per-warp candidate words][per-warp queue blocks]; the word blocks
    // start at a multiple of their size (30 KB = 15 x 2 KB)
    static constexpr uint32_t kAccAlign = 32u * KW * 4u;  // one warp's word block
    static constexpr uint32_t kAccOff = kSTWords * 4u;     // (+ up to kAccAlign - 1 at run time)
    static constexpr uint32_t kAccBytes = NWARP * 32u * KW * 4u + kAccAlign;
    // one queue block per warp -- [r = 0 queue][r = 1 queue][r >= 2 queue]
    // [claim counter, padded to 16 B] -- so every queue address is one per-warp
    // base plus a compile-time offset (separate arrays had the compiler
    // re-derive four bases from %tid and the shared window every scan: five
    // S2R and ~20 instructions per scan in the SASS)
    static constexpr uint32_t kQ1Rel = kCap0 * 2u;
    static constexpr uint32_t kQ2Rel = kQ1Rel + kCap1 * 2u;
    static constexpr uint32_t kQcRel = kQ2Rel + kCap2 * 4u;
    static constexpr uint32_t kQStride = kQcRel + 16u;
    static constexpr uint32_t kQOff = kAccOff + kAccBytes;
    static constexpr uint32_t kWorkBytes = kQOff + NWARP * kQStride;  // = planes offset
    static_assert(kWorkBytes % 128u == 0, "TMA destinations");
};

}  // namespace pms

namespace {

using namespace pms;

#ifdef PMS_TRACE
// tuning builds only (scripts/trace_tail.py): per warp of the last search
// launch [enter, ready, end (globaltimer ns), blocks, scans, hand-off
// candidates, most scans of one block, longest block (ns)]
__device__ unsigned long long g_pms_trace[8192 * 8];
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
#endif

// ------------------------------------------------------------- pre-pass
// Grid (n, G): CTA (i, y) stages sequence i's 2-bit codes in shared memory
// (checking every byte: windows are substrings of the input)
// and produces items [256 y, 256 y + 256) of the sequence's work list:
//   items [0, Wp): window k -> (1) its packed Bp32 word (rows padded to Wp
//     with copies of window W-1), (2) its r = 0 slot for block digits S
//     (byte offset of the candidate word in a warp's block | bit << 11);
//   items [Wp, Wp + LP*128): match plane (j, b, lane) of the prefix
//     positions (bit q: window lane*NWl + q has base b at position j).
// Thread 0 of CTA (0, 0) resets the step's state and the result counter.
template <int S>
__global__ void __launch_bounds__(kSlicePackThreads) pms_pack_slice(
    const uint8_t* __restrict__ seqs, int n, int t, int l, int W, int NWl, int LP,
    uint32_t* __restrict__ planes, uint16_t* __restrict__ slots, uint32_t* __restrict__ words,
    DevState* st, unsigned long long* nout, uint32_t epoch, uint32_t* spmask, uint32_t* spcnt,
    int sp_words, int sp_blocks) {
    constexpr int X = S - 5;
    __shared__ uint8_t code[1024 + 32];
    pdl_launch_dependents();
    const int i = blockIdx.x;
    if (sp_blocks) {  // sequence-parallel scratch: masks all ones, counters 0
        const int g = (int)(blockIdx.x * gridDim.y + blockIdx.y) * kSlicePackThreads + (int)threadIdx.x;
        const int gs = (int)(gridDim.x * gridDim.y) * kSlicePackThreads;
        for (int x = g; x < sp_words; x += gs) spmask[x] = kFull;
        for (int x = g; x < sp_blocks; x += gs) spcnt[x] = 0u;
    }
    if (i == 0 && blockIdx.y == 0 && threadIdx.x == 0) {
        *nout = 0ull;
        st->next = 0ull;
        st->extra = 0ull;
        st->block_scans = 0ull;
    }
    if (i >= n) return;
    const int Wp = 32 * NWl;
    const uint8_t* row = seqs + (long long)i * t;
    PMS_CHECK(t <= 1024 + 32);
    uint32_t bad = 0;
    for (int b = threadIdx.x; b < t; b += kSlicePackThreads) {
        const uint32_t u = row[b] & 0xDFu;  // upper-case; only 'x'/'X' map to 'X'
        const uint32_t c = u == 'A' ? 0u : u == 'C' ? 1u : u == 'G' ? 2u : u == 'T' ? 3u : 4u;
        bad |= c >> 2;
        code[b] = (uint8_t)c;
    }
    if (bad) *(volatile unsigned int*)&st->bad = epoch;
    __syncthreads();
    const int item = (int)blockIdx.y * kSlicePackThreads + (int)threadIdx.x;
    if (item < Wp) {
        const int k = item, src = min(k, W - 1);
        uint32_t H = 0, L = 0;
        for (int j = 0; j < l; ++j) {
            const uint32_t c = code[src + j] & 3u;
            H = (H << 1) | (c >> 1);
            L = (L << 1) | (c & 1u);
        }
        words[(long long)i * Wp + k] = (H << 16) | L;
        const uint32_t eH = H & ((1u << S) - 1u), eL = L & ((1u << S) - 1u);
        const uint32_t kw = ((eH >> 5) << X) | (eL >> 5);
        // slot = byte offset of the candidate's word in the warp's block
        // (word = k * 32 + lane, word-major; < 2 KB at S <= 7) | bit << 11
#if PMS_SLICE_SLOTS_QMAJOR
        const int kslot = (k % NWl) * 32 + k / NWl;
#else
        const int kslot = k;
#endif
        slots[(long long)i * Wp + kslot] =
            (uint16_t)(k < W ? (((kw * 32u + (eH & 31u)) * 4u) | ((eL & 31u) << 11)) : 0u);
    } else if (item < Wp + l * 128) {
        // positions j < LP: the staged prefix planes; j >= LP: the suffix
        // planes [n][S][4][32] after all prefix planes (sparse mode)
        const int idx = item - Wp;
        const int j = idx >> 7, b = (idx >> 5) & 3, ln = idx & 31;
        uint32_t v = 0;
        const int k0 = ln * NWl, nq = min(NWl, W - k0);
        for (int q = 0; q < nq; ++q)
            if (code[k0 + q + j] == (uint8_t)b) v |= 1u << q;
        if (j < LP) planes[(long long)i * LP * 128 + idx] = v;
        else planes[(long long)n * LP * 128 + (long long)i * S * 128 + (idx - LP * 128)] = v;
    }
}

// ----------------------------------------------------- carry-save counting
// Reduce N equal-weight bit planes to one (their sum mod 2); the carries
// (weight x2, N/2 of them) go to cy[0..N/2).  Full adder: sum = a^b^c (one
// LOP3), carry = maj(a,b,c) (one LOP3).
template <int N>
__device__ __forceinline__ uint32_t csa_col(uint32_t* v, uint32_t* cy) {
    if constexpr (N == 0) {
        return 0u;
    } else if constexpr (N == 1) {
        return v[0];
    } else if constexpr (N == 2) {
        cy[0] = v[0] & v[1];
        return v[0] ^ v[1];
    } else {
        const uint32_t a = v[0], b = v[1], c = v[2];
        cy[0] = (a & b) | (c & (a ^ b));
        v[2] = a ^ b ^ c;  // the sum joins the column again (queue order: balanced depth)
        return csa_col<N - 2>(v + 2, cy + 1);
    }
}

// K + (number of set planes among m[0..LP)) as five bit planes c[0..4],
// K given by its four bit masks (K = 16 - (LP - d) <= 15, so the total is at
// most 16 + d < 32 for d <= 15; the host checks d <= 15 and LP - d <= 16).
template <int LP>
__device__ __forceinline__ void slice_count(const uint32_t (&m)[LP], const uint32_t (&k)[4],
                                            uint32_t (&c)[5]) {
    constexpr int N0 = LP + 1, C0 = N0 / 2;
    constexpr int N1 = C0 + 1, C1 = N1 / 2;
    constexpr int N2 = C1 + 1, C2 = N2 / 2;
    constexpr int N3 = C2 + 1, C3 = N3 / 2;
    uint32_t v0[N0], y0[C0 > 0 ? C0 : 1];
#pragma unroll
    for (int j = 0; j < LP; ++j) v0[j] = m[j];
    v0[LP] = k[0];
    c[0] = csa_col<N0>(v0, y0);
    uint32_t v1[N1], y1[C1 > 0 ? C1 : 1];
#pragma unroll
    for (int j = 0; j < C0; ++j) v1[j] = y0[j];
    v1[C0] = k[1];
    c[1] = csa_col<N1>(v1, y1);
    uint32_t v2[N2], y2[C2 > 0 ? C2 : 1];
#pragma unroll
    for (int j = 0; j < C1; ++j) v2[j] = y1[j];
    v2[C1] = k[2];
    c[2] = csa_col<N2>(v2, y2);
    uint32_t v3[N3], y3[C3 > 0 ? C3 : 1];
#pragma unroll
    for (int j = 0; j < C2; ++j) v3[j] = y2[j];
    v3[C2] = k[3];
    c[3] = csa_col<N3>(v3, y3);
    uint32_t top = 0u;  // weight 16: at most one of these can be set (total < 32)
#pragma unroll
    for (int j = 0; j < C3; ++j) top |= y3[j];
    c[4] = top;
}


// ------------------------------------------------------ shared-space access
// 32-bit shared-window addresses and explicit ld/st/red.shared: the compiler
// otherwise re-derives generic->shared bases inside the hit loops.
__device__ __forceinline__ uint32_t lds16(uint32_t a) {
    uint32_t v;
    asm volatile("ld.shared.u16 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
    return v;
}
__device__ __forceinline__ uint32_t lds32(uint32_t a) {
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
    return v;
}
__device__ __forceinline__ void sts16(uint32_t a, uint32_t v) {
    asm volatile("st.shared.u16 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
__device__ __forceinline__ void sts32(uint32_t a, uint32_t v) {
    asm volatile("st.shared.u32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
__device__ __forceinline__ void red_or(uint32_t a, uint32_t v) {
    asm volatile("red.shared.or.b32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t atom_exch0(uint32_t a) {
    uint32_t r;
    asm volatile("atom.shared.exch.b32 %0, [%1], 0;" : "=r"(r) : "r"(a) : "memory");
    return r;
}
__device__ __forceinline__ uint32_t atom_add(uint32_t a, uint32_t v) {
    uint32_t r;
    asm volatile("atom.shared.add.u32 %0, [%1], %2;" : "=r"(r) : "r"(a), "r"(v) : "memory");
    return r;
}

// index of window (lane, bit q) in a sequence's slot row
__device__ __forceinline__ uint32_t slot_idx(uint32_t lane, uint32_t q, int NWl) {
#if PMS_SLICE_SLOTS_QMAJOR
    (void)NWl;
    return q * 32u + lane;
#else
    return lane * (uint32_t)NWl + q;
#endif
}

// r = d - p of the hit at bit q (the low four counter planes)
__device__ __forceinline__ uint32_t slice_r(const uint32_t (&c)[5], int q) {
    return ((c[0] >> q) & 1u) | (((c[1] >> q) & 1u) << 1) | (((c[2] >> q) & 1u) << 2) |
           (((c[3] >> q) & 1u) << 3);
}

// Word delta (word index = k * 32 + lane) of update u of a radius-1 ball:
// u = 0 the hit's own word, u = 1..5 the lanes one H bit away, u = 6.. the
// words one upper suffix position away (L bit, H bit, both).
template <int X>
__device__ __forceinline__ uint32_t r1_delta(uint32_t u) {
    if (u == 0) return 0u;
    if (u <= 5) return 1u << (u - 1);
    const uint32_t v = u - 6, pos = v / 3, alt = v % 3;
    const uint32_t kd = alt == 0 ? (1u << pos) : alt == 1 ? (1u << (X + pos)) : ((1u << pos) | (1u << (X + pos)));
    return kd * 32u;
}

// One r >= 2 hit (slot, r) applied by every lane to its own words: word ek
// gets T[r][el5][lane ^ eh5]; with X >= 1 the words one upper position away
// get T[r-1] and -- via `common`, ORed into every word at the end of the scan
// -- all words get T[r-X] (a superset-free bound: T[r-X] is within budget
// wherever X upper positions mismatch).
template <int X, bool CLAMP = true>
__device__ __forceinline__ void slice_bcast(uint32_t e, uint32_t lane4, uint32_t T_s,
                                            uint32_t acc_lane_s, uint32_t& common) {
    // e = slot | r << 16, slot = (ek * 32 + eh5) * 4 | el5 << 11.  Lane L's
    // word ek is at acc + ek * 128 + 4L (the block is aligned to its size);
    // T[rho][el5][L ^ eh5] at T + rho * 4096 + el5 * 128 + 4 (L ^ eh5)
    // (radius >= 5 covers all five positions: row 6 is all ones)
    if constexpr (!CLAMP) {
        // r <= d <= 6: every row r, r - 1, r - X exists (r >= 2 >= X), so the
        // three rows are one address and two immediate offsets:
        // (e >> 4) & 0xFF80 = r * 4096 + el5 * 128
        const uint32_t toff = T_s + ((e >> 4) & 0xFF80u) + ((e & 0x7Cu) ^ lane4);
        const uint32_t aw = acc_lane_s | (e & 0x780u);
        red_or(aw, lds32(toff));
        if constexpr (X >= 1) common |= lds32(toff - (uint32_t)X * 4096u);
        if constexpr (X >= 2) {
            const uint32_t b = lds32(toff - 4096u);
#pragma unroll
            for (int u = 0; u < 3 * X; ++u) red_or(aw ^ (r1_delta<X>(6u + (uint32_t)u) * 4u), b);
        }
        return;
    }
    const uint32_t r = e >> 16;
    const uint32_t toff = T_s + ((e >> 4) & 0xF80u) + ((e & 0x7Cu) ^ lane4);
    const uint32_t aw = acc_lane_s | (e & 0x780u);
    red_or(aw, lds32(toff + min(r, 6u) * 4096u));
    if constexpr (X >= 1) common |= lds32(toff + min(r - (uint32_t)X, 6u) * 4096u);
    if constexpr (X >= 2) {
        const uint32_t b = lds32(toff + min(r - 1u, 6u) * 4096u);
#pragma unroll
        for (int u = 0; u < 3 * X; ++u) red_or(aw ^ (r1_delta<X>(6u + (uint32_t)u) * 4u), b);
    }
}

// ------------------------------------------------------------ the search
// Per-warp state of the slice kernels: shared-window addresses of the warp's
// candidate words and queues, the tables, and lane constants.
template <int S, bool SMEM>
struct SliceWarp {
    using C = SliceCfg<S>;
    uint32_t lane, acc_s, wq_s, T_s, R1_s, slots_s;  // wq_s: the warp's queue block
    __device__ __forceinline__ uint32_t q0_s() const { return wq_s; }
    __device__ __forceinline__ uint32_t q1_s() const { return wq_s + C::kQ1Rel; }
    __device__ __forceinline__ uint32_t q2_s() const { return wq_s + C::kQ2Rel; }
    __device__ __forceinline__ uint32_t qc_s() const { return wq_s + C::kQcRel; }
    uint32_t lane4, acc_lane_s;  // 4 * lane; acc_s + 4 * lane (the lane's word 0)
    uint32_t planes_s;           // shared-window address of the staged planes (SMEM)
    const uint32_t* planes;  // shared (SMEM) or global
    const uint16_t* gslots;  // global slots (!SMEM)
    uint32_t vmask;          // this lane's real windows among its NWl
    bool rclamp;  // d > 6: r >= 2 broadcasts clamp their table rows (slice_bcast)
    uint32_t km[4];
    int NWl, Wp;
};

// Prologue shared by the slice kernels: shared-memory carve-up, zeroed
// candidate words and queue counters, TMA bulk copies of the ball table and
// (SMEM) the planes and slots, completion on an mbarrier.
template <int S, bool SMEM>
__device__ __forceinline__ SliceWarp<S, SMEM> slice_setup(const SliceArgs& a, uint32_t* sdyn,
                                                         uint64_t* bar) {
    using C = SliceCfg<S>;
    constexpr int KW = C::KW;
    SliceWarp<S, SMEM> w;
    w.lane = threadIdx.x & 31u;
    const uint32_t wid = threadIdx.x >> 5;
    const uint32_t dyn_s = smem_u32(sdyn);
    // word blocks aligned to their size at run time (the dynamic window's
    // base alignment is not guaranteed beyond 128 B)
    const uint32_t acc0_s = (dyn_s + C::kAccOff + C::kAccAlign - 1u) & ~(C::kAccAlign - 1u);
    w.acc_s = acc0_s + wid * C::kAccAlign;
    w.lane4 = w.lane * 4u;
    w.acc_lane_s = w.acc_s + w.lane4;
    w.wq_s = dyn_s + C::kQOff + wid * C::kQStride;
#if PMS_SLICE_PIN_WQ
    asm volatile("" : "+r"(w.wq_s));  // opaque: held in a register, not re-derived per scan
#endif
    PMS_CHECK((w.acc_s & (32u * KW * 4u - 1u)) == 0u);
#pragma unroll
    for (int k = 0; k < KW; ++k) sts32(w.acc_s + (k * 32u + w.lane) * 4u, 0u);
    if (w.lane == 0) sts32(w.qc_s(), 0u);
#ifdef PMS_DEBUG_CHECKS
    // protocol check: every queue entry starts poisoned and is
    // poisoned again once consumed, so a round that reads an entry nobody
    // wrote this scan (a missed __syncwarp, a bad claim) is counted
    for (int q = (int)w.lane; q < C::kCap0 + C::kCap1; q += 32) sts16(w.q0_s() + 2u * q, kPoison16);
    for (int q = (int)w.lane; q < C::kCap2; q += 32) sts32(w.q2_s() + 4u * q, kPoison32);
#endif
    uint32_t* splanes = sdyn + C::kWorkBytes / 4u;
    uint16_t* sslots = reinterpret_cast<uint16_t*>(reinterpret_cast<char*>(splanes) + a.plane_bytes);
    if (threadIdx.x == 0) mbar_init(bar, 1);
    __syncthreads();
    if (threadIdx.x == 0) {
        mbar_expect_tx(bar, kSTWords * 4u + (SMEM ? a.plane_bytes + a.slot_bytes : 0u));
        tma_bulk_g2s(sdyn, a.ball, kSTWords * 4u, bar);
        if (SMEM) {
            for (uint32_t off = 0; off < a.plane_bytes; off += 65536u)
                tma_bulk_g2s(reinterpret_cast<char*>(splanes) + off,
                             reinterpret_cast<const char*>(a.planes) + off,
                             min(65536u, a.plane_bytes - off), bar);
            for (uint32_t off = 0; off < a.slot_bytes; off += 65536u)
                tma_bulk_g2s(reinterpret_cast<char*>(sslots) + off,
                             reinterpret_cast<const char*>(a.slots) + off,
                             min(65536u, a.slot_bytes - off), bar);
        }
    }
    mbar_wait(bar, 0);
    w.planes = SMEM ? splanes : a.planes;
    w.gslots = a.slots;
#if PMS_SLICE_PIN_WQ
    // the table addresses as one opaque base plus offsets: the compiler
    // otherwise re-derives each from the shared window (S2R SR_CgaCtaId + MOV
    // + VIADD + LEA) wherever it is used, five times per scan in the SASS
    uint32_t base_s = dyn_s;
    asm volatile("" : "+r"(base_s));
    w.T_s = base_s;
    w.R1_s = base_s + 4u * kSR1Off;
    w.planes_s = base_s + C::kWorkBytes;
    w.slots_s = base_s + C::kWorkBytes + a.plane_bytes;
#else
    w.planes_s = smem_u32(splanes);
    w.T_s = dyn_s;
    w.R1_s = dyn_s + 4u * kSR1Off;
    w.slots_s = smem_u32(sslots);
#endif
    for (int b = 0; b < 4; ++b) w.km[b] = a.kmask[b];
    const int nvalid = min(a.NWl, max(0, a.W - (int)w.lane * a.NWl));
    w.vmask = nvalid >= 32 ? kFull : ((1u << nvalid) - 1u);
    w.rclamp = a.dp > 6u;
    w.NWl = a.NWl;
    w.Wp = a.Wp;
    return w;
}

// The block's plane offsets (bytes within a sequence's planes): the row of
// base b_j for each prefix position j.
template <int S, int LP>
__device__ __forceinline__ void slice_offsets(unsigned long long cbase, uint32_t lane,
                                              uint32_t (&po)[LP]) {
    constexpr int l = LP + S;
#pragma unroll
    for (int j = 0; j < LP; ++j) {
        const uint32_t bj = (uint32_t)(cbase >> (2 * (l - 1 - j))) & 3u;
        po[j] = ((uint32_t)(j * 128) + bj * 32u + lane) * 4u;
        asm volatile("" : "+r"(po[j]));  // keep in a register (no per-scan remat)
    }
}

// Pass 1 of a (block, sequence i) scan: the carry-save counter planes c and
// the class masks of this lane's windows (r = 0, r = 1, r >= 2 hits).
template <int S, int LP, bool SMEM>
__device__ __forceinline__ void slice_pass1(const SliceWarp<S, SMEM>& w, const uint32_t (&po)[LP],
                                            int i, uint32_t (&c)[5], uint32_t& r0m, uint32_t& r1m,
                                            uint32_t& r2m) {
    uint32_t m[LP];
    if constexpr (SMEM) {  // one IMAD for the sequence, one IADD per plane
        const uint32_t P = w.planes_s + (uint32_t)i * (uint32_t)(LP * 512);
#pragma unroll
        for (int j = 0; j < LP; ++j) {
            PMS_CHECK(po[j] < (uint32_t)(LP * 512));
            m[j] = lds32(P + po[j]);
        }
    } else {
        const char* P = reinterpret_cast<const char*>(w.planes) + (size_t)i * (LP * 512);
#pragma unroll
        for (int j = 0; j < LP; ++j) {
            PMS_CHECK(po[j] < (uint32_t)(LP * 512));
            m[j] = __ldg(reinterpret_cast<const uint32_t*>(P + po[j]));
        }
    }
    slice_count<LP>(m, w.km, c);
    const uint32_t hv = c[4] & w.vmask;
    const uint32_t up = c[1] | c[2] | c[3];
    r0m = hv & ~c[0] & ~up;
    r1m = hv & c[0] & ~up;
    r2m = hv & up;
}

// Pass 2 of a scan: every hit's candidates ORed into the warp's words (and
// `common`).  Returns nothing; the words are read by slice_finish.
template <int S, bool SMEM>
__device__ __forceinline__ void slice_pass2(const SliceWarp<S, SMEM>& w, int i,
                                            const uint32_t (&c)[5], uint32_t r0m, uint32_t r1m,
                                            uint32_t r2m, uint32_t& common) {
    using C = SliceCfg<S>;
    constexpr int X = C::X, NU = C::NU;
    const uint32_t lane = w.lane;
    // slot row of this lane's windows in sequence i
    const uint32_t srow = (uint32_t)(i * w.Wp) + slot_idx(lane, 0u, w.NWl);
    const uint32_t srow_s = w.slots_s + 2u * srow;
    auto slot_of = [&](int q) -> uint32_t {
        PMS_CHECK((int)lane * w.NWl + q < w.Wp && q < w.NWl);
        if constexpr (SMEM) return lds16(srow_s + 2u * slot_idx(0u, (uint32_t)q, w.NWl));
        else return __ldg(w.gslots + srow + slot_idx(0u, (uint32_t)q, w.NWl));
    };
#ifdef PMS_DEBUG_CHECKS
    // protocol check: the candidate words and the queue counter are clear at
    // the start of every scan (cleared by the previous scan's end)
#pragma unroll
    for (int k = 0; k < C::KW; ++k) PMS_CHECK(lds32(w.acc_s + (k * 32u + lane) * 4u) == 0u);
    if (lane == 0) PMS_CHECK(lds32(w.qc_s()) == 0u);
#endif
#if PMS_SLICE_R0_DIRECT
    // r = 0 hits (~80 %) resolved by the finding lane, no queue: one slot load
    // and one red per hit-iteration (~7 instructions) instead of a queue write
    // and a share of a round (~16); the kernel is issue-bound, not LSU-bound
    {
        const uint32_t acc = w.acc_s;
#if PMS_SLICE_R0_PAIR
        // two hits per iteration: both slot loads in flight together (the
        // second is a repeat of the first when the lane has one hit left)
        while (r0m) {
            const int q = msb(r0m);
            r0m ^= 1u << q;
            const int q2 = r0m ? msb(r0m) : q;
            r0m &= ~(1u << q2);
            const uint32_t sl = slot_of(q), sl2 = slot_of(q2);
            red_or(acc | (sl & 0x7FFu), 1u << (sl >> 11));
            red_or(acc | (sl2 & 0x7FFu), 1u << (sl2 >> 11));
        }
#else
        while (r0m) {
            const int q = msb(r0m);
            r0m ^= 1u << q;
            const uint32_t sl = slot_of(q);
            red_or(acc | (sl & 0x7FFu), 1u << (sl >> 11));
        }
#endif
#if PMS_SLICE_R1_DIRECT
        while (r1m) {
            const int q = msb(r1m);
            r1m ^= 1u << q;
            const uint32_t sl = slot_of(q);
            const uint32_t base = acc | (sl & 0x7FFu);
            const uint32_t row = w.R1_s + (sl >> 11) * (4u * kSR1Stride);
#pragma unroll
            for (int u = 0; u < NU; ++u)
                red_or(base ^ (r1_delta<X>((uint32_t)u) * 4u), lds32(row + (uint32_t)u * 4u));
        }
#endif
    }
#endif
    const uint32_t n012 =
        (uint32_t)__popc(r0m) | ((uint32_t)__popc(r1m) << 10) | ((uint32_t)__popc(r2m) << 20);
    const uint32_t tot = __reduce_add_sync(kFull, n012);
    const uint32_t t0 = tot & 1023u, t1 = (tot >> 10) & 1023u, t2 = tot >> 20;
    if (t0 <= (uint32_t)C::kCap0 && t1 <= (uint32_t)C::kCap1 && t2 <= (uint32_t)C::kCap2) {
        // queue the hits (one atomic claims all three queue positions; a
        // 5-step shuffle prefix sum instead measured +16 % at (15,4)), then
        // resolve them full-width
        if (n012) {
            const uint32_t pos = atom_add(w.qc_s(), n012);
            uint32_t a0 = w.q0_s() + 2u * (pos & 1023u);
            uint32_t a1 = w.q1_s() + 2u * ((pos >> 10) & 1023u);
            uint32_t a2 = w.q2_s() + 4u * (pos >> 20);
            while (r0m) {
                const int q = msb(r0m);
                r0m ^= 1u << q;
                sts16(a0, slot_of(q));
                a0 += 2u;
            }
            while (r1m) {
                const int q = msb(r1m);
                r1m ^= 1u << q;
                sts16(a1, slot_of(q));
                a1 += 2u;
            }
            while (r2m) {
                const int q = msb(r2m);
                r2m ^= 1u << q;
                sts32(a2, slot_of(q) | (slice_r(c, q) << 16));
                a2 += 4u;
            }
        }
        __syncwarp();
        if (lane == 0) sts32(w.qc_s(), 0u);  // claims are done; next use after __syncwarp
        // loop-invariant shared-window addresses, pinned in registers: under the
        // 64-register cap the compiler otherwise re-derives them every round
        uint32_t acc = w.acc_s, qa0 = w.q0_s() + 2u * lane;
        asm volatile("" : "+r"(acc), "+r"(qa0));
        // round loops with warp-uniform trip counts and predicated bodies: a
        // lane-dependent trip count let the warp run on diverged into the
        // broadcasts and the end of scan, executing both twice (measured)
#pragma unroll 1
        for (uint32_t b0 = 0; b0 < t0; b0 += 32u, qa0 += 64u) {
            if (b0 + lane < t0) {
                const uint32_t sl = lds16(qa0);
                PMS_CHECK(sl != kPoison16);
                red_or(acc | (sl & 0x7FFu), 1u << (sl >> 11));
            }
        }
        // hit-major rounds: lane L takes hit b + L and applies all NU updates of
        // its radius-1 ball, one red per update (the own word + 5 lane flips,
        // bits from its padded R1 row; the 3X upper words, centre bit).  Each
        // red instruction then touches one word per hit: few bank conflicts
        // (packing 6 updates of one hit into one instruction put the 3X upper
        // words of a hit -- same lane, same bank -- in one ~7-wavefront red),
        // and no per-lane update decode
        if (t1) {
            uint32_t qh = w.q1_s() + 2u * lane;
            asm volatile("" : "+r"(qh));
#pragma unroll 1
            for (uint32_t b1 = 0; b1 < t1; b1 += 32u, qh += 64u) {
                if (b1 + lane < t1) {
                    const uint32_t sl = lds16(qh);
                    PMS_CHECK(sl != kPoison16);
                    const uint32_t base = acc | (sl & 0x7FFu), e5 = sl >> 11;
                    const uint32_t row = w.R1_s + e5 * (4u * kSR1Stride);
#pragma unroll
                    for (int u = 0; u < 6; ++u)
                        red_or(base ^ (r1_delta<X>((uint32_t)u) * 4u), lds32(row + 4u * (uint32_t)u));
                    const uint32_t cb = 1u << e5;
#pragma unroll
                    for (int u = 6; u < C::NU; ++u) red_or(base ^ (r1_delta<X>((uint32_t)u) * 4u), cb);
                }
            }
        }
        __syncwarp();
        if (w.rclamp) {
#pragma unroll 1
            for (uint32_t b2 = 0; b2 < t2; ++b2) {
                const uint32_t e = lds32(w.q2_s() + 4u * b2);  // same address: broadcast
                PMS_CHECK(e != kPoison32);
                slice_bcast<X, true>(e, w.lane4, w.T_s, w.acc_lane_s, common);
            }
        } else {
#pragma unroll 1
            for (uint32_t b2 = 0; b2 < t2; ++b2) {
                const uint32_t e = lds32(w.q2_s() + 4u * b2);
                PMS_CHECK(e != kPoison32 && (e >> 16) <= 6u);
                slice_bcast<X, false>(e, w.lane4, w.T_s, w.acc_lane_s, common);
            }
        }
#ifdef PMS_DEBUG_CHECKS
        __syncwarp();  // every lane has read its entries: poison them again
        for (uint32_t q = lane; q < t0; q += 32u) sts16(w.q0_s() + 2u * q, kPoison16);
        for (uint32_t q = lane; q < t1; q += 32u) sts16(w.q1_s() + 2u * q, kPoison16);
        for (uint32_t q = lane; q < t2; q += 32u) sts32(w.q2_s() + 4u * q, kPoison32);
#endif
    } else {
        // dense hits (a queue would overflow): per-lane resolution
        while (r0m) {
            const int q = msb(r0m);
            r0m ^= 1u << q;
            const uint32_t sl = slot_of(q);
            red_or(w.acc_s | (sl & 0x7FFu), 1u << (sl >> 11));
        }
        while (r1m) {
            const int q = msb(r1m);
            r1m ^= 1u << q;
            const uint32_t sl = slot_of(q);
            const uint32_t base = w.acc_s | (sl & 0x7FFu);
#pragma unroll
            for (int u = 0; u < NU; ++u)
                red_or(base ^ (r1_delta<X>((uint32_t)u) * 4u),
                       lds32(w.R1_s + ((sl >> 11) * (uint32_t)kSR1Stride + (uint32_t)u) * 4u));
        }
        while (__any_sync(kFull, r2m != 0u)) {
            uint32_t rec = kFull;
            if (r2m) {
                const int q = msb(r2m);
                r2m ^= 1u << q;
                rec = slot_of(q) | (slice_r(c, q) << 16);
            }
            uint32_t who = __ballot_sync(kFull, rec != kFull);
            while (who) {
                const int src = msb(who);
                who ^= 1u << src;
                const uint32_t e = __shfl_sync(kFull, rec, src);
                slice_bcast<X>(e, w.lane4, w.T_s, w.acc_lane_s, common);
            }
        }
    }
}

// End of a scan: alive &= (the lane's words | common); the words are cleared
// for the next scan.  Returns the warp's number of alive candidates -- exact
// whenever it is at most `exact_upto` (the hand-off threshold); above that a
// lower bound > exact_upto is enough for the callers (skip rule: == 0;
// hand-off: <= threshold).  The bound is the popcount of the OR of the
// lane's words, summed over lanes (one POPC instead of KW).
template <int S, bool SMEM>
__device__ __forceinline__ int slice_finish(const SliceWarp<S, SMEM>& w, uint32_t common,
                                            uint32_t (&alive)[SliceCfg<S>::KW], int exact_upto) {
    constexpr int KW = SliceCfg<S>::KW;
    __syncwarp();
    uint32_t any = 0u;
#pragma unroll
    for (int k = 0; k < KW; ++k) {
        const uint32_t wa = w.acc_s + (k * 32u + w.lane) * 4u;
#if PMS_SLICE_EXCH
        alive[k] &= atom_exch0(wa) | common;  // read and clear in one instruction
#else
        alive[k] &= lds32(wa) | common;
        sts32(wa, 0u);
#endif
        any |= alive[k];
    }
    __syncwarp();
    const int lb = __reduce_add_sync(kFull, __popc(any));
    if (lb == 0 || lb > exact_upto) return lb;
    int na = 0;  // small: count exactly (a bit may be set in several words)
#pragma unroll
    for (int k = 0; k < KW; ++k) na += __popc(alive[k]);
    return __reduce_add_sync(kFull, na);
}

// Hand-off check of one candidate (the block's prefix P and the suffix in
// word k, lane `src`, bit `bit` of the block's mask) against sequences i0..n-1
// on the scan's own tables (per candidate, skip rule): P x
// matches sequence i iff some window w with prefix distance p <= d -- a
// pass-1 hit -- has Hamming(x, e_w) <= r = d - p.  The slot of a window holds
// its suffix planes (word k = eH>>5 << X | eL>>5, lane = eH & 31, bit =
// eL & 31), so slot ^ slot(x) gives the suffix mismatches directly.  Staged
// tables: no global-memory round trip per sequence (the packed-word check
// was ~2 us per sequence of L2 latency on a lone warp, the (13,3) tail).
template <int S>
__device__ __forceinline__ uint32_t slice_sfx_dist(uint32_t v) {
    constexpr int X = S - 5;
    uint32_t mm = ((v >> 2) | (v >> 11)) & 31u;
    if constexpr (X > 0) mm |= (((v >> 7) | (v >> (7 + X))) & ((1u << X) - 1u)) << 5;
    return (uint32_t)__popc(mm);
}

template <int S, int LP, bool SMEM>
__device__ __forceinline__ bool slice_check_one(const SliceWarp<S, SMEM>& w, const uint32_t (&po)[LP],
                                                int i0, int n, uint32_t k, uint32_t src,
                                                uint32_t bit, unsigned long long& scanned) {
    const uint32_t sx = ((k * 32u + src) * 4u) | (bit << 11);
    for (int i = i0; i < n; ++i) {
        uint32_t c[5], r0m, r1m, r2m;
        slice_pass1<S, LP, SMEM>(w, po, i, c, r0m, r1m, r2m);
        ++scanned;
        const uint32_t srow = (uint32_t)(i * w.Wp) + slot_idx(w.lane, 0u, w.NWl);
#if PMS_SLICE_CHECK_VOTE
        // The hit classes in the order an occurrence is most likely found --
        // r >= 2, r = 1, r = 0: a planted window at distance d has on average
        // d * LP / l of its mismatches in the prefix, while a chance prefix hit
        // is mostly at prefix distance d (r = 0) -- with warp-uniform trip
        // counts and a vote per iteration, so the warp stops at the first
        // match any lane finds instead of waiting for the lane with most hits
        // (this check is a lone warp's chain, the tail of the latency
        // instances; the result -- some window within d -- is the same)
        auto any_match = [&](uint32_t hv) -> bool {
            const uint32_t trips = __reduce_max_sync(kFull, (uint32_t)__popc(hv));
            for (uint32_t it = 0; it < trips; ++it) {
                bool f = false;
                if (hv) {
                    const int q = msb(hv);
                    hv ^= 1u << q;
                    PMS_CHECK((int)w.lane * w.NWl + q < w.Wp);
                    const uint32_t sl = SMEM ? lds16(w.slots_s + 2u * (srow + slot_idx(0u, (uint32_t)q, w.NWl)))
                                             : (uint32_t)__ldg(w.gslots + srow + slot_idx(0u, (uint32_t)q, w.NWl));
                    f = slice_sfx_dist<S>(sl ^ sx) <= slice_r(c, q);
                }
                if (__any_sync(kFull, f)) return true;
            }
            return false;
        };
        if (!(any_match(r2m) || any_match(r1m) || any_match(r0m))) return false;
#else
        bool f = false;
        uint32_t hv = r0m | r1m | r2m;
        while (hv && !f) {
            const int q = msb(hv);
            hv ^= 1u << q;
            PMS_CHECK((int)w.lane * w.NWl + q < w.Wp);
            const uint32_t sl = SMEM ? lds16(w.slots_s + 2u * (srow + slot_idx(0u, (uint32_t)q, w.NWl)))
                                     : (uint32_t)__ldg(w.gslots + srow + slot_idx(0u, (uint32_t)q, w.NWl));
            f = slice_sfx_dist<S>(sl ^ sx) <= slice_r(c, q);
        }
        if (!__any_sync(kFull, f)) return false;
#endif
    }
    return true;
}

// Sparse mode (the hand-off of the throughput instances): once
// at most a.handoff candidates of the block are alive, the remaining
// sequences are tested per candidate -- still per candidate and in input
// order (PAPER.md:63's skip rule), on the bit-sliced planes of all l
// positions: the block's prefix count (one pass 1 shared by the candidates,
// K + prefix matches, as slice_pass1) plus the candidate's own suffix match
// planes (global, L1/L2), so a window matches iff K + prefix + suffix
// matches >= 16 + S, i.e. at most d mismatches over all l positions -- for a
// lane's windows at once, no per-window or per-hit work.  The candidates'
// suffix codes are listed in the warp's word block (zero between scans), which
// is cleared again before the next block.
template <int N>
__device__ __forceinline__ void slice_count3(const uint32_t (&m)[N], uint32_t& s0, uint32_t& s1,
                                             uint32_t& s2) {
    static_assert(N >= 3 && N <= 7, "suffix digits");
    constexpr int N1 = N / 2, N2 = N1 / 2;
    uint32_t v0[N], y0[N1];
#pragma unroll
    for (int j = 0; j < N; ++j) v0[j] = m[j];
    s0 = csa_col<N>(v0, y0);
    uint32_t y1[N2 > 0 ? N2 : 1];
    s1 = csa_col<N1>(y0, y1);
    s2 = N2 > 0 ? y1[0] : 0u;
}

// One sparse-mode step: does each of the A listed candidates (suffix codes
// in the list at L_s) have a window within d in sequence i?  Bit j of the
// result: candidate j does.
template <int S, int LP, bool SMEM>
__device__ __forceinline__ uint32_t slice_sparse_step(const SliceWarp<S, SMEM>& w, const SliceArgs& a,
                                                      const uint32_t (&po)[LP], int i, uint32_t L_s,
                                                      uint32_t A) {
    constexpr uint32_t kGe = 16u + (uint32_t)S;  // K + matches >= 16 + S <=> <= d mismatches
    const uint32_t lane = w.lane;
    uint32_t m[LP], c[5];
    if constexpr (SMEM) {
        const uint32_t P = w.planes_s + (uint32_t)i * (uint32_t)(LP * 512);
#pragma unroll
        for (int j = 0; j < LP; ++j) m[j] = lds32(P + po[j]);
    } else {
        const char* P = reinterpret_cast<const char*>(w.planes) + (size_t)i * (LP * 512);
#pragma unroll
        for (int j = 0; j < LP; ++j) m[j] = __ldg(reinterpret_cast<const uint32_t*>(P + po[j]));
    }
    slice_count<LP>(m, w.km, c);
    const uint32_t* sp = a.splanes + (size_t)i * (S * 128) + lane;
    // does the candidate with suffix code x have a window within d here?
    // (t = c + suffix matches, five planes plus the carry out of bit 4: c <=
    // 16 + d and the suffix adds <= S, so t < 64; t >= 16 + S bit-sliced from
    // the low bit up, and any t >= 32 qualifies)
    auto test = [&](const uint32_t (&sm)[S]) -> uint32_t {
        uint32_t s0, s1, s2;
        slice_count3<S>(sm, s0, s1, s2);
        const uint32_t t0 = c[0] ^ s0;
        uint32_t k = c[0] & s0;
        const uint32_t t1 = c[1] ^ s1 ^ k;
        k = (c[1] & s1) | (k & (c[1] ^ s1));
        const uint32_t t2 = c[2] ^ s2 ^ k;
        k = (c[2] & s2) | (k & (c[2] ^ s2));
        const uint32_t t3 = c[3] ^ k;
        k = c[3] & k;
        const uint32_t t4 = c[4] ^ k;
        const uint32_t t5 = c[4] & k;  // t >= 32 (only when d + S >= 16)
        const uint32_t t[5] = {t0, t1, t2, t3, t4};
        uint32_t g = kFull;
#pragma unroll
        for (int b = 0; b < 5; ++b) g = ((kGe >> b) & 1u) ? (t[b] & g) : (t[b] | g);
        return (g | t5) & w.vmask;
    };
    uint32_t keep = 0;
    // (two candidates per step, their loads overlapped, measured slower:
    // (15,4) +4 %, (16,5) +1 %)
#pragma unroll 1
    for (uint32_t j = 0; j < A; ++j) {
        const uint32_t x = lds32(L_s + 4u * j);  // broadcast
        uint32_t sm[S];
#pragma unroll
        for (int q = 0; q < S; ++q)
            sm[q] = __ldg(sp + (q * 4 + ((x >> (2 * (S - 1 - q))) & 3u)) * 32u);
        keep |= (uint32_t)__any_sync(kFull, test(sm) != 0u) << j;
    }
    return keep;
}

template <int S, int LP, bool SMEM>
__device__ __forceinline__ void slice_sparse(const SliceWarp<S, SMEM>& w, const SliceArgs& a,
                                             const uint32_t (&po)[LP], int i0,
                                             const uint32_t (&alive)[SliceCfg<S>::KW],
                                             unsigned long long cbase, unsigned long long& scanned) {
    constexpr int KW = SliceCfg<S>::KW;
    const uint32_t lane = w.lane;
    const uint32_t L_s = w.acc_s;  // the list (the word block is zero here)
    uint32_t A = 0;                 // warp-uniform
#pragma unroll
    for (int k = 0; k < KW; ++k) {
        uint32_t hold = __ballot_sync(kFull, alive[k] != 0u);
        while (hold) {
            const int src = __ffs(hold) - 1;
            hold &= hold - 1;
            uint32_t bits = __shfl_sync(kFull, alive[k], src);
            while (bits) {
                const uint32_t b = (uint32_t)__ffs(bits) - 1u;
                bits &= bits - 1;
                PMS_CHECK(A < 32u);
                if (lane == 0) sts32(L_s + 4u * A, blk_sfx<Bp32, S>((uint32_t)src, (uint32_t)k, b));
                ++A;
            }
        }
    }
    __syncwarp();
    const uint32_t A0 = A;
    int i = i0;
    for (; i < a.n && A; ++i) {
        const uint32_t keep = slice_sparse_step<S, LP, SMEM>(w, a, po, i, L_s, A);
        // candidate checks in the low bits, steps from bit kSparseStepShift
        // (DevState.extra; the host splits them)
        scanned += A + (1ull << kSparseStepShift);
        // drop the candidates with no window within d in sequence i
        const uint32_t x = lane < A ? lds32(L_s + 4u * lane) : 0u;
        __syncwarp();
        if (lane < A && ((keep >> lane) & 1u)) sts32(L_s + 4u * (uint32_t)__popc(keep & ((1u << lane) - 1u)), x);
        __syncwarp();
        A = (uint32_t)__popc(keep);
    }
    if (A) {  // survivors of all n sequences
        PMS_CHECK(i == a.n);
        const uint32_t x = lane < A ? lds32(L_s + 4u * lane) : 0u;
        unsigned long long slot = 0;
        if (lane == 0) slot = atomicAdd(a.nout, (unsigned long long)A);
        slot = __shfl_sync(kFull, slot, 0) + lane;
        if (lane < A && slot < a.cap) {
            const unsigned long long code = cbase + x;
            if (a.out_wide) static_cast<unsigned long long*>(a.out)[slot] = code;
            else static_cast<uint32_t*>(a.out)[slot] = (uint32_t)code;
        }
    }
    __syncwarp();
    if (lane < A0) sts32(L_s + 4u * lane, 0u);  // the word block is zero again
    __syncwarp();
}

template <int S, int LP, bool SMEM, bool HT = false>
__global__ void __launch_bounds__(SliceCfg<S>::NT, 1) pms_search_slice(SliceArgs a) {
    using B = BlkTraits<S>;
    using C = SliceCfg<S>;
    constexpr int KW = C::KW;
    [[maybe_unused]] constexpr int NWARP = C::NWARP;  // (trace builds)
    static_assert(LP >= 1 && LP <= kSliceMaxLP, "prefix length");
    // [ball table][candidate words][queues][planes][slots] (SliceCfg); each
    // warp's word block is aligned to its size, so a word index XOR is an
    // address XOR (r = 1 rounds).  Only 128-B alignment of the dynamic window
    // is real (measured base 0xC00), so nothing larger is declared: the
    // compiler would fold it.
    extern __shared__ __align__(128) uint32_t sdyn[];
    __shared__ __align__(8) uint64_t bar;
#ifdef PMS_TRACE
    const unsigned long long tr_enter = gtimer();
    unsigned long long tr_blocks = 0, tr_hand = 0, tr_maxs = 0, tr_maxt = 0;
#endif
    pdl_wait();
    if (*(volatile unsigned int*)&a.st->bad == a.epoch) return;
    const SliceWarp<S, SMEM> w = slice_setup<S, SMEM>(a, sdyn, &bar);
    const uint32_t lane = w.lane;
    unsigned long long scanned = 0, bscans = 0;
#ifdef PMS_TRACE
    const unsigned long long tr_ready = gtimer();
#endif

    for (;;) {
        unsigned long long bgrab = 0;
        if (lane == 0) bgrab = atomicAdd(&a.st->next, (unsigned long long)a.batch);
        bgrab = __shfl_sync(kFull, bgrab, 0);
        if (bgrab >= a.span) break;
        for (int sb = 0; sb < a.batch; sb += B::C) {
            const unsigned long long cbase = a.lo_al + bgrab + sb;
            if (cbase >= a.hi) break;
#ifdef PMS_TRACE
            const unsigned long long tr_b0 = gtimer(), tr_s0 = bscans, tr_h0 = scanned;
            struct TrEnd {
                unsigned long long t0, s0, h0, *maxs, *maxt, *blocks, *hand;
                const unsigned long long *bs, *sc;
                __device__ ~TrEnd() {
                    const unsigned long long dt = gtimer() - t0;
                    if (*bs - s0 > *maxs) *maxs = *bs - s0;
                    if (dt > *maxt) *maxt = dt;
                    ++*blocks;
                    *hand += *sc - h0;
                }
            } tr_end{tr_b0, tr_s0, tr_h0, &tr_maxs, &tr_maxt, &tr_blocks, &tr_hand, &bscans, &scanned};
#endif
            uint32_t po[LP];
            slice_offsets<S, LP>(cbase, lane, po);
            uint32_t alive[KW];
#pragma unroll
            for (int k = 0; k < KW; ++k) alive[k] = kFull;
            if (cbase < a.lo || cbase + B::C > a.hi) {  // edge block of [lo, hi)
#pragma unroll 1
                for (int k = 0; k < KW; ++k) {
                    uint32_t m = 0u;
#pragma unroll 1
                    for (uint32_t bb = 0; bb < 32; ++bb) {
                        const unsigned long long c = cbase + blk_sfx<Bp32, S>(lane, k, bb);
                        if (c >= a.lo && c < a.hi) m |= 1u << bb;
                    }
#pragma unroll
                    for (int q = 0; q < KW; ++q)
                        if (q == k) alive[q] = m;
                }
            }
            int i = 0;
            bool dead = false;
            int nalive = B::C;
            for (; i < a.n; ++i) {
                if (i > 0 && a.skip && nalive <= a.handoff) break;
                uint32_t c[5], r0m, r1m, r2m, common = 0u;
                slice_pass1<S, LP, SMEM>(w, po, i, c, r0m, r1m, r2m);
                slice_pass2<S, SMEM>(w, i, c, r0m, r1m, r2m, common);
                nalive = slice_finish<S, SMEM>(w, common, alive, a.handoff);
                ++bscans;
                if (nalive == 0) {  // skip rule for the whole block
                    dead = true;
                    if (a.skip) break;
                }
            }
            if (dead) continue;
            if (i == a.n) {  // every alive candidate matched all n sequences
#pragma unroll
                for (int k = 0; k < KW; ++k) {
                    if (!alive[k]) continue;
                    unsigned long long slot = atomicAdd(a.nout, (unsigned long long)__popc(alive[k]));
                    for (uint32_t mm = alive[k]; mm; mm &= mm - 1, ++slot) {
                        const unsigned long long code = cbase + blk_sfx<Bp32, S>(lane, k, __ffs(mm) - 1);
                        if (slot < a.cap) {
                            if (a.out_wide) static_cast<unsigned long long*>(a.out)[slot] = code;
                            else static_cast<uint32_t*>(a.out)[slot] = (uint32_t)code;
                        }
                    }
                }
                continue;
            }
            if constexpr (!HT) {
                // throughput instances: sparse mode (the list of at most
                // a.handoff candidates, all remaining sequences)
                slice_sparse<S, LP, SMEM>(w, a, po, i, alive, cbase, scanned);
                continue;
            } else {
                // latency instances: at most a.handoff survivors, each finished
                // from sequence i by the whole warp on the staged tables (a lone
                // warp's chain is the run time here; no L2 round trips)
                for (;;) {
                    uint32_t pick = kFull;
#pragma unroll
                    for (int k = KW - 1; k >= 0; --k)
                        if (alive[k]) pick = ((uint32_t)k << 5) | (__ffs(alive[k]) - 1);
                    const uint32_t holder = __ballot_sync(kFull, pick != kFull);
                    if (!holder) break;
                    const int src = __ffs(holder) - 1;
                    const uint32_t pk = __shfl_sync(kFull, pick, src);
                    const uint32_t k = pk >> 5;
                    if ((int)lane == src) {
#pragma unroll
                        for (int q = 0; q < KW; ++q)
                            if (q == (int)k) alive[q] &= alive[q] - 1;
                    }
                    const unsigned long long code = cbase + blk_sfx<Bp32, S>(src, k, pk & 31u);
                    if (slice_check_one<S, LP, SMEM>(w, po, i, a.n, k, (uint32_t)src, pk & 31u, scanned) &&
                        lane == 0) {
                        const unsigned long long slot = atomicAdd(a.nout, 1ull);
                        if (slot < a.cap) {
                            if (a.out_wide) static_cast<unsigned long long*>(a.out)[slot] = code;
                            else static_cast<uint32_t*>(a.out)[slot] = (uint32_t)code;
                        }
                    }
                }
            }
        }
    }
    if (lane == 0) {
        if (scanned) atomicAdd(&a.st->extra, scanned);
        if (bscans) atomicAdd(&a.st->block_scans, bscans);
    }
#ifdef PMS_TRACE
    const unsigned long long wg = (unsigned long long)blockIdx.x * NWARP + (threadIdx.x >> 5);
    if (lane == 0 && wg < 8192) {
        unsigned long long* r = g_pms_trace + wg * 8;
        r[0] = tr_enter; r[1] = tr_ready; r[2] = gtimer(); r[3] = tr_blocks;
        r[4] = bscans; r[5] = tr_hand; r[6] = tr_maxs; r[7] = tr_maxt;
    }
#endif
}

// ------------------------------------------- sequence-parallel search
// For ranges with few blocks (e.g. (9,2): 256 blocks for 4,736 resident
// warps), the sequential per-block chain of scans is the whole run time.
// Here every (block, sequence) pair is its own work unit: a warp scans one
// sequence for one block (alive starts full), ANDs the result into the
// block's global mask, and the unit that completes the block's n-th sequence
// emits the survivors.  The set is the definition's (AND over sequences of
// "has a window within d"); the sequential skip rule is replaced by a dead
// flag: once a block's AND is empty its remaining units skip the scan.
template <int S, int LP>
__global__ void __launch_bounds__(SliceCfg<S>::NT, 1) pms_search_slice_sp(SliceArgs a) {
    using B = BlkTraits<S>;
    using C = SliceCfg<S>;
    constexpr int KW = C::KW;
    [[maybe_unused]] constexpr int NWARP = C::NWARP;  // (trace builds)
    extern __shared__ __align__(128) uint32_t sdyn[];
    __shared__ __align__(8) uint64_t bar;
#ifdef PMS_TRACE
    const unsigned long long tr_enter = gtimer();
    unsigned long long tr_units = 0;
#endif
    pdl_wait();
    if (*(volatile unsigned int*)&a.st->bad == a.epoch) return;
    const SliceWarp<S, true> w = slice_setup<S, true>(a, sdyn, &bar);
    const uint32_t lane = w.lane;
    const unsigned long long nunits = a.sp_blocks * (unsigned long long)a.n;
    unsigned long long bscans = 0;
#ifdef PMS_TRACE
    const unsigned long long tr_ready = gtimer();
#endif
    for (;;) {
        unsigned long long u = 0;
        if (lane == 0) u = atomicAdd(&a.st->next, 1ull);
        u = __shfl_sync(kFull, u, 0);
        if (u >= nunits) break;
#ifdef PMS_TRACE
        ++tr_units;
#endif
        const unsigned long long b = u / (unsigned)a.n;
        const int i = (int)(u - b * (unsigned)a.n);
        const unsigned long long cbase = a.lo_al + (b << (2 * S));
        uint32_t* gmask = a.spmask + b * (32ull * KW);
        uint32_t flag = 0;
        if (lane == 0) flag = *(volatile uint32_t*)&a.spcnt[b];
        flag = __shfl_sync(kFull, flag, 0);
        if (!(flag & kSpDead)) {
            uint32_t po[LP];
            slice_offsets<S, LP>(cbase, lane, po);
            uint32_t alive[KW];
#pragma unroll
            for (int k = 0; k < KW; ++k) alive[k] = kFull;
            if (cbase < a.lo || cbase + B::C > a.hi) {  // edge block of [lo, hi)
#pragma unroll 1
                for (int k = 0; k < KW; ++k) {
                    uint32_t m = 0u;
#pragma unroll 1
                    for (uint32_t bb = 0; bb < 32; ++bb) {
                        const unsigned long long c = cbase + blk_sfx<Bp32, S>(lane, k, bb);
                        if (c >= a.lo && c < a.hi) m |= 1u << bb;
                    }
#pragma unroll
                    for (int q = 0; q < KW; ++q)
                        if (q == k) alive[q] = m;
                }
            }
            uint32_t c[5], r0m, r1m, r2m, common = 0u;
            slice_pass1<S, LP, true>(w, po, i, c, r0m, r1m, r2m);
            slice_pass2<S, true>(w, i, c, r0m, r1m, r2m, common);
            slice_finish<S, true>(w, common, alive, 0);
            ++bscans;
            uint32_t left = 0u;
#pragma unroll
            for (int k = 0; k < KW; ++k) left |= atomicAnd(gmask + k * 32 + lane, alive[k]) & alive[k];
            if (!__any_sync(kFull, left != 0u) && lane == 0) atomicOr(&a.spcnt[b], kSpDead);
        }
        __threadfence();  // the AND is visible before this unit counts as done
        uint32_t done = 0;
        if (lane == 0) done = atomicAdd(&a.spcnt[b], 1u) & 0xFFFFu;
        done = __shfl_sync(kFull, done, 0);
        if (done == (uint32_t)a.n - 1u) {  // the block's last unit: emit its survivors
            __threadfence();
#pragma unroll
            for (int k = 0; k < KW; ++k) {
                const uint32_t m = __ldcg(gmask + k * 32 + lane);
                if (!m) continue;
                unsigned long long slot = atomicAdd(a.nout, (unsigned long long)__popc(m));
                for (uint32_t mm = m; mm; mm &= mm - 1, ++slot) {
                    const unsigned long long code = cbase + blk_sfx<Bp32, S>(lane, k, __ffs(mm) - 1);
                    if (slot < a.cap) {
                        if (a.out_wide) static_cast<unsigned long long*>(a.out)[slot] = code;
                        else static_cast<uint32_t*>(a.out)[slot] = (uint32_t)code;
                    }
                }
            }
        }
    }
    if (lane == 0 && bscans) atomicAdd(&a.st->block_scans, bscans);
#ifdef PMS_TRACE
    const unsigned long long wg = (unsigned long long)blockIdx.x * NWARP + (threadIdx.x >> 5);
    if (lane == 0 && wg < 8192) {  // [enter, ready, end, units, scans, 0, 0, 0]
        unsigned long long* r = g_pms_trace + wg * 8;
        r[0] = tr_enter; r[1] = tr_ready; r[2] = gtimer(); r[3] = tr_units;
        r[4] = bscans; r[5] = 0; r[6] = 0; r[7] = 0;
    }
#endif
}

// ------------------------------------------------- roofline microbenchmark
// The search kernel's per-scan code on the same tables, with everything
// dynamic removed: no work counter, no skip rule, no hand-off, no output.
// Warp g walks blocks g, g + warps, g + 2 warps, ... (as the search's
// one-block grabs do: the warps running at any time hold neighbouring blocks,
// which share most plane rows) and scans each against sequences 0 ..
// depth-1, depth = the last execution's scans per block (the mix the skip
// rule produced); every warp stays busy for `scans` scans.  Both matter
// when the tables are read through L1/L2.
//   MODE 0: pass 1 only (plane loads + carry-save classification) -> R_pass1
//   MODE 1: pass 1 + hit resolution + end of scan at the instance's own hit
//           mix (alive reset each scan) -> R_scan
//   MODE 2: sparse-mode steps, a list of a.handoff candidates per step (the
//           last execution's mean list size) -> R_sparse
//   MODE 3: the launch's own mix: MODE 1 scans with a.batch / 65536 sparse
//           steps interleaved per scan (the last execution's ratio) -> R_mix
template <int S, int LP, bool SMEM, int MODE>
__global__ void __launch_bounds__(SliceCfg<S>::NT, 1) pms_roofline_slice(SliceArgs a, int scans,
                                                                        int depth,
                                                                        unsigned long long nblocks,
                                                                        unsigned long long* sink) {
    using C = SliceCfg<S>;
    constexpr int KW = C::KW, NWARP = C::NWARP;
    extern __shared__ __align__(128) uint32_t sdyn[];
    __shared__ __align__(8) uint64_t bar;
    const SliceWarp<S, SMEM> w = slice_setup<S, SMEM>(a, sdyn, &bar);
    const unsigned long long warps = (unsigned long long)gridDim.x * NWARP;
    const unsigned long long g = (unsigned long long)blockIdx.x * NWARP + (threadIdx.x >> 5);
    uint32_t acc = 0;
    unsigned long long blk = g % nblocks;
    const unsigned long long bstep = warps % nblocks;
    int i = 0;
    const uint32_t A = (uint32_t)min(max(a.handoff, 1), 32);
    // a fixed pseudo-random candidate list per warp (modes 2, 3)
    const uint32_t xl = (uint32_t)((g * 32u + w.lane) * 2654435761ull) & ((1u << (2 * S)) - 1u);
    if (MODE == 2 && w.lane < A) sts32(w.acc_s + 4u * w.lane, xl);
    __syncwarp();
    // mode 3: sparse steps owed, 16.16 fixed point (a.batch per scan); the
    // warps start at staggered fractions, so their sparse steps do not all
    // fall on the same scans (in the search they come whenever a block's
    // survivors drop below the threshold)
    uint32_t credit = (uint32_t)(g * 40503u) & 0xFFFFu;
    // the block's plane offsets change with the block, not with the scan (as in
    // the search kernel: computed once per block)
    uint32_t po[LP];
    slice_offsets<S, LP>(blk << (2 * S), w.lane, po);
#pragma unroll 1
    for (int k = 0; k < scans; ++k) {
        if (i == 0 && k) slice_offsets<S, LP>(blk << (2 * S), w.lane, po);
        if constexpr (MODE == 2) {
            acc ^= slice_sparse_step<S, LP, SMEM>(w, a, po, i, w.acc_s, A);
            if (++i == depth) {
                i = 0;
                blk += bstep;  // = (blk + warps) % nblocks without a 64-bit division per block
                if (blk >= nblocks) blk -= nblocks;
            }
            continue;
        }
        uint32_t c[5], r0m, r1m, r2m, common = 0u;
        slice_pass1<S, LP, SMEM>(w, po, i, c, r0m, r1m, r2m);
        if (MODE == 0) {
            acc ^= r0m ^ (r1m << 1) ^ (r2m << 2);
        } else {
            slice_pass2<S, SMEM>(w, i, c, r0m, r1m, r2m, common);
            // (alive reset every scan: keeping it live across a block's scans,
            // as the search must, measured 3.7 % slower -- register pressure --
            // so this is the higher, more conservative ceiling)
            uint32_t alive[KW];
#pragma unroll
            for (int q = 0; q < KW; ++q) alive[q] = kFull;
            acc += (uint32_t)slice_finish<S, SMEM>(w, common, alive, a.handoff);
            if constexpr (MODE == 3) {
                // the launch's own mix: a.batch / 65536 sparse steps per dense
                // scan, interleaved, the list written into the (zero) word
                // block and cleared again as the search kernel does
                credit += (uint32_t)a.batch;
                if (credit >= 65536u) {
                    if (w.lane < A) sts32(w.acc_s + 4u * w.lane, xl);
                    __syncwarp();
                    do {
                        credit -= 65536u;
                        acc ^= slice_sparse_step<S, LP, SMEM>(w, a, po, i, w.acc_s, A);
                    } while (credit >= 65536u);
                    __syncwarp();
                    if (w.lane < A) sts32(w.acc_s + 4u * w.lane, 0u);
                    __syncwarp();
                }
            }
        }
        if (++i == depth) {
            i = 0;
            blk += bstep;  // = (blk + warps) % nblocks without a 64-bit division per block
            if (blk >= nblocks) blk -= nblocks;
        }
    }
    if (acc == 0x9E3779B9u) sink[0] = acc;  // keeps the work live
}

}  // namespace
