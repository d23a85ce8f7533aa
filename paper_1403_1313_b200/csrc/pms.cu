// pms.cu -- B200 (sm_100a) Skip-Brute-Force planted (l,d) motif search:
// device pre-pass, persistent search kernels, roofline microbenchmark, and
// the host orchestration behind the C ABI of include/pms.h.
//
// Hot path:
//   a1 validate + stage        host checks (PMS_E_ARG), H2D copy
//   a2 pack pre-pass           pms_pack_kernel: bytes -> bit-plane window words,
//                              byte check (PMS_E_CHAR) -- PAPER.md:63, :77
//   a3 candidate enumeration   64-bit atomic work counter over code ranges;
//                              the candidate is generated from its index
//   a4 Hamming test            XOR / XOR-OR fold with rotated operands / POPC
//   a5 per-sequence match      lanes split windows, warp vote; the skip rule
//      + skip rule             abandons a candidate at the first sequence with no
//                              window within d
//   a6 result append           atomicAdd slot + store ("output the motif")
//   a7 finish                  D2H count + codes, host sort (ascending codes)
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <new>
#include <vector>

#include "pms.h"
#include "pms_device.cuh"

using namespace pms;

namespace {

#define PMS_NW_LIST(X) \
    X(1) X(2) X(3) X(4) X(5) X(6) X(7) X(8) X(10) X(12) X(14) X(16) X(19) X(22) X(25) X(28) \
    X(31) X(34) X(37) X(40) X(44) X(48)

constexpr int kSub = 256;          // candidates per aligned sub-block (4 low digits)
constexpr int kBlock = 256;        // threads per CTA (8 warps)
constexpr uint32_t kFull = 0xFFFFFFFFu;

// Diagnostics for PMS_E_CUDA: the source line and the CUDA error string of the
// last failure on this host thread (pms_last_error).
thread_local char g_last_error[256] = "";
int fail_cuda(int line, cudaError_t e = cudaSuccess) {
    if (e == cudaSuccess) e = cudaPeekAtLastError();
    snprintf(g_last_error, sizeof(g_last_error), "pms.cu:%d: %s", line,
             e == cudaSuccess ? "(no CUDA error pending)" : cudaGetErrorString(e));
    return PMS_E_CUDA;
}

// bit-plane word of every 4-digit value i (the low 4 digits of a candidate)
__constant__ uint32_t c_bp256[kSub];

struct SearchArgs {
    const uint32_t* tab;            // packed table [n][Wp] (global)
    int n, W, Wp;
    uint32_t d2;                    // 2*min(d, l): popc(x|rot16(x)) = 2*Hamming
    unsigned long long lo, hi;      // candidate code range [lo, hi)
    unsigned long long lo_al;       // lo rounded down to the plan unit (256 or 4^S)
    unsigned long long span;        // hi - lo_al
    int batch;                      // candidates per atomic grab (multiple of kSub)
    int in_smem;                    // stage the table into shared memory (TMA bulk)
    int skip;                       // 1 = skip rule (skip-BF); 0 = plain brute force
    int handoff;                    // block family: <= this many survivors -> per-candidate
    uint32_t tab_bytes;
    DevState* st;
    unsigned long long* nout;       // result counter (caller's d_count)
    uint32_t* out;                  // result buffer, capacity cap
    unsigned long long cap;
};

// ------------------------------------------------------------------ a2 pre-pass
// One thread per (sequence i, window k < Wp).  Window k (the length-l
// substring starting at k, k in [0, W)) is packed into a bit-plane word; rows
// are padded to Wp (multiple of 32) with copies of window W-1, which cannot
// change "some window is within d".  Every byte lies in at least one window,
// so the byte check covers the whole input.
__global__ void pms_pack_kernel(const uint8_t* __restrict__ seqs, int n, int t, int l, int W,
                                int Wp, uint32_t* __restrict__ tab, DevState* st) {
    const long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (idx >= (long long)n * Wp) return;
    const int i = (int)(idx / Wp);
    const int k = (int)(idx - (long long)i * Wp);
    const uint8_t* p = seqs + (long long)i * t + min(k, W - 1);
    uint32_t H = 0, L = 0, bad = 0;
    PMS_CHECK(min(k, W - 1) + l <= t);
    for (int j = 0; j < l; ++j) {
        const uint32_t u = p[j] & 0xDFu;  // upper-case; only 'x'/'X' map to 'X'
        const uint32_t code = u == 'A' ? 0u : u == 'C' ? 1u : u == 'G' ? 2u : u == 'T' ? 3u : 4u;
        bad |= code >> 2;
        H = (H << 1) | ((code >> 1) & 1u);
        L = (L << 1) | (code & 1u);
    }
    tab[idx] = (H << 16) | L;
    if (bad) atomicOr(&st->bad, 1u);
}

// ------------------------------------------------------------- shared pieces
// Stage the packed table into shared memory with one TMA bulk copy per 64 KB,
// completion tracked by an mbarrier (transaction bytes).
__device__ __forceinline__ void stage_table(const SearchArgs& a, uint32_t* stab, uint64_t* bar) {
    if (threadIdx.x == 0) mbar_init(bar, 1);
    __syncthreads();
    if (threadIdx.x == 0) {
        mbar_expect_tx(bar, a.tab_bytes);
        constexpr uint32_t kChunk = 65536;
        for (uint32_t off = 0; off < a.tab_bytes; off += kChunk) {
            const uint32_t bytes = min(kChunk, a.tab_bytes - off);
            tma_bulk_g2s(reinterpret_cast<char*>(stab) + off,
                         reinterpret_cast<const char*>(a.tab) + off, bytes, bar);
        }
    }
    mbar_wait(bar, 0);
}

// a4+a5 for sequences [i0, n) with the whole warp on one candidate: lanes take
// windows k = lane, lane+32, ...; one vote per sequence; the first sequence
// with no window within d abandons the candidate (skip rule).
__device__ __forceinline__ bool check_sequences(const uint32_t* tab, int i0, int n, int Wp,
                                                uint32_t cb, uint32_t d2, int lane,
                                                unsigned long long& scanned, bool skip = true) {
    const uint32_t cr = rot16(cb);
    bool all = true;
    for (int i = i0; i < n; ++i) {
        const uint32_t* row = tab + (size_t)i * Wp;
        uint32_t m = 0xFFu;
#pragma unroll 4
        for (int k = lane; k < Wp; k += 32) {
            PMS_CHECK(i < n && k < Wp);
            const uint32_t w = row[k];
            m = min(m, mism2(cb, cr, w, rot16(w)));
        }
        ++scanned;
        if (!__any_sync(kFull, m <= d2)) {
            all = false;
            if (skip) return false;  // skip rule: abandon at the first failing sequence
        }
    }
    return all;
}

// a6: atomic-append compaction
__device__ __forceinline__ void append(const SearchArgs& a, uint32_t code) {
    const unsigned long long slot = atomicAdd(a.nout, 1ull);
    if (slot < a.cap) a.out[slot] = code;
}

// -------------------------------------------------- a3-a6 persistent search
// Register-resident variant.  G lanes per candidate (G = 16: two candidates
// per warp iteration; G = 32: one); each lane keeps NW windows of sequence 0
// (k = hl + G*j, clamped to W-1) and their rotations in registers, since
// sequence 0 is scanned for every candidate.  Survivors of sequence 0 are
// checked against sequences 1..n-1 from shared memory by the whole warp.
template <int G, int NW, bool SMEM>
__global__ void __launch_bounds__(kBlock) pms_search_reg(SearchArgs a) {
    extern __shared__ __align__(128) uint32_t stab[];
    __shared__ __align__(8) uint64_t bar;
    if (*(volatile unsigned int*)&a.st->bad) return;  // invalid input: no work
    if (SMEM) stage_table(a, stab, &bar);
    const uint32_t* tab = SMEM ? stab : a.tab;

    constexpr int CPI = 32 / G;  // candidates per warp iteration
    const int lane = threadIdx.x & 31;
    const uint32_t half = (G == 32) ? 0u : (uint32_t)(lane / G);
    const int hl = lane % G;
    uint32_t w[NW], wr[NW];
#pragma unroll
    for (int j = 0; j < NW; ++j) {
        w[j] = tab[min(hl + G * j, a.W - 1)];
        wr[j] = rot16(w[j]);
    }
    unsigned long long scanned = 0;
    for (;;) {
        unsigned long long b = 0;
        if (lane == 0) b = atomicAdd(&a.st->next, (unsigned long long)a.batch);
        b = __shfl_sync(kFull, b, 0);
        if (b >= a.span) break;
        for (int sb = 0; sb < a.batch; sb += kSub) {
            const unsigned long long cbase = a.lo_al + b + sb;
            if (cbase >= a.hi) break;
            const uint32_t ubp = code_to_bp((uint32_t)cbase);
            const bool whole = cbase >= a.lo && cbase + kSub <= a.hi;
            for (int it = 0; it < kSub; it += CPI) {
                const uint32_t cb = ubp | c_bp256[it] | half;
                const uint32_t cr = rot16(cb);
                uint32_t m = 0xFFu;
#pragma unroll
                for (int j = 0; j < NW; ++j) m = min(m, mism2(cb, cr, w[j], wr[j]));
                bool hit = m <= a.d2;
                if (!whole) {
                    const unsigned long long code = cbase + it + half;
                    hit = hit && code >= a.lo && code < a.hi;
                }
                const uint32_t bal = __ballot_sync(kFull, hit);
                if (bal) {
#pragma unroll
                    for (int h = 0; h < CPI; ++h) {
                        const uint32_t hb = (G == 32) ? bal : ((bal >> (16 * h)) & 0xFFFFu);
                        if (hb) {
                            const uint32_t cbh = ubp | c_bp256[it] | (uint32_t)h;
                            if (check_sequences(tab, 1, a.n, a.Wp, cbh, a.d2, lane, scanned) &&
                                lane == 0)
                                append(a, (uint32_t)(cbase + it + h));
                        }
                    }
                }
            }
        }
    }
    if (lane == 0 && scanned) atomicAdd(&a.st->extra, scanned);
}

// Generic variant (any W; table in shared or global memory): the whole warp
// takes one candidate and scans sequences 0..n-1 with the skip rule (or, with
// a.skip == 0, without it: the plain brute force the skip rule enhances).
template <bool SMEM>
__global__ void __launch_bounds__(kBlock) pms_search_generic(SearchArgs a) {
    extern __shared__ __align__(128) uint32_t stab[];
    __shared__ __align__(8) uint64_t bar;
    if (*(volatile unsigned int*)&a.st->bad) return;
    if (SMEM) stage_table(a, stab, &bar);
    const uint32_t* tab = SMEM ? stab : a.tab;
    const int lane = threadIdx.x & 31;
    unsigned long long scanned = 0;
    for (;;) {
        unsigned long long b = 0;
        if (lane == 0) b = atomicAdd(&a.st->next, (unsigned long long)a.batch);
        b = __shfl_sync(kFull, b, 0);
        if (b >= a.span) break;
        for (int sb = 0; sb < a.batch; sb += kSub) {
            const unsigned long long cbase = a.lo_al + b + sb;
            if (cbase >= a.hi) break;
            const uint32_t ubp = code_to_bp((uint32_t)cbase);
            for (int it = 0; it < kSub; ++it) {
                const unsigned long long code = cbase + it;
                if (code < a.lo || code >= a.hi) continue;
                if (check_sequences(tab, 0, a.n, a.Wp, ubp | c_bp256[it], a.d2, lane, scanned,
                                    a.skip != 0) &&
                    lane == 0)
                    append(a, (uint32_t)code);
            }
        }
    }
    if (lane == 0 && scanned) atomicAdd(&a.st->extra, scanned);
}

// ------------------------------------------------- PMS_ALGO_BLOCK search
// The 4^S candidates of a 4^S-aligned code block (S = 5 or 6) share their
// first l-S digits (the prefix P) and differ in the last S (the suffix x).
// For a window w, Hamming(P x, w) = Hamming(P, w[0..l-S)) + Hamming(x,
// w[l-S..l)), so one XOR / XOR-OR fold / POPC of the prefix against w gives p,
// and the block candidates that match w (distance <= d) are
// exactly the suffixes within Hamming distance d - p of w's suffix.  After a
// sequence, alive &= acc (the candidates with a window within d in it); the
// block is abandoned at the first sequence that leaves no candidate alive --
// the skip rule on 4^S candidates at once -- and a lone survivor is finished
// by the whole warp (check_sequences).
//
// Candidates are indexed in BIT-PLANE order.  A suffix has planes (H, L) of S
// bits (H = high bits, L = low bits of its base codes, position l-S in bit
// S-1); its distance to a window suffix (eH, eL) is popc((H ^ eH) | (L ^ eL)).
// With X = S - 5: lane = H >> X, mask word k = (H & (2^X-1)) << X | (L >> 5)
// (4^X words per lane), bit = L & 31.
//   * a hit with no budget left (p == d, ~80 % of hits) matches only the
//     window's own suffix: the finding lane sets bit eL & 31 of word
//     (eH << X) | (eL >> 5) of the warp's shared-memory mask (one atomic OR);
//   * other hits are broadcast (one SHFL) and every lane ORs, per word, the
//     table entry T[r-1][eL & 31][mm] with mm = (H ^ eH) | ((L >> 5 ^ eL >> 5) << 5):
//     bit b set iff popc(mm | (b ^ (eL & 31))) <= r.  mm is the fastest index,
//     so a broadcast reads (nearly) distinct banks.
constexpr int kUnitMax = 4096;              // largest block (S = 6)
static_assert(kUnitMax % kSub == 0, "batches hold whole 256-candidate sub-blocks");
constexpr int kBlockB = 512;                // max threads per CTA of the block kernel
constexpr int kBlkMinL = 5;                 // the block family needs l >= 5

template <int S>
struct BlkTraits {
    static constexpr int X = S - 5;
    static constexpr int C = 1 << (2 * S);               // candidates per block
    static constexpr int KW = 1 << (2 * X);              // mask words per lane
    static constexpr uint32_t M = (1u << S) - 1u;        // suffix plane mask
    static constexpr uint32_t SFX = M | (M << 16);       // suffix bits of a word
    static constexpr int TROW = 32 << S;                 // words per budget row
    static constexpr int TWORDS = S * TROW;              // rows r = 1..S (r = S: all)
};

template <int S>
__device__ __forceinline__ void build_suffix_table(uint32_t* T) {
    using B = BlkTraits<S>;
    for (int idx = threadIdx.x; idx < B::TWORDS; idx += blockDim.x) {
        const uint32_t mm = idx & B::M, eL = (idx >> S) & 31;
        const int r = idx / B::TROW + 1;
        uint32_t word = 0;
        for (uint32_t b = 0; b < 32; ++b)
            if ((int)__popc(mm | (b ^ eL)) <= r) word |= 1u << b;
        T[idx] = word;
    }
}

// Suffix code (S digits, big-endian base 4) of the suffix with planes (H, L).
__device__ __forceinline__ uint32_t sfx_code(uint32_t h, uint32_t l) {
    return (spread_even(h) << 1) | spread_even(l);
}

// Process every pending hit of every lane (hm bits index the lane's windows
// row[lane + 32*j]) and OR the matching candidates into the lane's acc words.
template <int S>
__device__ __forceinline__ void drain_hits(uint32_t hm, const uint32_t* row, int wp, uint32_t cb,
                                           uint32_t d2, int lane, const uint32_t* T,
                                           uint32_t* wmask,
                                           uint32_t (&acc)[BlkTraits<S>::KW]) {
    (void)wp;  // row length (windows), used by the debug bounds checks
    using B = BlkTraits<S>;
    while (__any_sync(kFull, hm != 0u)) {
        uint32_t mine = kFull;
        if (hm) {
            const int j = __ffs(hm) - 1;
            hm &= hm - 1;
            PMS_CHECK(lane + 32 * j < wp);
            const uint32_t w = row[lane + 32 * j];
            const uint32_t x = (cb ^ w) & ~B::SFX;
            const uint32_t p2 = __popc(x | rot16(x));
            const uint32_t eH = (w >> 16) & B::M, eL = w & B::M;
            if (p2 == d2) {
                PMS_CHECK(((eH << B::X) | (eL >> 5)) < 32u * B::KW);
                atomicOr(&wmask[(eH << B::X) | (eL >> 5)], 1u << (eL & 31u));
            } else {  // record: (r-1) row, eL & 31, eH in the low S bits, eL >> 5 on top
                const uint32_t r = min((d2 - p2) >> 1, (uint32_t)S);
                mine = ((((r - 1) << 5) | (eL & 31u)) << S) | eH | ((eL >> 5) << 24);
            }
        }
        uint32_t who = __ballot_sync(kFull, mine != kFull);
        while (who) {
            const int src = __ffs(who) - 1;
            who &= who - 1;
            const uint32_t v = __shfl_sync(kFull, mine, src);
            if (B::X == 0) {
                PMS_CHECK((v ^ (uint32_t)lane) < (uint32_t)B::TWORDS);
                acc[0] |= T[v ^ (uint32_t)lane];
            } else {
                const uint32_t vx = v & 0x00FFFFFFu, eLt = v >> 24;
#pragma unroll
                for (int k = 0; k < B::KW; ++k) {
                    const uint32_t hk = ((uint32_t)lane << B::X) | ((uint32_t)k >> B::X);
                    const uint32_t lt = (uint32_t)k & ((1u << B::X) - 1u);
                    PMS_CHECK(((vx ^ hk) | ((lt ^ eLt) << 5)) < (uint32_t)B::TWORDS);
                    acc[k] |= T[(vx ^ hk) | ((lt ^ eLt) << 5)];
                }
            }
        }
    }
    __syncwarp();
#pragma unroll
    for (int k = 0; k < B::KW; ++k) {
        acc[k] |= wmask[lane * B::KW + k];
        wmask[lane * B::KW + k] = 0u;
    }
    __syncwarp();
}

// NW > 0: rows are padded to 32*NW windows and the window loops are fully
// unrolled; for NW <= kReg0Max the lane also keeps windows lane + 32j of
// sequence 0 in registers, pre-masked (suffix bits cleared) and pre-rotated
// (larger NW would cost occupancy: all sequences then stream from smem).
constexpr int kReg0Max = 24;
template <int S, bool SMEM, int NW>
__global__ void __launch_bounds__(kBlockB, 2) pms_search_block(SearchArgs a) {
    using B = BlkTraits<S>;
    constexpr bool kReg0 = NW > 0 && NW <= kReg0Max;
    extern __shared__ __align__(128) uint32_t stab[];  // [T][table if SMEM]
    __shared__ __align__(8) uint64_t bar;
    __shared__ uint32_t wmasks[kBlockB / 32][32 * B::KW];  // per-warp single-candidate hits
    if (*(volatile unsigned int*)&a.st->bad) return;
    uint32_t* T = stab;
    uint32_t* wmask = wmasks[threadIdx.x >> 5];
#pragma unroll
    for (int k = 0; k < B::KW; ++k) wmask[(threadIdx.x & 31) * B::KW + k] = 0u;
    uint32_t* tsm = stab + B::TWORDS;  // 128-B aligned for the bulk copy
    if (SMEM) {  // start the table's TMA bulk copy, build the suffix table meanwhile
        if (threadIdx.x == 0) mbar_init(&bar, 1);
        __syncthreads();
        if (threadIdx.x == 0) {
            mbar_expect_tx(&bar, a.tab_bytes);
            constexpr uint32_t kChunk = 65536;
            for (uint32_t off = 0; off < a.tab_bytes; off += kChunk)
                tma_bulk_g2s(reinterpret_cast<char*>(tsm) + off,
                             reinterpret_cast<const char*>(a.tab) + off,
                             min(kChunk, a.tab_bytes - off), &bar);
        }
    }
    build_suffix_table<S>(T);
    __syncthreads();
    if (SMEM) mbar_wait(&bar, 0);
    const uint32_t* tab = SMEM ? tsm : a.tab;
    const int lane = threadIdx.x & 31;
    uint32_t wm[kReg0 ? NW : 1], wmr[kReg0 ? NW : 1];
#pragma unroll
    for (int j = 0; j < (kReg0 ? NW : 0); ++j) {
        wm[j] = tab[min(lane + 32 * j, a.W - 1)] & ~B::SFX;
        wmr[j] = rot16(wm[j]);
    }
    unsigned long long scanned = 0, bscans = 0;

    for (;;) {
        unsigned long long b = 0;
        if (lane == 0) b = atomicAdd(&a.st->next, (unsigned long long)a.batch);
        b = __shfl_sync(kFull, b, 0);
        if (b >= a.span) break;
        for (int sb = 0; sb < a.batch; sb += B::C) {
            const unsigned long long cbase = a.lo_al + b + sb;
            if (cbase >= a.hi) break;
            const uint32_t cb = code_to_bp((uint32_t)cbase);  // suffix bits are zero
            const uint32_t cr = rot16(cb);
            // this lane's candidates inside [lo, hi)
            uint32_t alive[B::KW];
#pragma unroll
            for (int k = 0; k < B::KW; ++k) alive[k] = kFull;
            if (cbase < a.lo || cbase + B::C > a.hi) {  // edge block of [lo, hi)
#pragma unroll
                for (int k = 0; k < B::KW; ++k) {
                    const uint32_t h = ((uint32_t)lane << B::X) | ((uint32_t)k >> B::X);
                    const uint32_t lt = (uint32_t)k & ((1u << B::X) - 1u);
                    uint32_t m = 0u;
                    for (uint32_t bb = 0; bb < 32; ++bb) {
                        const unsigned long long c = cbase + sfx_code(h, (lt << 5) | bb);
                        if (c >= a.lo && c < a.hi) m |= 1u << bb;
                    }
                    alive[k] = m;
                }
            }
            int i = 0;
            bool dead = false;
            for (; i < a.n; ++i) {
                if (i > 0 && a.skip) {
                    int na = 0;
#pragma unroll
                    for (int k = 0; k < B::KW; ++k) na += __popc(alive[k]);
                    if (__reduce_add_sync(kFull, na) <= a.handoff) break;
                }
                const uint32_t* row = tab + (size_t)i * a.Wp;
                uint32_t acc[B::KW];
#pragma unroll
                for (int k = 0; k < B::KW; ++k) acc[k] = 0u;
                // pass 1: prefix distance of each window; hits recorded per lane
                if (NW > 0) {
                    uint32_t hm = 0;
                    if (kReg0 && i == 0) {
#pragma unroll
                        for (int j = 0; j < (kReg0 ? NW : 0); ++j)
                            if (__popc((cb ^ wm[j]) | (cr ^ wmr[j])) <= a.d2) hm |= 1u << j;
                    } else {
#pragma unroll
                        for (int j = 0; j < NW; ++j) {
                            PMS_CHECK(lane + 32 * j < a.Wp && i < a.n);
                            const uint32_t x = (cb ^ row[lane + 32 * j]) & ~B::SFX;
                            if (__popc(x | rot16(x)) <= a.d2) hm |= 1u << j;
                        }
                    }
                    // pass 2: resolve the hits into each lane's candidate words
                    drain_hits<S>(hm, row, a.Wp, cb, a.d2, lane, T, wmask, acc);
                } else {
                    for (int k0 = 0; k0 < a.Wp; k0 += 32 * 32) {  // 32 windows per lane per chunk
                        uint32_t hm = 0;
                        const int nj = min(a.Wp - k0, 32 * 32) / 32;
                        for (int j = 0; j < nj; ++j) {
                            PMS_CHECK(k0 + lane + 32 * j < a.Wp && i < a.n);
                            const uint32_t x = (cb ^ row[k0 + lane + 32 * j]) & ~B::SFX;
                            if (__popc(x | rot16(x)) <= a.d2) hm |= 1u << j;
                        }
                        drain_hits<S>(hm, row + k0, a.Wp - k0, cb, a.d2, lane, T, wmask, acc);
                    }
                }
                uint32_t any = 0;
#pragma unroll
                for (int k = 0; k < B::KW; ++k) {
                    alive[k] &= acc[k];
                    any |= alive[k];
                }
                ++bscans;
                if (!__any_sync(kFull, any != 0u)) {  // skip rule for the whole block
                    dead = true;
                    if (a.skip) break;  // (a.skip == 0: plain brute force scans on)
                }
            }
            if (dead) continue;
            if (i == a.n) {  // every alive candidate matched all n sequences
#pragma unroll
                for (int k = 0; k < B::KW; ++k) {
                    if (!alive[k]) continue;
                    const uint32_t h = ((uint32_t)lane << B::X) | ((uint32_t)k >> B::X);
                    const uint32_t lt = (uint32_t)k & ((1u << B::X) - 1u);
                    unsigned long long slot = atomicAdd(a.nout, (unsigned long long)__popc(alive[k]));
                    for (uint32_t m = alive[k]; m; m &= m - 1, ++slot)
                        if (slot < a.cap)
                            a.out[slot] = (uint32_t)(cbase + sfx_code(h, (lt << 5) | (__ffs(m) - 1)));
                }
                continue;
            }
            // at most a.handoff survivors left: the whole warp finishes each one
            // from sequence i on with the per-candidate check
            for (;;) {
                uint32_t pick = kFull;  // (k << 5) | bit of this lane's first alive candidate
#pragma unroll
                for (int k = B::KW - 1; k >= 0; --k)
                    if (alive[k]) pick = ((uint32_t)k << 5) | (__ffs(alive[k]) - 1);
                const uint32_t holder = __ballot_sync(kFull, pick != kFull);
                if (!holder) break;
                const int src = __ffs(holder) - 1;
                const uint32_t pk = __shfl_sync(kFull, pick, src);
                const uint32_t k = pk >> 5;
                if (lane == src) {
#pragma unroll
                    for (int q = 0; q < B::KW; ++q)
                        if (q == (int)k) alive[q] &= alive[q] - 1;  // clear the picked bit
                }
                const uint32_t h = ((uint32_t)src << B::X) | (k >> B::X);
                const uint32_t l5 = ((k & ((1u << B::X) - 1u)) << 5) | (pk & 31u);
                const uint32_t code = (uint32_t)(cbase + sfx_code(h, l5));
                if (check_sequences(tab, i, a.n, a.Wp, code_to_bp(code), a.d2, lane, scanned) &&
                    lane == 0)
                    append(a, code);
            }
        }
    }
    if (lane == 0) {
        if (scanned) atomicAdd(&a.st->extra, scanned);
        if (bscans) atomicAdd(&a.st->block_scans, bscans);
    }
}

using BlockFn = void (*)(SearchArgs);
struct BlockKernel {
    int S, NW;
    BlockFn fn_smem, fn_global;
};
#define PMS_BLK5(nw) {5, nw, pms_search_block<5, true, nw>, pms_search_block<5, false, nw>},
#define PMS_BLK6(nw) {6, nw, pms_search_block<6, true, nw>, pms_search_block<6, false, nw>},
const BlockKernel kBlockKernels[] = {
    {5, 0, pms_search_block<5, true, 0>, pms_search_block<5, false, 0>},
    {6, 0, pms_search_block<6, true, 0>, pms_search_block<6, false, 0>},
    PMS_NW_LIST(PMS_BLK5) PMS_NW_LIST(PMS_BLK6)};

// ---------------------------------------------------- roofline microbenchmark
// The exact per-compare sequence of pms_search_reg<G,NW> (same register-
// resident windows, same candidate generation, same vote), with no early exit
// and no survivor path: compares/clk/SM of this loop is R_mix.
template <int G, int NW>
__global__ void __launch_bounds__(kBlock) pms_roofline_kernel(const uint32_t* __restrict__ tab,
                                                              int iters, uint32_t d2,
                                                              unsigned long long* sink) {
    constexpr int CPI = 32 / G;
    const int lane = threadIdx.x & 31;
    const uint32_t half = (G == 32) ? 0u : (uint32_t)(lane / G);
    const int hl = lane % G;
    uint32_t w[NW], wr[NW];
#pragma unroll
    for (int j = 0; j < NW; ++j) {
        w[j] = tab[hl + G * j];
        wr[j] = rot16(w[j]);
    }
    uint32_t hits = 0;
    const uint32_t ubp0 = code_to_bp(blockIdx.x * 65536u + (threadIdx.x >> 5) * 1024u);
    for (int sb = 0; sb < iters; sb += kSub) {
        const uint32_t ubp = ubp0 + (uint32_t)sb;  // varies the candidate stream
        for (int it = 0; it < kSub; it += CPI) {
            const uint32_t cb = ubp | c_bp256[it] | half;
            const uint32_t cr = rot16(cb);
            uint32_t m = 0xFFu;
#pragma unroll
            for (int j = 0; j < NW; ++j) m = min(m, mism2(cb, cr, w[j], wr[j]));
            hits += __ballot_sync(kFull, m <= d2) != 0u;
        }
    }
    if (hits == 0xFFFFFFFFu) sink[0] = hits;  // never true; keeps the work live
}

// ------------------------------------------------------ kernel instance table
using SearchFn = void (*)(SearchArgs);
struct RegKernel {
    int G, NW;
    SearchFn fn_smem, fn_global;
};
#define PMS_REG16(nw) {16, nw, pms_search_reg<16, nw, true>, pms_search_reg<16, nw, false>},
#define PMS_REG32(nw) {32, nw, pms_search_reg<32, nw, true>, pms_search_reg<32, nw, false>},
const RegKernel kRegKernels[] = {PMS_NW_LIST(PMS_REG16) PMS_NW_LIST(PMS_REG32)};

bool pick_reg_kernel(int W, int force_g, RegKernel* best) {
    bool found = false;
    int best_waste = 0;
    for (const RegKernel& k : kRegKernels) {
        if (force_g && k.G != force_g) continue;
        if (k.G * k.NW < W) continue;
        const int waste = k.G * k.NW - W;
        // smallest NW per G is the first that fits (list ascending); prefer less
        // padding, then G = 32 (half the registers for the same padding)
        if (!found || waste < best_waste || (waste == best_waste && k.G > best->G)) {
            *best = k;
            best_waste = waste;
            found = true;
        }
    }
    return found;
}

int ensure_constants() {
    static thread_local int dev_done[64] = {0};
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return fail_cuda(__LINE__);
    if (dev_done[dev]) return PMS_OK;
    uint32_t h[kSub];
    for (int i = 0; i < kSub; ++i) h[i] = code_to_bp((uint32_t)i);
    if (cudaMemcpyToSymbol(c_bp256, h, sizeof(h)) != cudaSuccess) return fail_cuda(__LINE__);
    dev_done[dev] = 1;
    return PMS_OK;
}

}  // namespace

// ========================================================================
//                                   plan
// ========================================================================
struct pms_plan {
    int n = 0, t = 0, l = 0, d = 0, W = 0, Wp = 0;
    int dev = 0, sms = 0;
    pms_launch launch{};
    uint32_t* d_table = nullptr;
    DevState* d_state = nullptr;
    DevState* h_state = nullptr;  // pinned mirror, filled after each execution
    cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};  // start, packed, searched, state copied
    SearchFn fn = nullptr;
    int G = 32, NW = 0, generic = 0, in_smem = 0, algo = PMS_ALGO_CANDIDATE, S = 0;
    uint32_t tab_bytes = 0, smem_bytes = 0;
    int grid = 0, block = kBlock, batch = kSub;
    unsigned long long last_lo = 0, last_hi = 0;
    bool executed = false;
};

namespace {

int check_shape(int32_t n, int32_t t, int32_t l, int32_t d) {
    if (n < 1 || t < 1 || l < 1 || l > PMS_MAX_L || l > t || d < 0) return PMS_E_ARG;
    if ((long long)n * t > 0x7FFFFFFFLL) return PMS_E_TOO_LARGE;
    const long long W = t - l + 1, Wp = (W + 31) / 32 * 32;
    if (n * Wp * 4 > 0x7FFFFFFFLL) return PMS_E_TOO_LARGE;
    return PMS_OK;
}

void destroy_plan(pms_plan* p) {
    if (!p) return;
    cudaFree(p->d_table);
    cudaFree(p->d_state);
    cudaFreeHost(p->h_state);
    for (cudaEvent_t e : p->ev)
        if (e) cudaEventDestroy(e);
    delete p;
}

}  // namespace

extern "C" int pms_plan_create(int32_t n, int32_t t, int32_t l, int32_t d,
                               const pms_launch* launch, pms_plan** plan) {
    if (!plan) return PMS_E_ARG;
    *plan = nullptr;
    int st = check_shape(n, t, l, d);
    if (st != PMS_OK) return st;
    pms_plan* p = new (std::nothrow) pms_plan();
    if (!p) return fail_cuda(__LINE__);
    p->n = n; p->t = t; p->l = l; p->d = d;
    p->W = t - l + 1;
    p->Wp = (p->W + 31) / 32 * 32;
    if (launch) p->launch = *launch;
    int smem_optin = 0;
    if (cudaGetDevice(&p->dev) != cudaSuccess ||
        cudaDeviceGetAttribute(&p->sms, cudaDevAttrMultiProcessorCount, p->dev) != cudaSuccess ||
        cudaDeviceGetAttribute(&smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, p->dev) !=
            cudaSuccess ||
        ensure_constants() != PMS_OK) {
        destroy_plan(p);
        return fail_cuda(__LINE__);
    }
    // block family: AUTO or explicit; with no_skip only when asked for explicitly
    // (AUTO + no_skip keeps the per-candidate plain brute force)
    const bool block_algo =
        (p->launch.algo == PMS_ALGO_BLOCK || (p->launch.algo == PMS_ALGO_AUTO && !p->launch.no_skip)) &&
        l >= kBlkMinL;
    // block digits S: 6 (4096-candidate blocks) when there are enough blocks to
    // keep every warp busy (l >= 13: >= 16k blocks), else 5
    int S = p->launch.block_digits == 5 || p->launch.block_digits == 6 ? p->launch.block_digits
                                                                        : (l >= 13 ? 6 : 5);
    if (S > l) S = 5;
    const BlockKernel* bk = nullptr;
    if (block_algo) {
        for (const BlockKernel& k : kBlockKernels)  // generic (NW = 0) of this S first
            if (k.S == S && k.NW == 0) { bk = &k; break; }
        if (!p->launch.force_generic)
            for (const BlockKernel& k : kBlockKernels)  // smallest register tile covering W
                if (k.S == S && k.NW > 0 && 32 * k.NW >= p->W) {
                    bk = &k;
                    p->Wp = 32 * k.NW;  // rows padded to the tile (re-read on hits)
                    break;
                }
        p->S = S;
    }
    p->tab_bytes = (uint32_t)((size_t)n * p->Wp * 4);
    const uint32_t static_smem = 12288;  // mbarrier, per-warp hit masks, slack
    const uint32_t ball_bytes =
        block_algo ? (uint32_t)(S == 6 ? BlkTraits<6>::TWORDS : BlkTraits<5>::TWORDS) * 4u : 0u;
    p->in_smem = !p->launch.table_global &&
                 p->tab_bytes + ball_bytes + static_smem <= (uint32_t)smem_optin;
    // block family: a table that leaves room for only one CTA per SM is read
    // through L1/L2 instead -- two resident CTAs win (measured at (16,5):
    // 8.6 ms vs 9.9 ms); 228 KB of shared memory per SM, 1 KB reserved per CTA
    if (block_algo && p->in_smem && 2u * (p->tab_bytes + ball_bytes + static_smem + 1024u) > 233472u)
        p->in_smem = 0;
    p->smem_bytes = ball_bytes + (p->in_smem ? p->tab_bytes : 0);

    RegKernel rk{};
    const int force_g = (p->launch.lanes_per_cand == 16 || p->launch.lanes_per_cand == 32)
                            ? p->launch.lanes_per_cand
                            : 0;
    if (block_algo) {
        p->fn = p->in_smem ? bk->fn_smem : bk->fn_global;
        p->G = 32; p->NW = bk->NW; p->generic = 0; p->algo = PMS_ALGO_BLOCK;
    } else if (!p->launch.force_generic && !p->launch.no_skip &&
               pick_reg_kernel(p->W, force_g, &rk)) {
        p->fn = p->in_smem ? rk.fn_smem : rk.fn_global;
        p->G = rk.G; p->NW = rk.NW; p->generic = 0; p->algo = PMS_ALGO_CANDIDATE;
    } else {
        p->fn = p->in_smem ? pms_search_generic<true> : pms_search_generic<false>;
        p->G = 32; p->NW = 0; p->generic = 1; p->algo = PMS_ALGO_CANDIDATE;
    }
    const int max_block = p->algo == PMS_ALGO_BLOCK ? kBlockB : kBlock;  // __launch_bounds__
    p->block = p->launch.warps_per_cta > 0 ? 32 * std::min(p->launch.warps_per_cta, 32)
                                           : (p->algo == PMS_ALGO_BLOCK ? kBlockB : kBlock);
    if (p->block > max_block) p->block = max_block;
    // The attribute is per kernel, shared by every plan (and pooled context)
    // that launches it: raise it to the device maximum, never to this plan's
    // size, or a later smaller plan would break an earlier larger one.
    cudaFuncAttributes fa{};
    if (cudaFuncGetAttributes(&fa, (const void*)p->fn) != cudaSuccess ||
        p->smem_bytes + fa.sharedSizeBytes > (size_t)smem_optin ||
        cudaFuncSetAttribute((const void*)p->fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             smem_optin - (int)fa.sharedSizeBytes) != cudaSuccess) {
        destroy_plan(p);
        return fail_cuda(__LINE__);
    }
    int occ = 0;
    if (p->algo == PMS_ALGO_BLOCK && p->launch.warps_per_cta <= 0) {
        // block family: pick the CTA size with the most resident warps per SM
        int best = 0;
        for (int blk = kBlockB; blk >= 256; blk -= 64) {
            int o = 0;
            if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, (const void*)p->fn, blk,
                                                              p->smem_bytes) != cudaSuccess)
                continue;
            if (o * blk > best) { best = o * blk; p->block = blk; occ = o; }
        }
    } else if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, (const void*)p->fn, p->block,
                                                             p->smem_bytes) != cudaSuccess) {
        occ = 0;
    }
    if (occ < 1) {
        destroy_plan(p);
        return fail_cuda(__LINE__);
    }
    if (p->launch.ctas_per_sm > 0) occ = std::min(occ, (int)p->launch.ctas_per_sm);
    p->grid = p->sms * occ;
    if (p->launch.grid_ctas > 0) p->grid = std::min((int)p->launch.grid_ctas, p->grid);
    if (cudaMalloc(&p->d_table, p->tab_bytes) != cudaSuccess ||
        cudaMalloc(&p->d_state, sizeof(DevState)) != cudaSuccess ||
        cudaMallocHost(&p->h_state, sizeof(DevState)) != cudaSuccess) {
        destroy_plan(p);
        return fail_cuda(__LINE__);
    }
    for (cudaEvent_t& e : p->ev)
        if (cudaEventCreate(&e) != cudaSuccess) {
            destroy_plan(p);
            return fail_cuda(__LINE__);
        }
    *plan = p;
    return PMS_OK;
}

extern "C" void pms_plan_destroy(pms_plan* plan) { destroy_plan(plan); }

extern "C" int pms_plan_execute(pms_plan* p, const uint8_t* d_seqs, uint64_t lo, uint64_t hi,
                                uint32_t* d_out, uint64_t cap, uint64_t* d_count, void* stream) {
    if (!p || !d_seqs || !d_count || (!d_out && cap > 0)) return PMS_E_ARG;
    const unsigned long long total = 1ull << (2 * p->l);
    if (hi > total) hi = total;
    if (lo > hi) return PMS_E_ARG;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    // batches and lo are aligned to the plan's unit: one block (4^S candidates)
    // for the block family, a 256-candidate sub-block for the candidate family
    const unsigned long long kUnit =
        p->algo == PMS_ALGO_BLOCK ? (1ull << (2 * p->S)) : (unsigned long long)kSub;
    const unsigned long long lo_al = lo / kUnit * kUnit;
    const unsigned long long span = hi - lo_al;

    // batch: aim for >= 8 grabs per warp, multiple of kSub, at most 16 sub-blocks
    const unsigned long long warps = (unsigned long long)p->grid * (p->block / 32);
    int batch = p->launch.batch > 0 ? (int)((p->launch.batch + kUnit - 1) / kUnit * kUnit) : 0;
    if (batch == 0) {
        unsigned long long b = span / (warps * 8);
        b = (b + kUnit - 1) / kUnit * kUnit;
        batch = (int)std::min<unsigned long long>(std::max<unsigned long long>(b, kUnit),
                                                  std::max<unsigned long long>(4 * kUnit, 4096));
    }
    p->batch = batch;
    p->last_lo = lo;
    p->last_hi = hi;

    SearchArgs a{};
    a.tab = p->d_table; a.n = p->n; a.W = p->W; a.Wp = p->Wp;
    a.d2 = 2u * (uint32_t)std::min(p->d, p->l);
    a.lo = lo; a.hi = hi; a.lo_al = lo_al; a.span = span; a.batch = batch;
    a.in_smem = p->in_smem; a.tab_bytes = p->tab_bytes;
    a.skip = p->launch.no_skip ? 0 : 1;
    a.handoff = p->launch.handoff > 0 ? p->launch.handoff : (p->d >= 5 ? 3 : 1);  // measured
    a.st = p->d_state; a.nout = reinterpret_cast<unsigned long long*>(d_count);
    a.out = d_out; a.cap = cap;

    if (cudaEventRecord(p->ev[0], s) != cudaSuccess) return fail_cuda(__LINE__);
    if (cudaMemsetAsync(p->d_state, 0, sizeof(DevState), s) != cudaSuccess ||
        cudaMemsetAsync(d_count, 0, sizeof(uint64_t), s) != cudaSuccess)
        return fail_cuda(__LINE__);
    const long long cells = (long long)p->n * p->Wp;
    pms_pack_kernel<<<(unsigned)((cells + 255) / 256), 256, 0, s>>>(d_seqs, p->n, p->t, p->l, p->W,
                                                                     p->Wp, p->d_table, p->d_state);
    const cudaError_t e_pack = cudaGetLastError();
    if (e_pack != cudaSuccess) return fail_cuda(__LINE__, e_pack);
    if (cudaEventRecord(p->ev[1], s) != cudaSuccess) return fail_cuda(__LINE__);
    if (span > 0) {
        p->fn<<<p->grid, p->block, p->smem_bytes, s>>>(a);
        const cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return fail_cuda(__LINE__, e);
    }
    if (cudaEventRecord(p->ev[2], s) != cudaSuccess) return fail_cuda(__LINE__);
    if (cudaMemcpyAsync(p->h_state, p->d_state, sizeof(DevState), cudaMemcpyDeviceToHost, s) !=
        cudaSuccess)
        return fail_cuda(__LINE__);
    if (cudaEventRecord(p->ev[3], s) != cudaSuccess) return fail_cuda(__LINE__);
    p->executed = true;
    return PMS_OK;
}

extern "C" int pms_plan_wait(pms_plan* p, pms_stats* stats) {
    if (!p || !p->executed) return PMS_E_ARG;
    if (cudaEventSynchronize(p->ev[3]) != cudaSuccess) return fail_cuda(__LINE__);
    if (stats) {
        float pack = 0.f, search = 0.f, tot = 0.f;
        cudaEventElapsedTime(&pack, p->ev[0], p->ev[1]);
        cudaEventElapsedTime(&search, p->ev[1], p->ev[2]);
        cudaEventElapsedTime(&tot, p->ev[0], p->ev[2]);
        stats->pack_ms = pack;
        stats->search_ms = search;
        stats->total_ms = tot;
        const unsigned long long cands = p->last_hi - p->last_lo;
        stats->candidates = cands;
        const unsigned long long W = (unsigned long long)p->W;
        // candidate family: W compares per candidate on sequence 0 (register
        // path) + W per further sequence scanned.  Block family: W prefix
        // compares per (block, sequence) scan + W per per-candidate scan.
        const bool seq0_implicit = !p->generic && p->algo == PMS_ALGO_CANDIDATE;
        stats->issued_compares =
            p->h_state->bad ? 0
                            : (seq0_implicit ? cands * W : 0) +
                                  (p->h_state->extra + p->h_state->block_scans) * W;
        stats->algo = p->algo;
        stats->block_scans = p->h_state->block_scans;
        stats->block_digits = p->S;
        stats->motifs = 0;
        stats->grid = p->grid;
        stats->block = p->block;
        stats->lanes_per_cand = p->G;
        stats->windows_per_lane = p->NW;
        stats->generic = p->generic;
        stats->table_in_smem = p->in_smem;
        stats->smem_bytes = p->smem_bytes;
    }
    return p->h_state->bad ? PMS_E_CHAR : PMS_OK;
}

// ========================================================================
//                              host entry points
// ========================================================================
namespace {

// A reusable host-call context: plan + device buffers + stream + pinned count.
// pms_find/pms_find_ex keep idle contexts in a small process-wide pool keyed
// by (device, shape, launch) so repeated calls skip allocation and setup.
struct CallCtx {
    int dev = 0;
    int32_t n = 0, t = 0, l = 0, d = 0;
    pms_launch launch{};
    pms_plan* plan = nullptr;
    uint8_t* d_seqs = nullptr;
    uint32_t* d_out = nullptr;
    unsigned long long out_cap = 0;
    uint64_t* d_count = nullptr;
    uint64_t* h_count = nullptr;  // pinned
    uint8_t* h_seqs = nullptr;    // pinned staging of the input (n*t bytes)
    uint32_t* h_out = nullptr;    // pinned staging of small result sets
    static constexpr unsigned long long kHostOutCap = 1ull << 16;
    cudaStream_t stream = nullptr;

    bool matches(int dv, int32_t n_, int32_t t_, int32_t l_, int32_t d_,
                 const pms_launch& L) const {
        return dev == dv && n == n_ && t == t_ && l == l_ && d == d_ &&
               std::memcmp(&launch, &L, sizeof(L)) == 0;
    }
    void release_resources() {
        destroy_plan(plan);
        cudaFree(d_seqs);
        cudaFree(d_out);
        cudaFree(d_count);
        cudaFreeHost(h_count);
        cudaFreeHost(h_seqs);
        cudaFreeHost(h_out);
        if (stream) cudaStreamDestroy(stream);
    }
};

std::mutex g_pool_mu;
std::vector<CallCtx*> g_pool;
constexpr size_t kPoolMax = 8;

void ctx_destroy(CallCtx* c) {
    if (!c) return;
    c->release_resources();
    delete c;
}

int ctx_acquire(int32_t n, int32_t t, int32_t l, int32_t d, const pms_launch& L, CallCtx** out) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return fail_cuda(__LINE__);
    {
        std::lock_guard<std::mutex> lk(g_pool_mu);
        for (size_t i = 0; i < g_pool.size(); ++i)
            if (g_pool[i]->matches(dev, n, t, l, d, L)) {
                *out = g_pool[i];
                g_pool.erase(g_pool.begin() + (long)i);
                return PMS_OK;
            }
    }
    CallCtx* c = new (std::nothrow) CallCtx();
    if (!c) return fail_cuda(__LINE__);
    c->dev = dev; c->n = n; c->t = t; c->l = l; c->d = d; c->launch = L;
    int st = pms_plan_create(n, t, l, d, &L, &c->plan);
    if (st != PMS_OK) {
        delete c;
        return st;
    }
    if (cudaMalloc(&c->d_seqs, (size_t)n * t) != cudaSuccess ||
        cudaMalloc(&c->d_count, sizeof(uint64_t)) != cudaSuccess ||
        cudaMallocHost(&c->h_count, sizeof(uint64_t)) != cudaSuccess ||
        cudaMallocHost(&c->h_seqs, (size_t)n * t) != cudaSuccess ||
        cudaMallocHost(&c->h_out, CallCtx::kHostOutCap * sizeof(uint32_t)) != cudaSuccess ||
        cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking) != cudaSuccess) {
        ctx_destroy(c);
        return fail_cuda(__LINE__);
    }
    *out = c;
    return PMS_OK;
}

void ctx_release(CallCtx* c) {
    std::lock_guard<std::mutex> lk(g_pool_mu);
    if (g_pool.size() < kPoolMax) {
        g_pool.push_back(c);
        return;
    }
    ctx_destroy(c);
}

}  // namespace

extern "C" int pms_find_ex(const uint8_t* seqs, int32_t n, int32_t t, int32_t l, int32_t d,
                           uint64_t lo, uint64_t hi, const pms_launch* launch, uint32_t* out_codes,
                           uint64_t max_out, uint64_t* count, pms_stats* stats) {
    // a1: argument checks in the documented order
    if (!seqs || !count || (!out_codes && max_out > 0)) return PMS_E_ARG;
    int st = check_shape(n, t, l, d);
    if (st != PMS_OK) return st;
    const unsigned long long total = 1ull << (2 * l);
    if (hi > total) hi = total;
    if (lo > hi) return PMS_E_ARG;
    *count = 0;

    const pms_launch L = launch ? *launch : pms_launch{};
    CallCtx* c = nullptr;
    st = ctx_acquire(n, t, l, d, L, &c);
    if (st != PMS_OK) return st;
    bool healthy = true;
    struct Guard {
        CallCtx* c;
        bool* healthy;
        ~Guard() {
            if (*healthy) ctx_release(c);
            else ctx_destroy(c);
        }
    } guard{c, &healthy};

    const unsigned long long cap = std::min<unsigned long long>(max_out, hi - lo);
    if (cap > c->out_cap) {  // grow the result buffer (kept for the next call)
        cudaFree(c->d_out);
        c->d_out = nullptr;
        c->out_cap = 0;
        if (cudaMalloc(&c->d_out, cap * sizeof(uint32_t)) != cudaSuccess) {
            healthy = false;
            return fail_cuda(__LINE__);
        }
        c->out_cap = cap;
    }
    cudaStream_t s = c->stream;
    std::memcpy(c->h_seqs, seqs, (size_t)n * t);  // pinned staging: the H2D is a true async DMA
    if (cudaMemcpyAsync(c->d_seqs, c->h_seqs, (size_t)n * t, cudaMemcpyHostToDevice, s) !=
        cudaSuccess) {
        healthy = false;
        return fail_cuda(__LINE__);
    }
    st = pms_plan_execute(c->plan, c->d_seqs, lo, hi, c->d_out, cap, c->d_count, s);
    if (st != PMS_OK) {
        healthy = false;
        return st;
    }
    if (cudaMemcpyAsync(c->h_count, c->d_count, sizeof(uint64_t), cudaMemcpyDeviceToHost, s) !=
        cudaSuccess) {
        healthy = false;
        return fail_cuda(__LINE__);
    }
    st = pms_plan_wait(c->plan, stats);
    if (cudaStreamSynchronize(s) != cudaSuccess) {
        healthy = false;
        return fail_cuda(__LINE__);
    }
    if (st == PMS_E_CUDA) healthy = false;
    if (st != PMS_OK) return st;
    const uint64_t found = *c->h_count;
    if (stats) stats->motifs = found;
    *count = found;
    if (found > max_out) return PMS_E_TRUNCATED;
    // a7: D2H of the codes, host sort (ascending code = lexicographic order)
    if (found > 0) {
        const bool staged = found <= CallCtx::kHostOutCap;
        if (cudaMemcpyAsync(staged ? c->h_out : out_codes, c->d_out, found * sizeof(uint32_t),
                            cudaMemcpyDeviceToHost, s) != cudaSuccess ||
            cudaStreamSynchronize(s) != cudaSuccess) {
            healthy = false;
            return fail_cuda(__LINE__);
        }
        if (staged) std::memcpy(out_codes, c->h_out, found * sizeof(uint32_t));
        std::sort(out_codes, out_codes + found);
    }
    return PMS_OK;
}

extern "C" int pms_find(const uint8_t* seqs, int32_t n, int32_t t, int32_t l, int32_t d,
                        uint32_t* out_codes, uint64_t max_out, uint64_t* count) {
    return pms_find_ex(seqs, n, t, l, d, 0, ~0ull, nullptr, out_codes, max_out, count, nullptr);
}

extern "C" int pms_roofline(int32_t iters, double* compares_per_s, double* compares_per_clk_sm,
                            double* ms) {
    if (iters < kSub || !compares_per_s) return PMS_E_ARG;
    iters = iters / kSub * kSub;
    constexpr int G = 16, NW = 37;  // the (15,4) n=20 t=600 headline shape (W = 586)
    int dev = 0, sms = 0, clk = 0;
    if (cudaGetDevice(&dev) != cudaSuccess ||
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess ||
        cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev) != cudaSuccess ||
        ensure_constants() != PMS_OK)
        return fail_cuda(__LINE__);
    uint32_t h[G * NW];
    uint32_t x = 0x9E3779B9u;
    for (int i = 0; i < G * NW; ++i) {  // arbitrary 15-mer windows
        x = x * 1664525u + 1013904223u;
        h[i] = code_to_bp(x >> 2);
    }
    uint32_t* tab = nullptr;
    unsigned long long* sink = nullptr;
    if (cudaMalloc(&tab, sizeof(h)) != cudaSuccess ||
        cudaMalloc(&sink, sizeof(unsigned long long)) != cudaSuccess) {
        cudaFree(tab);
        return fail_cuda(__LINE__);
    }
    cudaMemcpy(tab, h, sizeof(h), cudaMemcpyHostToDevice);
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, pms_roofline_kernel<G, NW>, kBlock, 0);
    const int grid = sms * std::max(occ, 1);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    pms_roofline_kernel<G, NW><<<grid, kBlock>>>(tab, kSub, 8u, sink);  // warm-up
    float best = 1e30f;
    for (int r = 0; r < 3; ++r) {
        cudaEventRecord(e0);
        pms_roofline_kernel<G, NW><<<grid, kBlock>>>(tab, iters, 8u, sink);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float t = 0.f;
        cudaEventElapsedTime(&t, e0, e1);
        best = std::min(best, t);
    }
    const cudaError_t err = cudaGetLastError();
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(tab);
    cudaFree(sink);
    if (err != cudaSuccess) return fail_cuda(__LINE__);
    // compares per launch: warps * (iters / CPI) iterations * 32 lanes * NW slots
    const double warps = (double)grid * (kBlock / 32);
    const double cmp = warps * ((double)iters / (32 / G)) * 32.0 * NW;
    *compares_per_s = cmp / (best * 1e-3);
    if (compares_per_clk_sm) *compares_per_clk_sm = *compares_per_s / ((double)sms * clk * 1e3);
    if (ms) *ms = best;
    return PMS_OK;
}

extern "C" const char* pms_last_error(void) { return g_last_error; }

extern "C" int64_t pms_debug_violations(int32_t reset) {
#ifdef PMS_DEBUG_CHECKS
    if (cudaDeviceSynchronize() != cudaSuccess) return -2;
    unsigned int v = 0;
    if (cudaMemcpyFromSymbol(&v, pms::g_pms_violations, sizeof(v)) != cudaSuccess) return -2;
    if (reset) {
        const unsigned int z = 0;
        cudaMemcpyToSymbol(pms::g_pms_violations, &z, sizeof(z));
    }
    return (int64_t)v;
#else
    (void)reset;
    return -1;
#endif
}

extern "C" const char* pms_strerror(int status) {
    switch (status) {
        case PMS_OK: return "ok";
        case PMS_E_ARG: return "invalid argument";
        case PMS_E_CHAR: return "byte outside ACGTacgt in the input";
        case PMS_E_TOO_LARGE: return "input too large";
        case PMS_E_CUDA: return "CUDA device error (no device, allocation, launch or runtime)";
        case PMS_E_TRUNCATED: return "more motifs than max_out (count is exact)";
        default: return "unknown status";
    }
}

extern "C" int pms_device_info(int32_t* sms, int32_t* smem_optin_bytes, int32_t* clock_khz) {
    int dev = 0, a = 0, b = 0, c = 0;
    if (cudaGetDevice(&dev) != cudaSuccess ||
        cudaDeviceGetAttribute(&a, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess ||
        cudaDeviceGetAttribute(&b, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) != cudaSuccess ||
        cudaDeviceGetAttribute(&c, cudaDevAttrClockRate, dev) != cudaSuccess)
        return fail_cuda(__LINE__);
    if (sms) *sms = a;
    if (smem_optin_bytes) *smem_optin_bytes = b;
    if (clock_khz) *clock_khz = c;
    return PMS_OK;
}
