// pms_kernels.cuh -- the search kernels shared by both window-word widths.
//
// Included by pms.cu (32-bit words, l <= 16) and pms64.cu (64-bit words,
// l <= 31); each translation unit instantiates its own word policy, so the
// kernel templates live in an anonymous namespace (TU-local stubs) while the
// argument / table types shared with the host code live in namespace pms.
//
// Word policies:
//   Bp32  one uint32 per window: H plane in bits 16..31, L plane in 0..15;
//         distances come out doubled (popc over both rotated halves).
//   Bp64  one uint2 per window: .x = H plane, .y = L plane, position j of the
//         l-mer at bit l-1-j of each plane (l <= 31); the
//         distance is popc((cH ^ wH) | (cL ^ wL)) (PAPER.md:63 Hamming).
// Both expose a candidate as a uint2 register pair so a compare is always
// popc((c.x ^ e.x) | (c.y ^ e.y)) on an "expanded" window e.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "pms_device.cuh"

namespace pms {

struct SearchArgs {
    const void* tab;                // packed table [n][Wp] of P::word (global)
    int n, W, Wp;
    uint32_t dd;                    // candidate-family register kernel: 2*min(d, l) (mism2 is doubled)
    uint32_t dp;                    // every other test: min(d, l) (plain Hamming)
    unsigned long long lo, hi;      // candidate code range [lo, hi)
    unsigned long long lo_al;       // lo rounded down to the plan unit (256 or 4^S)
    unsigned long long span;        // hi - lo_al
    int batch;                      // candidates per atomic grab (multiple of the unit)
    int in_smem;                    // stage the table into shared memory (TMA bulk)
    int skip;                       // 1 = skip rule (skip-BF); 0 = plain brute force
    int handoff;                    // block family: <= this many survivors -> per-candidate
    int out_wide;                   // 1 = result codes are uint64, 0 = uint32
    uint32_t tab_bytes;
    const uint32_t* ball;           // the ball table T in global memory (built once per device)
    DevState* st;
    uint32_t epoch;                 // this step's id; st->bad == epoch: invalid input
    unsigned long long* nout;       // result counter (caller's d_count)
    void* out;                      // result buffer, capacity cap (uint32 or uint64)
    unsigned long long cap;
};

using SearchFn = void (*)(SearchArgs);
using PackFn = void (*)(const uint8_t*, int, int, int, int, int, void*, DevState*,
                        unsigned long long*, uint32_t);

struct BlockKernel {
    int S, NW;
    SearchFn fn_smem, fn_global;
};

constexpr int kBlock = 256;        // threads per CTA of the candidate family (8 warps)
#ifndef PMS_BLK_MAX_THREADS
#define PMS_BLK_MAX_THREADS 512
#endif
constexpr int kBlockB = PMS_BLK_MAX_THREADS;  // max threads per CTA of the block family
constexpr int kUnitMax = 4096;     // largest block (S = 6)
constexpr int kBlkMinL = 5;        // the block family needs l >= 5
// Sequence 0 streams from shared memory like the other sequences: a
// register-resident copy (38 registers at NW = 19) forced the drain loop to
// rematerialise addresses under the 64-register cap (measured at (15,4):
// 0.563 ms with it, 0.520 ms without).
// Block family, register-tile path: balanced (queue) hit drain
#ifndef PMS_QUEUE_DRAIN
#define PMS_QUEUE_DRAIN 1
#endif
#ifndef PMS_BLK_MIN_CTAS
#define PMS_BLK_MIN_CTAS 2
#endif
constexpr uint32_t kFull = 0xFFFFFFFFu;

// 64-bit code (l <= 31) -> 32-bit plane of its even bits
__host__ __device__ __forceinline__ uint32_t compress_even64(unsigned long long c) {
    return compress_even((uint32_t)c) | (compress_even((uint32_t)(c >> 32)) << 16);
}

struct Bp32 {
    using word = uint32_t;
    static constexpr int kMaxL = 16;
    __device__ static __forceinline__ uint2 prep(unsigned long long code) {
        const uint32_t c = code_to_bp((uint32_t)code);
        return make_uint2(c, rot16(c));
    }
    // Hamming distance of a candidate and a window: with x = c ^ w the
    // upper half of x | x << 16 is the per-position mismatch mask (the
    // shift is a multiply on the FMA pipe; OR + mask are one LOP3)
    __device__ static __forceinline__ uint32_t full_dist(uint2 c, word w) {
        const uint32_t x = c.x ^ w;
        return __popc((x | (x * 65536u)) & 0xFFFF0000u);
    }
    // Hamming distance of the prefix (positions before the last S): with
    // x = c ^ w, (x | x << 16) holds the per-position mismatch in its upper
    // half; x << 16 is a multiply (FMA pipe), the OR and the prefix mask are
    // one LOP3, so the test costs two ALU-pipe ops.
    template <int S>
    __device__ static __forceinline__ uint32_t prefix_dist(uint2 c, word w) {
        constexpr uint32_t PM = 0xFFFF0000u & ~(((1u << S) - 1u) << 16);
        const uint32_t x = c.x ^ w;
        return __popc((x | (x * 65536u)) & PM);
    }
    template <int S>
    __device__ static __forceinline__ uint32_t sfx_h(word w) { return (w >> 16) & ((1u << S) - 1u); }
    template <int S>
    __device__ static __forceinline__ uint32_t sfx_l(word w) { return w & ((1u << S) - 1u); }
    // suffix planes (bit S-1 = first suffix base) -> suffix code (S digits)
    template <int S>
    __device__ static __forceinline__ uint32_t sfx_code(uint32_t h, uint32_t l) {
        return (spread_even(h) << 1) | spread_even(l);
    }
    // pre-pass: planes of one window (position j at bit l-1-j) -> word
    __device__ static __forceinline__ word pack(uint32_t H, uint32_t L, int) { return (H << 16) | L; }
};

struct Bp64 {
    using word = uint2;
    static constexpr int kMaxL = 31;
    // Planes are TOP-aligned: position j of the l-mer sits at bit 32 - l + j
    // (the last base in bit 31), so the suffix is the top S bits of each plane
    // and a left shift -- a multiply, on the FMA pipe -- drops it.
    __device__ static __forceinline__ uint2 prep(unsigned long long code) {
        return make_uint2(__brev(compress_even64(code >> 1)), __brev(compress_even64(code)));
    }
    __device__ static __forceinline__ uint32_t full_dist(uint2 c, word w) {
        return __popc((c.x ^ w.x) | (c.y ^ w.y));
    }
    template <int S>
    __device__ static __forceinline__ uint32_t prefix_dist(uint2 c, word w) {
        return __popc(((c.x ^ w.x) | (c.y ^ w.y)) * (1u << S));
    }
    // suffix planes: bit i = suffix position i (first suffix base in bit 0)
    template <int S>
    __device__ static __forceinline__ uint32_t sfx_h(word w) { return w.x >> (32 - S); }
    template <int S>
    __device__ static __forceinline__ uint32_t sfx_l(word w) { return w.y >> (32 - S); }
    template <int S>
    __device__ static __forceinline__ uint32_t sfx_code(uint32_t h, uint32_t l) {
        return (spread_even(__brev(h) >> (32 - S)) << 1) | spread_even(__brev(l) >> (32 - S));
    }
    // pre-pass: planes with position j at bit l-1-j -> position j at bit
    // 32-l+j (bit reversal)
    __device__ static __forceinline__ word pack(uint32_t H, uint32_t L, int) {
        return make_uint2(__brev(H), __brev(L));
    }
};

}  // namespace pms

namespace {

using namespace pms;


// ------------------------------------------------------------------ a2 pre-pass
// One thread per (sequence i, window k < Wp).  Window k (the length-l
// substring starting at k, k in [0, W)) is packed into a bit-plane word; rows
// are padded to Wp with copies of window W-1, which cannot change "some window
// is within d".  A CTA takes kPackThreads consecutive windows of one row: its
// bytes are staged (one independent load each, so a cold input costs one HBM
// latency instead of l dependent ones) and checked once per byte; every byte
// lies in at least one window, so the byte check covers the whole input.
// Thread 0 also resets the step's state and the caller's result counter (no
// memset launch); an invalid byte stores the step's epoch in st->bad, so a
// stale flag of an earlier step never needs clearing.
constexpr int kPackThreads = 256;
template <class P>
__global__ void __launch_bounds__(kPackThreads) pms_pack_kernel(
    const uint8_t* __restrict__ seqs, int n, int t, int l, int W, int Wp, void* __restrict__ tab_,
    DevState* st, unsigned long long* nout, uint32_t epoch) {
    __shared__ uint8_t code[kPackThreads + 32];  // 2-bit codes of the CTA's bytes, 4 = invalid
    pdl_launch_dependents();
    typename P::word* tab = static_cast<typename P::word*>(tab_);
    const int chunks = (Wp + kPackThreads - 1) / kPackThreads;
    const int i = (int)(blockIdx.x / (unsigned)chunks);
    const int k0 = (int)(blockIdx.x - (unsigned)i * chunks) * kPackThreads;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        *nout = 0ull;
        st->next = 0ull;
        st->extra = 0ull;
        st->block_scans = 0ull;
    }
    if (i >= n) return;
    // bytes [s0, s1) of row i feed windows k0 .. k0 + kPackThreads - 1 (clamped to W-1)
    const int s0 = min(k0, W - 1);
    const int s1 = min(k0 + kPackThreads - 1, W - 1) + l;
    PMS_CHECK(s1 <= t && s1 - s0 <= kPackThreads + 32);
    const uint8_t* row = seqs + (long long)i * t;
    uint32_t bad = 0;
    for (int b = s0 + (int)threadIdx.x; b < s1; b += kPackThreads) {
        const uint32_t u = row[b] & 0xDFu;  // upper-case; only 'x'/'X' map to 'X'
        const uint32_t c = u == 'A' ? 0u : u == 'C' ? 1u : u == 'G' ? 2u : u == 'T' ? 3u : 4u;
        bad |= c >> 2;
        code[b - s0] = (uint8_t)c;
    }
    if (bad) *(volatile unsigned int*)&st->bad = epoch;
    __syncthreads();
    const int k = k0 + (int)threadIdx.x;
    if (k >= Wp) return;
    const uint8_t* q = code + (min(k, W - 1) - s0);
    uint32_t H = 0, L = 0;
    for (int j = 0; j < l; ++j) {
        const uint32_t c = q[j];
        H = (H << 1) | ((c >> 1) & 1u);
        L = (L << 1) | (c & 1u);
    }
    tab[(long long)i * Wp + k] = P::pack(H, L, l);
}

// ------------------------------------------------------------- shared pieces
// Stage the packed table into shared memory with one TMA bulk copy per 64 KB,
// completion tracked by an mbarrier (transaction bytes).
__device__ __forceinline__ void issue_table_copy(const SearchArgs& a, void* stab, uint64_t* bar) {
    mbar_expect_tx(bar, a.tab_bytes);
    constexpr uint32_t kChunk = 65536;
    for (uint32_t off = 0; off < a.tab_bytes; off += kChunk)
        tma_bulk_g2s(static_cast<char*>(stab) + off, static_cast<const char*>(a.tab) + off,
                     min(kChunk, a.tab_bytes - off), bar);
}

__device__ __forceinline__ void stage_table(const SearchArgs& a, void* stab, uint64_t* bar) {
    if (threadIdx.x == 0) mbar_init(bar, 1);
    __syncthreads();
    if (threadIdx.x == 0) issue_table_copy(a, stab, bar);
    mbar_wait(bar, 0);
}

// a4+a5 for sequences [i0, n) with the whole warp on one candidate: lanes take
// windows k = lane, lane+32, ...; one vote per sequence; the first sequence
// with no window within d abandons the candidate (skip rule).
template <class P>
__device__ __forceinline__ bool check_sequences(const typename P::word* tab, int i0, int n, int Wp,
                                                uint2 cb, uint32_t d, int lane,
                                                unsigned long long& scanned, bool skip = true) {
    bool all = true;
    for (int i = i0; i < n; ++i) {
        const typename P::word* row = tab + (size_t)i * Wp;
        uint32_t m = 0xFFu;
#pragma unroll 4
        for (int k = lane; k < Wp; k += 32) {
            PMS_CHECK(i < n && k < Wp);
            m = min(m, P::full_dist(cb, row[k]));
        }
        ++scanned;
        if (!__any_sync(kFull, m <= d)) {
            all = false;
            if (skip) return false;  // skip rule: abandon at the first failing sequence
        }
    }
    return all;
}

// a6: result store (uint32 or uint64 codes) and atomic-append compaction
__device__ __forceinline__ void store_code(const SearchArgs& a, unsigned long long slot,
                                           unsigned long long code) {
    if (slot >= a.cap) return;
    if (a.out_wide) static_cast<unsigned long long*>(a.out)[slot] = code;
    else static_cast<uint32_t*>(a.out)[slot] = (uint32_t)code;
}

__device__ __forceinline__ void append(const SearchArgs& a, unsigned long long code) {
    store_code(a, atomicAdd(a.nout, 1ull), code);
}

// Generic candidate-family variant (any W; table in shared or global memory):
// the whole warp takes one candidate and scans sequences 0..n-1 with the skip
// rule (or, with a.skip == 0, without it: the plain brute force the skip rule
// enhances).
template <class P, bool SMEM>
__global__ void __launch_bounds__(kBlock) pms_search_generic(SearchArgs a) {
    using word = typename P::word;
    extern __shared__ __align__(128) unsigned char gsm[];
    __shared__ __align__(8) uint64_t bar;
    pdl_wait();
    if (*(volatile unsigned int*)&a.st->bad == a.epoch) return;
    if (SMEM) stage_table(a, gsm, &bar);
    const word* tab = SMEM ? reinterpret_cast<const word*>(gsm) : static_cast<const word*>(a.tab);
    const int lane = threadIdx.x & 31;
    constexpr int kSub = 256;
    unsigned long long scanned = 0;
    for (;;) {
        unsigned long long b = 0;
        if (lane == 0) b = atomicAdd(&a.st->next, (unsigned long long)a.batch);
        b = __shfl_sync(kFull, b, 0);
        if (b >= a.span) break;
        for (int sb = 0; sb < a.batch; sb += kSub) {
            const unsigned long long cbase = a.lo_al + b + sb;
            if (cbase >= a.hi) break;
            for (int it = 0; it < kSub; ++it) {
                const unsigned long long code = cbase + it;
                if (code < a.lo || code >= a.hi) continue;
                if (check_sequences<P>(tab, 0, a.n, a.Wp, P::prep(code), a.dp, lane, scanned,
                                       a.skip != 0) &&
                    lane == 0)
                    append(a, code);
            }
        }
    }
    if (lane == 0 && scanned) atomicAdd(&a.st->extra, scanned);
}

// ------------------------------------------------- PMS_ALGO_BLOCK search
// The 4^S candidates of a 4^S-aligned code block (S = 5 or 6) share their
// first l-S digits (the prefix P) and differ in the last S (the suffix x).
// For a window w, Hamming(P x, w) = Hamming(P, w[0..l-S)) + Hamming(x,
// w[l-S..l)), so one XOR / OR-fold / POPC of the prefix against w gives p,
// and the block candidates that match w (distance <= d) are
// exactly the suffixes within Hamming distance d - p of w's suffix.  After a
// sequence, alive &= (the candidates with a window within d in it); the
// block is abandoned at the first sequence that leaves no candidate alive --
// the skip rule on 4^S candidates at once -- and at most `handoff` survivors
// are finished one by one by the whole warp (check_sequences).
//
// Candidates are indexed in BIT-PLANE order.  A suffix has planes (H, L) of S
// bits (H = high bits, L = low bits of its base codes, position l-S in bit
// S-1); its distance to a window suffix (eH, eL) is popc((H ^ eH) | (L ^ eL)).
// The last five positions (plane bits 0..4) spread over lanes and bits, the
// positions above them (S = 6: one) over a lane's mask words:
//   lane = H & 31, bit = L & 31, word k = (H >> 5) << X | (L >> 5)  (X = S - 5,
//   4^X words per lane).
// A hit (window w, prefix distance p <= d, budget r = d - p) matches the
// block candidates within distance r of w's suffix (eH, eL); pass 2
// (drain_queue / resolve_hit / apply_broadcasts below) ORs them into the
// warp's shared-memory words:
//   * r = 0 (~80 % of hits): only the window's own suffix -- one atomic OR of
//     bit eL & 31 into word k(eH, eL) of lane eH & 31;
//   * r = 1 (~18 %): the radius-1 ball, ORed by the finding lane itself with
//     6 + 3X atomics (ball-table rows, below);
//   * r >= 2: broadcast (one SHFL) to all lanes, which read two words of the
//     ball table T[rho][e][m] (bit b set iff popc(m | (b ^ e)) <= rho, five
//     positions): A = T[r][eL & 31][lane ^ (eH & 31)] for the word whose upper
//     position matches w's, B = T[r-1][...] for the other words (one mismatch
//     spent there).  B is the same for all of a lane's words, so it goes into
//     one `common` register; A into the one matching word (an atomic OR on
//     the lane's own word).  m is the fastest index: a broadcast reads 32
//     distinct banks.
template <int S>
struct BlkTraits {
    static constexpr int X = S - 5;
    static constexpr int C = 1 << (2 * S);               // candidates per block
    static constexpr int KW = 1 << (2 * X);              // mask words per lane (1, 4, 16)
    static constexpr uint32_t M = (1u << S) - 1u;        // suffix plane mask
};
constexpr int kTRows = 7;                                // rho = 0..6 (5, 6: all ones)
// + 32 x 8 words: the six radius-1 words resolve_hit needs per e = eL & 31,
// T[1][e][m] for m = 0, 1, 2, 4, 8, 16 (two pad words), packed for two 16-B
// loads (the rows of T itself would put every lane's T[1][e][0] in one bank)
constexpr int kR1Off = kTRows * 1024;
constexpr int kTWords = kR1Off + 32 * 8;                 // 29 KB ball table

// Suffix code (S digits, big-endian base 4) of the block candidate at
// (lane, word k, bit b).
template <class P, int S>
__device__ __forceinline__ uint32_t blk_sfx(uint32_t lane, uint32_t k, uint32_t b) {
    constexpr int X = S - 5;
    return P::template sfx_code<S>(lane | ((k >> X) << 5), b | ((k & ((1u << X) - 1u)) << 5));
}

// Per-warp r = 0 / ball word of lane `ln`, word k.  Lane-major (ln * KW + k,
// default) lets a lane read its words with 16-B accesses; word-major
// (k * 32 + ln) has fewer bank conflicts among the hit atomics.  Measured:
// equal at (15,4), lane-major 1.4 % faster at (16,5), word-major 2-3 % faster
// at (17,6) / (19,7).
#ifndef PMS_WMASK_KMAJOR
#define PMS_WMASK_KMAJOR 0
#endif
template <int S>
__device__ __forceinline__ uint32_t widx(uint32_t ln, uint32_t k) {
    return PMS_WMASK_KMAJOR ? k * 32u + ln : ln * (uint32_t)BlkTraits<S>::KW + k;
}

// ---- hit resolution (pass 2), shared by both drains ----------------------
// Words of the upper suffix positions (X of them) that differ from a hit's
// word ek in exactly one position: ek ^ kUp1[u] (X = 1: 3 words, X = 2: 6).
__device__ __forceinline__ uint32_t up1_delta(int X, int u) {
    // u = 3*pos + alt; alt 0: L bit, 1: H bit, 2: both
    const uint32_t pos = (uint32_t)u / 3u, alt = (uint32_t)u % 3u;
    const uint32_t lb = 1u << pos, hb = 1u << (X + pos);
    return alt == 0 ? lb : alt == 1 ? hb : (lb | hb);
}

// One hit (window w with prefix distance p <= d) of the finding lane:
//   r = 0: one atomic OR (the window's own suffix);
//   r = 1: the radius-1 ball, ORed by this lane with 6 + 3X atomics: its own
//          word with the five low positions flipped (T[1][eL & 31][0]), the
//          five lanes with one H bit flipped (T[1][eL & 31][1 << q]), and the
//          3X words one upper position away (centre bit only);
//   r >= 2: returns a broadcast record (byte offset of T[r][eL & 31][eH & 31],
//          word ek on top), else kFull.
template <class P, int S>
__device__ __forceinline__ uint32_t resolve_hit(typename P::word w, uint2 cb, uint32_t dp,
                                                const uint32_t* T, uint32_t* wmask) {
    using B = BlkTraits<S>;
    const uint32_t p = P::template prefix_dist<S>(cb, w);
    const uint32_t eH = P::template sfx_h<S>(w), eL = P::template sfx_l<S>(w);
    const uint32_t ek = ((eH >> 5) << B::X) | (eL >> 5);  // word of w's upper positions
    const uint32_t eh5 = eH & 31u, el5 = eL & 31u;
    if (p == dp) {
        PMS_CHECK(widx<S>(eh5, ek) < 32u * B::KW);
        atomicOr(wmask + widx<S>(eh5, ek), 1u << el5);
        return kFull;
    }
    if (p + 1u == dp) {
        const uint4* R = reinterpret_cast<const uint4*>(T + kR1Off + (el5 << 3));
        const uint4 r0 = R[0], r1 = R[1];
        const uint32_t t1[6] = {r0.x, r0.y, r0.z, r0.w, r1.x, r1.y};  // m = 0, 1, 2, 4, 8, 16
        atomicOr(wmask + widx<S>(eh5, ek), t1[0]);
#pragma unroll
        for (int q = 0; q < 5; ++q) atomicOr(wmask + widx<S>(eh5 ^ (1u << q), ek), t1[q + 1]);
#pragma unroll
        for (int u = 0; u < 3 * B::X; ++u)
            atomicOr(wmask + widx<S>(eh5, ek ^ up1_delta(B::X, u)), 1u << el5);
        return kFull;
    }
    const uint32_t r = min(dp - p, (uint32_t)(kTRows - 1));
    return (((r << 10) | (el5 << 5) | eh5) << 2) | (ek << 16);
}

// Apply every broadcast record of the warp (one SHFL each): per lane, word ek
// gets T[r] (A), the words one upper position away T[r-1] (B), and -- as
// `common`, which every word receives at the end of the scan -- the row for
// all X upper positions mismatched, T[r-X].  X = 0: A only.
template <int S>
__device__ __forceinline__ void apply_broadcasts(uint32_t mine, int lane, const uint32_t* T,
                                                 uint32_t* wmask, uint32_t& common) {
    using B = BlkTraits<S>;
    const char* Tb = reinterpret_cast<const char*>(T);
    const uint32_t lane4 = (uint32_t)lane << 2;
    uint32_t who = __ballot_sync(kFull, mine != kFull);
    while (who) {
        const int src = msb(who);
        who &= ~(1u << src);
        const uint32_t v = __shfl_sync(kFull, mine, src);
        const uint32_t off = (v ^ lane4) & 0xFFFFu;
        PMS_CHECK(off < 4u * kTWords && off + 1u > 4096u * B::X);
        const uint32_t a = *reinterpret_cast<const uint32_t*>(Tb + off);
        const uint32_t ek = v >> 16;
        atomicOr(wmask + widx<S>(lane, ek), a);  // the lane's own word: conflict-free
        if (B::X > 0) {
            common |= *reinterpret_cast<const uint32_t*>(Tb + off - 4096 * B::X);
            if (B::X > 1) {
                const uint32_t b = *reinterpret_cast<const uint32_t*>(Tb + off - 4096);
#pragma unroll
                for (int u = 0; u < 3 * B::X; ++u)
                    atomicOr(wmask + widx<S>(lane, ek ^ up1_delta(B::X, u)), b);
            }
        }
    }
}

// End of a (block, sequence) scan: alive &= (the lane's words | common); the
// words are cleared for the next scan.
template <int S>
__device__ __forceinline__ void finish_scan(uint32_t* wmask, int lane, uint32_t common,
                                            uint32_t (&alive)[BlkTraits<S>::KW]) {
    using B = BlkTraits<S>;
    __syncwarp();
    if (B::KW % 4 == 0 && !PMS_WMASK_KMAJOR) {  // lane-major: 16-B accesses
        uint4* wv = reinterpret_cast<uint4*>(wmask + lane * B::KW);
#pragma unroll
        for (int q = 0; q < B::KW / 4; ++q) {
            const uint4 m = wv[q];
            wv[q] = make_uint4(0u, 0u, 0u, 0u);
            alive[(4 * q + 0) % B::KW] &= m.x | common;
            alive[(4 * q + 1) % B::KW] &= m.y | common;
            alive[(4 * q + 2) % B::KW] &= m.z | common;
            alive[(4 * q + 3) % B::KW] &= m.w | common;
        }
    } else {
#pragma unroll
        for (int k = 0; k < B::KW; ++k) {
            alive[k] &= wmask[widx<S>(lane, k)] | common;
            wmask[widx<S>(lane, k)] = 0u;
        }
    }
    __syncwarp();
}

// Per-lane drain (NW = 0 streaming path): each lane resolves its own hits,
// one per round (bit q of hm marks window row[lane + 32 * (top - q)]).
template <class P, int S>
__device__ __forceinline__ void drain_hits(uint32_t hm, int top, const typename P::word* row,
                                           int wp, uint2 cb, uint32_t dp, int lane,
                                           const uint32_t* T, uint32_t* wmask, uint32_t& common) {
    (void)wp;
    while (__any_sync(kFull, hm != 0u)) {
        uint32_t mine = kFull;
        if (hm) {
            const int q = msb(hm);  // any order
            hm &= ~(1u << q);
            PMS_CHECK(lane + 32 * (top - q) < wp && top - q >= 0);
            mine = resolve_hit<P, S>(row[lane + 32 * (top - q)], cb, dp, T, wmask);
        }
        apply_broadcasts<S>(mine, lane, T, wmask, common);
    }
}

// Balanced drain (NW > 0): the warp's hits are first compacted into a
// per-warp shared-memory queue of window indices (exclusive prefix sum of the
// lanes' hit counts, then each lane writes its own), and the queue is
// processed 32 hits per round -- typically one or two rounds, where the
// per-lane drain needs max-over-lanes(hits) rounds of the same work.
// Queue slots by a shared-memory atomic per lane (1) or a warp prefix sum
// (0); default (-1): atomic for 32-bit words (measured -0.6 % at (15,4),
// -0.7 % at (16,5)), prefix sum for 64-bit words (atomic: +5..7 % at (17,6),
// (19,7), whose scans carry many more hits).
#ifndef PMS_QUEUE_ATOMIC
#define PMS_QUEUE_ATOMIC -1
#endif
template <class P, int S>
__device__ __forceinline__ void drain_queue(uint32_t hm, int top, const typename P::word* row,
                                            uint16_t* queue, uint32_t* qcnt, uint2 cb, uint32_t dp,
                                            int lane, const uint32_t* T, uint32_t* wmask,
                                            uint32_t& common) {
    constexpr bool kAtomic =
        PMS_QUEUE_ATOMIC > 0 || (PMS_QUEUE_ATOMIC < 0 && sizeof(typename P::word) == 4);
    const uint32_t nh = __popc(hm);
    uint32_t pos, total;
    if (kAtomic) {
        // lanes claim their queue slots with one shared-memory atomic each
        // (any order of the lanes is a valid queue); the warp's counter is
        // reset once the slots are claimed
        pos = atomicAdd(qcnt, nh);
        total = __reduce_add_sync(kFull, nh);
    } else {
        uint32_t inc = nh;  // inclusive prefix sum of the hit counts over lanes
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t v = __shfl_up_sync(kFull, inc, o);
            if (lane >= o) inc += v;
        }
        total = __shfl_sync(kFull, inc, 31);
        pos = inc - nh;
    }
    const int qbase = lane + 32 * top;  // window of hit bit q: qbase - 32 q
    while (hm) {
        const int q = msb(hm);
        hm ^= 1u << q;
        queue[pos++] = (uint16_t)(qbase - 32 * q);
    }
    __syncwarp();
    if (kAtomic && lane == 0) *qcnt = 0u;  // next use is after finish_scan's __syncwarp
    for (uint32_t base = 0; base < total; base += 32) {
        uint32_t mine = kFull;
        if (base + lane < total) mine = resolve_hit<P, S>(row[queue[base + lane]], cb, dp, T, wmask);
        apply_broadcasts<S>(mine, lane, T, wmask, common);
    }
}

// NW > 0: rows are padded to 32*NW windows and the window loops are fully
// unrolled; NW = 0: any row length, 32 windows per lane per chunk.
template <class P, int S, bool SMEM, int NW>
__global__ void __launch_bounds__(kBlockB, PMS_BLK_MIN_CTAS) pms_search_block(SearchArgs a) {
    using B = BlkTraits<S>;
    using word = typename P::word;
    static_assert(NW <= 32, "the per-lane hit mask holds 32 windows");
    extern __shared__ __align__(128) uint32_t stab[];  // [ball table T][window table if SMEM]
    __shared__ __align__(8) uint64_t bar;
    __shared__ __align__(16) uint32_t wmasks[kBlockB / 32][32 * B::KW];  // per-warp r = 0 hits
    __shared__ uint32_t qcnts[kBlockB / 32];  // per-warp queue counters (atomic slots)
    pdl_wait();
    if (*(volatile unsigned int*)&a.st->bad == a.epoch) return;
    uint32_t* T = stab;
    uint32_t* wmask = wmasks[threadIdx.x >> 5];
#pragma unroll
    for (int k = 0; k < B::KW; ++k) wmask[widx<S>(threadIdx.x & 31, k)] = 0u;
    if ((threadIdx.x & 31) == 0) qcnts[threadIdx.x >> 5] = 0u;
    word* tsm = reinterpret_cast<word*>(stab + kTWords);  // 128-B aligned for the bulk copy
    // prologue: TMA bulk copies of the ball table (28 KB, precomputed once per
    // device) and, when staged, the window table into shared memory
    if (threadIdx.x == 0) mbar_init(&bar, 1);
    __syncthreads();
    if (threadIdx.x == 0) {
        mbar_expect_tx(&bar, kTWords * 4u + (SMEM ? a.tab_bytes : 0u));
        tma_bulk_g2s(T, a.ball, kTWords * 4u, &bar);
        if (SMEM)
            for (uint32_t off = 0; off < a.tab_bytes; off += 65536u)
                tma_bulk_g2s(reinterpret_cast<char*>(tsm) + off,
                             static_cast<const char*>(a.tab) + off, min(65536u, a.tab_bytes - off),
                             &bar);
    }
    mbar_wait(&bar, 0);
    const word* tab = SMEM ? tsm : static_cast<const word*>(a.tab);
    const int lane = threadIdx.x & 31;
    // per-warp hit queue (NW > 0): 32*NW window indices after the tables
    uint16_t* queue = reinterpret_cast<uint16_t*>(
        reinterpret_cast<char*>(stab) + kTWords * 4 + (SMEM ? a.tab_bytes : 0u)) +
        (threadIdx.x >> 5) * 32 * (NW > 0 ? NW : 1);
    unsigned long long scanned = 0, bscans = 0;
    const uint32_t dp1 = a.dp + 1u;
    // register tile: hit bits of this lane's real windows (lane + 32j < W; the
    // padding repeats window W-1 and would only re-deliver its hits)
    uint32_t real = kFull;
    if (NW > 0) {
        const int nreal = min(NW, max(0, (a.W - lane + 31) / 32));
        real = (nreal == 0) ? 0u : ((nreal >= 32 ? kFull : ((1u << nreal) - 1u)) << (NW - nreal));
    }

    for (;;) {
        unsigned long long b = 0;
        if (lane == 0) b = atomicAdd(&a.st->next, (unsigned long long)a.batch);
        b = __shfl_sync(kFull, b, 0);
        if (b >= a.span) break;
        for (int sb = 0; sb < a.batch; sb += B::C) {
            const unsigned long long cbase = a.lo_al + b + sb;
            if (cbase >= a.hi) break;
            const uint2 cb = P::prep(cbase);  // suffix bits are zero
            // this lane's candidates inside [lo, hi)
            uint32_t alive[B::KW];
#pragma unroll
            for (int k = 0; k < B::KW; ++k) alive[k] = kFull;
            if (cbase < a.lo || cbase + B::C > a.hi) {  // edge block of [lo, hi)
#pragma unroll
                for (int k = 0; k < B::KW; ++k) {
                    uint32_t m = 0u;
                    for (uint32_t bb = 0; bb < 32; ++bb) {
                        const unsigned long long c = cbase + blk_sfx<P, S>(lane, k, bb);
                        if (c >= a.lo && c < a.hi) m |= 1u << bb;
                    }
                    alive[k] = m;
                }
            }
            int i = 0;
            bool dead = false;
            int nalive = B::C;  // the block's alive candidates (warp total) after sequence i-1
            for (; i < a.n; ++i) {
                if (i > 0 && a.skip && nalive <= a.handoff) break;
                const word* row = tab + (size_t)i * a.Wp;
                uint32_t common = 0u;  // ball words every candidate word of the lane gets
                // pass 1: prefix distance of each window; a hit (p <= d) makes
                // p - (d + 1) negative, and its sign bit is shifted into hm
                // (one funnel shift per window, no compare / select)
                if (NW > 0) {
                    uint32_t hm = 0;
#pragma unroll
                    for (int j = 0; j < NW; ++j) {
                        PMS_CHECK(lane + 32 * j < a.Wp && i < a.n);
                        hm = __funnelshift_l(P::template prefix_dist<S>(cb, row[lane + 32 * j]) - dp1,
                                             hm, 1);
                    }
                    hm &= real;
                    // pass 2: resolve the hits into each lane's candidate words
                    if (PMS_QUEUE_DRAIN)
                        drain_queue<P, S>(hm, NW - 1, row, queue, &qcnts[threadIdx.x >> 5], cb, a.dp,
                                          lane, T, wmask, common);
                    else
                        drain_hits<P, S>(hm, NW - 1, row, a.Wp, cb, a.dp, lane, T, wmask, common);
                } else {
                    for (int k0 = 0; k0 < a.Wp; k0 += 32 * 32) {  // 32 windows per lane per chunk
                        uint32_t hm = 0;
                        const int nj = min(a.Wp - k0, 32 * 32) / 32;
                        for (int j = 0; j < nj; ++j) {
                            PMS_CHECK(k0 + lane + 32 * j < a.Wp && i < a.n);
                            hm = __funnelshift_l(
                                P::template prefix_dist<S>(cb, row[k0 + lane + 32 * j]) - dp1, hm, 1);
                        }
                        drain_hits<P, S>(hm, nj - 1, row + k0, a.Wp - k0, cb, a.dp, lane, T, wmask,
                                         common);
                    }
                }
                finish_scan<S>(wmask, lane, common, alive);
                ++bscans;
                {  // one warp reduction gives the skip rule and the hand-off test
                    int na = 0;
#pragma unroll
                    for (int k = 0; k < B::KW; ++k) na += __popc(alive[k]);
                    nalive = __reduce_add_sync(kFull, na);
                }
                if (nalive == 0) {  // skip rule for the whole block
                    dead = true;
                    if (a.skip) break;  // (a.skip == 0: plain brute force scans on)
                }
            }
            if (dead) continue;
            if (i == a.n) {  // every alive candidate matched all n sequences
#pragma unroll
                for (int k = 0; k < B::KW; ++k) {
                    if (!alive[k]) continue;
                    unsigned long long slot = atomicAdd(a.nout, (unsigned long long)__popc(alive[k]));
                    for (uint32_t m = alive[k]; m; m &= m - 1, ++slot)
                        store_code(a, slot, cbase + blk_sfx<P, S>(lane, k, __ffs(m) - 1));
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
                const unsigned long long code = cbase + blk_sfx<P, S>(src, k, pk & 31u);
                if (check_sequences<P>(tab, i, a.n, a.Wp, P::prep(code), a.dp, lane, scanned) &&
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

}  // namespace
