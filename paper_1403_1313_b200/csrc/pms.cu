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
//
// This translation unit holds the 32-bit-word kernels (l <= 16) and the host
// code; pms64.cu holds the 64-bit-word instances (l <= 31).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <new>
#include <vector>

#include "pms.h"
#include "pms_device.cuh"
#include "pms_kernels.cuh"
#include "pms_slice.cuh"

namespace pms {  // defined in pms64.cu
const BlockKernel* block_kernels64(int* count);
SearchFn generic_kernel64(bool smem);
PackFn pack_kernel64();
int64_t debug_violations64(int reset);
}  // namespace pms

namespace {

#define PMS_NW_LIST(X) \
    X(1) X(2) X(3) X(4) X(5) X(6) X(7) X(8) X(10) X(12) X(14) X(16) X(19) X(22) X(25) X(28) \
    X(31) X(34) X(37) X(40) X(44) X(48)

constexpr int kSub = 256;          // candidates per aligned sub-block (4 low digits)
static_assert(kUnitMax % kSub == 0, "batches hold whole 256-candidate sub-blocks");

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
    pdl_wait();
    if (*(volatile unsigned int*)&a.st->bad == a.epoch) return;  // invalid input: no work
    if (SMEM) stage_table(a, stab, &bar);
    const uint32_t* tab = SMEM ? stab : static_cast<const uint32_t*>(a.tab);

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
                bool hit = m <= a.dd;
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
                            if (check_sequences<Bp32>(tab, 1, a.n, a.Wp, make_uint2(cbh, rot16(cbh)), a.dp,
                                                          lane, scanned) &&
                                lane == 0)
                                append(a, cbase + it + h);
                        }
                    }
                }
            }
        }
    }
    if (lane == 0 && scanned) atomicAdd(&a.st->extra, scanned);
}

// ------------------------------------------------ block-family instances
#define PMS_BLK5(nw) {5, nw, pms_search_block<Bp32, 5, true, nw>, pms_search_block<Bp32, 5, false, nw>},
#define PMS_BLK6(nw) {6, nw, pms_search_block<Bp32, 6, true, nw>, pms_search_block<Bp32, 6, false, nw>},
// Block-family register tiles stop at 32 windows per lane (the per-lane hit
// mask is one 32-bit word); longer rows stream through the NW = 0 kernel.
#define PMS_NWB_LIST(X) \
    X(1) X(2) X(3) X(4) X(5) X(6) X(7) X(8) X(10) X(12) X(14) X(16) X(19) X(22) X(25) X(28) \
    X(31) X(32)
// per S: the generic (NW = 0) instance first, then register tiles ascending
// (S = 7 -- 16 words per lane -- was measured slower: (15,4) 0.46-0.52 ms vs
// 0.378, (16,5) 8.7-10.2 ms vs 4.8; its scans cost 4.7x an S = 6 scan)
const BlockKernel kBlockKernels[] = {
    {5, 0, pms_search_block<Bp32, 5, true, 0>, pms_search_block<Bp32, 5, false, 0>},
    {6, 0, pms_search_block<Bp32, 6, true, 0>, pms_search_block<Bp32, 6, false, 0>},
    PMS_NWB_LIST(PMS_BLK5) PMS_NWB_LIST(PMS_BLK6)};

int kSliceThreadsFor(int S) { return S == 7 ? SliceCfg<7>::NT : SliceCfg<6>::NT; }

// PMS_ALGO_SLICE instances (pms_slice.cu) and their roofline kernels
// (pms_roof.cu): block digits S x prefix length LP = l - S
const SliceKernel* find_slice_kernel(int S, int LP) {
    int cnt = 0;
    const SliceKernel* ks = slice_kernels(&cnt);
    for (int q = 0; q < cnt; ++q)
        if (ks[q].S == S && ks[q].LP == LP) return &ks[q];
    ks = slice_kernels_wide(&cnt);  // l = 17..31
    for (int q = 0; q < cnt; ++q)
        if (ks[q].S == S && ks[q].LP == LP) return &ks[q];
    return nullptr;
}

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

// The ball table T[rho][e][m] (bit b set iff popc(m | (b ^ e)) <= rho over five
// positions, rho = 0..kTRows-1): computed once per device on the host and
// bulk-copied into each CTA's shared memory by the block kernels.
std::mutex g_ball_mu;
uint32_t* g_ball[64] = {nullptr};

const uint32_t* ensure_ball_table(int dev) {
    std::lock_guard<std::mutex> lk(g_ball_mu);
    if (dev < 0 || dev >= 64) return nullptr;
    if (!g_ball[dev]) {
        std::vector<uint32_t> h(kTWords, 0u);
        for (int idx = 0; idx < kR1Off; ++idx) {
            const uint32_t m = idx & 31u, e = (idx >> 5) & 31u;
            const int rho = idx >> 10;
            uint32_t w = 0;
            for (uint32_t b = 0; b < 32; ++b)
                if (__builtin_popcount(m | (b ^ e)) <= rho) w |= 1u << b;
            h[idx] = w;
        }
        static const int kM[6] = {0, 1, 2, 4, 8, 16};  // radius-1 rows, packed (see kR1Off)
        for (int e = 0; e < 32; ++e)
            for (int j = 0; j < 6; ++j) h[kR1Off + e * 8 + j] = h[1024 + e * 32 + kM[j]];
        uint32_t* d = nullptr;
        if (cudaMalloc(&d, kTWords * 4) != cudaSuccess) return nullptr;
        if (cudaMemcpy(d, h.data(), kTWords * 4, cudaMemcpyHostToDevice) != cudaSuccess ||
            cudaDeviceSynchronize() != cudaSuccess) {
            cudaFree(d);
            return nullptr;
        }
        g_ball[dev] = d;
    }
    return g_ball[dev];
}

// The slice family's ball table (pms_slice.cuh): the rows of T, then the
// radius-1 rows R1[e][u] (kSR1Stride words apart).  Once per device, like g_ball.
uint32_t* g_sball[64] = {nullptr};

const uint32_t* ensure_slice_ball_table(int dev) {
    std::lock_guard<std::mutex> lk(g_ball_mu);
    if (dev < 0 || dev >= 64) return nullptr;
    if (!g_sball[dev]) {
        std::vector<uint32_t> h(kSTWords, 0u);
        for (int idx = 0; idx < kSR1Off; ++idx) {
            const uint32_t m = idx & 31u, e = (idx >> 5) & 31u;
            const int rho = idx >> 10;
            uint32_t w = 0;
            for (uint32_t b = 0; b < 32; ++b)
                if (__builtin_popcount(m | (b ^ e)) <= rho) w |= 1u << b;
            h[idx] = w;
        }
        for (int e = 0; e < 32; ++e) {
            uint32_t* r = &h[kSR1Off + e * kSR1Stride];
            r[0] = h[1024 + e * 32 + 0];
            for (int q = 0; q < 5; ++q) r[1 + q] = h[1024 + e * 32 + (1 << q)];
            for (int u = 6; u < 15; ++u) r[u] = 1u << e;
        }
        uint32_t* d = nullptr;
        if (cudaMalloc(&d, kSTWords * 4) != cudaSuccess) return nullptr;
        if (cudaMemcpy(d, h.data(), kSTWords * 4, cudaMemcpyHostToDevice) != cudaSuccess ||
            cudaDeviceSynchronize() != cudaSuccess) {
            cudaFree(d);
            return nullptr;
        }
        g_sball[dev] = d;
    }
    return g_sball[dev];
}

int ensure_constants() {
    static thread_local int dev_done[64] = {0};
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return fail_cuda(__LINE__);
    if (dev_done[dev]) return PMS_OK;
    uint32_t h[kSub];
    for (int i = 0; i < kSub; ++i) h[i] = code_to_bp((uint32_t)i);
    if (cudaMemcpyToSymbol(c_bp256, h, sizeof(h)) != cudaSuccess ||
        cudaDeviceSynchronize() != cudaSuccess)
        return fail_cuda(__LINE__);
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
    void* d_table = nullptr;        // packed windows [n][Wp]: uint32 (Bp32) or uint2 (Bp64)
    const uint32_t* d_ball = nullptr;  // the device's ball table (block family; not owned)
    DevState* d_state = nullptr;
    DevState* h_state = nullptr;  // pinned mirror, read back by pms_plan_wait
    bool state_external = false;  // d_state lives in a pms_find context's result block
    uint32_t epoch = 0;           // id of the last step (h_state->bad == epoch: invalid input)
    cudaEvent_t ev[3] = {nullptr, nullptr, nullptr};  // start, packed, searched
    cudaStream_t aux = nullptr;   // private stream for the state read-back
    SearchFn fn = nullptr;
    PackFn pack = nullptr;
    int wide = 0;                   // 64-bit window words (l > 16 or pms_launch.wide_words)
    int G = 32, NW = 0, generic = 0, in_smem = 0, algo = PMS_ALGO_CANDIDATE, S = 0;
    uint32_t tab_bytes = 0, smem_bytes = 0;
    int grid = 0, block = kBlock, batch = kSub;
    unsigned long long last_lo = 0, last_hi = 0;
    bool executed = false;
    bool last_timed = true;       // the last execution recorded the pre-pass/search event
    // PMS_ALGO_SLICE (pms_slice.cuh): match planes, r = 0 slots, kernel
    void* d_planes = nullptr;
    void* d_slots = nullptr;
    int NWl = 0, LP = 0;
    uint32_t plane_bytes = 0, slot_bytes = 0;
    SliceFn sfn = nullptr;
    SliceFn sfn_ht = nullptr;  // the same search, hand-off on the staged tables (few blocks)
    int last_ht = 0;
    int sparse_handoff = 2;    // sparse-mode threshold (alive candidates) of the other instances
    int seqpar = 0;                 // sequence-parallel slice kernel (pms_search_slice_sp)
    uint32_t* d_spmask = nullptr;   // its per-block masks and counters
    uint32_t* d_spcnt = nullptr;
};

namespace {

// max_l: PMS_MAX_L for the uint32-code entry points, PMS_MAX_L64 otherwise
int check_shape(int32_t n, int32_t t, int32_t l, int32_t d, int32_t max_l) {
    if (n < 1 || t < 1 || l < 1 || l > max_l || l > t || d < 0) return PMS_E_ARG;
    if ((long long)n * t > 0x7FFFFFFFLL) return PMS_E_TOO_LARGE;
    const long long W = t - l + 1, Wp = (W + 31) / 32 * 32;
    if (n * Wp * 8 > 0x7FFFFFFFLL) return PMS_E_TOO_LARGE;
    return PMS_OK;
}

void destroy_plan(pms_plan* p) {
    if (!p) return;
    cudaFree(p->d_table);
    cudaFree(p->d_planes);
    cudaFree(p->d_slots);
    cudaFree(p->d_spmask);
    cudaFree(p->d_spcnt);
    if (!p->state_external) cudaFree(p->d_state);
    cudaFreeHost(p->h_state);
    for (cudaEvent_t e : p->ev)
        if (e) cudaEventDestroy(e);
    if (p->aux) cudaStreamDestroy(p->aux);
    delete p;
}

}  // namespace

extern "C" int pms_plan_create(int32_t n, int32_t t, int32_t l, int32_t d,
                               const pms_launch* launch, pms_plan** plan) {
    if (!plan) return PMS_E_ARG;
    *plan = nullptr;
    int st = check_shape(n, t, l, d, PMS_MAX_L64);
    if (st != PMS_OK) return st;
    pms_plan* p = new (std::nothrow) pms_plan();
    if (!p) return fail_cuda(__LINE__);
    p->n = n; p->t = t; p->l = l; p->d = d;
    p->W = t - l + 1;
    p->Wp = (p->W + 31) / 32 * 32;
    if (launch) p->launch = *launch;
    // window words: 32-bit (two 16-bit planes) up to l = 16, else 64-bit (two
    // 32-bit planes, l <= 31); wide_words forces 64-bit words at any l
    p->wide = (l > PMS_MAX_L || p->launch.wide_words) ? 1 : 0;
    int nbk = 0;
    const BlockKernel* bks = kBlockKernels;
    if (p->wide) bks = block_kernels64(&nbk);
    else nbk = (int)(sizeof(kBlockKernels) / sizeof(kBlockKernels[0]));
    const size_t word_bytes = p->wide ? 8 : 4;
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
        (p->launch.algo == PMS_ALGO_BLOCK || p->launch.algo == PMS_ALGO_SLICE ||
         (p->launch.algo == PMS_ALGO_AUTO && !p->launch.no_skip)) &&
        l >= kBlkMinL;
    // block digits S: 6 (4096-candidate blocks) when there are enough blocks to
    // keep every warp busy (l >= 13: >= 16k blocks), else 5
    int S = p->launch.block_digits == 5 || p->launch.block_digits == 6 ? p->launch.block_digits
                                                                        : (l >= 13 ? 6 : 5);
    if (S > l) S = 5;
    // slice family: S = 7 (16384-candidate blocks, slice family only) from
    // l = 13 (measured: (15,4) 168 us vs 328 at S = 6, (13,3) 48 vs 51; at
    // (11,3) S = 7 leaves most warps idle: 343 us vs 45), else the block
    // family's rule
    const int S_slice = p->launch.block_digits >= 5 && p->launch.block_digits <= 7
                            ? p->launch.block_digits
                            : (l >= 13 ? 7 : S);
    // PMS_ALGO_SLICE (the default where it applies): l <= 31, rows of at most
    // 1024 windows, a prefix of LP = l - S digits with d below it (otherwise
    // every window would hit), within the prefix counter's range (LP - d <= 16,
    // d <= 15: K + LP <= 31) and an instance for (S, LP) (l = 17..31: S = 7,
    // pms_slice_wide.cu); wide_words asks for the block family's 64-bit words;
    // elsewhere the block family runs
    if (block_algo && p->launch.algo != PMS_ALGO_BLOCK && !p->launch.wide_words && p->W <= 1024 &&
        l - S_slice >= 1 && d < l - S_slice && l - S_slice - d <= 16 && d <= 15 &&
        find_slice_kernel(S_slice, l - S_slice)) {
        S = S_slice;
        const SliceKernel* sk = find_slice_kernel(S, l - S);
        p->algo = PMS_ALGO_SLICE;
        p->S = S;
        p->LP = l - S;
        p->NWl = (p->W + 31) / 32;
        p->Wp = 32 * p->NWl;
        p->tab_bytes = (uint32_t)((size_t)n * p->Wp * 4);
        p->plane_bytes = (uint32_t)((size_t)n * p->LP * 512);
        p->slot_bytes = (uint32_t)(((size_t)n * p->Wp * 2 + 15) / 16 * 16);
        cudaFuncAttributes fs{};
        if (cudaFuncGetAttributes(&fs, (const void*)sk->fn_smem) != cudaSuccess) {
            destroy_plan(p);
            return fail_cuda(__LINE__);
        }
        // ball table + per-warp words and queues (SliceCfg<S>::kWorkBytes)
        const size_t ball_bytes = S == 5 ? SliceCfg<5>::kWorkBytes
                                  : S == 6 ? SliceCfg<6>::kWorkBytes : SliceCfg<7>::kWorkBytes;
        p->in_smem = !p->launch.table_global &&
                     ball_bytes + p->plane_bytes + p->slot_bytes + fs.sharedSizeBytes <= (size_t)smem_optin;
        p->smem_bytes = (uint32_t)ball_bytes + (p->in_smem ? p->plane_bytes + p->slot_bytes : 0u);
        p->sfn = p->in_smem ? sk->fn_smem : sk->fn_global;
        // sequence-parallel when the range has few blocks for the resident
        // warps (auto: blocks < warps / 4; measured at (9,2): one block's
        // sequential chain of scans is ~45 of the ~52 us)
        const int warps_total = p->sms * (kSliceThreadsFor(S) / 32);
        const unsigned long long nblk = 1ull << (2 * (l - S));
        const SliceFn spf = slice_seqpar_kernel(S, l - S);
        if (spf && p->in_smem && p->launch.seq_parallel >= 0 &&
            (p->launch.seq_parallel == 1 || nblk * 4ull < (unsigned long long)warps_total) &&
            nblk <= (1ull << 16)) {
            p->seqpar = 1;
            p->sfn = spf;
        }
        if (p->in_smem && !p->seqpar) p->sfn_ht = slice_ht_kernel(S, l - S);
        // sparse mode pays per candidate what a dense scan pays per hit: its
        // threshold follows the expected pass-1 hits per scan, W * P(prefix
        // within d) for iid uniform bases (a tuning knob; the set is the same).
        // Measured: (15,4) ~67 hits/scan best at 2 (155.6 us; 8: 161.8),
        // (16,5) ~163 hits/scan best at 8-12 (1.98 ms; 2: 2.14)
        {
            double ph = 0.0;  // P(Binomial(LP, 1/4) >= LP - d)
            const int LPs = l - S;
            for (int m = std::max(0, LPs - d); m <= LPs; ++m) {
                double c = 1.0;
                for (int q = 0; q < m; ++q) c = c * (LPs - q) / (q + 1);
                ph += c * std::pow(0.25, m) * std::pow(0.75, LPs - m);
            }
            const double hits = p->W * ph;
            p->sparse_handoff = std::max(2, std::min(12, (int)(hits / 20.0)));
        }
        p->G = 32; p->NW = p->NWl; p->generic = 0;
        p->block = kSliceThreadsFor(S);
        p->d_ball = ensure_slice_ball_table(p->dev);
        cudaFuncAttributes fh{};
        if (p->sfn_ht &&
            (cudaFuncGetAttributes(&fh, (const void*)p->sfn_ht) != cudaSuccess ||
             p->smem_bytes + fh.sharedSizeBytes > (size_t)smem_optin ||
             cudaFuncSetAttribute((const void*)p->sfn_ht, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  smem_optin - (int)fh.sharedSizeBytes) != cudaSuccess)) {
            destroy_plan(p);
            return fail_cuda(__LINE__);
        }
        cudaFuncAttributes fa{};
        int occ = 0;
        if (!p->d_ball || cudaFuncGetAttributes(&fa, (const void*)p->sfn) != cudaSuccess ||
            p->smem_bytes + fa.sharedSizeBytes > (size_t)smem_optin ||
            cudaFuncSetAttribute((const void*)p->sfn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 smem_optin - (int)fa.sharedSizeBytes) != cudaSuccess ||
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, (const void*)p->sfn, p->block,
                                                          p->smem_bytes) != cudaSuccess ||
            occ < 1) {
            destroy_plan(p);
            return fail_cuda(__LINE__);
        }
        if (p->launch.ctas_per_sm > 0) occ = std::min(occ, (int)p->launch.ctas_per_sm);
        p->grid = p->sms * occ;
        if (p->launch.grid_ctas > 0) p->grid = std::min((int)p->launch.grid_ctas, p->grid);
        const size_t sp_words = p->seqpar ? (size_t)nblk * 32 * (1u << (2 * (S - 5))) : 0;
        if (p->seqpar &&
            (cudaMalloc(&p->d_spmask, sp_words * 4) != cudaSuccess ||
             cudaMalloc(&p->d_spcnt, (size_t)nblk * 4) != cudaSuccess)) {
            destroy_plan(p);
            return fail_cuda(__LINE__);
        }
        if (cudaMalloc(&p->d_table, p->tab_bytes) != cudaSuccess ||
            // prefix planes [n][LP][4][32] (staged), then the suffix planes
            // [n][S][4][32] (sparse mode, read through L1/L2)
            cudaMalloc(&p->d_planes, (size_t)p->n * p->l * 512) != cudaSuccess ||
            cudaMalloc(&p->d_slots, p->slot_bytes) != cudaSuccess ||
            cudaMalloc(&p->d_state, sizeof(DevState)) != cudaSuccess ||
            cudaMallocHost(&p->h_state, sizeof(DevState)) != cudaSuccess ||
            cudaMemset(p->d_state, 0, sizeof(DevState)) != cudaSuccess ||
            cudaMemset(p->d_slots, 0, p->slot_bytes) != cudaSuccess ||
            cudaDeviceSynchronize() != cudaSuccess) {
            destroy_plan(p);
            return fail_cuda(__LINE__);
        }
        for (cudaEvent_t& e : p->ev)
            if (cudaEventCreate(&e) != cudaSuccess) {
                destroy_plan(p);
                return fail_cuda(__LINE__);
            }
        if (cudaStreamCreateWithFlags(&p->aux, cudaStreamNonBlocking) != cudaSuccess) {
            destroy_plan(p);
            return fail_cuda(__LINE__);
        }
        *plan = p;
        return PMS_OK;
    }
    const BlockKernel* bk = nullptr;
    if (block_algo) {
        for (int q = 0; q < nbk; ++q)  // generic (NW = 0) of this S first
            if (bks[q].S == S && bks[q].NW == 0) { bk = &bks[q]; break; }
        if (!p->launch.force_generic)
            for (int q = 0; q < nbk; ++q)  // smallest register tile covering W (list ascending)
                if (bks[q].S == S && bks[q].NW > 0 && 32 * bks[q].NW >= p->W) {
                    bk = &bks[q];
                    p->Wp = 32 * bks[q].NW;  // rows padded to the tile (re-read on hits)
                    break;
                }
        p->S = S;
    }
    p->tab_bytes = (uint32_t)((size_t)n * p->Wp * word_bytes);
    // static shared memory of the chosen kernel (mbarrier, per-warp hit masks)
    uint32_t static_smem = 12288;
    if (block_algo) {
        cudaFuncAttributes fb{};
        if (cudaFuncGetAttributes(&fb, (const void*)bk->fn_smem) != cudaSuccess) {
            destroy_plan(p);
            return fail_cuda(__LINE__);
        }
        static_smem = (uint32_t)fb.sharedSizeBytes;
    }
    const uint32_t ball_bytes =
        block_algo ? (uint32_t)kTWords * 4u : 0u;  // ball table (29 KB)
    // block family with a register tile: per-warp hit queue (u16 window
    // indices, 32*NW per warp, sized for the largest CTA)
    const uint32_t queue_bytes =
        (block_algo && PMS_QUEUE_DRAIN && bk->NW > 0) ? (uint32_t)(kBlockB / 32) * 64u * bk->NW : 0u;
    p->in_smem = !p->launch.table_global &&
                 p->tab_bytes + ball_bytes + queue_bytes + static_smem <= (uint32_t)smem_optin;
    // block family: a table that leaves room for only one CTA per SM is read
    // through L1/L2 instead -- two resident CTAs win (measured at (16,5):
    // 8.6 ms vs 9.9 ms); 228 KB of shared memory per SM, 1 KB reserved per CTA
    if (block_algo && p->in_smem &&
        2u * (p->tab_bytes + ball_bytes + queue_bytes + static_smem + 1024u) > 233472u)
        p->in_smem = 0;
    p->smem_bytes = ball_bytes + (p->in_smem ? p->tab_bytes : 0) + queue_bytes;
    if (block_algo && !(p->d_ball = ensure_ball_table(p->dev))) {
        destroy_plan(p);
        return fail_cuda(__LINE__);
    }

    RegKernel rk{};
    const int force_g = (p->launch.lanes_per_cand == 16 || p->launch.lanes_per_cand == 32)
                            ? p->launch.lanes_per_cand
                            : 0;
    if (block_algo) {
        p->fn = p->in_smem ? bk->fn_smem : bk->fn_global;
        p->G = 32; p->NW = bk->NW; p->generic = 0; p->algo = PMS_ALGO_BLOCK;
    } else if (!p->wide && !p->launch.force_generic && !p->launch.no_skip &&
               pick_reg_kernel(p->W, force_g, &rk)) {
        p->fn = p->in_smem ? rk.fn_smem : rk.fn_global;
        p->G = rk.G; p->NW = rk.NW; p->generic = 0; p->algo = PMS_ALGO_CANDIDATE;
    } else {
        if (p->wide) p->fn = generic_kernel64(p->in_smem != 0);
        else p->fn = p->in_smem ? pms_search_generic<Bp32, true> : pms_search_generic<Bp32, false>;
        p->G = 32; p->NW = 0; p->generic = 1; p->algo = PMS_ALGO_CANDIDATE;
    }
    p->pack = p->wide ? pack_kernel64() : pms_pack_kernel<Bp32>;
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
        cudaMallocHost(&p->h_state, sizeof(DevState)) != cudaSuccess ||
        cudaMemset(p->d_state, 0, sizeof(DevState)) != cudaSuccess ||
        // one-time setup above ran on the legacy stream (cudaMemset, the ball
        // table and constant copies); the work streams are non-blocking, so
        // wait for it here rather than rely on stream ordering
        cudaDeviceSynchronize() != cudaSuccess) {
        destroy_plan(p);
        return fail_cuda(__LINE__);
    }
    for (cudaEvent_t& e : p->ev)
        if (cudaEventCreate(&e) != cudaSuccess) {
            destroy_plan(p);
            return fail_cuda(__LINE__);
        }
    if (cudaStreamCreateWithFlags(&p->aux, cudaStreamNonBlocking) != cudaSuccess) {
        destroy_plan(p);
        return fail_cuda(__LINE__);
    }
    *plan = p;
    return PMS_OK;
}

extern "C" void pms_plan_destroy(pms_plan* plan) { destroy_plan(plan); }

namespace {

// DevState.extra: per-candidate sequence checks (low bits) | the slice
// family's sparse-mode steps << kSparseStepShift
unsigned long long extra_checks(const DevState& s) {
    return s.extra & ((1ull << kSparseStepShift) - 1ull);
}

// The slice kernels' arguments that depend on the plan only (tables, shape,
// threshold masks, skip rule and hand-off).
SliceArgs slice_args(const pms_plan* p) {
    SliceArgs sa{};
    sa.planes = static_cast<const uint32_t*>(p->d_planes);
    sa.splanes = static_cast<const uint32_t*>(p->d_planes) + p->plane_bytes / 4;
    sa.slots = static_cast<const uint16_t*>(p->d_slots);
    sa.words = static_cast<const uint32_t*>(p->d_table);
    sa.ball = p->d_ball;
    sa.n = p->n; sa.W = p->W; sa.Wp = p->Wp; sa.NWl = p->NWl;
    sa.dp = (uint32_t)std::min(p->d, p->l);
    const uint32_t K = 16u - (uint32_t)(p->LP - p->d);  // 1 <= LP - d <= LP
    for (int b = 0; b < 4; ++b) sa.kmask[b] = ((K >> b) & 1u) ? 0xFFFFFFFFu : 0u;
    sa.skip = p->launch.no_skip ? 0 : 1;
    sa.handoff = p->launch.handoff > 0 ? p->launch.handoff : (p->d >= 5 ? 2 : 1);
    sa.plane_bytes = p->plane_bytes; sa.slot_bytes = p->slot_bytes;
    return sa;
}

// out_wide: d_out holds uint64 codes (pms_plan_execute64) instead of uint32
// timed = false (pms_find* without stats): no event between the pre-pass and
// the search kernel, so the programmatic dependent launch overlaps them.
int plan_execute(pms_plan* p, const uint8_t* d_seqs, uint64_t lo, uint64_t hi, void* d_out,
                 int out_wide, uint64_t cap, uint64_t* d_count, void* stream, bool timed = true) {
    if (!p || !d_seqs || !d_count || (!d_out && cap > 0)) return PMS_E_ARG;
    if (!out_wide && p->l > PMS_MAX_L) return PMS_E_ARG;  // codes would not fit uint32
    const unsigned long long total = 1ull << (2 * p->l);
    if (hi > total) hi = total;
    if (lo > hi) return PMS_E_ARG;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    // batches and lo are aligned to the plan's unit: one block (4^S candidates)
    // for the block family, a 256-candidate sub-block for the candidate family
    const unsigned long long kUnit = (p->algo == PMS_ALGO_BLOCK || p->algo == PMS_ALGO_SLICE)
                                         ? (1ull << (2 * p->S))
                                         : (unsigned long long)kSub;
    const unsigned long long lo_al = lo / kUnit * kUnit;
    const unsigned long long span = hi - lo_al;

    // batch: aim for >= 8 grabs per warp, multiple of kSub, at most 16 sub-blocks
    const unsigned long long warps = (unsigned long long)p->grid * (p->block / 32);
    int batch = p->launch.batch > 0 ? (int)((p->launch.batch + kUnit - 1) / kUnit * kUnit) : 0;
    if (batch == 0 && p->algo == PMS_ALGO_SLICE) {
        batch = (int)kUnit;  // one block per grab (measured: (16,5) -1.4 %, (15,4) equal)
    } else if (batch == 0) {
        unsigned long long b = span / (warps * 8);
        b = (b + kUnit - 1) / kUnit * kUnit;
        batch = (int)std::min<unsigned long long>(std::max<unsigned long long>(b, kUnit),
                                                  std::max<unsigned long long>(4 * kUnit, 4096));
    }
    p->batch = batch;
    p->last_lo = lo;
    p->last_hi = hi;
    p->last_timed = timed;

    SearchArgs a{};
    a.tab = p->d_table; a.n = p->n; a.W = p->W; a.Wp = p->Wp;
    a.dd = 2u * (uint32_t)std::min(p->d, p->l);
    a.dp = (uint32_t)std::min(p->d, p->l);
    a.lo = lo; a.hi = hi; a.lo_al = lo_al; a.span = span; a.batch = batch;
    a.in_smem = p->in_smem; a.tab_bytes = p->tab_bytes;
    a.skip = p->launch.no_skip ? 0 : 1;
    a.handoff = p->launch.handoff > 0 ? p->launch.handoff : (p->d >= 5 ? 2 : 1);  // measured
    a.st = p->d_state; a.nout = reinterpret_cast<unsigned long long*>(d_count);
    a.out = d_out; a.out_wide = out_wide; a.cap = cap;
    a.ball = p->d_ball;
    if (++p->epoch == 0) p->epoch = 1;  // 0 is the reset value of st->bad
    a.epoch = p->epoch;
    static const bool no_pdl = std::getenv("PMS_NO_PDL") != nullptr;
    if (p->algo == PMS_ALGO_SLICE) {
        SliceArgs sa = slice_args(p);
        sa.lo = lo; sa.hi = hi; sa.lo_al = lo_al; sa.span = span; sa.batch = batch;
        sa.out_wide = out_wide;
        sa.st = p->d_state; sa.epoch = p->epoch;
        sa.nout = reinterpret_cast<unsigned long long*>(d_count);
        sa.out = d_out; sa.cap = cap;
        // hand-off checks on the staged tables (the HT instance) when the
        // range has fewer than two blocks per resident warp (measured: (13,3)
        // 48 -> 35 us); with many blocks per warp the packed-word check's
        // fewer instructions win.  PMS_HANDOFF_TABLES=0/1 forces either.
        static const char* ht_env = std::getenv("PMS_HANDOFF_TABLES");
        const bool ht = p->sfn_ht && (ht_env ? std::atoi(ht_env) != 0 : span / kUnit < 2ull * warps);
        p->last_ht = ht ? 1 : 0;
        // hand-off threshold: the tables check takes one candidate at a time
        // (1, or 2 for d >= 5); sparse mode (the other instances) takes up to
        // kSparseHandoff candidates together
        if (p->launch.handoff <= 0) sa.handoff = ht ? (p->d >= 5 ? 2 : 1) : p->sparse_handoff;
        if (!ht && sa.handoff > 32) sa.handoff = 32;  // one sparse list entry per lane
        int sp_words = 0, sp_blocks = 0;
        if (p->seqpar) {
            sa.spmask = p->d_spmask;
            sa.spcnt = p->d_spcnt;
            sa.sp_blocks = (span + kUnit - 1) / kUnit;
            sp_blocks = (int)sa.sp_blocks;
            sp_words = sp_blocks * 32 * (1 << (2 * (p->S - 5)));
        }
        if (cudaEventRecord(p->ev[0], s) != cudaSuccess) return fail_cuda(__LINE__);
        const SlicePackFn pack = slice_pack_kernel(p->S);
        const unsigned pack_y =
            (unsigned)((p->Wp + p->l * 128 + kSlicePackThreads - 1) / kSlicePackThreads);
        pack<<<dim3((unsigned)p->n, pack_y), kSlicePackThreads, 0, s>>>(
            d_seqs, p->n, p->t, p->l, p->W, p->NWl, p->LP, static_cast<uint32_t*>(p->d_planes),
            static_cast<uint16_t*>(p->d_slots), static_cast<uint32_t*>(p->d_table), p->d_state,
            reinterpret_cast<unsigned long long*>(d_count), p->epoch, p->d_spmask, p->d_spcnt,
            sp_words, sp_blocks);
        const cudaError_t e_pack = cudaGetLastError();
        if (e_pack != cudaSuccess) return fail_cuda(__LINE__, e_pack);
        if (timed && cudaEventRecord(p->ev[1], s) != cudaSuccess) return fail_cuda(__LINE__);
        if (span > 0) {
            cudaLaunchConfig_t cfg{};
            cfg.gridDim = dim3((unsigned)p->grid);
            cfg.blockDim = dim3((unsigned)p->block);
            cfg.dynamicSmemBytes = (size_t)p->smem_bytes;
            cfg.stream = s;
            cudaLaunchAttribute attr[1];
            attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
            attr[0].val.programmaticStreamSerializationAllowed = 1;
            cfg.attrs = attr;
            cfg.numAttrs = no_pdl ? 0 : 1;
            const cudaError_t e = cudaLaunchKernelEx(&cfg, ht ? p->sfn_ht : p->sfn, sa);
            if (e != cudaSuccess) return fail_cuda(__LINE__, e);
        }
        if (cudaEventRecord(p->ev[2], s) != cudaSuccess) return fail_cuda(__LINE__);
        p->executed = true;
        return PMS_OK;
    }

    // device work of a step: pre-pass (which also resets the state and the
    // result counter), search; the state read-back is pms_plan_wait's
    if (cudaEventRecord(p->ev[0], s) != cudaSuccess) return fail_cuda(__LINE__);
    const long long pack_ctas = (long long)p->n * ((p->Wp + kPackThreads - 1) / kPackThreads);
    p->pack<<<(unsigned)pack_ctas, kPackThreads, 0, s>>>(d_seqs, p->n, p->t, p->l, p->W, p->Wp,
                                                             p->d_table, p->d_state,
                                                             reinterpret_cast<unsigned long long*>(d_count),
                                                             p->epoch);
    const cudaError_t e_pack = cudaGetLastError();
    if (e_pack != cudaSuccess) return fail_cuda(__LINE__, e_pack);
    if (timed && cudaEventRecord(p->ev[1], s) != cudaSuccess) return fail_cuda(__LINE__);
    if (span > 0) {
        // programmatic dependent launch after the pre-pass (PMS_NO_PDL: plain)
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3((unsigned)p->grid);
        cfg.blockDim = dim3((unsigned)p->block);
        cfg.dynamicSmemBytes = (size_t)p->smem_bytes;
        cfg.stream = s;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = attr;
        cfg.numAttrs = no_pdl ? 0 : 1;
        const cudaError_t e = cudaLaunchKernelEx(&cfg, p->fn, a);
        if (e != cudaSuccess) return fail_cuda(__LINE__, e);
    }
    if (cudaEventRecord(p->ev[2], s) != cudaSuccess) return fail_cuda(__LINE__);
    p->executed = true;
    return PMS_OK;
}

}  // namespace

extern "C" int pms_plan_execute(pms_plan* p, const uint8_t* d_seqs, uint64_t lo, uint64_t hi,
                                uint32_t* d_out, uint64_t cap, uint64_t* d_count, void* stream) {
    return plan_execute(p, d_seqs, lo, hi, d_out, 0, cap, d_count, stream,
                        !(p && p->launch.overlap_prepass));
}

extern "C" int pms_plan_execute64(pms_plan* p, const uint8_t* d_seqs, uint64_t lo, uint64_t hi,
                                  uint64_t* d_out, uint64_t cap, uint64_t* d_count, void* stream) {
    return plan_execute(p, d_seqs, lo, hi, d_out, 1, cap, d_count, stream,
                        !(p && p->launch.overlap_prepass));
}

namespace {

// Fill *stats from the plan's events and its (already read back) state.
void fill_stats(pms_plan* p, pms_stats* stats) {
    float pack = 0.f, search = 0.f, tot = 0.f;
    cudaEventElapsedTime(&tot, p->ev[0], p->ev[2]);
    if (p->last_timed) {
        cudaEventElapsedTime(&pack, p->ev[0], p->ev[1]);
        cudaEventElapsedTime(&search, p->ev[1], p->ev[2]);
    } else {
        search = tot;  // (no boundary event: the two kernels overlap)
    }
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
        p->h_state->bad == p->epoch ? 0
                        : (seq0_implicit ? cands * W : 0) +
                              (extra_checks(*p->h_state) + p->h_state->block_scans) * W;
    stats->algo = p->algo;
    stats->block_scans = p->h_state->block_scans;
    stats->sparse_steps = p->h_state->extra >> kSparseStepShift;
    stats->block_digits = p->S;
    stats->mode_flags = (p->seqpar ? 1 : 0) | (p->last_ht ? 2 : 0);
    stats->motifs = 0;
    stats->grid = p->grid;
    stats->block = p->block;
    stats->lanes_per_cand = p->G;
    stats->windows_per_lane = p->NW;
    stats->generic = p->generic;
    stats->table_in_smem = p->in_smem;
    stats->smem_bytes = p->smem_bytes;
}

}  // namespace

extern "C" int pms_plan_wait(pms_plan* p, pms_stats* stats) {
    if (!p || !p->executed) return PMS_E_ARG;
    // read the state back on the plan's own stream once the search is done
    if (cudaStreamWaitEvent(p->aux, p->ev[2], 0) != cudaSuccess ||
        cudaMemcpyAsync(p->h_state, p->d_state, sizeof(DevState), cudaMemcpyDeviceToHost,
                        p->aux) != cudaSuccess ||
        cudaStreamSynchronize(p->aux) != cudaSuccess)
        return fail_cuda(__LINE__);
    if (stats) fill_stats(p, stats);
    return p->h_state->bad == p->epoch ? PMS_E_CHAR : PMS_OK;
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
    // one device block [plan state | count | codes]: a single D2H brings back
    // the state, the count and the first kSpecCodes codes
    static constexpr size_t kHead = 128;
    static constexpr unsigned long long kSpecCodes = 1024;  // codes copied back with the count
    char* d_buf = nullptr;            // kHead + out_bytes
    void* d_out = nullptr;            // result codes (uint32 or uint64) = d_buf + kHead
    unsigned long long out_bytes = 0;
    uint64_t* d_count = nullptr;      // = d_buf + 64
    char* h_head = nullptr;           // pinned mirror of the block's first kHead + 8 kSpecCodes bytes
    uint64_t* h_count = nullptr;      // = h_head + 64
    uint8_t* h_seqs = nullptr;    // pinned staging of the input (n*t bytes)
    void* h_out = nullptr;        // pinned staging of small result sets
    static constexpr unsigned long long kHostOutBytes = 1ull << 19;
    cudaStream_t stream = nullptr;
    // the call's device work (H2D, pre-pass, search, D2H) as one CUDA graph,
    // re-captured when the range, capacity, code width or buffers change
    cudaGraphExec_t gexec = nullptr;
    unsigned long long g_lo = 0, g_hi = 0, g_cap = 0;
    int g_wide = -1, g_disabled = 0;
    void* g_out = nullptr;
    uint32_t g_epoch = 0;  // the plan step id baked into the graph's pre-pass
    // previous call's parameters: a graph is captured only for a repeat
    unsigned long long p_lo = ~0ull, p_hi = 0, p_cap = 0;
    int p_wide = -1;

    bool matches(int dv, int32_t n_, int32_t t_, int32_t l_, int32_t d_,
                 const pms_launch& L) const {
        return dev == dv && n == n_ && t == t_ && l == l_ && d == d_ &&
               std::memcmp(&launch, &L, sizeof(L)) == 0;
    }
    void release_resources() {
        if (gexec) cudaGraphExecDestroy(gexec);
        destroy_plan(plan);
        cudaFree(d_seqs);
        cudaFree(d_buf);
        cudaFreeHost(h_head);
        cudaFreeHost(h_seqs);
        cudaFreeHost(h_out);
        if (stream) cudaStreamDestroy(stream);
    }
};

// codes copied back speculatively with the count (one host round trip when
// the result set is small, as it is for planted-motif instances)
constexpr unsigned long long kSpecCodes = CallCtx::kSpecCodes;

// (Re)allocate the context's result block for `bytes` of codes; its head holds
// the plan's state (zeroed: no stale invalid-input flag) and the count.
int ctx_grow(CallCtx* c, unsigned long long bytes) {
    cudaFree(c->d_buf);
    c->d_buf = nullptr;
    c->d_out = nullptr;
    c->d_count = nullptr;
    c->out_bytes = 0;
    if (cudaMalloc(&c->d_buf, CallCtx::kHead + bytes) != cudaSuccess ||
        cudaMemset(c->d_buf, 0, CallCtx::kHead) != cudaSuccess ||
        cudaDeviceSynchronize() != cudaSuccess)  // (legacy-stream memset vs the context's stream)
        return fail_cuda(__LINE__);
    c->d_out = c->d_buf + CallCtx::kHead;
    c->d_count = reinterpret_cast<uint64_t*>(c->d_buf + 64);
    c->out_bytes = bytes;
    if (!c->plan->state_external) cudaFree(c->plan->d_state);
    c->plan->d_state = reinterpret_cast<DevState*>(c->d_buf);
    c->plan->state_external = true;
    return PMS_OK;
}
static_assert(kSpecCodes * 8 <= (1ull << 19), "fits the pinned staging buffer");

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
    int st = pms_plan_create(n, t, l, d, &L, &c->plan);  // (plan keyed by shape + launch)
    if (st != PMS_OK) {
        delete c;
        return st;
    }
    static_assert(sizeof(DevState) <= 64, "state + count fit the result block's head");
    if (cudaMalloc(&c->d_seqs, (size_t)n * t) != cudaSuccess ||
        cudaMallocHost(&c->h_head, CallCtx::kHead + 8 * kSpecCodes) != cudaSuccess ||
        cudaMallocHost(&c->h_seqs, (size_t)n * t) != cudaSuccess ||
        cudaMallocHost(&c->h_out, CallCtx::kHostOutBytes) != cudaSuccess ||
        cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking) != cudaSuccess) {
        ctx_destroy(c);
        return fail_cuda(__LINE__);
    }
    c->h_count = reinterpret_cast<uint64_t*>(c->h_head + 64);
    st = ctx_grow(c, 8 * kSpecCodes);
    if (st != PMS_OK) {
        ctx_destroy(c);
        return st;
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

namespace {

// One complete search from host buffers for code type Code (uint32_t: l <= 16;
// uint64_t: l <= 31): a1 checks, H2D, plan execution, D2H, a7 host sort.
template <class Code>
int find_host(const uint8_t* seqs, int32_t n, int32_t t, int32_t l, int32_t d, uint64_t lo,
              uint64_t hi, const pms_launch* launch, Code* out_codes, uint64_t max_out,
              uint64_t* count, pms_stats* stats) {
    constexpr int kWide = sizeof(Code) == 8;
    // a1: argument checks in the documented order
    if (!seqs || !count || (!out_codes && max_out > 0)) return PMS_E_ARG;
    int st = check_shape(n, t, l, d, kWide ? PMS_MAX_L64 : PMS_MAX_L);
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
    if (cap * sizeof(Code) > c->out_bytes) {  // grow the result block (kept for the next call)
        st = ctx_grow(c, cap * sizeof(Code));
        if (st != PMS_OK) {
            healthy = false;
            return st;
        }
    }
    cudaStream_t s = c->stream;
    std::memcpy(c->h_seqs, seqs, (size_t)n * t);  // pinned staging: the H2D is a true async DMA
    // one round trip: state, count and (speculatively) the first codes come
    // back with a single synchronisation; a second copy only for large sets
    const unsigned long long spec = std::min<unsigned long long>(cap, kSpecCodes);
    pms_plan* pl = c->plan;
    // the call's device work: H2D, pre-pass + search (plan_execute), D2H
    auto enqueue = [&]() -> int {
        if (cudaMemcpyAsync(c->d_seqs, c->h_seqs, (size_t)n * t, cudaMemcpyHostToDevice, s) !=
            cudaSuccess)
            return fail_cuda(__LINE__);
        const int e = plan_execute(pl, c->d_seqs, lo, hi, c->d_out, kWide, cap, c->d_count, s,
                                   stats != nullptr);
        if (e != PMS_OK) return e;
        if (cudaMemcpyAsync(c->h_head, c->d_buf, CallCtx::kHead + spec * sizeof(Code),
                            cudaMemcpyDeviceToHost, s) != cudaSuccess)
            return fail_cuda(__LINE__);
        return PMS_OK;
    };
    // replayed as a CUDA graph (one launch instead of ~8 API calls) unless
    // PMS_NO_GRAPH is set or capture is unavailable
    static const bool no_graph = std::getenv("PMS_NO_GRAPH") != nullptr;
    bool graphed = false;
    const bool repeat = c->p_lo == lo && c->p_hi == hi && c->p_cap == cap && c->p_wide == kWide;
    c->p_lo = lo; c->p_hi = hi; c->p_cap = cap; c->p_wide = kWide;
    const bool have = c->gexec && c->g_lo == lo && c->g_hi == hi && c->g_cap == cap &&
                      c->g_wide == kWide && c->g_out == c->d_out;
    // (not when stats are requested: the per-kernel event timings stay those of
    // an ordinary enqueue)
    if (!no_graph && !stats && !c->g_disabled && (have || repeat)) {
        if (!have) {
            if (c->gexec) cudaGraphExecDestroy(c->gexec);
            c->gexec = nullptr;
            cudaGraph_t g = nullptr;
            if (cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal) == cudaSuccess) {
                const int e = enqueue();
                const cudaError_t ee = cudaStreamEndCapture(s, &g);
                if (e == PMS_OK && ee == cudaSuccess && g &&
                    cudaGraphInstantiate(&c->gexec, g, 0) == cudaSuccess) {
                    c->g_lo = lo; c->g_hi = hi; c->g_cap = cap; c->g_wide = kWide;
                    c->g_out = c->d_out;
                    c->g_epoch = pl->epoch;
                } else {
                    c->gexec = nullptr;
                    c->g_disabled = 1;
                }
                if (g) cudaGraphDestroy(g);
            } else {
                c->g_disabled = 1;
            }
            cudaGetLastError();  // clear a failed capture's error state
        }
        if (c->gexec) {
            if (cudaGraphLaunch(c->gexec, s) != cudaSuccess) {
                healthy = false;
                return fail_cuda(__LINE__);
            }
            graphed = true;
            pl->epoch = c->g_epoch;  // the step id the graph's pre-pass stores on bad input
        }
    }
    if (!graphed) {
        st = enqueue();
        if (st != PMS_OK) {
            healthy = false;
            return st;
        }
    }
    if (cudaStreamSynchronize(s) != cudaSuccess) {
        healthy = false;
        return fail_cuda(__LINE__);
    }
    std::memcpy(pl->h_state, c->h_head, sizeof(DevState));
    if (stats) fill_stats(pl, stats);
    if (pl->h_state->bad == pl->epoch) {
        // a replayed graph reuses its step id: clear the flag for the next call
        if (cudaMemsetAsync(&pl->d_state->bad, 0, sizeof(unsigned int), s) != cudaSuccess ||
            cudaStreamSynchronize(s) != cudaSuccess) {
            healthy = false;
            return fail_cuda(__LINE__);
        }
        return PMS_E_CHAR;
    }
    const uint64_t found = *c->h_count;
    if (stats) stats->motifs = found;
    *count = found;
    if (found > max_out) return PMS_E_TRUNCATED;
    // a7: D2H of the codes, host sort (ascending code = lexicographic order)
    if (found > 0) {
        if (found > spec) {
            const bool staged = found * sizeof(Code) <= CallCtx::kHostOutBytes;
            if (cudaMemcpyAsync(staged ? c->h_out : (void*)out_codes, c->d_out,
                                found * sizeof(Code), cudaMemcpyDeviceToHost, s) != cudaSuccess ||
                cudaStreamSynchronize(s) != cudaSuccess) {
                healthy = false;
                return fail_cuda(__LINE__);
            }
            if (staged) std::memcpy(out_codes, c->h_out, found * sizeof(Code));
        } else {
            std::memcpy(out_codes, c->h_head + CallCtx::kHead, found * sizeof(Code));
        }
        std::sort(out_codes, out_codes + found);
    }
    return PMS_OK;
}

}  // namespace

extern "C" int pms_find_ex(const uint8_t* seqs, int32_t n, int32_t t, int32_t l, int32_t d,
                           uint64_t lo, uint64_t hi, const pms_launch* launch, uint32_t* out_codes,
                           uint64_t max_out, uint64_t* count, pms_stats* stats) {
    return find_host<uint32_t>(seqs, n, t, l, d, lo, hi, launch, out_codes, max_out, count, stats);
}

extern "C" int pms_find(const uint8_t* seqs, int32_t n, int32_t t, int32_t l, int32_t d,
                        uint32_t* out_codes, uint64_t max_out, uint64_t* count) {
    return pms_find_ex(seqs, n, t, l, d, 0, ~0ull, nullptr, out_codes, max_out, count, nullptr);
}

extern "C" int pms_find64_ex(const uint8_t* seqs, int32_t n, int32_t t, int32_t l, int32_t d,
                             uint64_t lo, uint64_t hi, const pms_launch* launch,
                             uint64_t* out_codes, uint64_t max_out, uint64_t* count,
                             pms_stats* stats) {
    return find_host<uint64_t>(seqs, n, t, l, d, lo, hi, launch, out_codes, max_out, count, stats);
}

extern "C" int pms_find64(const uint8_t* seqs, int32_t n, int32_t t, int32_t l, int32_t d,
                          uint64_t* out_codes, uint64_t max_out, uint64_t* count) {
    return pms_find64_ex(seqs, n, t, l, d, 0, ~0ull, nullptr, out_codes, max_out, count, nullptr);
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

extern "C" int pms_plan_roofline(pms_plan* p, int32_t mode, int32_t scans_per_warp,
                                 double* tests_per_s, double* scans_per_s, double* ms) {
    if (!p || !tests_per_s || p->algo != PMS_ALGO_SLICE || !p->executed || mode < 0 ||
        mode > 3 || scans_per_warp < 1)
        return PMS_E_ARG;
    const SliceRoofFn fn = slice_roofline_kernel(p->S, p->LP, mode, p->in_smem != 0);
    if (!fn) return PMS_E_ARG;
    // the tables of the plan's last execution (its pre-pass) must be complete;
    // its scans per block set the sequence mix the microbenchmark visits
    DevState hs{};
    if (cudaEventSynchronize(p->ev[2]) != cudaSuccess ||
        cudaMemcpy(&hs, p->d_state, sizeof(hs), cudaMemcpyDeviceToHost) != cudaSuccess)
        return fail_cuda(__LINE__);
    const double blocks_run =
        std::max(1.0, std::ceil((double)(p->last_hi - p->last_lo) / (double)(1ull << (2 * p->S))));
    const int depth = std::max(1, std::min(p->n, (int)std::llround((double)hs.block_scans / blocks_run)));
    int smem_optin = 0;
    cudaFuncAttributes fa{};
    if (cudaDeviceGetAttribute(&smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, p->dev) !=
            cudaSuccess ||
        cudaFuncGetAttributes(&fa, (const void*)fn) != cudaSuccess ||
        cudaFuncSetAttribute((const void*)fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             smem_optin - (int)fa.sharedSizeBytes) != cudaSuccess)
        return fail_cuda(__LINE__);
    SliceArgs sa = slice_args(p);
    // mode 2: lists of the last execution's mean sparse list size
    const unsigned long long ssteps = hs.extra >> kSparseStepShift;
    const int list = ssteps
                         ? std::max(1, std::min(32, (int)std::llround((double)extra_checks(hs) / ssteps)))
                         : std::max(1, std::min(32, p->sparse_handoff));
    if (mode >= 2) sa.handoff = list;
    // mode 3: sparse steps per dense scan of the last execution, 16.16
    const double ratio = hs.block_scans ? (double)ssteps / (double)hs.block_scans : 0.0;
    const uint32_t ratio_fp = (uint32_t)std::min(65536.0 * 64, std::llround(ratio * 65536.0) * 1.0);
    if (mode == 3) sa.batch = (int)ratio_fp;
    unsigned long long* sink = nullptr;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (cudaMalloc(&sink, sizeof(unsigned long long)) != cudaSuccess ||
        cudaEventCreate(&e0) != cudaSuccess || cudaEventCreate(&e1) != cudaSuccess) {
        cudaFree(sink);
        return fail_cuda(__LINE__);
    }
    const unsigned long long nblocks = 1ull << (2 * p->LP);
    cudaStream_t s = p->aux;
    float best = 1e30f;
    for (int r = 0; r < 4; ++r) {  // one warm-up, best of three
        cudaEventRecord(e0, s);
        fn<<<p->grid, p->block, p->smem_bytes, s>>>(sa, r == 0 ? 1 : scans_per_warp, depth, nblocks,
                                                    sink);
        cudaEventRecord(e1, s);
        if (cudaEventSynchronize(e1) != cudaSuccess) break;
        float t = 0.f;
        cudaEventElapsedTime(&t, e0, e1);
        if (r > 0) best = std::min(best, t);
    }
    const cudaError_t err = cudaGetLastError();
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(sink);
    if (err != cudaSuccess) return fail_cuda(__LINE__, err);
    // modes 0, 1: (block, sequence) scans of W window tests; mode 2: sparse
    // steps of `list` candidate-sequence checks (W window tests each)
    const double warps = (double)p->grid * (p->block / 32);
    const double scans = warps * scans_per_warp;
    // mode 3: the warps' sparse steps, as their credit loops count them
    // (warp g starts with credit (g * 40503) mod 2^16)
    double steps3 = 0.0;
    for (uint64_t g = 0; g < (uint64_t)warps; ++g)
        steps3 += (double)((((g * 40503u) & 0xFFFFu) + (uint64_t)scans_per_warp * ratio_fp) >> 16);
    *tests_per_s = (mode == 2   ? scans * list
                    : mode == 3 ? scans + steps3 * list
                                : scans) *
                   p->W / (best * 1e-3);
    if (scans_per_s) *scans_per_s = scans / (best * 1e-3);
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
    int64_t total = (int64_t)v;
    for (int64_t x : {pms::debug_violations64(reset), pms::debug_violations_slice(reset),
                      pms::debug_violations_roof(reset),
                      pms::debug_violations_ht(reset),
                      pms::debug_violations_wide(reset)}) {  // the other TUs' counters
        if (x < 0) return x;
        total += x;
    }
    return total;
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
