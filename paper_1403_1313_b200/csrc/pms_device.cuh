// pms_device.cuh -- device building blocks of the sm_100a skip-BF search.
//
// Window / candidate word ("bit-plane" 2-bit encoding):
//   base code A=0 C=1 G=2 T=3; position j of an l-mer
//   (j = 0 is the first base) sits at bit (l-1-j) of two 16-bit planes:
//     bits [16,32): high bit of each base code   (plane H)
//     bits [ 0,16): low  bit of each base code   (plane L)
//   A position mismatches iff it differs in H or in L.  With x = c ^ w and
//   r = rot16(x), (x | r) holds the mismatch mask in BOTH halves, so
//   popc(x | r) = 2 * Hamming(c, w)  (PAPER.md:63 Hamming distance).
//   With the rotated operands precomputed (cr = rot16(c), wr = rot16(w)) the
//   per-compare work is LOP3(c^w) + LOP3((cr^wr)|x) + POPC + 1/2 VIMNMX3.
//
// Candidate code (big-endian base 4) <-> bit-plane word:
//   L = even bits of the code compressed, H = odd bits compressed.
#pragma once
#include <cstdint>

namespace pms {

// Debug builds (-DPMS_DEBUG_CHECKS, libpms_b200_debug.so) count every failed
// check (out-of-range index, protocol violation) in a device counter the host
// reads with pms_debug_violations().  A check is a detector, not a guard: the
// access it precedes still runs (a bad index can still fault), but the count
// makes a silent slip visible.  Release builds compile the checks away.
#ifdef PMS_DEBUG_CHECKS
static __device__ unsigned int g_pms_violations;  // one per translation unit
#define PMS_CHECK(cond)                                          \
    do {                                                         \
        if (!(cond)) atomicAdd(&::pms::g_pms_violations, 1u);    \
    } while (0)
#else
#define PMS_CHECK(cond) \
    do {                \
    } while (0)
#endif

constexpr int kSparseStepShift = 40;  // DevState.extra: candidate checks | steps << 40
struct DevState {
    unsigned long long next;    // work counter: candidates handed out, from lo_al
    unsigned long long extra;   // sequences scanned beyond sequence 0 (survivors); the slice
                                // family's sparse-mode steps count from bit kSparseStepShift

    unsigned long long block_scans;  // PMS_ALGO_BLOCK (block, sequence) scans
    unsigned int bad;           // = the step's epoch: its pre-pass saw a byte outside ACGTacgt
    unsigned int pad[3];
};

__host__ __device__ __forceinline__ uint32_t compress_even(uint32_t x) {
    x &= 0x55555555u;
    x = (x | (x >> 1)) & 0x33333333u;
    x = (x | (x >> 2)) & 0x0F0F0F0Fu;
    x = (x | (x >> 4)) & 0x00FF00FFu;
    x = (x | (x >> 8)) & 0x0000FFFFu;
    return x;
}

__host__ __device__ __forceinline__ uint32_t spread_even(uint32_t x) {
    x &= 0x0000FFFFu;
    x = (x | (x << 8)) & 0x00FF00FFu;
    x = (x | (x << 4)) & 0x0F0F0F0Fu;
    x = (x | (x << 2)) & 0x33333333u;
    x = (x | (x << 1)) & 0x55555555u;
    return x;
}

// code -> bit-plane word
__host__ __device__ __forceinline__ uint32_t code_to_bp(uint32_t c) {
    return (compress_even(c >> 1) << 16) | compress_even(c);
}

// bit-plane word -> code
__host__ __device__ __forceinline__ uint32_t bp_to_code(uint32_t w) {
    return (spread_even(w >> 16) << 1) | spread_even(w);
}

__device__ __forceinline__ uint32_t rot16(uint32_t x) { return __funnelshift_r(x, x, 16); }

// Position of the most significant set bit (x != 0): one FLO, where
// 31 - __clz(x) costs three instructions.
__device__ __forceinline__ int msb(uint32_t x) {
    uint32_t r;
    asm("bfind.u32 %0, %1;" : "=r"(r) : "r"(x));
    return (int)r;
}

// 2 * Hamming(c, w) for bit-plane words, given the rotated operands.
__device__ __forceinline__ uint32_t mism2(uint32_t c, uint32_t cr, uint32_t w, uint32_t wr) {
    return __popc((c ^ w) | (cr ^ wr));
}

// ---------------------------------------------------------------- PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
                 : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}

// TMA bulk copy global -> shared (no tensor map; 16-B aligned, size % 16 == 0),
// completion signalled on the mbarrier as transaction bytes.
__device__ __forceinline__ void tma_bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                             uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
            "r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

// Programmatic dependent launch: the pre-pass lets the search kernel launch
// early; the search kernel waits here until the pre-pass grid has completed
// and its writes are visible (a no-op when launched without the attribute).
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch_dependents() {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
    uint32_t done = 0;
    while (!done) {
        asm volatile(
            "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; "
            "selp.u32 %0, 1, 0, p; }"
            : "=r"(done)
            : "r"(smem_u32(bar)), "r"(phase)
            : "memory");
    }
}

}  // namespace pms
