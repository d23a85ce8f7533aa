// pms64.cu -- 64-bit-word instances of the search kernels:
// l = 17..31 (SPEC.md:117 caps l at 31 so a code fits 64 bits), or any l with
// pms_launch.wide_words.  A window is a uint2 of two 32-bit bit planes; the
// kernels are the templates of pms_kernels.cuh instantiated with Bp64.  A
// separate translation unit so it compiles in parallel with pms.cu.
#include <cuda_runtime.h>

#include <cstdint>

#include "pms_device.cuh"
#include "pms_kernels.cuh"

namespace {

#define PMS_NW64_LIST(X) X(1) X(2) X(4) X(8) X(12) X(16) X(19) X(24) X(32)
#define PMS_BLK64(S, nw) {S, nw, pms_search_block<Bp64, S, true, nw>, pms_search_block<Bp64, S, false, nw>},
#define PMS_BLK64_5(nw) PMS_BLK64(5, nw)
#define PMS_BLK64_6(nw) PMS_BLK64(6, nw)
// per S: the generic (NW = 0) instance, then register tiles ascending
const BlockKernel kBlockKernels64[] = {
    PMS_BLK64(5, 0) PMS_BLK64(6, 0) PMS_NW64_LIST(PMS_BLK64_5) PMS_NW64_LIST(PMS_BLK64_6)};

}  // namespace

namespace pms {

const BlockKernel* block_kernels64(int* count) {
    *count = (int)(sizeof(kBlockKernels64) / sizeof(kBlockKernels64[0]));
    return kBlockKernels64;
}

SearchFn generic_kernel64(bool smem) {
    return smem ? pms_search_generic<Bp64, true> : pms_search_generic<Bp64, false>;
}

PackFn pack_kernel64() { return pms_pack_kernel<Bp64>; }

int64_t debug_violations64(int reset) {
#ifdef PMS_DEBUG_CHECKS
    unsigned int v = 0;
    if (cudaMemcpyFromSymbol(&v, g_pms_violations, sizeof(v)) != cudaSuccess) return -2;
    if (reset) {
        const unsigned int z = 0;
        cudaMemcpyToSymbol(g_pms_violations, &z, sizeof(z));
    }
    return (int64_t)v;
#else
    (void)reset;
    return 0;
#endif
}

}  // namespace pms
