// pms_slice_wide.cu -- slice search instances for l = 17..31 (64-bit codes):
// S = 7 blocks, prefixes of LP = 10..24 digits.  The kernel is the same
// template as pms_slice.cu's (pms_slice.cuh): the prefix test counts LP match
// planes into the 5-bit carry-save counter (K + matches <= 16 + d <= 31 for
// d <= 15, K = 16 - (LP - d) >= 0 for LP - d <= 16: the host checks both), the
// suffix stays 7 digits, and codes are cbase + suffix in 64 bits.  Own
// translation unit: compiles in parallel with the rest.
#include <cuda_runtime.h>

#include <cstdint>

#include "pms_device.cuh"
#include "pms_kernels.cuh"
#include "pms_slice.cuh"

namespace {

#define PMS_SLICE_W(LP) {7, LP, pms_search_slice<7, LP, true>, pms_search_slice<7, LP, false>},
const pms::SliceKernel kSliceKernelsWide[] = {
    PMS_SLICE_W(10) PMS_SLICE_W(11) PMS_SLICE_W(12) PMS_SLICE_W(13) PMS_SLICE_W(14)
    PMS_SLICE_W(15) PMS_SLICE_W(16) PMS_SLICE_W(17) PMS_SLICE_W(18) PMS_SLICE_W(19)
    PMS_SLICE_W(20) PMS_SLICE_W(21) PMS_SLICE_W(22) PMS_SLICE_W(23) PMS_SLICE_W(24)};

}  // namespace

namespace pms {

const SliceKernel* slice_kernels_wide(int* count) {
    *count = (int)(sizeof(kSliceKernelsWide) / sizeof(kSliceKernelsWide[0]));
    return kSliceKernelsWide;
}

int64_t debug_violations_wide(int reset) {
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
