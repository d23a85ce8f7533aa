// pms_slice_ht.cu -- slice search instances whose hand-off checks run on the
// staged planes and slots (slice_check_one) instead of the packed words: the
// host launches them when the range has fewer than two blocks per resident
// warp, where a lone warp's hand-off chain is the kernel's run time
// (DESIGN.md 6c).  Own translation unit: compiles in parallel with the rest.
#include <cuda_runtime.h>

#include <cstdint>

#include "pms_device.cuh"
#include "pms_kernels.cuh"
#include "pms_slice.cuh"

namespace {

struct HtKernel {
    int S, LP;
    pms::SliceFn fn;
};
#define PMS_HT(S, LP) {S, LP, pms_search_slice<S, LP, true, true>},
#define PMS_HT5(LP) PMS_HT(5, LP)
#define PMS_HT6(LP) PMS_HT(6, LP)
#define PMS_HT7(LP) PMS_HT(7, LP)
#define PMS_HT_LIST(X) X(1) X(2) X(3) X(4) X(5) X(6) X(7) X(8) X(9)
const HtKernel kHtKernels[] = {PMS_HT_LIST(PMS_HT5) PMS_HT5(10) PMS_HT5(11)
                               PMS_HT_LIST(PMS_HT6) PMS_HT6(10)
                               PMS_HT_LIST(PMS_HT7)};

}  // namespace

namespace pms {

SliceFn slice_ht_kernel(int S, int LP) {
    for (const HtKernel& k : kHtKernels)
        if (k.S == S && k.LP == LP) return k.fn;
    return nullptr;
}

int64_t debug_violations_ht(int reset) {
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

#ifdef PMS_TRACE
// tuning builds only: the trace of this translation unit's instances
extern "C" int pms_trace_read_ht(unsigned long long* host, int nwarps) {
    if (nwarps > 8192) nwarps = 8192;
    if (cudaDeviceSynchronize() != cudaSuccess) return -1;
    return cudaMemcpyFromSymbol(host, g_pms_trace, (size_t)nwarps * 64) == cudaSuccess ? 0 : -1;
}
#endif
