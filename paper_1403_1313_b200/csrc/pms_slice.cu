// pms_slice.cu -- the PMS_ALGO_SLICE kernel instances (pms_slice.cuh): the
// pre-pass per block size S and the search kernel per (S, prefix length LP,
// table placement).  A separate translation unit so the instances compile in
// parallel with the host code (pms.cu).
#include <cuda_runtime.h>

#include <cstdint>

#include "pms_device.cuh"
#include "pms_kernels.cuh"
#include "pms_slice.cuh"

namespace {

#define PMS_SLICE(S, LP) {S, LP, pms_search_slice<S, LP, true>, pms_search_slice<S, LP, false>},
#define PMS_SLICE5(LP) PMS_SLICE(5, LP)
#define PMS_SLICE6(LP) PMS_SLICE(6, LP)
#define PMS_SLICE7(LP) PMS_SLICE(7, LP)
#define PMS_LP_LIST(X) X(1) X(2) X(3) X(4) X(5) X(6) X(7) X(8) X(9)
// l <= 16: LP = l - S <= 11 (S = 5), 10 (S = 6), 9 (S = 7)
const pms::SliceKernel kSliceKernels[] = {PMS_LP_LIST(PMS_SLICE5) PMS_SLICE5(10) PMS_SLICE5(11)
                                          PMS_LP_LIST(PMS_SLICE6) PMS_SLICE6(10)
                                          PMS_LP_LIST(PMS_SLICE7)};

// sequence-parallel instances (few blocks: small l), staged tables only
struct SpKernel {
    int S, LP;
    pms::SliceFn fn;
};
#define PMS_SP(S, LP) {S, LP, pms_search_slice_sp<S, LP>},
#define PMS_SP5(LP) PMS_SP(5, LP)
#define PMS_SP6(LP) PMS_SP(6, LP)
const SpKernel kSpKernels[] = {PMS_LP_LIST(PMS_SP5) PMS_SP5(10) PMS_SP5(11)
                               PMS_LP_LIST(PMS_SP6) PMS_SP6(10)};

}  // namespace

namespace pms {

SliceFn slice_seqpar_kernel(int S, int LP) {
    for (const SpKernel& k : kSpKernels)
        if (k.S == S && k.LP == LP) return k.fn;
    return nullptr;
}

const SliceKernel* slice_kernels(int* count) {
    *count = (int)(sizeof(kSliceKernels) / sizeof(kSliceKernels[0]));
    return kSliceKernels;
}

SlicePackFn slice_pack_kernel(int S) {
    return S == 5 ? pms_pack_slice<5> : S == 6 ? pms_pack_slice<6> : pms_pack_slice<7>;
}

int64_t debug_violations_slice(int reset) {
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
// tuning builds only: copy the per-warp trace of the last slice search launch
extern "C" int pms_trace_read(unsigned long long* host, int nwarps) {
    if (nwarps > 8192) nwarps = 8192;
    if (cudaDeviceSynchronize() != cudaSuccess) return -1;
    return cudaMemcpyFromSymbol(host, g_pms_trace, (size_t)nwarps * 64) == cudaSuccess ? 0 : -1;
}
#endif
