// pms_roof.cu -- roofline microbenchmark instances of the slice family
// (pms_roofline_slice in pms_slice.cuh): for each (S, LP), MODE 0 (pass 1
// only, R_pass1), MODE 1 (the whole per-scan code at the instance's hit
// mix, R_scan), MODE 2 (sparse-mode steps, R_sparse) and MODE 3 (the two
// interleaved at the launch's own ratio, R_mix), with the tables staged in shared memory or read through
// L1/L2 like the plan's search kernel.  Own translation unit: it only
// compiles in parallel with the others.
#include <cuda_runtime.h>

#include <cstdint>

#include "pms_device.cuh"
#include "pms_kernels.cuh"
#include "pms_slice.cuh"

namespace {

struct RoofKernel {
    int S, LP;
    pms::SliceRoofFn fn[2][4];  // [tables in smem][mode]
};
#define PMS_ROOF(S, LP)                                                                       \
    {S, LP, {{pms_roofline_slice<S, LP, false, 0>, pms_roofline_slice<S, LP, false, 1>,       \
              pms_roofline_slice<S, LP, false, 2>, pms_roofline_slice<S, LP, false, 3>},      \
             {pms_roofline_slice<S, LP, true, 0>, pms_roofline_slice<S, LP, true, 1>,         \
              pms_roofline_slice<S, LP, true, 2>, pms_roofline_slice<S, LP, true, 3>}}},
#define PMS_ROOF5(LP) PMS_ROOF(5, LP)
#define PMS_ROOF6(LP) PMS_ROOF(6, LP)
#define PMS_ROOF7(LP) PMS_ROOF(7, LP)
#define PMS_LP_LIST(X) X(1) X(2) X(3) X(4) X(5) X(6) X(7) X(8) X(9)
const RoofKernel kRoofKernels[] = {PMS_LP_LIST(PMS_ROOF5) PMS_ROOF5(10) PMS_ROOF5(11)
                                   PMS_LP_LIST(PMS_ROOF6) PMS_ROOF6(10) PMS_LP_LIST(PMS_ROOF7)};

}  // namespace

namespace pms {

SliceRoofFn slice_roofline_kernel(int S, int LP, int mode, bool smem) {
    if (mode < 0 || mode > 3) return nullptr;
    for (const RoofKernel& k : kRoofKernels)
        if (k.S == S && k.LP == LP) return k.fn[smem ? 1 : 0][mode];
    return nullptr;
}

int64_t debug_violations_roof(int reset) {
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
