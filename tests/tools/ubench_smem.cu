// ubench_smem.cu -- hand-run microbenchmark (not part of the product): the
// per-SM throughput of the shared-memory and warp operations the block
// kernel's hit resolution uses, at full occupancy (148 SMs x 32 warps), with
// 8 independent operations per iteration and register-resident addresses, so
// the kernel design can be costed in SM cycles instead of guessed.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/ubench_smem tests/tools/ubench_smem.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

enum { ATOM_RAND, ATOM_OWN, RED_RAND, LDS_RAND, LDS_ROW, LDS128, STS_RAND, RMW_RAND, SHFL, ALU2,
       POPC1, FLO1 };

template <int MODE>
__global__ void __launch_bounds__(1024, 1) kern(int iters, int act, uint32_t* sink) {
    __shared__ __align__(16) uint32_t m[32][128];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int k = lane; k < 128; k += 32) m[w][k] = k;
    __syncwarp();
    uint32_t a[8], acc = 0;
    uint32_t x = threadIdx.x * 2654435761u + blockIdx.x;
#pragma unroll
    for (int u = 0; u < 8; ++u) { x = x * 1664525u + 1013904223u; a[u] = x >> 25; }
    const bool on = lane < act;
    uint32_t* base = m[w];
#pragma unroll 1
    for (int it = 0; it < iters; ++it) {
        const uint32_t s = (uint32_t)it;
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const uint32_t idx = (a[u] ^ s) & 127u;
            if (MODE == ATOM_RAND) { if (on) atomicOr(base + idx, 1u << (idx & 31)); }
            if (MODE == ATOM_OWN) { if (on) atomicOr(base + (lane * 4 + (u & 3)), 1u << (idx & 31)); }
            if (MODE == RED_RAND) { if (on) asm volatile("red.shared.or.b32 [%0], %1;" :: "r"((uint32_t)__cvta_generic_to_shared(base + idx)), "r"(1u << (idx & 31)) : "memory"); }
            if (MODE == LDS_RAND) { if (on) acc += base[idx]; }
            if (MODE == LDS_ROW) { if (on) acc += base[(lane + 32 * (u & 3)) ^ (s & 32)]; }
            if (MODE == LDS128) { if (on) { const uint4 v = reinterpret_cast<const uint4*>(base)[(lane ^ s) & 31]; acc += v.x ^ v.w; } }
            if (MODE == STS_RAND) { if (on) base[idx] = s; }
            if (MODE == RMW_RAND) { if (on) { base[idx] |= 1u << (idx & 31); } }
            if (MODE == SHFL) { acc += __shfl_sync(0xFFFFFFFFu, a[u] ^ acc, (int)(idx & 31)); }
            if (MODE == ALU2) { acc = (acc ^ idx) | (acc >> 3); }
            if (MODE == POPC1) { acc += __popc(idx ^ acc); }
            if (MODE == FLO1) { acc ^= 31 - __clz(idx | 1); }
        }
    }
    __syncwarp();
    if (acc == 0x12345678u) sink[0] = acc;
    if (lane == 0 && base[0] == 0x9u) sink[1] = 1;
}

template <int MODE>
void run(const char* name, int act, int sms, int ops_per_u) {
    uint32_t* sink;
    cudaMalloc(&sink, 8);
    const int iters = 4000;
    kern<MODE><<<sms, 1024>>>(10, act, sink);
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a);
    kern<MODE><<<sms, 1024>>>(iters, act, sink);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0; cudaEventElapsedTime(&ms, a, b);
    const double warp_ops = (double)sms * 32 * iters * 8;  // warp instructions of the op
    const double cyc = ms * 1e-3 * 1.965e9;                 // at the max SM clock
    printf("%-26s act=%2d %7.3f ms  SM-cycles per warp-op=%6.2f  (ops/u=%d)\n", name, act, ms,
           cyc * sms / warp_ops, ops_per_u);
    cudaFree(sink);
}

int main() {
    int sms = 0; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    run<ALU2>("ALU (xor/or/shift) ref", 32, sms, 3);
    for (int act : {32, 8, 1}) run<ATOM_RAND>("ATOMS.OR random", act, sms, 1);
    for (int act : {32, 1}) run<ATOM_OWN>("ATOMS.OR own word", act, sms, 1);
    for (int act : {32, 8, 1}) run<RED_RAND>("red.shared.or random", act, sms, 1);
    for (int act : {32, 1}) run<LDS_RAND>("LDS random", act, sms, 1);
    run<LDS_ROW>("LDS row (conflict-free)", 32, sms, 1);
    run<LDS128>("LDS.128 conflict-free", 32, sms, 1);
    for (int act : {32, 1}) run<STS_RAND>("STS random", act, sms, 1);
    for (int act : {32, 8}) run<RMW_RAND>("LDS+OR+STS random", act, sms, 2);
    run<SHFL>("SHFL.IDX", 32, sms, 1);
    run<POPC1>("POPC", 32, sms, 1);
    run<FLO1>("FLO", 32, sms, 1);
    return 0;
}
