// dip_ubench.cu -- the integer-pipe microbenchmark behind the scorer's ALU roofline:
// the B200's sustained issue rate of the instructions the longest-path wavefront is made of
// (IADD3, IMNMX, ISETP + SEL, SHFL, 64-bit add, IMAD), measured on the box the bench runs on,
// instead of a figure taken from a guide. Each thread runs 8 independent dependency chains
// (enough in flight to hide the ALU latency at full occupancy); the grid fills every SM.
#include <cuda_runtime.h>
#include <stdint.h>

#include "dip_host_internal.h"

namespace {

constexpr int UB_ITERS = 2048;
constexpr int UB_CHAINS = 8;

template <int KIND>
__global__ void __launch_bounds__(256) ub_kernel(uint32_t seed, uint32_t *sink) {
    uint32_t a[UB_CHAINS], b = seed ^ threadIdx.x, c = seed * 7u + blockIdx.x;
    unsigned long long w[UB_CHAINS];
#pragma unroll
    for (int k = 0; k < UB_CHAINS; k++) { a[k] = seed + k * 977u + threadIdx.x; w[k] = a[k]; }
    for (int it = 0; it < UB_ITERS; it++) {
#pragma unroll
        for (int k = 0; k < UB_CHAINS; k++) {
            if constexpr (KIND == 0) {            // IADD3: a = a + b + c
                asm volatile("add.u32 %0, %0, %1;\n\tadd.u32 %0, %0, %2;" : "+r"(a[k]) : "r"(b), "r"(c));
            } else if constexpr (KIND == 1) {     // IMNMX: a = min(a, b) ^ ... (max then min)
                asm volatile("min.u32 %0, %0, %1;\n\tmax.u32 %0, %0, %2;" : "+r"(a[k]) : "r"(b), "r"(c));
            } else if constexpr (KIND == 2) {     // ISETP + SEL: a = a < b ? a + c : a - c (select)
                asm volatile("{ .reg .pred p; setp.lt.u32 p, %0, %1; selp.u32 %0, %2, %0, p; }"
                             : "+r"(a[k]) : "r"(b), "r"(c));
            } else if constexpr (KIND == 3) {     // SHFL
                a[k] = __shfl_xor_sync(0xffffffffu, a[k], 1 + (k & 15)) + 1u;
            } else if constexpr (KIND == 4) {     // 64-bit add (IADD3 + IADD3.X)
                asm volatile("add.u64 %0, %0, %1;" : "+l"(w[k]) : "l"((unsigned long long)b << 20 | c));
            } else {                              // IMAD: a = a * b + c
                asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(a[k]) : "r"(b | 1u), "r"(c));
            }
        }
    }
    uint32_t acc = 0;
#pragma unroll
    for (int k = 0; k < UB_CHAINS; k++) acc ^= a[k] ^ (uint32_t)w[k] ^ (uint32_t)(w[k] >> 32);
    if (acc == 0x9E3779B9u) sink[blockIdx.x] = acc;   // never true in practice; keeps the chains live
}

// SASS instructions per chain step of each kind (cuobjdump -sass of this file for sm_100a: the two
// adds fuse into one IADD3; min + max = 2 VIMNMX; ISETP + SEL; SHFL.BFLY + an add; IADD3 +
// IADD3.X; one IMAD) -- the rate reported is thread-level instructions per second
constexpr double OPS_PER_STEP[6] = {1.0, 2.0, 2.0, 2.0, 2.0, 1.0};

}  // namespace

extern "C" dip_status dip_ubench_int(uint32_t kind, int device, double *ops_per_s, double *ms) {
    using namespace diph;
    if (kind > 5 || !ops_per_s) return fail(DIP_EINVAL, "kind in 0..5");
    CUDA_TRY(cudaSetDevice(device));
    cudaDeviceProp prop;
    CUDA_TRY(cudaGetDeviceProperties(&prop, device));
    uint32_t *sink = nullptr;
    const int blocks = prop.multiProcessorCount * 8;
    CUDA_TRY(cudaMalloc(&sink, blocks * 4));
    cudaEvent_t e0, e1;
    CUDA_TRY(cudaEventCreate(&e0));
    CUDA_TRY(cudaEventCreate(&e1));
    auto launch = [&](uint32_t seed) {
        switch (kind) {
        case 0: ub_kernel<0><<<blocks, 256>>>(seed, sink); break;
        case 1: ub_kernel<1><<<blocks, 256>>>(seed, sink); break;
        case 2: ub_kernel<2><<<blocks, 256>>>(seed, sink); break;
        case 3: ub_kernel<3><<<blocks, 256>>>(seed, sink); break;
        case 4: ub_kernel<4><<<blocks, 256>>>(seed, sink); break;
        default: ub_kernel<5><<<blocks, 256>>>(seed, sink); break;
        }
    };
    launch(1);                               // warm-up
    float best = 1e30f;
    for (int rep = 0; rep < 5; rep++) {
        cudaEventRecord(e0);
        launch(2 + rep);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float t = 0.f;
        cudaEventElapsedTime(&t, e0, e1);
        best = t < best ? t : best;
    }
    cudaError_t e = cudaGetLastError();
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(sink);
    if (e != cudaSuccess) return fail(DIP_ECUDA, cudaGetErrorString(e));
    const double threads = (double)blocks * 256.0;
    *ops_per_s = threads * UB_ITERS * UB_CHAINS * OPS_PER_STEP[kind] / (best * 1e-3);
    if (ms) *ms = best;
    g_launches += 6;
    return DIP_OK;
}
