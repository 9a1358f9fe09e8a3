/* crn_ubench.cu -- int16x2 ALU throughput microbenchmark (DESIGN.md "ALU peak",
 * SURVEY G8): the roofline denominator of the decoder.  Each thread runs a ring
 * of 8 independent registers through one opcode so the loop body is 8 x the
 * opcode under test plus the loop overhead (checked with cuobjdump -sass).
 * Launched at full occupancy (148 SMs x 2048 threads). */
#include <cuda_runtime.h>
#include <stdint.h>

#include "crn_internal.h"

namespace {
template <int OP>
__device__ __forceinline__ uint32_t op(uint32_t a, uint32_t b, uint32_t c) {
    if (OP == 0) return __vadd2(a, b);                 /* VIADD.16x2      */
    if (OP == 1) return __vmaxs2(a, b);                /* VIMNMX.S16x2    */
    if (OP == 2) return __vimax3_s16x2(a, b, c);       /* VIMNMX3.S16x2   */
    return __viaddmax_s16x2(a, b, c);                  /* VIADDMNMX.S16x2 */
}

template <int OP>
__global__ void ubench_kernel(uint32_t *out, int iters, uint32_t seed, long long *cycles) {
    uint32_t x[8];
#pragma unroll
    for (int k = 0; k < 8; k++) x[k] = seed * (threadIdx.x + 7 * k + 1) + k;
    __syncthreads();
    long long t0 = clock64();
    for (int i = 0; i < iters; i++) {
#pragma unroll
        for (int r = 0; r < 4; r++) {
#pragma unroll
            for (int k = 0; k < 8; k++) x[k] = op<OP>(x[k], x[(k + 1) & 7], x[(k + 2) & 7]);
        }
    }
    __syncthreads();
    long long t1 = clock64();
    uint32_t acc = 0;
#pragma unroll
    for (int k = 0; k < 8; k++) acc ^= x[k];
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
}
}  // namespace

extern "C" int crn_launch_ubench(int32_t opcode, int64_t *lane_instr, float *ms, int64_t *cycles_per_block) {
    int dev, sms;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int threads = 256, blocks = sms * 8, iters = 4096;
    uint32_t *out;
    long long *cyc;
    if (cudaMalloc(&out, sizeof(uint32_t) * threads * blocks) != cudaSuccess) return CRN_ENOMEM;
    if (cudaMalloc(&cyc, sizeof(long long) * blocks) != cudaSuccess) { cudaFree(out); return CRN_ENOMEM; }
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    auto run = [&]() {
        switch (opcode) {
            case 0: ubench_kernel<0><<<blocks, threads>>>(out, iters, 12345u, cyc); break;
            case 1: ubench_kernel<1><<<blocks, threads>>>(out, iters, 12345u, cyc); break;
            case 2: ubench_kernel<2><<<blocks, threads>>>(out, iters, 12345u, cyc); break;
            default: ubench_kernel<3><<<blocks, threads>>>(out, iters, 12345u, cyc); break;
        }
    };
    run();                                   /* warm-up */
    cudaEventRecord(e0);
    run();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(ms, e0, e1);
    long long h[4096];
    int nb = blocks < 4096 ? blocks : 4096;
    cudaMemcpy(h, cyc, sizeof(long long) * nb, cudaMemcpyDeviceToHost);
    long long mx = 0;
    for (int b = 0; b < nb; b++) mx = h[b] > mx ? h[b] : mx;
    *cycles_per_block = mx;
    *lane_instr = (int64_t)blocks * threads * (int64_t)iters * 32;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(out);
    cudaFree(cyc);
    return cudaGetLastError() == cudaSuccess ? CRN_OK : CRN_ECUDA;
}
