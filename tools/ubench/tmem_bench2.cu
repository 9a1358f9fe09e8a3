// TMEM correctness + throughput with 6 or 8 warps, one CTA per SM forced by 200 KB dynamic smem.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void k(uint32_t* out, long long* cyc, int iters, int ncols_per_warp_group) {
    extern __shared__ uint32_t dyn[];
    __shared__ uint32_t s_taddr;
    const int warp = threadIdx.x / 32;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" :: "r"(smem_u32(&s_taddr)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tbase = s_taddr;
    const uint32_t ta = tbase + (((warp % 4) * 32) << 16) + (warp / 4) * 256;
    uint32_t bad = 0;
    for (int c = 0; c < 256; c += 16) {
        uint32_t v = (threadIdx.x << 16) | c;
        asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};"
            :: "r"(ta + c), "r"(v), "r"(v+1), "r"(v+2), "r"(v+3), "r"(v+4), "r"(v+5), "r"(v+6), "r"(v+7), "r"(v+8), "r"(v+9),
               "r"(v+10), "r"(v+11), "r"(v+12), "r"(v+13), "r"(v+14), "r"(v+15));
    }
    asm volatile("tcgen05.wait::st.sync.aligned;");
    __syncthreads();
    long long t0 = clock64();
    uint32_t acc = 0;
    for (int i = 0; i < iters; i++) {
        const int c = (i * 16) & 255;
        uint32_t r[16];
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                     : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                       "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
                     : "r"(ta + c));
        asm volatile("tcgen05.wait::ld.sync.aligned;");
        for (int q = 0; q < 16; q++) { bad += r[q] != ((threadIdx.x << 16) | (c + q)); acc += r[q]; }
    }
    long long t1 = clock64();
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
    if (bad) atomicAdd(&out[0], 0x40000000u);
    if (bad && (threadIdx.x % 32) == 0) printf("blk %d warp %d bad %u\n", blockIdx.x, warp, bad);
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" :: "r"(tbase));
}

int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    uint32_t* out; long long* cyc; cudaMalloc(&out, sms * 256 * 4); cudaMalloc(&cyc, sms * 8);
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    long long h[256];
    for (int nw : {4, 6, 8}) {
        int iters = 8192;
        cudaMemset(out, 0, sms * 256 * 4);
        k<<<sms, nw * 32, 200 * 1024>>>(out, cyc, iters, 0);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("warps=%d error %s\n", nw, cudaGetErrorString(e)); return 1; }
        cudaMemcpy(h, cyc, sms * 8, cudaMemcpyDeviceToHost);
        uint32_t o0; cudaMemcpy(&o0, out, 4, cudaMemcpyDeviceToHost);
        long long mx = 0; for (int i = 0; i < sms; i++) mx = h[i] > mx ? h[i] : mx;
        printf("warps=%d ld.x16+wait cycles/iter=%.1f bytes/clk/SM=%.1f bad=%u\n", nw, (double)mx / iters,
               16.0 * 4 * 32 * nw * iters / mx, o0 >> 30);
    }
    return 0;
}
