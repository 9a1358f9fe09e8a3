// TMEM (tcgen05.ld/st) throughput + correctness microbenchmark for sm_100a.
// One CTA per SM, 4..8 warps; each warp accesses its lane quadrant (warp % 4).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int NW>
__global__ void tmem_kernel(uint32_t* out, long long* cyc, int iters, int mode) {
    __shared__ uint32_t s_taddr;
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" :: "r"(smem_u32(&s_taddr)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tbase = s_taddr;
    const uint32_t quad = (warp % 4) * 32, colbase = (warp / 4) * 256;
    const uint32_t ta = tbase + (quad << 16) + colbase;
    // write pattern: value = (thread << 16) | col
    for (int c = 0; c < 256; c += 4) {
        uint32_t v0 = (threadIdx.x << 16) | c, v1 = v0 + 1, v2 = v0 + 2, v3 = v0 + 3;
        asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %2, %3, %4};" :: "r"(ta + c), "r"(v0), "r"(v1), "r"(v2), "r"(v3));
    }
    asm volatile("tcgen05.wait::st.sync.aligned;");
    // correctness: read back
    uint32_t bad = 0;
    for (int c = 0; c < 256; c += 2) {
        uint32_t r0, r1;
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0, %1}, [%2];" : "=r"(r0), "=r"(r1) : "r"(ta + c));
        asm volatile("tcgen05.wait::ld.sync.aligned;");
        bad += (r0 != ((threadIdx.x << 16) | c)) + (r1 != ((threadIdx.x << 16) | (c + 1)));
    }
    __syncthreads();
    long long t0 = clock64();
    uint32_t acc = 0;
    if (mode == 0) {            // ld x2, dependent use each iteration (latency-ish)
        for (int i = 0; i < iters; i++) {
            uint32_t r0, r1;
            asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0, %1}, [%2];" : "=r"(r0), "=r"(r1) : "r"(ta + ((i * 2 + acc) & 255)));
            asm volatile("tcgen05.wait::ld.sync.aligned;");
            acc += r0 ^ r1;
        }
    } else if (mode == 1) {     // ld x16 throughput (4 loads in flight, one wait)
        for (int i = 0; i < iters; i++) {
            uint32_t r[16];
            asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                         : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                           "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
                         : "r"(ta + ((i * 16) & 255)));
            asm volatile("tcgen05.wait::ld.sync.aligned;");
#pragma unroll
            for (int k = 0; k < 16; k++) acc += r[k];
        }
    } else {                    // st x16 throughput
        for (int i = 0; i < iters; i++) {
            uint32_t v = i + threadIdx.x;
            asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1};"
                         :: "r"(ta + ((i * 16) & 255)), "r"(v));
        }
        asm volatile("tcgen05.wait::st.sync.aligned;");
    }
    long long t1 = clock64();
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc + bad * 0x10000000u;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
    if (threadIdx.x == 0 && bad) printf("block %d thread 0 bad %u\n", blockIdx.x, bad);
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" :: "r"(tbase));
}

int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    uint32_t* out; long long* cyc; cudaMalloc(&out, sms * 256 * 4); cudaMalloc(&cyc, sms * 8);
    long long h[256];
    const char* names[3] = {"ld.x2 dependent (latency)", "ld.x16 + wait", "st.x16"};
    for (int nw : {4, 8}) for (int mode = 0; mode < 3; mode++) {
        int iters = 4096;
        if (nw == 4) tmem_kernel<4><<<sms, 128>>>(out, cyc, iters, mode); else tmem_kernel<8><<<sms, 256>>>(out, cyc, iters, mode);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
        cudaMemcpy(h, cyc, sms * 8, cudaMemcpyDeviceToHost);
        long long mx = 0; for (int i = 0; i < sms; i++) mx = h[i] > mx ? h[i] : mx;
        double words = (mode == 0 ? 2.0 : 16.0) * iters * 32 * nw;   // 32-bit words per SM
        printf("warps=%d %-28s cycles/iter=%.1f  bytes/clk/SM=%.1f\n", nw, names[mode], (double)mx / iters, words * 4 / mx);
    }
    return 0;
}
