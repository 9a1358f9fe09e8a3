// Per-trellis-step cost of the decoder's recursions for a lone warp vs several
// warps per SM sub-partition (DESIGN.md §10 "TTI latency"): one CTA of NW warps
// runs N steps of
//   mode 0: alpha_step_d only (the dependent ACS + normalisation chain)
//   mode 1: + one tcgen05.st of the 8 metrics per step (phase 1 store)
//   mode 2: the phase-1 step of siso_split: gathered + plane LDS, branch-metric
//           STS, tcgen05.st, alpha_step_d
//   mode 3: the phase-2 step: tcgen05.ld one step ahead + wait, LDS of the
//           branch-metric chunk and parity, lambda_le + STS, beta_step_d
//   mode 4: mode 2 in four distinct code copies (alpha / beta x two gather
//           halves) run in rotation: the decoder's phase-1 code footprint
// using the kernel's own helpers (this file includes crn_decode.cu).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr
//        -I paper_1905_01141_b200/csrc tools/ubench/step_lat.cu -o tools/ubench/step_lat
#include "../../paper_1905_01141_b200/csrc/crn_decode.cu"

#include <cstdio>

namespace {

template <int V>
__device__ __forceinline__ void phase1_copy(u32 (&m)[NS], const u32 (&sn)[HW], const u32 (&qq)[HW], u32 lp_s, uint2 *ch,
                                            u32 ta) {
    u32 av[HW], pv[HW];
    const u32 off = (V & 1) ? 4u * 512u : 0u;
    av[0] = lds_at(qq[0] + off);
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(pv[0]) : "r"(lp_s));
#pragma unroll
    for (int s = 0; s < HW; s++) {
        if (s + 1 < HW) {
            av[s + 1] = lds_at(qq[s + 1] + off);
            asm volatile("ld.shared.u32 %0, [%1];" : "=r"(pv[s + 1]) : "r"(lp_s + 4 * (s + 1) * 384));
        }
        const u32 d = vadd(sn[s], av[s]);
        const u32 x = vadd(vadd(d, pv[s]), pv[s]);
        ch[s * 256] = make_uint2(x, d);
        tm_store8(ta + s * 8, m);
        if (V & 2) beta_step_d<false>(m, pv[s], x, d);
        else alpha_step_d<false>(m, pv[s], x, d);
    }
    tm_wait_st();
}

template <int MODE>
__global__ void __launch_bounds__(384, 1) steplat(u32 *out, long long *cyc, int nsteps) {
    extern __shared__ __align__(16) u32 sm[];
    __shared__ u32 s_t;
    const int tid = threadIdx.x, warp = tid >> 5;
    for (int i = tid; i < 16384; i += blockDim.x) sm[i] = (u32)(i * 2654435761u) & 0x03FF03FFu;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_addr(&s_t)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const u32 ta = s_t + ((u32)((warp & 3) * 32) << 16) + (u32)((warp >> 2) * 128);
    u32 m[NS], sn[HW], qq[HW];
#pragma unroll
    for (int s = 0; s < NS; s++) m[s] = (u32)(tid * 7 + s) & 0x00FF00FFu;
    const u32 base = smem_addr(sm);
#pragma unroll
    for (int s = 0; s < HW; s++) {
        sn[s] = (u32)(tid * 13 + s * 5) & 0x01FF01FFu;
        qq[s] = base + 4u * (u32)((s * 384 + ((tid * 37 + s * 11) % 384)) & 8191);   /* gather: some row word */
    }
    const u32 lp_s = base + 4u * (8192u + (u32)tid);
    uint2 *ch = reinterpret_cast<uint2 *>(sm + 16384) + (tid & 255);
    u32 *le = sm + 4096 + tid;
    __syncthreads();
    const long long t0 = clock64();
    for (int it = 0; it < nsteps; it += HW) {
        if (MODE == 4) {
            const int r = (it / HW) & 3;
            if (r == 0) phase1_copy<0>(m, sn, qq, lp_s, ch, ta);
            else if (r == 1) phase1_copy<1>(m, sn, qq, lp_s, ch, ta);
            else if (r == 2) phase1_copy<2>(m, sn, qq, lp_s, ch, ta);
            else phase1_copy<3>(m, sn, qq, lp_s, ch, ta);
        } else if (MODE <= 2) {
            u32 av[HW], pv[HW];
            if (MODE == 2) {
                av[0] = lds_at(qq[0]);
                asm volatile("ld.shared.u32 %0, [%1];" : "=r"(pv[0]) : "r"(lp_s));
            }
#pragma unroll
            for (int s = 0; s < HW; s++) {
                u32 x, d, p;
                if (MODE == 2) {
                    if (s + 1 < HW) {
                        av[s + 1] = lds_at(qq[s + 1]);
                        asm volatile("ld.shared.u32 %0, [%1];" : "=r"(pv[s + 1]) : "r"(lp_s + 4 * (s + 1) * 384));
                    }
                    d = vadd(sn[s], av[s]);
                    x = vadd(vadd(d, pv[s]), pv[s]);
                    p = pv[s];
                    ch[s * 256] = make_uint2(x, d);
                } else {
                    d = sn[s];
                    p = sn[(s + 3) & 15];
                    x = vadd(vadd(d, p), p);
                }
                if (MODE >= 1) tm_store8(ta + s * 8, m);
                alpha_step_d<false>(m, p, x, d);
            }
            if (MODE >= 1) tm_wait_st();
        } else {
            u32 bufA[NS], bufB[NS];
            tm_load8(ta + (HW - 1) * 8, bufA);
#pragma unroll 2
            for (int s = HW - 1; s >= 0; s -= 2) {
#pragma unroll
                for (int h = 0; h < 2; h++) {
                    const int ss = s - h;
                    u32 *cur = h ? bufB : bufA, *nx = h ? bufA : bufB;
                    const uint2 g = ch[ss * 256];
                    u32 p;
                    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(p) : "r"(lp_s + 4 * ss * 384));
                    tm_wait_ld8(cur);
                    tm_load8(ta + (ss > 0 ? ss - 1 : 0) * 8, nx);
                    le[ss * 384] = lambda_le<false>(cur, m, p);
                    beta_step_d<false>(m, p, g.x, g.y);
                }
            }
            tm_wait_ld8(bufA);
        }
    }
    const long long t1 = clock64();
    u32 acc = 0;
#pragma unroll
    for (int s = 0; s < NS; s++) acc ^= m[s];
    out[blockIdx.x * blockDim.x + tid] = acc;
    if ((tid & 31) == 0) cyc[blockIdx.x * 12 + warp] = t1 - t0;
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(s_t));
}

}  // namespace

int main() {
    u32 *out;
    long long *cyc;
    cudaMalloc(&out, 4 * 384 * 148);
    cudaMalloc(&cyc, 8 * 12 * 148);
    const int N = 4096;
    const void *ks[5] = {(const void *)steplat<0>, (const void *)steplat<1>, (const void *)steplat<2>,
                         (const void *)steplat<3>, (const void *)steplat<4>};
    for (int k = 0; k < 5; k++) cudaFuncSetAttribute(ks[k], cudaFuncAttributeMaxDynamicSharedMemorySize, 32768 * 4);
    printf("{\"steps\": %d, \"cycles_per_step\": {", N);
    const int nws[3] = {1, 4, 12};
    for (int mode = 0; mode < 5; mode++) {
        for (int w = 0; w < 3; w++) {
            const int nt = 32 * nws[w];
            for (int rep = 0; rep < 2; rep++) {
                switch (mode) {
                    case 0: steplat<0><<<1, nt, 32768 * 4>>>(out, cyc, N); break;
                    case 1: steplat<1><<<1, nt, 32768 * 4>>>(out, cyc, N); break;
                    case 2: steplat<2><<<1, nt, 32768 * 4>>>(out, cyc, N); break;
                    case 3: steplat<3><<<1, nt, 32768 * 4>>>(out, cyc, N); break;
                    default: steplat<4><<<1, nt, 32768 * 4>>>(out, cyc, N); break;
                }
            }
            long long h[12];
            cudaError_t e = cudaMemcpy(h, cyc, 8 * 12, cudaMemcpyDeviceToHost);
            if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
            long long mx = 0;
            for (int i = 0; i < nws[w]; i++) mx = h[i] > mx ? h[i] : mx;
            printf("%s\"mode%d_warps%d\": %.1f", (mode || w) ? ", " : "", mode, nws[w], (double)mx / N);
        }
    }
    printf("}}\n");
    return 0;
}
