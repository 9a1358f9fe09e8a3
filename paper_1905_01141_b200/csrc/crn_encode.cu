/* crn_encode.cu -- rate-1/3 LTE turbo encoder on the device (the paper's
 * downlink "encoding function"; NEXT row f3 of DESIGN.md).
 * One thread per code block: optional CRC24A/B attach over the first K-24 bits
 * (fillers counted as 0), RSC 1 over c, RSC 2 over c'_i = c_{Pi(i)} with Pi
 * advanced by the QPP forward recurrence, 12 tail bits column-wise (R11).
 * Used by bench.py to build its synthetic uplink inputs on the GPU. */
#include <cuda_runtime.h>
#include <stdint.h>

#include <mutex>

#include "crn_internal.h"
#include "qpp_table.h"

namespace {
__constant__ int16_t c_f1[CRN_NUM_K], c_f2[CRN_NUM_K];

/* index of K in the ascending size table (closed form of SPEC.md:217's set) */
__device__ __forceinline__ int crn_k_index_dev(int K) {
    if (K <= 512) return (K - 40) / 8;
    if (K <= 1024) return 60 + (K - 528) / 16;
    if (K <= 2048) return 92 + (K - 1056) / 32;
    return 124 + (K - 2112) / 64;
}

struct CbView {
    const uint8_t *info;
    int K, F, L;           /* L = number of attached CRC bits (0 or 24) */
    uint32_t crc;
    __device__ uint32_t bit(int n) const {
        if (n < F) return 0u;
        if (n < K - L) return info[n] & 1u;
        return (crc >> (23 - (n - (K - L)))) & 1u;
    }
};

__device__ __forceinline__ void rsc(uint32_t &r1, uint32_t &r2, uint32_t &r3, uint32_t u, uint32_t &z) {
    uint32_t a = u ^ r2 ^ r3;
    z = a ^ r1 ^ r3;
    r3 = r2; r2 = r1; r1 = a;
}

__global__ void encode_kernel(const crn_cb_desc *__restrict__ desc, int n_cb, const uint8_t *__restrict__ info,
                              int attach, uint8_t *d0, uint8_t *d1, uint8_t *d2) {
    const int cb = blockIdx.x * blockDim.x + threadIdx.x;
    if (cb >= n_cb) return;
    const crn_cb_desc d = desc[cb];
    CbView v{info + d.ext_off, d.K, d.F, attach ? 24 : 0, 0u};
    if (attach) {
        const uint32_t poly = d.crc_kind == CRN_CRC24A ? 0x864CFBu : 0x800063u;
        uint32_t reg = 0;
        for (int n = 0; n < d.K - 24; n++) {
            uint32_t fb = ((reg >> 23) ^ v.bit(n)) & 1u;
            reg = ((reg << 1) & 0xFFFFFFu) ^ (fb ? poly : 0u);
        }
        v.crc = reg;
    }
    uint8_t *o0 = d0 + d.llr_off, *o1 = d1 + d.llr_off, *o2 = d2 + d.llr_off;
    const int K = d.K;
    uint32_t r1 = 0, r2 = 0, r3 = 0, z;
    for (int n = 0; n < K; n++) {
        uint32_t u = v.bit(n);
        rsc(r1, r2, r3, u, z);
        o0[n] = (uint8_t)u;
        o1[n] = (uint8_t)z;
    }
    uint8_t t[12];
    for (int k = 0; k < 3; k++) {           /* termination: u = r2^r3, z = r1^r3 */
        uint32_t u = r2 ^ r3;
        t[2 * k] = (uint8_t)u;
        t[2 * k + 1] = (uint8_t)(r1 ^ r3);
        r3 = r2; r2 = r1; r1 = 0;
    }
    const int ki = crn_k_index_dev(K);
    const int64_t f1 = c_f1[ki], f2 = c_f2[ki];
    int64_t pi = 0, g = (f1 + f2) % K;      /* Pi(x+1) = Pi(x) + g(x), g(x+1) = g(x) + 2 f2 (mod K) */
    r1 = r2 = r3 = 0;
    for (int i = 0; i < K; i++) {
        rsc(r1, r2, r3, v.bit((int)pi), z);
        o2[i] = (uint8_t)z;
        pi += g; if (pi >= K) pi -= K;
        g += 2 * f2; g %= K;
    }
    for (int k = 0; k < 3; k++) {
        uint32_t u = r2 ^ r3;
        t[6 + 2 * k] = (uint8_t)u;
        t[6 + 2 * k + 1] = (uint8_t)(r1 ^ r3);
        r3 = r2; r2 = r1; r1 = 0;
    }
    for (int m = 0; m < 12; m++) {
        uint8_t *o = (m % 3 == 0) ? o0 : (m % 3 == 1) ? o1 : o2;
        o[K + m / 3] = t[m];
    }
}
}  // namespace

extern "C" int crn_launch_encode(const crn_cb_desc *d_desc, int32_t n_cb, const uint8_t *info, int32_t attach,
                                 uint8_t *d0, uint8_t *d1, uint8_t *d2, const crn_tables *, void *stream) {
    static std::mutex mu;
    static uint64_t done = 0;                   /* bit d: the QPP constants are on device d */
    int dev;
    if (cudaGetDevice(&dev) != cudaSuccess) return CRN_ECUDA;
    {
        std::lock_guard<std::mutex> lk(mu);
        if (dev >= 64 || !((done >> dev) & 1u)) {
            if (cudaMemcpyToSymbol(c_f1, crn_qpp_f1, sizeof(crn_qpp_f1)) != cudaSuccess ||
                cudaMemcpyToSymbol(c_f2, crn_qpp_f2, sizeof(crn_qpp_f2)) != cudaSuccess)
                return CRN_ECUDA;
            if (dev < 64) done |= 1ull << dev;
        }
    }
    encode_kernel<<<(n_cb + 127) / 128, 128, 0, (cudaStream_t)stream>>>(d_desc, n_cb, info, attach, d0, d1, d2);
    return cudaGetLastError() == cudaSuccess ? CRN_OK : CRN_ECUDA;
}
