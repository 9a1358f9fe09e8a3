/* crn_encode.cu -- rate-1/3 LTE turbo encoder on the device (the paper's
 * downlink "encoding function"; NEXT row f3 of DESIGN.md).
 * One warp per code block: optional CRC24A/B attach over the first K-24 bits
 * (fillers counted as 0; per-lane CRC registers combined by a GF(2) multiply),
 * RSC 1 over c, RSC 2 over c'_i = c_{Pi(i)} with Pi advanced by the QPP
 * forward recurrence, each split into 32 chunks by linearity (below), 12 tail
 * bits column-wise (R11).  Also builds bench.py's synthetic uplink inputs. */
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

/* ---- warp-per-CB encoder.  The RSC code is linear over GF(2): with state
 * s = 4 r1 + 2 r2 + r3, one step is s' = A s + 4u and z = c.s + u, and A has
 * order 7 (feedback 1 + D^2 + D^3 is primitive), so A^L = A^(L mod 7).  Each
 * lane encodes a contiguous chunk of the CB twice: from state 0 to learn the
 * chunk's input-driven end state f, then -- after a 32-step scan of
 * s_{l+1} = A^{L_l} s_l + f_l gives every chunk's true start state -- again,
 * emitting its parity bits.  Bits are staged per warp in shared memory (the
 * second encoder gathers c_{Pi(i)} there) and written out coalesced. */
constexpr int ENC_WARPS = 4;
constexpr int ENC_STAGE = 6144 + 2 * 6148;      /* per warp: c, then parity bytes of both encoders */

__device__ __forceinline__ int rsc_A(int s) {       /* zero-input step */
    const int r1 = (s >> 2) & 1, r2 = (s >> 1) & 1, r3 = s & 1;
    return ((r2 ^ r3) << 2) | (r1 << 1) | r2;
}

__device__ __forceinline__ int rsc_Apow(int s, int L) {
    for (int i = L % 7; i > 0; i--) s = rsc_A(s);
    return s;
}

__device__ __forceinline__ uint32_t mulmod24(uint32_t a, uint32_t b, uint32_t poly) {
    uint32_t acc = 0;
    for (int k = 23; k >= 0; k--) {
        acc = ((acc << 1) & 0xFFFFFFu) ^ ((acc & 0x800000u) ? poly : 0u);
        if ((b >> k) & 1u) acc ^= a;
    }
    return acc;
}

__device__ __forceinline__ uint32_t xpow24(int64_t e, uint32_t poly) {
    uint32_t r = 1, base = 2;
    while (e > 0) {
        if (e & 1) r = mulmod24(r, base, poly);
        base = mulmod24(base, base, poly);
        e >>= 1;
    }
    return r;
}

/* one RSC encoder over the warp's staged input: pass 1 (zero start), scan, pass 2 */
template <bool INTERLEAVED>
__device__ __forceinline__ int rsc_warp(const uint8_t *c, uint8_t *z_out, int K, int lane, int64_t f1, int64_t f2) {
    const int per = (K + 31) / 32, c0 = min(K, lane * per), c1 = min(K, c0 + per), L = c1 - c0;
    const int64_t f2x2 = (2 * f2) % K;
    auto input = [&](int k, int64_t &pi, int64_t &g) -> int {
        if (!INTERLEAVED) return c[k];
        const int v = c[pi];
        pi += g;
        if (pi >= K) pi -= K;
        g += f2x2;                                    /* 2 f2 mod K: 2 f2 itself may exceed K */
        if (g >= K) g -= K;
        return v;
    };
    auto pi0 = [&](int64_t &pi, int64_t &g) {       /* Pi(c0) and the recurrence increment g(c0) */
        const int64_t k = c0;
        pi = (f1 * k + f2 * ((k * k) % K)) % K;
        g = (f1 + f2 * ((2 * k + 1) % K)) % K;
    };
    int64_t pi = 0, g = 0;
    if (INTERLEAVED) pi0(pi, g);
    int s = 0;
    for (int k = c0; k < c1; k++) {
        const int u = input(k, pi, g), r2 = (s >> 1) & 1, r3 = s & 1;
        s = (((u ^ r2 ^ r3) & 1) << 2) | (((s >> 2) & 1) << 1) | r2;
    }
    /* start state of every chunk: s_{l+1} = A^{L_l} s_l + f_l (lane 0 -> 31) */
    int start = 0, run = 0;
    for (int l = 0; l < 32; l++) {
        const int fl = __shfl_sync(0xFFFFFFFFu, s, l), Ll = __shfl_sync(0xFFFFFFFFu, L, l);
        if (l == lane) start = run;
        run = rsc_Apow(run, Ll) ^ fl;
    }
    if (INTERLEAVED) pi0(pi, g);
    s = start;
    for (int k = c0; k < c1; k++) {
        const int u = input(k, pi, g), r1 = (s >> 2) & 1, r2 = (s >> 1) & 1, r3 = s & 1;
        const int a = u ^ r2 ^ r3;
        z_out[k] = (uint8_t)(a ^ r1 ^ r3);
        s = (a << 2) | (r1 << 1) | r2;
    }
    return run;                                       /* the state after all K inputs */
}

__global__ void __launch_bounds__(32 * ENC_WARPS)
encode_kernel(const crn_cb_desc *__restrict__ desc, int n_cb, const uint8_t *__restrict__ info,
              int attach, uint8_t *d0, uint8_t *d1, uint8_t *d2) {
    extern __shared__ uint8_t enc_sm[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int cb = blockIdx.x * ENC_WARPS + warp;
    if (cb >= n_cb) return;                           /* whole warps */
    const crn_cb_desc d = desc[cb];
    const int K = d.K, F = d.F, L = attach ? 24 : 0;
    uint8_t *c = enc_sm + (size_t)warp * ENC_STAGE, *z1 = c + 6144, *z2 = z1 + 6148;
    const uint8_t *src = info + d.ext_off;
    for (int n = lane; n < K - L; n += 32) c[n] = n < F ? 0 : (src[n] & 1u);
    __syncwarp();
    if (attach) {                                     /* CRC of bits [0, K-24): chunk registers combined */
        const uint32_t poly = d.crc_kind == CRN_CRC24A ? 0x864CFBu : 0x800063u;
        const int N = K - 24, per = (N + 31) / 32, b0 = min(N, lane * per), b1 = min(N, b0 + per);
        uint32_t reg = 0;
        for (int n = b0; n < b1; n++) {
            const uint32_t fb = ((reg >> 23) ^ c[n]) & 1u;
            reg = ((reg << 1) & 0xFFFFFFu) ^ (fb ? poly : 0u);
        }
        uint32_t part = b0 < b1 ? mulmod24(reg, xpow24(N - b1, poly), poly) : 0u;
        for (int o = 16; o > 0; o >>= 1) part ^= __shfl_xor_sync(0xFFFFFFFFu, part, o);
        if (lane < 24) c[N + lane] = (uint8_t)((part >> (23 - lane)) & 1u);
        __syncwarp();
    }
    const int ki = crn_k_index_dev(K);
    const int64_t f1 = c_f1[ki], f2 = c_f2[ki];
    const int s1 = rsc_warp<false>(c, z1, K, lane, f1, f2);
    const int s2 = rsc_warp<true>(c, z2, K, lane, f1, f2);
    __syncwarp();
    uint8_t *o0 = d0 + d.llr_off, *o1 = d1 + d.llr_off, *o2 = d2 + d.llr_off;
    for (int n = lane; n < K; n += 32) {
        o0[n] = c[n];
        o1[n] = z1[n];
        o2[n] = z2[n];
    }
    if (lane == 0) {                                  /* termination: u = r2^r3, x = u, z = r1^r3 (R11) */
        uint8_t t[12];
        int s = s1;
        for (int k = 0; k < 3; k++) {
            const int r1 = (s >> 2) & 1, r2 = (s >> 1) & 1, r3 = s & 1;
            t[2 * k] = (uint8_t)(r2 ^ r3);
            t[2 * k + 1] = (uint8_t)(r1 ^ r3);
            s = (r1 << 1) | r2;
        }
        s = s2;
        for (int k = 0; k < 3; k++) {
            const int r1 = (s >> 2) & 1, r2 = (s >> 1) & 1, r3 = s & 1;
            t[6 + 2 * k] = (uint8_t)(r2 ^ r3);
            t[6 + 2 * k + 1] = (uint8_t)(r1 ^ r3);
            s = (r1 << 1) | r2;
        }
        for (int m = 0; m < 12; m++) {
            uint8_t *o = (m % 3 == 0) ? o0 : (m % 3 == 1) ? o1 : o2;
            o[K + m / 3] = t[m];
        }
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
    static bool attr = false;
    if (!attr) {
        if (cudaFuncSetAttribute(encode_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, ENC_WARPS * ENC_STAGE) !=
            cudaSuccess)
            return CRN_ECUDA;
        attr = true;
    }
    encode_kernel<<<(n_cb + ENC_WARPS - 1) / ENC_WARPS, 32 * ENC_WARPS, ENC_WARPS * ENC_STAGE, (cudaStream_t)stream>>>(
        d_desc, n_cb, info, attach, d0, d1, d2);
    return cudaGetLastError() == cudaSuccess ? CRN_OK : CRN_ECUDA;
}
