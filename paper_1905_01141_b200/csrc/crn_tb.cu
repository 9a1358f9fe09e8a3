/* crn_tb.cu -- TB post-processing on the device (the
 * paper's "post-processing (combination of CBs)", and its TB
 * rule "a TB can be successfully decoded only when all CBs have been
 * individually decoded").
 *
 * One CTA per transport block.  The TB's bit stream b[0 .. tbs+24) is the
 * concatenation over its CBs r (segment order) of the decoded bits
 * [F_r, K_r - L) (fillers and CB CRC24B stripped; 36.212 5.1.2 read
 * backwards).  Thread j owns 32-bit output words [w0_j, w1_j) of that stream:
 * it gathers the bits from the CBs' packed words, writes the payload words
 * (LSB-first, the decoder's convention, R19) and runs the CRC24A
 * register over its bits in stream (MSB-first) order; the per-thread registers
 * are combined as crc(A||B) = crc(A) x^|B| + crc(B) mod g(x) (zero initial
 * register, so the CRC is linear) with x^e mod g by square-and-multiply.
 * tb_ok = (every CB's crc_ok) AND (combined register == 0).
 */
#include <cuda_runtime.h>
#include <stdint.h>

#include "crn_internal.h"

namespace {

constexpr int TB_THREADS = 256;
constexpr uint32_t POLY_A = 0x864CFBu;

__device__ __forceinline__ uint32_t mulmod(uint32_t a, uint32_t b) {   /* a(x) b(x) mod g_A(x) */
    uint32_t acc = 0;
    for (int k = 23; k >= 0; k--) {
        acc = ((acc << 1) & 0xFFFFFFu) ^ ((acc & 0x800000u) ? POLY_A : 0u);
        if ((b >> k) & 1u) acc ^= a;
    }
    return acc;
}

__device__ __forceinline__ uint32_t xpow(int64_t e) {                  /* x^e mod g_A(x) */
    uint32_t r = 1, base = 2;                                          /* x^0, x^1 */
    while (e > 0) {
        if (e & 1) r = mulmod(r, base);
        base = mulmod(base, base);
        e >>= 1;
    }
    return r;
}

/* n <= 32 bits of a CB starting at its bit k (LSB-first packed words), as the low bits */
__device__ __forceinline__ uint32_t cb_bits(const uint32_t *__restrict__ w, int64_t k, int n) {
    const int64_t wi = k >> 5;
    const int sh = (int)(k & 31);
    uint32_t v = __ldg(w + wi) >> sh;
    if (sh && sh + n > 32) v |= __ldg(w + wi + 1) << (32 - sh);
    return n >= 32 ? v : (v & ((1u << n) - 1u));
}

__global__ void __launch_bounds__(TB_THREADS)
tb_kernel(const crn_tb_desc *__restrict__ tbs, const crn_cb_desc *__restrict__ desc,
          const uint32_t *__restrict__ cb_words, const uint8_t *__restrict__ crc_ok, uint8_t *__restrict__ tb_ok,
          uint32_t *__restrict__ tb_words) {
    __shared__ int64_t s_start[CRN_TB_MAX_CB + 1];   /* stream position where CB r's bits begin */
    __shared__ int s_F[CRN_TB_MAX_CB];
    __shared__ int64_t s_woff[CRN_TB_MAX_CB];
    __shared__ uint32_t s_crc;
    __shared__ int s_all;
    const crn_tb_desc t = tbs[blockIdx.x];
    const int L = t.n_cb > 1 ? 24 : 0, tid = threadIdx.x;
    if (tid == 0) {
        int64_t p = 0;
        int all = 1;
        for (int r = 0; r < t.n_cb; r++) {
            const crn_cb_desc &d = desc[t.cb0 + r];
            s_start[r] = p;
            s_F[r] = d.F;
            s_woff[r] = d.bit_off;
            p += d.K - d.F - L;
            all &= crc_ok[t.cb0 + r] != 0;
        }
        s_start[t.n_cb] = p;
        s_crc = 0;
        s_all = all;
    }
    __syncthreads();
    const int64_t N = t.tbs + 24;                    /* payload + TB CRC24A */
    const int64_t nw = (N + 31) / 32;
    const int64_t per = (nw + TB_THREADS - 1) / TB_THREADS;
    const int64_t w0 = tid * per, w1 = w0 + per < nw ? w0 + per : nw;
    uint32_t reg = 0;
    int r = 0;
    for (int64_t w = w0; w < w1; w++) {
        const int64_t p0 = 32 * w, p1 = p0 + 32 < N ? p0 + 32 : N;
        /* the word's bits come from at most two CB segments: funnel-shift them out */
        while (p0 >= s_start[r + 1]) r++;
        const int n1 = (int)((s_start[r + 1] < p1 ? s_start[r + 1] : p1) - p0);
        uint32_t word = cb_bits(cb_words + s_woff[r], s_F[r] + (p0 - s_start[r]), n1);
        if (p0 + n1 < p1) word |= cb_bits(cb_words + s_woff[r + 1], s_F[r + 1], (int)(p1 - p0 - n1)) << n1;
        const int nb = (int)(p1 - p0);
        for (int i = 0; i < nb; i++) {               /* CRC24A register, stream (MSB-first) order */
            const uint32_t fb = ((reg >> 23) ^ (word >> i)) & 1u;
            reg = ((reg << 1) & 0xFFFFFFu) ^ (fb ? POLY_A : 0u);
        }
        if (tb_words) {                              /* payload words only (the CRC24A tail is not output) */
            const int64_t pw = (t.tbs + 31) / 32;
            if (w < pw) {
                const int64_t keep = t.tbs - p0;    /* payload bits in this word */
                tb_words[t.word_off + w] = keep >= 32 ? word : (word & ((1u << keep) - 1u));
            }
        }
    }
    if (w0 < w1) {
        const int64_t end = 32 * w1 < N ? 32 * w1 : N;
        atomicXor(&s_crc, mulmod(reg, xpow(N - end)));
    }
    __syncthreads();
    if (tid == 0) tb_ok[blockIdx.x] = (uint8_t)(s_all && s_crc == 0);
}

}  // namespace

extern "C" int crn_launch_tb(const crn_tb_desc *d_tbs, int32_t n_tb, const crn_cb_desc *d_desc,
                             const uint32_t *cb_words, const uint8_t *crc_ok, uint8_t *tb_ok, uint32_t *tb_words,
                             void *stream) {
    tb_kernel<<<n_tb, TB_THREADS, 0, (cudaStream_t)stream>>>(d_tbs, d_desc, cb_words, crc_ok, tb_ok, tb_words);
    return cudaGetLastError() == cudaSuccess ? CRN_OK : CRN_ECUDA;
}
