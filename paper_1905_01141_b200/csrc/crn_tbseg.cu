/* crn_tbseg.cu -- transport-block conditioning on the device: the "code block
 * creation, segmentation" pre-processing the paper times before its channel
 * coding (Performance captor KPIs) and the first step of its
 * encoding function (the TB is split into CBs, each then
 * turbo encoded), per TS 36.212 5.1.1-5.1.2 (R4, R6, R7):
 *
 *   b = payload || CRC24A(payload);  CB r = [F_r filler zeros][K_r - L - F_r bits
 *   of b][CRC24B of the CB's first K_r - 24 bits, if C > 1]
 *
 * with the segmentation (C, K+, K-, C-, F, L) from crn_segment_tb on the host
 * (O(1) per TB, like the decoder's bucketing).  One CTA per TB:
 *   tables   the byte-table CRCs and x^(32 m) mod g: built once per device
 *            (tbseg_init_kernel), copied into shared memory per CTA;
 *   pack     the payload (one bit per byte) into MSB-first words in shared
 *            memory, front-padded so it ends on a word boundary (leading zeros
 *            do not change a zero-initialised CRC), eight positions per thread;
 *   CRC24A   every thread runs the byte-table CRC over its run of words and
 *            multiplies its register by x^(32 m) mod g (m = words after the run,
 *            square-and-multiply over x^(32 2^k)), XOR-reduced over the CTA;
 *   CBs      all threads write the CB bytes (fillers, b's bits, the CRC24A bits
 *            for C = 1) coalesced, eight bytes per thread;
 *   CRC24B   a warp per CB: 32-bit segments of the CB's data aligned to its end,
 *            byte-table CRC each, times x^(32 m) (table), XOR-reduced by shuffles.
 * The CB contents are exactly crn_tb_build_cbs's (one bit per byte), ready for
 * crn_encode_batch. */
#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

#include <mutex>

#include "crn_internal.h"

namespace {

constexpr int SEG_THREADS = 256;
constexpr uint32_t POLY_A = 0x864CFBu, POLY_B = 0x800063u;
constexpr int XP_LOG = 16;                  /* x^(32 2^k), k < 16: up to 2^16 words (2 Mbit) */
constexpr int XPB_N = 6144 / 32 + 1;        /* x^(32 m) mod g_B, m <= 192 (one CB) */

__device__ __forceinline__ uint32_t crc_step_bit(uint32_t reg, uint32_t poly) {   /* reg x mod g */
    return ((reg << 1) & 0xFFFFFFu) ^ ((reg & 0x800000u) ? poly : 0u);
}

__device__ __forceinline__ uint32_t mulmod24(uint32_t a, uint32_t b, uint32_t poly) {   /* a b mod g */
    uint32_t acc = 0;
    for (int k = 23; k >= 0; k--) {
        acc = crc_step_bit(acc, poly);
        if ((b >> k) & 1u) acc ^= a;
    }
    return acc;
}

struct SegSmem {
    uint32_t tab[2][256];                   /* byte-at-a-time CRC24A / CRC24B, MSB-first */
    uint32_t xp2[2][XP_LOG];                /* x^(32 2^k) mod g */
    uint32_t xpb[XPB_N];                    /* x^(32 m) mod g_B */
    uint32_t red[SEG_THREADS / 32];
    uint32_t crc_a;
    uint32_t w[1];                          /* packed b (dynamic length) */
};

__device__ __forceinline__ uint32_t crc_bytes(uint32_t reg, uint32_t word, const uint32_t *tab) {
#pragma unroll
    for (int k = 0; k < 4; k++) {           /* the word's bytes, most significant first */
        const uint32_t byte = (word >> (24 - 8 * k)) & 0xFFu;
        reg = ((reg << 8) & 0xFFFFFFu) ^ tab[((reg >> 16) ^ byte) & 0xFFu];
    }
    return reg;
}

/* x^(32 m) mod g from the x^(32 2^k) table */
__device__ __forceinline__ uint32_t xpow32(const uint32_t *xp2, uint32_t m, uint32_t poly) {
    uint32_t r = 1;                         /* x^0 */
    for (int k = 0; m; k++, m >>= 1)
        if (m & 1u) r = mulmod24(r, xp2[k], poly);
    return r;
}

/* SegSmem's leading tables (tab, xp2, xpb: one contiguous run of words), per device */
constexpr int SEG_TAB_WORDS = 2 * 256 + 2 * XP_LOG + XPB_N;
__device__ uint32_t g_seg_tab[SEG_TAB_WORDS];

__global__ void __launch_bounds__(SEG_THREADS) tbseg_init_kernel() {
    __shared__ uint32_t xp2[2][XP_LOG];
    const int tid = threadIdx.x;
    uint32_t *tab = g_seg_tab, *gxp2 = g_seg_tab + 2 * 256, *xpb = gxp2 + 2 * XP_LOG;
    for (int e = tid; e < 2 * 256; e += SEG_THREADS) {
        const uint32_t poly = (e >> 8) ? POLY_B : POLY_A;
        uint32_t reg = (uint32_t)(e & 255) << 16;
        for (int k = 0; k < 8; k++) reg = crc_step_bit(reg, poly);
        tab[e] = reg;
    }
    if (tid < 2) {
        const uint32_t poly = tid ? POLY_B : POLY_A;
        uint32_t r = 1;
        for (int k = 0; k < 32; k++) r = crc_step_bit(r, poly);     /* x^32 */
        for (int k = 0; k < XP_LOG; k++) {
            xp2[tid][k] = r;
            gxp2[tid * XP_LOG + k] = r;
            r = mulmod24(r, r, poly);
        }
    }
    __syncthreads();
    for (int m = tid; m < XPB_N; m += SEG_THREADS) xpb[m] = xpow32(xp2[1], (uint32_t)m, POLY_B);
}

__global__ void __launch_bounds__(SEG_THREADS)
tbseg_kernel(const crn_tbseg *__restrict__ tbs, int n_tb, const uint8_t *__restrict__ payload,
             uint8_t *__restrict__ cb_bits) {
    extern __shared__ __align__(16) uint8_t seg_raw[];
    SegSmem &S = *reinterpret_cast<SegSmem *>(seg_raw);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    /* the CRC tables: built once per device by tbseg_init_kernel, copied per CTA */
    static_assert(offsetof(SegSmem, red) == 4 * SEG_TAB_WORDS, "tab, xp2, xpb lead SegSmem");
    for (int e = tid; e < SEG_TAB_WORDS; e += SEG_THREADS) reinterpret_cast<uint32_t *>(seg_raw)[e] = g_seg_tab[e];
    __syncthreads();

    for (int t = blockIdx.x; t < n_tb; t += gridDim.x) {
        const crn_tbseg T = tbs[t];
        const int64_t B = T.tbs;
        const int pad = (int)((32 - (B & 31)) & 31);             /* payload bit i at padded position pad + i */
        const int nwa = (int)((B + pad) >> 5);                    /* words of the padded payload */
        const uint8_t *src = payload + T.payload_off;
        /* ---- pack: word k holds padded positions 32k..32k+31, MSB first.  A thread
         * packs eight positions into one byte of S.w: two aligned 8-byte loads funnelled
         * to the payload's byte alignment, the eight 0/1 bytes gathered into eight bits
         * by one multiply (byte j -> bit 63 - j: no two products share a bit); the groups
         * at the payload's two ends (positions before it, the last 15 bytes) bit by bit */
        {
            uint8_t *wb = reinterpret_cast<uint8_t *>(S.w);
            const int ng = nwa * 4;
            for (int q = tid; q < ng; q += SEG_THREADS) {
                const int64_t i0 = 8 * (int64_t)q - pad;
                uint32_t b8 = 0;
                if (i0 >= 0 && i0 + 16 <= B) {
                    const uintptr_t a = reinterpret_cast<uintptr_t>(src + i0);
                    const unsigned long long *al = reinterpret_cast<const unsigned long long *>(a & ~(uintptr_t)7);
                    const int sh = (int)(a & 7) * 8;
                    const unsigned long long lo = __ldg(al), hi = __ldg(al + 1);
                    const unsigned long long x = sh ? (lo >> sh) | (hi << (64 - sh)) : lo;
                    b8 = (uint32_t)(((x & 0x0101010101010101ull) * 0x8040201008040201ull) >> 56);
                } else {
                    for (int j = 0; j < 8; j++) {
                        const int64_t i = i0 + j;
                        if (i >= 0 && i < B && (__ldg(src + i) & 1u)) b8 |= 0x80u >> j;
                    }
                }
                wb[q ^ 3] = (uint8_t)b8;                          /* word q/4, its bytes most significant first */
            }
        }
        __syncthreads();
        /* ---- CRC24A over the padded payload */
        {
            const int per = (nwa + SEG_THREADS - 1) / SEG_THREADS;
            const int w0 = min(nwa, tid * per), w1 = min(nwa, w0 + per);
            uint32_t reg = 0;
            for (int k = w0; k < w1; k++) reg = crc_bytes(reg, S.w[k], S.tab[0]);
            if (w1 > w0 && w1 < nwa) reg = mulmod24(reg, xpow32(S.xp2[0], (uint32_t)(nwa - w1), POLY_A), POLY_A);
            for (int o = 16; o; o >>= 1) reg ^= __shfl_xor_sync(0xFFFFFFFFu, reg, o);
            if (lane == 0) S.red[warp] = reg;
        }
        __syncthreads();
        if (tid == 0) {
            uint32_t c = 0;
            for (int k = 0; k < SEG_THREADS / 32; k++) c ^= S.red[k];
            S.crc_a = c;
            S.w[nwa] = c << 8;                                    /* b's last 24 bits, MSB first */
            S.w[nwa + 1] = 0;
        }
        __syncthreads();
        /* ---- CB contents: fillers, then b; the CRC24B positions (C > 1) after */
        const int C = T.C, Km = T.Kminus, Kp = T.Kplus, Cm = T.Cminus, F = T.F, L = T.L;
        const int64_t total = (int64_t)Cm * Km + (int64_t)(C - Cm) * Kp;
        uint8_t *dst = cb_bits + T.cb_bit0;
        if ((reinterpret_cast<uintptr_t>(dst) & 7) == 0) {
            /* K, L and every CB offset are multiples of 8: a thread writes eight bytes
             * of one CB from eight bits of b (no per-byte division).  Positions before
             * the payload (CB 0's fillers) read the zero front padding or fall before
             * word 0 */
            int64_t cb0 = 0;
            for (int r = 0; r < C; r++) {
                const int Kr = r < Cm ? Km : Kp, Fr = r == 0 ? F : 0;
                const int64_t srcr = (r <= Cm ? (int64_t)r * (Km - L) : (int64_t)Cm * (Km - L) + (int64_t)(r - Cm) * (Kp - L))
                                     - (r > 0 ? F : 0);
                unsigned long long *d8 = reinterpret_cast<unsigned long long *>(dst + cb0);
                for (int k8 = 8 * tid; k8 < Kr - L; k8 += 8 * SEG_THREADS) {
                    const int64_t P = pad + srcr + (k8 - Fr);
                    uint32_t b8;                                  /* positions P..P+7, first one in bit 7 */
                    if (P >= 0) {
                        const uint32_t hi = S.w[P >> 5], lo = S.w[(P >> 5) + 1];
                        b8 = __funnelshift_l(lo, hi, (int)(P & 31)) >> 24;
                    } else
                        b8 = P > -8 ? (S.w[0] >> 24) >> (int)(-P) : 0u;
                    const unsigned long long x = (unsigned long long)(__brev(b8) >> 24);      /* byte j's bit in bit j */
                    const unsigned long long v = (x * 0x0101010101010101ull) & 0x8040201008040201ull;
                    d8[k8 >> 3] = ((v + 0x7F7F7F7F7F7F7F7Full) >> 7) & 0x0101010101010101ull;
                }
                cb0 += Kr;
            }
        } else
        for (int64_t p = tid; p < total; p += SEG_THREADS) {
            int r, k;
            if (p < (int64_t)Cm * Km) { r = (int)(p / Km); k = (int)(p - (int64_t)r * Km); }
            else { const int64_t q = p - (int64_t)Cm * Km; r = Cm + (int)(q / Kp); k = (int)(q - (int64_t)(r - Cm) * Kp); }
            const int Kr = r < Cm ? Km : Kp, Fr = r == 0 ? F : 0;
            if (k >= Kr - L) continue;                            /* the CB's CRC24B: below */
            uint8_t v = 0;
            if (k >= Fr) {
                /* src_r = sum over s < r of (K_s - L - F_s) */
                const int64_t srcr = (r <= Cm ? (int64_t)r * (Km - L) : (int64_t)Cm * (Km - L) + (int64_t)(r - Cm) * (Kp - L))
                                     - (r > 0 ? F : 0);
                const int64_t P = pad + srcr + (k - Fr);
                v = (uint8_t)((S.w[P >> 5] >> (31 - (P & 31))) & 1u);
            }
            dst[p] = v;
        }
        if (C > 1) {
            for (int r = warp; r < C; r += SEG_THREADS / 32) {
                const int Kr = r < Cm ? Km : Kp, Fr = r == 0 ? F : 0, n = Kr - 24 - Fr;
                const int64_t srcr = (r <= Cm ? (int64_t)r * (Km - L) : (int64_t)Cm * (Km - L) + (int64_t)(r - Cm) * (Kp - L))
                                     - (r > 0 ? F : 0);
                const int ns = (n + 31) >> 5;
                uint32_t reg = 0;
                for (int s = lane; s < ns; s += 32) {
                    const int ps = n - 32 * (ns - s);                 /* first data position of the segment */
                    const int64_t P = pad + srcr + ps;
                    uint32_t seg;
                    if (P < 0) seg = S.w[0] >> (int)(-P);
                    else {
                        const int sh = (int)(P & 31);
                        const uint32_t hi = S.w[P >> 5], lo = S.w[(P >> 5) + 1];
                        seg = sh ? (hi << sh) | (lo >> (32 - sh)) : hi;
                    }
                    if (ps < 0) seg &= 0xFFFFFFFFu >> (-ps);          /* positions before the CB's data: 0 */
                    uint32_t c = crc_bytes(0, seg, S.tab[1]);
                    const int m = ns - 1 - s;
                    if (m) c = mulmod24(c, S.xpb[m], POLY_B);
                    reg ^= c;
                }
                for (int o = 16; o; o >>= 1) reg ^= __shfl_xor_sync(0xFFFFFFFFu, reg, o);
                const int64_t off = (r <= Cm ? (int64_t)r * Km : (int64_t)Cm * Km + (int64_t)(r - Cm) * Kp) + Kr - 24;
                if (lane < 24) dst[off + lane] = (uint8_t)((reg >> (23 - lane)) & 1u);
            }
        }
        __syncthreads();                                          /* S.w reused by the next TB */
    }
}

}  // namespace

size_t crn_tbseg_smem_bytes(int64_t max_words) {
    return sizeof(SegSmem) + 4 * (size_t)(max_words + 2);
}

extern "C" int crn_launch_tbseg(const crn_tbseg *d_tbs, int32_t n_tb, int64_t max_tbs, const uint8_t *payload,
                                uint8_t *cb_bits, void *stream) {
    static std::mutex mu;
    static size_t attr_bytes = 0;
    int dev, sms = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return CRN_ECUDA;
    const int64_t max_words = (max_tbs + 31) / 32 + 1;
    const size_t smem = crn_tbseg_smem_bytes(max_words);
    if (smem > 227 * 1024) return CRN_EINVAL;
    {
        std::lock_guard<std::mutex> lk(mu);
        if (smem > attr_bytes) {
            if (cudaFuncSetAttribute(tbseg_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024) !=
                cudaSuccess)
                return CRN_ECUDA;
            attr_bytes = 227 * 1024;
        }
    }
    {   /* first use on this device: build the tables and wait for them, so a later
         * call on any other stream finds them complete */
        static bool tab_ready[64] = {};
        std::lock_guard<std::mutex> lk(mu);
        if (dev < 0 || dev >= 64) return CRN_EINVAL;
        if (!tab_ready[dev]) {
            tbseg_init_kernel<<<1, SEG_THREADS, 0, (cudaStream_t)stream>>>();
            if (cudaGetLastError() != cudaSuccess || cudaStreamSynchronize((cudaStream_t)stream) != cudaSuccess)
                return CRN_ECUDA;
            tab_ready[dev] = true;
        }
    }
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int per_sm = (int)((228 * 1024) / (smem + 1024));
    const int cap = sms * (per_sm > 0 ? per_sm : 1);
    const int grid = n_tb < cap ? n_tb : cap;
    tbseg_kernel<<<grid, SEG_THREADS, smem, (cudaStream_t)stream>>>(d_tbs, n_tb, payload, cb_bits);
    return cudaGetLastError() == cudaSuccess ? CRN_OK : CRN_ECUDA;
}
