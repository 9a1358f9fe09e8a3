/* crn_encode.cu -- rate-1/3 LTE turbo encoder on the device (the paper's
 * downlink "encoding function"; NEXT row f3 of DESIGN.md).
 * A warp per code block, bit-packed in shared memory: optional CRC24A/B attach
 * over the first K-24 bits (fillers counted as 0), RSC 1 over c, RSC 2 over
 * c'_i = c_{Pi(i)}, 12 tail bits column-wise (R11), one bit per output byte.
 * Also builds bench.py's synthetic uplink inputs.
 *
 * Work per CB is a few instructions per bit:
 *   input    K bytes (one bit each) -> packed words: 8-byte loads, 8 bits per
 *            load by a multiply (or a ballot per 32 bytes when unaligned);
 *   CRC      byte-table CRC over word-aligned lane chunks, the 32 lane
 *            registers combined as crc(A||B) = crc(A) x^|B| + crc(B) with
 *            x^(32 m) mod g from a per-CTA table;
 *   c'       c_{Pi(i)} gathered bit by bit with the QPP forward recurrence
 *            Pi(i+1) = Pi(i) + g(i), g(i+1) = g(i) + 2 f2 (mod K), two
 *            add-and-fold steps per bit;
 *   RSC      the code is linear over GF(2): with state s = 4 r1 + 2 r2 + r3 one
 *            step is s' = A s + 4u, A of order 7 (1 + D^2 + D^3 is primitive).
 *            Each lane runs its chunk a byte at a time through a (state, input
 *            byte) -> (next state, 8 parity bits) table, first from state 0 to
 *            learn the chunk's input-driven end state f, then -- after a 32-step
 *            scan s_{l+1} = A^{L_l} s_l + f_l gives every chunk's true start
 *            state -- again, emitting parity;
 *   output   4 bits -> 4 bytes by a multiply, 32-bit coalesced stores.
 * A persistent grid; each CTA builds its tables once. */
#include <cuda_runtime.h>
#include <stdint.h>

#include <mutex>

#include "crn_internal.h"
#include "qpp_table.h"

namespace {
__constant__ int16_t c_f1[CRN_NUM_K], c_f2[CRN_NUM_K];

constexpr int ENC_WARPS = 8;
constexpr int ENC_THREADS = 32 * ENC_WARPS;
constexpr int ENC_WORDS = 6144 / 32;                 /* packed words of the largest CB */
constexpr uint32_t POLY_A = 0x864CFBu, POLY_B = 0x800063u;

/* index of K in the ascending size table (closed form of SPEC.md:217's set) */
__device__ __forceinline__ int crn_k_index_dev(int K) {
    if (K <= 512) return (K - 40) / 8;
    if (K <= 1024) return 60 + (K - 528) / 16;
    if (K <= 2048) return 92 + (K - 1056) / 32;
    return 124 + (K - 2112) / 64;
}

__device__ __forceinline__ int rsc_A(int s) {       /* zero-input step */
    const int r1 = (s >> 2) & 1, r2 = (s >> 1) & 1, r3 = s & 1;
    return ((r2 ^ r3) << 2) | (r1 << 1) | r2;
}

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

struct EncShared {
    uint16_t rsc[8 * 256];                /* (state, input byte) -> parity byte | next state << 8 */
    uint32_t crc_tab[2][256];             /* byte-at-a-time CRC24A / CRC24B (MSB-first) */
    uint32_t xp[2][ENC_WORDS + 1];        /* x^(32 m) mod g_A / g_B */
    uint8_t apow[8 * 8];                  /* A^e s, index 8 e + s, e in [0, 7) */
    struct Warp {
        uint32_t c[ENC_WORDS + 2];        /* c, packed LSB-first */
        uint32_t ci[ENC_WORDS];           /* c' = c_{Pi(i)} */
        uint32_t z1[ENC_WORDS + 2], z2[ENC_WORDS + 2];   /* (+ the tail word of the packed write-out) */
    } w[ENC_WARPS];
};

__device__ void build_tables(EncShared &S) {
    for (int e = threadIdx.x; e < 8 * 256; e += ENC_THREADS) {
        int s = e >> 8;
        const int b = e & 255;
        uint32_t z = 0;
        for (int k = 0; k < 8; k++) {
            const int u = (b >> k) & 1, r1 = (s >> 2) & 1, r2 = (s >> 1) & 1, r3 = s & 1;
            const int a = u ^ r2 ^ r3;
            z |= (uint32_t)(a ^ r1 ^ r3) << k;
            s = (a << 2) | (r1 << 1) | r2;
        }
        S.rsc[e] = (uint16_t)(z | (uint32_t)s << 8);
    }
    if (threadIdx.x < 56) {
        int s = threadIdx.x & 7;
        for (int k = threadIdx.x >> 3; k > 0; k--) s = rsc_A(s);
        S.apow[threadIdx.x] = (uint8_t)s;
    }
    for (int e = threadIdx.x; e < 2 * 256; e += ENC_THREADS) {
        const uint32_t poly = (e >> 8) ? POLY_B : POLY_A;
        uint32_t reg = (uint32_t)(e & 255) << 16;
        for (int k = 0; k < 8; k++) reg = crc_step_bit(reg, poly);
        S.crc_tab[e >> 8][e & 255] = reg;
    }
    for (int e = threadIdx.x; e < 2 * (ENC_WORDS + 1); e += ENC_THREADS) {
        const int p = e / (ENC_WORDS + 1), m = e % (ENC_WORDS + 1);
        const uint32_t poly = p ? POLY_B : POLY_A;
        uint32_t r = 1, base = 1;                                  /* x^0; base -> x^32 mod g */
        for (int k = 0; k < 32; k++) base = crc_step_bit(base, poly);
        for (int q = m; q > 0; q >>= 1) {                          /* square-and-multiply */
            if (q & 1) r = mulmod24(r, base, poly);
            base = mulmod24(base, base, poly);
        }
        S.xp[p][m] = r;
    }
    __syncthreads();
}

/* K bits (one per byte at src) -> packed words c[0 .. ceil(K/32)), zero beyond K */
__device__ __forceinline__ void load_bits(const uint8_t *src, int K, uint32_t *c, int lane) {
    const int nw = (K + 31) >> 5;
    if ((reinterpret_cast<uintptr_t>(src) & 7u) == 0) {             /* K = 0 mod 8: K/8 whole 8-byte units */
        const uint2 *s8 = reinterpret_cast<const uint2 *>(src);
        uint8_t *cb = reinterpret_cast<uint8_t *>(c);
        const int nu = K >> 3;
        constexpr int U = 8;
        for (int u0 = lane; u0 < nu; u0 += 32 * U) {
            uint2 v[U];
#pragma unroll
            for (int j = 0; j < U; j++)
                if (u0 + 32 * j < nu) v[j] = __ldg(s8 + u0 + 32 * j);
#pragma unroll
            for (int j = 0; j < U; j++)
                if (u0 + 32 * j < nu) {
                    const uint32_t lo = ((v[j].x & 0x01010101u) * 0x01020408u) >> 24;
                    const uint32_t hi = ((v[j].y & 0x01010101u) * 0x01020408u) >> 24;
                    cb[u0 + 32 * j] = (uint8_t)(lo | hi << 4);
                }
        }
        /* (the last word's bytes past K are masked by the caller) */
    } else {
        for (int t = 0; t < nw; t++) {
            const int n = 32 * t + lane;
            const uint32_t w = __ballot_sync(0xFFFFFFFFu, n < K && (__ldg(src + n) & 1u));
            if (lane == 0) c[t] = w;
        }
    }
    __syncwarp();
}

/* K bits at bit offset off of a packed LSB-first array -> c[0 .. ceil(K/32)) (bits past K
 * in the last word are the source's; the caller masks them) */
__device__ __forceinline__ void load_bits_packed(const uint32_t *src, int64_t off, int K, uint32_t *c, int lane) {
    const int nw = (K + 31) >> 5, sh = (int)(off & 31);
    const uint32_t *s = src + (off >> 5);
    for (int t = lane; t < nw; t += 32) {
        const uint32_t a = __ldg(s + t);
        const uint32_t b = (sh && 32 * t + 32 - sh < K) ? __ldg(s + t + 1) : 0u;   /* the next word only if needed */
        c[t] = __funnelshift_r(a, b, sh);
    }
    __syncwarp();
}

/* src bits [0, nbits) -> dst bits [off, off + nbits) (packed LSB-first); words the
 * range covers only in part are merged with two atomics (neighbouring CBs share
 * them), whole words are plain stores.  src must hold ceil(nbits / 32) + 1 words. */
__device__ __forceinline__ void store_bits_packed(uint32_t *dst, int64_t off, const uint32_t *src, int nbits,
                                                  int lane) {
    const int sh = (int)(off & 31), end = (int)((off + nbits) & 31);
    const int nwd = (sh + nbits + 31) >> 5;                            /* destination words touched */
    uint32_t *d = dst + (off >> 5);
    for (int i = lane; i < nwd; i += 32) {
        const uint32_t v = sh ? __funnelshift_l(i ? src[i - 1] : 0u, src[i], sh) : src[i];  /* dest bit b <- src bit 32 i - sh + b */
        if (i > 0 && i < nwd - 1) {
            d[i] = v;                                                  /* interior: a whole word */
        } else {
            uint32_t mask = ~0u;
            if (i == 0) mask &= ~0u << sh;
            if (i == nwd - 1 && end) mask &= ~0u >> (32 - end);
            if (mask == ~0u) {
                d[i] = v;
            } else {
                atomicAnd(d + i, ~mask);
                atomicOr(d + i, v & mask);
            }
        }
    }
}

/* PACKED = false: one bit per byte in and out (info at ext_off, streams at llr_off);
 * PACKED = true: packed LSB-first bits (info at bit offset ext_off, each stream's
 * K + 4 bits at bit offset llr_off). */
template <bool PACKED>
__global__ void __launch_bounds__(ENC_THREADS)
encode_kernel(const crn_cb_desc *__restrict__ desc, int n_cb, const void *__restrict__ info_v, int attach,
              void *d0_v, void *d1_v, void *d2_v) {
    const uint8_t *info = static_cast<const uint8_t *>(info_v);
    uint8_t *d0 = static_cast<uint8_t *>(d0_v), *d1 = static_cast<uint8_t *>(d1_v), *d2 = static_cast<uint8_t *>(d2_v);
    extern __shared__ __align__(16) uint8_t enc_raw[];
    EncShared &S = *reinterpret_cast<EncShared *>(enc_raw);
    build_tables(S);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    EncShared::Warp &W = S.w[warp];
    for (int cb = blockIdx.x * ENC_WARPS + warp; cb < n_cb; cb += gridDim.x * ENC_WARPS) {
        const crn_cb_desc d = desc[cb];
        const int K = d.K, F = d.F, nw = (K + 31) >> 5;
        if (PACKED) load_bits_packed(static_cast<const uint32_t *>(info_v), d.ext_off, K, W.c, lane);
        else load_bits(info + d.ext_off, K, W.c, lane);
        /* fillers read as 0; with attach the last 24 bits are recomputed */
        const int N = attach ? K - 24 : K;
        for (int t = lane; t < nw; t += 32) {
            uint32_t w = W.c[t];
            const int b0 = 32 * t;
            if (b0 < F) w &= F - b0 >= 32 ? 0u : ~0u << (F - b0);
            if (b0 + 32 > N) w &= N - b0 <= 0 ? 0u : ~0u >> (32 - (N - b0));
            W.c[t] = w;
        }
        if (lane == 0) W.c[nw] = 0;
        __syncwarp();
        const int per = (nw + 31) >> 5;                            /* words per lane chunk */
        const int w0 = min(nw, lane * per), w1 = min(nw, w0 + per);
        if (attach) {
            /* CRC register of bits [32 w0, min(32 w1, N)) from zero, a byte at a time */
            const int p = d.crc_kind == CRN_CRC24A ? 0 : 1;
            const uint32_t poly = p ? POLY_B : POLY_A;
            const uint32_t *tab = S.crc_tab[p];
            const int e1 = min(32 * w1, N);
            uint32_t reg = 0;
            for (int t = w0; 32 * t < e1; t++) {
                const uint32_t rw = __brev(W.c[t]);                 /* first bit -> MSB */
                const int nb = min(4, (e1 - 32 * t) >> 3);          /* N = 0 mod 8 */
                for (int k = 0; k < nb; k++) {
                    const uint32_t byte = (rw >> (24 - 8 * k)) & 0xFFu;
                    reg = ((reg << 8) & 0xFFFFFFu) ^ tab[((reg >> 16) ^ byte) & 0xFFu];
                }
            }
            /* times x^(N - e1): x^(32 m) from the table, then 0..3 zero bytes */
            uint32_t part = 0;
            if (32 * w0 < e1) {
                const int ex = N - e1, m = ex >> 5;
                part = m ? mulmod24(reg, S.xp[p][m], poly) : reg;
                for (int k = 0; k < ((ex & 31) >> 3); k++) part = ((part << 8) & 0xFFFFFFu) ^ tab[(part >> 16) & 0xFFu];
            }
            for (int o = 16; o > 0; o >>= 1) part ^= __shfl_xor_sync(0xFFFFFFFFu, part, o);
            if (lane == 0) {                                        /* bits N .. N+23, MSB of the CRC first */
                const uint32_t bits = __brev(part << 8);            /* crc bit 23-i at position i */
                const int t = N >> 5, sh = N & 31;
                W.c[t] |= bits << sh;
                if (sh) W.c[t + 1] |= bits >> (32 - sh);
            }
            __syncwarp();
        }
        /* c'_i = c_{Pi(i)} for the lane's words.  With K = 0 mod 64 the two halves
         * go together: Pi(i + K/2) = Pi(i) + K/2 mod K (f1 odd, f2 even), so one
         * recurrence step serves bit i and bit i + K/2 */
        {
            const int ki = crn_k_index_dev(K);
            const int f1 = c_f1[ki], f2 = c_f2[ki];
            const uint32_t f2x2 = (uint32_t)((2 * f2) % K);
            const bool halves = (K & 63) == 0;
            const int nwh = halves ? nw >> 1 : nw;               /* words the recurrence walks */
            const int perh = (nwh + 31) >> 5;
            const int h0 = min(nwh, lane * perh), h1 = min(nwh, h0 + perh);
            const int i0 = 32 * h0;
            uint32_t pi = (uint32_t)((f1 * i0 + f2 * ((i0 * i0) % K)) % K);
            uint32_t g = (uint32_t)((f1 + f2 * ((2 * i0 + 1) % K)) % K);
            if (halves) {
                const uint32_t Kh = (uint32_t)(K >> 1);
                for (int t = h0; t < h1; t++) {
                    uint32_t acc = 0, acc2 = 0;
#pragma unroll
                    for (int k = 0; k < 32; k++) {
                        const uint32_t pj = min(pi + Kh, pi - Kh);        /* Pi(i + K/2) */
                        const uint32_t v = W.c[pi >> 5], v2 = W.c[pj >> 5];
                        acc = __funnelshift_r(acc, __funnelshift_r(v, v, pi), 1);
                        acc2 = __funnelshift_r(acc2, __funnelshift_r(v2, v2, pj), 1);
                        pi = min(pi + g, pi + g - (uint32_t)K);
                        g = min(g + f2x2, g + f2x2 - (uint32_t)K);
                    }
                    W.ci[t] = acc;
                    W.ci[t + nwh] = acc2;
                }
            } else {
                for (int t = h0; t < h1; t++) {
                    uint32_t acc = 0;
                    const int nbit = min(32, K - 32 * t);                /* 32, or 8/16/24 in the last word */
                    auto step = [&]() {
                        const uint32_t v = W.c[pi >> 5];
                        acc = __funnelshift_r(acc, __funnelshift_r(v, v, pi), 1);   /* bit pi -> acc MSB */
                        pi = min(pi + g, pi + g - (uint32_t)K);                     /* (pi + g) mod K */
                        g = min(g + f2x2, g + f2x2 - (uint32_t)K);
                    };
                    if (nbit == 32) {
#pragma unroll
                        for (int k = 0; k < 32; k++) step();
                    } else {
                        for (int k = 0; k < nbit; k++) step();
                        acc >>= 32 - nbit;
                    }
                    W.ci[t] = acc;
                }
            }
        }
        __syncwarp();
        /* both RSC encoders: pass 1 from state 0 (end state), scan, pass 2 with parity */
        const int L = max(0, min(32 * w1, K) - 32 * w0);              /* chunk bits, 0 mod 8 */
        const int nbytes = L >> 3;
        const uint8_t *cb1 = reinterpret_cast<const uint8_t *>(W.c) + 4 * w0;
        const uint8_t *cb2 = reinterpret_cast<const uint8_t *>(W.ci) + 4 * w0;
        int s1 = 0, s2 = 0;
        for (int k = 0; k < nbytes; k++) {
            s1 = S.rsc[(s1 << 8) | cb1[k]] >> 8;
            s2 = S.rsc[(s2 << 8) | cb2[k]] >> 8;
        }
        /* chunk l maps its start state s to A^{L_l} s + f_l: an affine map over GF(2)^3
         * whose linear part is a power of A (order 7), so maps compose as
         * (e2, b2) o (e1, b1) = (e1 + e2 mod 7, A^{e2} b1 + b2).  Inclusive scan over
         * the lanes; lane l starts from lane l-1's b (the map of chunks < l applied
         * to state 0), the CB ends in lane 31's. */
        int e = L % 7, b1 = s1, b2 = s2;
        for (int o = 1; o < 32; o <<= 1) {
            const int pe = __shfl_up_sync(0xFFFFFFFFu, e, o), pb1 = __shfl_up_sync(0xFFFFFFFFu, b1, o),
                      pb2 = __shfl_up_sync(0xFFFFFFFFu, b2, o);
            if (lane >= o) {
                b1 ^= S.apow[8 * e + pb1];
                b2 ^= S.apow[8 * e + pb2];
                e = e + pe >= 7 ? e + pe - 7 : e + pe;
            }
        }
        const int u1 = __shfl_up_sync(0xFFFFFFFFu, b1, 1), u2 = __shfl_up_sync(0xFFFFFFFFu, b2, 1);
        const int st1 = lane ? u1 : 0, st2 = lane ? u2 : 0;
        const int run1 = __shfl_sync(0xFFFFFFFFu, b1, 31), run2 = __shfl_sync(0xFFFFFFFFu, b2, 31);
        s1 = st1;
        s2 = st2;
        uint8_t *z1b = reinterpret_cast<uint8_t *>(W.z1) + 4 * w0, *z2b = reinterpret_cast<uint8_t *>(W.z2) + 4 * w0;
        for (int k = 0; k < nbytes; k++) {
            const uint32_t v1 = S.rsc[(s1 << 8) | cb1[k]], v2 = S.rsc[(s2 << 8) | cb2[k]];
            z1b[k] = (uint8_t)v1;
            z2b[k] = (uint8_t)v2;
            s1 = v1 >> 8;
            s2 = v2 >> 8;
        }
        __syncwarp();
        if (PACKED) {
            /* the 4 termination bits of each stream (R11) go to bits K .. K+3 of its
             * words (K = 0 mod 8: one word), then each stream's K + 4 bits are stored */
            if (lane == 0) {
                uint32_t tb[3] = {0u, 0u, 0u};
                int s = run1;
                for (int k = 0; k < 3; k++) {
                    const int r1 = (s >> 2) & 1, r2 = (s >> 1) & 1, r3 = s & 1;
                    const int m0 = 2 * k, m1 = 2 * k + 1;                /* t[m] -> stream m % 3, bit K + m / 3 */
                    tb[m0 % 3] |= (uint32_t)(r2 ^ r3) << (m0 / 3);
                    tb[m1 % 3] |= (uint32_t)(r1 ^ r3) << (m1 / 3);
                    s = (r1 << 1) | r2;
                }
                s = run2;
                for (int k = 0; k < 3; k++) {
                    const int r1 = (s >> 2) & 1, r2 = (s >> 1) & 1, r3 = s & 1;
                    const int m0 = 6 + 2 * k, m1 = 6 + 2 * k + 1;
                    tb[m0 % 3] |= (uint32_t)(r2 ^ r3) << (m0 / 3);
                    tb[m1 % 3] |= (uint32_t)(r1 ^ r3) << (m1 / 3);
                    s = (r1 << 1) | r2;
                }
                const int t = K >> 5, sh = K & 31;
                const uint32_t keep = sh ? (1u << sh) - 1u : 0u;       /* bits below K in the word */
                W.c[t] = (W.c[t] & keep) | (tb[0] << sh);
                W.z1[t] = (W.z1[t] & keep) | (tb[1] << sh);
                W.z2[t] = (W.z2[t] & keep) | (tb[2] << sh);
            }
            __syncwarp();
            store_bits_packed(static_cast<uint32_t *>(d0_v), d.llr_off, W.c, K + 4, lane);
            store_bits_packed(static_cast<uint32_t *>(d1_v), d.llr_off, W.z1, K + 4, lane);
            store_bits_packed(static_cast<uint32_t *>(d2_v), d.llr_off, W.z2, K + 4, lane);
            __syncwarp();                                 /* W is rewritten by the next CB */
            continue;
        }
        /* write-out: bit n -> byte n of each stream, four bytes per store */
        uint8_t *o0 = d0 + d.llr_off, *o1 = d1 + d.llr_off, *o2 = d2 + d.llr_off;
        const bool al = ((reinterpret_cast<uintptr_t>(o0) | reinterpret_cast<uintptr_t>(o1) |
                          reinterpret_cast<uintptr_t>(o2)) & 3u) == 0;
        if (al) {
            /* packed byte q = bits 8q .. 8q+7 -> output bytes 8q .. 8q+7 (two words, or one
             * 8-byte store when the streams are 8-byte aligned) */
            const uint8_t *n0 = reinterpret_cast<const uint8_t *>(W.c), *n1 = reinterpret_cast<const uint8_t *>(W.z1),
                          *n2 = reinterpret_cast<const uint8_t *>(W.z2);
            const bool al8 = ((reinterpret_cast<uintptr_t>(o0) | reinterpret_cast<uintptr_t>(o1) |
                               reinterpret_cast<uintptr_t>(o2)) & 7u) == 0;
            auto expand = [](uint32_t b) {
                return make_uint2(((b & 0xFu) * 0x00204081u) & 0x01010101u, ((b >> 4) * 0x00204081u) & 0x01010101u);
            };
            for (int q = lane; q < (K >> 3); q += 32) {
                const uint2 a = expand(n0[q]), b = expand(n1[q]), c = expand(n2[q]);
                if (al8) {
                    reinterpret_cast<uint2 *>(o0)[q] = a;
                    reinterpret_cast<uint2 *>(o1)[q] = b;
                    reinterpret_cast<uint2 *>(o2)[q] = c;
                } else {
                    uint32_t *p0 = reinterpret_cast<uint32_t *>(o0) + 2 * q, *p1 = reinterpret_cast<uint32_t *>(o1) + 2 * q,
                             *p2 = reinterpret_cast<uint32_t *>(o2) + 2 * q;
                    p0[0] = a.x; p0[1] = a.y;
                    p1[0] = b.x; p1[1] = b.y;
                    p2[0] = c.x; p2[1] = c.y;
                }
            }
        } else {
            for (int n = lane; n < K; n += 32) {
                o0[n] = (uint8_t)((W.c[n >> 5] >> (n & 31)) & 1u);
                o1[n] = (uint8_t)((W.z1[n >> 5] >> (n & 31)) & 1u);
                o2[n] = (uint8_t)((W.z2[n >> 5] >> (n & 31)) & 1u);
            }
        }
        if (lane == 0) {                                  /* termination: u = r2^r3, x = u, z = r1^r3 (R11) */
            uint8_t t[12];
            int s = run1;
            for (int k = 0; k < 3; k++) {
                const int r1 = (s >> 2) & 1, r2 = (s >> 1) & 1, r3 = s & 1;
                t[2 * k] = (uint8_t)(r2 ^ r3);
                t[2 * k + 1] = (uint8_t)(r1 ^ r3);
                s = (r1 << 1) | r2;
            }
            s = run2;
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
        __syncwarp();                                     /* W is rewritten by the next CB */
    }
}
}  // namespace

extern "C" int crn_launch_encode(const crn_cb_desc *d_desc, int32_t n_cb, const void *info, int32_t attach,
                                 void *d0, void *d1, void *d2, int32_t packed, const crn_tables *, void *stream) {
    static std::mutex mu;
    static uint64_t done = 0;                   /* bit d: the QPP constants are on device d */
    static int grid_max = 0;
    int dev;
    if (cudaGetDevice(&dev) != cudaSuccess) return CRN_ECUDA;
    {
        std::lock_guard<std::mutex> lk(mu);
        if (dev >= 64 || !((done >> dev) & 1u)) {
            if (cudaMemcpyToSymbol(c_f1, crn_qpp_f1, sizeof(crn_qpp_f1)) != cudaSuccess ||
                cudaMemcpyToSymbol(c_f2, crn_qpp_f2, sizeof(crn_qpp_f2)) != cudaSuccess)
                return CRN_ECUDA;
            if (cudaFuncSetAttribute(encode_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)sizeof(EncShared)) != cudaSuccess ||
                cudaFuncSetAttribute(encode_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)sizeof(EncShared)) != cudaSuccess)
                return CRN_ECUDA;
            int sms = 0, per_sm = 0;
            if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess ||
                cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, encode_kernel<false>, ENC_THREADS,
                                                              sizeof(EncShared)) != cudaSuccess)
                return CRN_ECUDA;
            grid_max = sms * (per_sm > 0 ? per_sm : 1);
            if (dev < 64) done |= 1ull << dev;
        }
    }
    const int need = (n_cb + ENC_WARPS - 1) / ENC_WARPS;
    const int grid = need < grid_max ? need : grid_max;
    if (packed)
        encode_kernel<true><<<grid, ENC_THREADS, sizeof(EncShared), (cudaStream_t)stream>>>(d_desc, n_cb, info, attach,
                                                                                           d0, d1, d2);
    else
        encode_kernel<false><<<grid, ENC_THREADS, sizeof(EncShared), (cudaStream_t)stream>>>(d_desc, n_cb, info, attach,
                                                                                            d0, d1, d2);
    return cudaGetLastError() == cudaSuccess ? CRN_OK : CRN_ECUDA;
}
