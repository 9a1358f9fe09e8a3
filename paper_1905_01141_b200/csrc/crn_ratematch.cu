/* crn_ratematch.cu -- TS 36.212 5.1.4.1 rate matching / de-matching for
 * turbo-coded channels on the device (R30):
 * the input side of the decoder -- the received data R(x_i) of PAPER.md:289
 * are the E rate-matched soft values of a CB.
 *
 * Geometry per CB: D = K + 4 bits per stream, R = ceil(D/32) rows, Kpi = 32 R,
 * ND = Kpi - D dummy bits, circular buffer w of Ncb = 3 Kpi positions (v0, then
 * v1/v2 interlaced), k0 = R (2 ceil(Ncb / 8R) rv + 2).  The dummy positions are
 * few (<= 97) and sit only at row 0 of a column (plus one wrapped position
 * of v2), so the rank of a position -- its index among non-dummy positions
 * counted circularly from k0 -- is closed-form from a 64-entry table
 * (build_ranks).  One CTA per CB; the CB's E values (or 3D bits) are staged in
 * shared memory in rank order, so both global sides are coalesced:
 *   de-matching: stage[r] = sum over m >= 0 of e[r + m 3D] (repetition; exact
 *     int32; 0 for punctured ranks r >= E), then every output (stream s, bit
 *     n) reads stage[rank(s, n)], saturated once (onto the previous HARQ
 *     buffer when combining), so the result does not depend on any order.
 *   matching: stage[rank(s, n)] = d_s[n], then e[k] = stage[k mod 3D].
 */
#include <cuda_runtime.h>

#include <atomic>
#include <stdint.h>

#include "crn_internal.h"

namespace {

constexpr int RM_THREADS = 512;

__device__ __forceinline__ int bitrev5(int c) { return (int)(__brev((unsigned)c) >> 27); }

struct Geo {
    int D, R, Kpi, ND, Ncb, k0, nn;   /* nn = non-dummy positions = 3D */
};

__device__ __forceinline__ Geo geo(int K, int rv) {
    Geo g;
    g.D = K + 4;
    g.R = (g.D + 31) / 32;
    g.Kpi = 32 * g.R;
    g.ND = g.Kpi - g.D;
    g.Ncb = 3 * g.Kpi;
    g.k0 = g.R * (2 * ((g.Ncb + 8 * g.R - 1) / (8 * g.R)) * rv + 2);
    g.nn = 3 * g.D;
    return g;
}

/* Dummy positions lie only at row 0 of a column (v0: w = cR if P(c) < ND; v1:
 * Kpi + 2cR under the same condition; v2: Kpi + 2cR + 1 if P(c) + 1 < ND) plus,
 * when ND > 0, the last position of w (v2's wrapped y = 0).  So for any
 * NON-dummy position p in column c the number of dummies below p is a function
 * of (region, c) alone -- every row-0 dummy of columns <= c in its region and of
 * the regions before it (a row-0 dummy of the same column lies below p, or p is
 * itself that dummy or precedes only dummies: a2 implies a0).  Warp 0 builds
 * the 64 counts nb[region][c] and base = k0 - (dummies below k0), so a CB
 * position's rank counted circularly from k0 is p - nb - base (mod 3D); it keeps
 * the rank of row 0 of each of the 96 columns and the row-0 dummy masks. */
struct RankTab {
    int r0[96];           /* rank of row 0 of column (s, c), index 32 s + c, in [0, 3D) */
    uint32_t dmask[3];    /* bit c of dmask[s]: row 0 of column (s, c) is a dummy */
};

__device__ void build_ranks(const Geo &g, RankTab *t) {
    if (threadIdx.x < 32) {
        const int c = threadIdx.x, P = bitrev5(c);
        const int a0 = P < g.ND, a2 = P + 1 < g.ND;
        int s0 = a0, s12 = a0 + a2;                                   /* inclusive scans over c */
        for (int o = 1; o < 32; o <<= 1) {
            const int u0 = __shfl_up_sync(0xFFFFFFFFu, s0, o), u12 = __shfl_up_sync(0xFFFFFFFFu, s12, o);
            if (c >= o) { s0 += u0; s12 += u12; }
        }
        const int N0 = __shfl_sync(0xFFFFFFFFu, s0, 31);
        /* dummies strictly below k0 (the wrapped last position never is) */
        const int below = (a0 && c * g.R < g.k0) + (a0 && g.Kpi + 2 * c * g.R < g.k0) +
                          (a2 && g.Kpi + 2 * c * g.R + 1 < g.k0);
        int tot = below;
        for (int o = 16; o > 0; o >>= 1) tot += __shfl_xor_sync(0xFFFFFFFFu, tot, o);
        const int base = g.k0 - tot;
        /* rank of a non-dummy p in column c: p - nb - base; row 0's (or, for a dummy
         * row 0, the next real position's) folded into [0, 3D): p - nb in [-1, 3D) */
        const int nb[3] = {s0, N0 + s12, N0 + s12};
        for (int s = 0; s < 3; s++) {
            const int p0 = (s ? g.Kpi + (s - 1) : 0) + (s ? 2 : 1) * c * g.R;
            int r = p0 - nb[s] - base;
            if (r < 0) r += g.nn;
            t->r0[32 * s + c] = r;
        }
        const uint32_t m0 = __ballot_sync(0xFFFFFFFFu, a0), m2 = __ballot_sync(0xFFFFFFFFu, a2);
        if (c == 0) { t->dmask[0] = m0; t->dmask[1] = m0; t->dmask[2] = m2; }
    }
    __syncthreads();
}


/* ---- staging.  The CB's input range is brought into shared memory by one
 * bulk copy (cp.async.bulk, completion on an mbarrier) of the 16-byte blocks
 * that hold it -- never a byte outside those blocks, so never a page the range
 * does not touch.  It is then re-laid out as T[s][c][row]: sub-block s's bit in
 * column c (after the inter-column permutation) and row, column stride Rp
 * chosen so that both walks over T are bank-conflict-free -- stream order n
 * (y = n + ND, or y - 1 for v2, lies in column c = P(y mod 32), row y / 32: a
 * warp's 32 consecutive y hit 32 distinct c, and c (Rp / elements-per-word) is
 * a bijection mod 32 when that quotient is odd) and circular-buffer order (a
 * column's rows are consecutive elements and consecutive ranks). */
constexpr int RM_MAXR = (6144 + 4 + 31) / 32;                         /* 193 rows at most */

/* (volatile: computed once and kept in a register, not re-derived per access) */
__device__ __forceinline__ uint32_t smem_addr(const void *p) {
    uint32_t a;
    asm volatile("{ .reg .u64 t; cvta.to.shared.u64 t, %1; cvt.u32.u64 %0, t; }" : "=r"(a) : "l"(p));
    return a;
}

__device__ __forceinline__ void bar_init(uint64_t *bar) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(bar)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void bar_expect(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes) : "memory");
}

__device__ __forceinline__ void bar_wait0(uint64_t *bar) {
    uint32_t done = 0;
    while (!done)
        asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0, 1, 0, p; }"
                     : "=r"(done) : "r"(smem_addr(bar)) : "memory");
}

/* shared-memory accesses by 32-bit shared address (keeps the compiler from
 * re-deriving a generic window address at every access) */
__device__ __forceinline__ uint32_t ld_s8(uint32_t a) {
    uint32_t v;
    asm volatile("ld.shared.u8 %0, [%1];" : "=r"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ int32_t ld_s16(uint32_t a) {
    int32_t v;
    asm volatile("ld.shared.s16 %0, [%1];" : "=r"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ void st_s8(uint32_t a, uint32_t v) {
    asm volatile("st.shared.u8 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
__device__ __forceinline__ void st_s8_if(uint32_t a, uint32_t v, bool p) {
    asm volatile("{ .reg .pred q; setp.ne.u32 q, %2, 0; @q st.shared.u8 [%0], %1; }" ::"r"(a), "r"(v),
                 "r"((uint32_t)p) : "memory");
}
__device__ __forceinline__ void st_s16_if(uint32_t a, int32_t v, bool p) {
    asm volatile("{ .reg .pred q; setp.ne.u32 q, %2, 0; @q st.shared.u16 [%0], %1; }" ::"r"(a), "r"(v),
                 "r"((uint32_t)p) : "memory");
}

struct Blocks {           /* the 16-byte blocks holding [src, src + len) */
    const uint8_t *a0;
    uint32_t bytes;
    int lead;
};

__device__ __forceinline__ Blocks blocks_of(const void *src, int64_t len) {
    const uintptr_t a = reinterpret_cast<uintptr_t>(src), a0 = a & ~(uintptr_t)15;
    const uintptr_t a1 = (a + (uintptr_t)len + 15) & ~(uintptr_t)15;
    return Blocks{reinterpret_cast<const uint8_t *>(a0), (uint32_t)(a1 - a0), (int)(a - a0)};
}

__device__ __forceinline__ void bulk_load(void *dst, const Blocks &b, uint64_t *bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(smem_addr(dst)), "l"(b.a0), "r"(b.bytes), "r"(smem_addr(bar)) : "memory");
}

/* smallest Rp >= R with Rp / q odd (q = elements per 32-bit word) */
__device__ __forceinline__ int pad_rows(int R, int q) {
    int Rp = (R + q - 1) / q * q;
    if (((Rp / q) & 1) == 0) Rp += q;
    return Rp;
}

__device__ __forceinline__ int t_index(const Geo &g, int Rp, int s, int n) {
    int y = n + g.ND;
    if (s == 2) y = y == 0 ? g.Kpi - 1 : y - 1;                    /* y = (P(col) + 32 row + 1) mod Kpi */
    return (s * 32 + bitrev5(y & 31)) * Rp + (y >> 5);
}

/* Calls f(T index, rank, in_range, real) for the circular-buffer positions, a
 * warp per column, lanes over rows: the rank grows by 1 (v0) or 2 (v1/v2) per
 * row, the T index by 1.  Rows run to 32 ceil(R / 32) so the loop is
 * warp-uniform: in_range = row < R, real = in_range and not a dummy (a dummy's
 * or an out-of-range row's "rank" is some rank in [0, 3D) of a real position). */
template <class F>
__device__ __forceinline__ void for_each_position(const Geo &g, const RankTab &t, int Rp, F &&f) {
    const int lane = threadIdx.x & 31;
    const int nrow32 = (g.R + 31) >> 5;
    for (int col = threadIdx.x >> 5; col < 96; col += RM_THREADS / 32) {
        const int s = col >> 5, c = col & 31;
        const int mul = s ? 2 : 1, inc = 32 * mul;
        int r = t.r0[col] + mul * lane;                              /* mul lane <= 62 < 3D */
        if (r >= g.nn) r -= g.nn;
        const int skip0 = ((t.dmask[s] >> c) & 1u) ? 0 : -1;                        /* dummy rows */
        const int skip1 = (col == 95 && g.ND > 0) ? g.R - 1 : -1;                   /* the wrapped dummy */
        int ix = col * Rp + lane;
#pragma unroll
        for (int i = 0; i < (RM_MAXR + 31) / 32; i++) {
            if (i < nrow32) {
                const int row = lane + 32 * i;
                const bool in_range = row < g.R;
                f(ix, r, in_range, in_range && row != skip0 && row != skip1);
            }
            ix += 32;
            r += inc;
            if (r >= g.nn) r -= g.nn;
        }
    }
}

constexpr int DM_RAW = (2 * 3 * (6144 + 4) + 32 + 15) / 16 * 16;      /* E <= 3D int16 + two partial blocks */
constexpr int DM_T16 = 96 * 194 * 2;                                  /* pad_rows(193, 2) = 194 */
constexpr int DM_SMEM = DM_RAW + DM_T16;                              /* 74,160 B: 3 CTAs per SM */
static_assert(96 * (RM_MAXR | 1) * 4 <= DM_SMEM, "int32 T (repetition) fits the same space");
constexpr int MT_RAW = (6144 + 4 + 32 + 15) / 16 * 16;                /* one stream + two partial blocks */
constexpr int MT_T8 = 96 * 196 + 256;                                /* pad_rows(193, 4) = 196, + over-read slack */
constexpr int MT_SMEM = 3 * MT_RAW + MT_T8;                           /* 37,648 B; Q (3D bytes) reuses the raw area */
static_assert(3 * MT_RAW >= 3 * (6144 + 4), "Q fits the raw area");

/* De-matching.  E <= 3D (no repetition): e is bulk-copied, re-laid out into
 * int16 T in circular-buffer order (rank r's value e[r], 0 if punctured, r >=
 * E), then the three streams are written in stream order, saturated once (onto
 * the previous HARQ buffer when combining).  E > 3D: T holds the exact int32
 * sums of e[r + m 3D] over m, read from global memory.  Order-independent. */
__global__ void __launch_bounds__(RM_THREADS)
dematch_kernel(const crn_rm_desc *__restrict__ desc, const int16_t *__restrict__ e, int combine,
               int16_t *__restrict__ h0, int16_t *__restrict__ h1, int16_t *__restrict__ h2) {
    extern __shared__ __align__(16) uint8_t dm_sm[];
    __shared__ RankTab tab;
    __shared__ __align__(8) uint64_t bar;
    const crn_rm_desc d = desc[blockIdx.x];
    const Geo g = geo(d.K, d.rv);
    const int16_t *ec = e + d.e_off;
    const int E = d.E, nn = g.nn;
    const bool rep = E > nn;
    const Blocks blk = blocks_of(ec, 2 * (int64_t)E);
    if (!rep && threadIdx.x == 0) {
        bar_init(&bar);
        bar_expect(&bar, blk.bytes);
        bulk_load(dm_sm, blk, &bar);
    }
    build_ranks(g, &tab);                                             /* ends with __syncthreads */
    int16_t *T16 = reinterpret_cast<int16_t *>(dm_sm + DM_RAW);
    int32_t *T32 = reinterpret_cast<int32_t *>(dm_sm);
    const int Rp = rep ? (g.R | 1) : pad_rows(g.R, 2);
    if (!rep) {
        bar_wait0(&bar);
        const uint32_t raw = smem_addr(dm_sm) + blk.lead, t16 = smem_addr(T16);
        for_each_position(g, tab, Rp, [&](int ix, int r, bool in_range, bool) {
            const int32_t v = ld_s16(raw + 2 * min(r, E - 1));
            st_s16_if(t16 + 2 * ix, r < E ? v : 0, in_range);
        });
    } else {
        for_each_position(g, tab, Rp, [&](int ix, int r, bool in_range, bool) {
            if (!in_range) return;
            int32_t v = 0;
            for (int k = r; k < E; k += nn) v += __ldg(ec + k);
            T32[ix] = v;
        });
    }
    __syncthreads();
    /* stream order: a thread's n advances by 2 x RM_THREADS = 1024, i.e. 32 rows of
     * the same column, so its T index advances by 32 */
    const int half = g.D >> 1;                                        /* D = K + 4 is even */
#pragma unroll 1
    for (int s = 0; s < 3; s++) {
        int16_t *h = (s == 0 ? h0 : s == 1 ? h1 : h2) + d.llr_off;
        int i = threadIdx.x;
        if (i >= half) continue;
        int ia = t_index(g, Rp, s, 2 * i), ib = t_index(g, Rp, s, 2 * i + 1);
        if (!rep && !combine && (reinterpret_cast<uintptr_t>(h) & 3u) == 0) {
            uint32_t *hw = reinterpret_cast<uint32_t *>(h);
            const uint32_t t16 = smem_addr(T16);
            for (; i < half; i += RM_THREADS, ia += 32, ib += 32)
                hw[i] = (uint32_t)(uint16_t)ld_s16(t16 + 2 * ia) | ((uint32_t)ld_s16(t16 + 2 * ib) << 16);
        } else {
            for (; i < half; i += RM_THREADS, ia += 32, ib += 32) {
                int32_t va = rep ? T32[ia] : (int32_t)T16[ia], vb = rep ? T32[ib] : (int32_t)T16[ib];
                if (combine) { va += h[2 * i]; vb += h[2 * i + 1]; }
                h[2 * i] = (int16_t)max(-32768, min(32767, va));
                h[2 * i + 1] = (int16_t)max(-32768, min(32767, vb));
            }
        }
    }
}

/* Matching: the three coded streams are bulk-copied, re-laid out into byte T in
 * stream order, and each circular-buffer position's bit is written to e[r + m
 * 3D] for every m with r + m 3D < E (punctured ranks: none). */
__global__ void __launch_bounds__(RM_THREADS)
match_kernel(const crn_rm_desc *__restrict__ desc, const uint8_t *__restrict__ d0, const uint8_t *__restrict__ d1,
             const uint8_t *__restrict__ d2, uint8_t *__restrict__ e) {
    extern __shared__ __align__(16) uint8_t mt_sm[];
    __shared__ RankTab tab;
    __shared__ __align__(8) uint64_t bar;
    const crn_rm_desc d = desc[blockIdx.x];
    const Geo g = geo(d.K, d.rv);
    const Blocks b0 = blocks_of(d0 + d.llr_off, g.D), b1 = blocks_of(d1 + d.llr_off, g.D),
                 b2 = blocks_of(d2 + d.llr_off, g.D);
    if (threadIdx.x == 0) {
        bar_init(&bar);
        bar_expect(&bar, b0.bytes + b1.bytes + b2.bytes);
        bulk_load(mt_sm, b0, &bar);
        bulk_load(mt_sm + MT_RAW, b1, &bar);
        bulk_load(mt_sm + 2 * MT_RAW, b2, &bar);
    }
    build_ranks(g, &tab);                                             /* ends with __syncthreads */
    uint8_t *T8 = mt_sm + 3 * MT_RAW;
    const int Rp = pad_rows(g.R, 4);
    bar_wait0(&bar);
    /* stream order: a thread's n advances by RM_THREADS = 512 = 16 rows */
#pragma unroll 1
    for (int s = 0; s < 3; s++) {
        const uint32_t raw = smem_addr(mt_sm) + s * MT_RAW + (s == 0 ? b0.lead : s == 1 ? b1.lead : b2.lead);
        int n = threadIdx.x;
        if (n >= g.D) continue;
        for (uint32_t ta = smem_addr(T8) + t_index(g, Rp, s, n); n < g.D; n += RM_THREADS, ta += 16)
            st_s8(ta, ld_s8(raw + n));
    }
    __syncthreads();
    /* circular-buffer order: Q[r] = bit of rank r (Q reuses the raw area) */
    uint8_t *Q = mt_sm;
    const uint32_t qa = smem_addr(Q), t8 = smem_addr(T8);
    for_each_position(g, tab, Rp, [&](int ix, int r, bool, bool real) { st_s8_if(qa + r, ld_s8(t8 + ix), real); });
    __syncthreads();
    /* e[k] = Q[k mod 3D]: whole words when e is word-aligned (3D = 0 mod 4) */
    uint8_t *ec = e + d.e_off;
    const int E = d.E, nn = g.nn;
    if ((reinterpret_cast<uintptr_t>(ec) & 3u) == 0) {
        const uint32_t *qw = reinterpret_cast<const uint32_t *>(Q);
        uint32_t *ew = reinterpret_cast<uint32_t *>(ec);
        const int nw = E >> 2, nnw = nn >> 2;
        int w = threadIdx.x, j = w % nnw;
        const int jinc = RM_THREADS % nnw;
        for (; w < nw; w += RM_THREADS) {
            ew[w] = qw[j];
            j += jinc;
            if (j >= nnw) j -= nnw;
        }
        for (int k = 4 * nw + threadIdx.x; k < E; k += RM_THREADS) ec[k] = Q[k % nn];
    } else {
        for (int k = threadIdx.x; k < E; k += RM_THREADS) ec[k] = Q[k % nn];
    }
}

/* Matching with packed bits (one bit per bit, LSB-first words): CB i's three
 * streams are bits [llr_off, llr_off + K + 4) of d0 / d1 / d2, its E output bits go
 * to bits [e_off, e_off + E) of e.  The same walk as match_kernel on byte-wide T
 * and Q in shared memory; the stream words come in with plain coalesced loads (a
 * few hundred words), and the output is assembled a word per warp instruction by
 * a ballot -- whole words stored, the (at most two) words shared with
 * neighbouring CBs merged with atomics. */
constexpr int MP_RAW_W = RM_MAXR + 2;                                 /* words covering one stream at any bit offset */
constexpr int MP_Q = (3 * (6144 + 4) + 15) / 16 * 16;
constexpr int MP_SMEM = 3 * MP_RAW_W * 4 + MT_T8 + MP_Q;              /* 39,864 B */

__global__ void __launch_bounds__(RM_THREADS)
match_packed_kernel(const crn_rm_desc *__restrict__ desc, const uint32_t *__restrict__ d0,
                    const uint32_t *__restrict__ d1, const uint32_t *__restrict__ d2, uint32_t *e) {
    extern __shared__ __align__(16) uint8_t mp_sm[];
    __shared__ RankTab tab;
    const crn_rm_desc d = desc[blockIdx.x];
    const Geo g = geo(d.K, d.rv);
    uint32_t *raw = reinterpret_cast<uint32_t *>(mp_sm);             /* [3][MP_RAW_W] */
    uint8_t *T8 = mp_sm + 3 * MP_RAW_W * 4, *Q = T8 + MT_T8;
    const int sh = (int)(d.llr_off & 31);
    const int64_t w0 = d.llr_off >> 5;
    const int nwr = (sh + g.D + 31) >> 5;                              /* words holding the stream's bits */
    for (int i = threadIdx.x; i < 3 * nwr; i += RM_THREADS) {
        const int s = i / nwr, k = i - s * nwr;
        raw[s * MP_RAW_W + k] = __ldg((s == 0 ? d0 : s == 1 ? d1 : d2) + w0 + k);
    }
    build_ranks(g, &tab);                                             /* ends with __syncthreads */
    const int Rp = pad_rows(g.R, 4);
    /* stream order: a thread's n advances by RM_THREADS = 512 = 16 rows */
#pragma unroll 1
    for (int s = 0; s < 3; s++) {
        const uint32_t *rw = raw + s * MP_RAW_W;
        int n = threadIdx.x;
        if (n >= g.D) continue;
        for (uint32_t ta = smem_addr(T8) + t_index(g, Rp, s, n); n < g.D; n += RM_THREADS, ta += 16) {
            const int b = sh + n;
            st_s8(ta, (rw[b >> 5] >> (b & 31)) & 1u);
        }
    }
    __syncthreads();
    const uint32_t qa = smem_addr(Q), t8 = smem_addr(T8);
    for_each_position(g, tab, Rp, [&](int ix, int r, bool, bool real) { st_s8_if(qa + r, ld_s8(t8 + ix), real); });
    __syncthreads();
    /* e bit e_off + k = Q[k mod 3D]: a warp per output word, lane = bit (32
     * consecutive rank bytes: conflict-free), one ballot; the lane's rank advances
     * by a constant per word, so no division in the loop */
    const int lane = threadIdx.x & 31, nn = g.nn, sh0 = (int)(d.e_off & 31), E = d.E;
    const int nwd = (sh0 + E + 31) >> 5;
    uint32_t *ec = e + (d.e_off >> 5);
    int k = 32 * (int)(threadIdx.x >> 5) + lane - sh0;
    int rr = k % nn;
    if (rr < 0) rr += nn;
    const int kinc = 32 * (RM_THREADS / 32), rinc = kinc % nn;
    for (int i = threadIdx.x >> 5; i < nwd; i += RM_THREADS / 32) {
        const bool in = k >= 0 && k < E;
        const uint32_t word = __ballot_sync(0xFFFFFFFFu, in && Q[rr] != 0), mask = __ballot_sync(0xFFFFFFFFu, in);
        if (lane == 0) {
            if (mask == 0xFFFFFFFFu) {
                ec[i] = word;
            } else {
                atomicAnd(ec + i, ~mask);
                atomicOr(ec + i, word);
            }
        }
        k += kinc;
        rr += rinc;
        if (rr >= nn) rr -= nn;
    }
}

/* the kernels' dynamic shared-memory attribute, set once per device (a bit per
 * device id; the attribute is per device context) */
template <class K>
int rm_smem_attr(K kernel, int bytes, std::atomic<uint64_t> &done) {
    int dev;
    if (cudaGetDevice(&dev) != cudaSuccess) return CRN_ECUDA;
    if (dev < 64 && ((done.load() >> dev) & 1u)) return CRN_OK;
    if (cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes) != cudaSuccess)
        return CRN_ECUDA;
    if (dev < 64) done.fetch_or(1ull << dev);
    return CRN_OK;
}

}  // namespace

extern "C" int crn_launch_dematch(const crn_rm_desc *d_desc, int32_t n_cb, const int16_t *e, int32_t combine,
                                  int16_t *h0, int16_t *h1, int16_t *h2, void *stream) {
    static std::atomic<uint64_t> done{0};
    const int attr = rm_smem_attr(dematch_kernel, DM_SMEM, done);
    if (attr) return attr;
    dematch_kernel<<<n_cb, RM_THREADS, DM_SMEM, (cudaStream_t)stream>>>(d_desc, e, combine, h0, h1, h2);
    return cudaGetLastError() == cudaSuccess ? CRN_OK : CRN_ECUDA;
}

extern "C" int crn_launch_match(const crn_rm_desc *d_desc, int32_t n_cb, const uint8_t *d0, const uint8_t *d1,
                                const uint8_t *d2, uint8_t *e, void *stream) {
    static std::atomic<uint64_t> done{0};
    const int attr = rm_smem_attr(match_kernel, MT_SMEM, done);
    if (attr) return attr;
    match_kernel<<<n_cb, RM_THREADS, MT_SMEM, (cudaStream_t)stream>>>(d_desc, d0, d1, d2, e);
    return cudaGetLastError() == cudaSuccess ? CRN_OK : CRN_ECUDA;
}

extern "C" int crn_launch_match_packed(const crn_rm_desc *d_desc, int32_t n_cb, const uint32_t *d0, const uint32_t *d1,
                                       const uint32_t *d2, uint32_t *e, void *stream) {
    static std::atomic<uint64_t> done{0};
    const int attr = rm_smem_attr(match_packed_kernel, MP_SMEM, done);
    if (attr) return attr;
    match_packed_kernel<<<n_cb, RM_THREADS, MP_SMEM, (cudaStream_t)stream>>>(d_desc, d0, d1, d2, e);
    return cudaGetLastError() == cudaSuccess ? CRN_OK : CRN_ECUDA;
}
