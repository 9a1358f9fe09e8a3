/* crn_decode.cu -- the hot path of arxiv 1905.01141's uplink channel decoding
 * as one persistent sm_100a kernel: batched LTE turbo
 * decoding, int16 max-log-MAP on the 8-state RSC trellis, QPP interleaver,
 * M_K parallel windows with next-iteration initialisation, fixed or CRC
 * early-terminated iterations, hard decision + CRC (rows a2..a9 of DESIGN.md).
 *
 * Layout.  A CTA task holds n_pairs pairs of equal-K code blocks; the two CBs of
 * a pair live in the low / high int16 half of every 32-bit register and word
 * (pair-SIMD: VIADD.16x2, VIMNMX(3).S16x2, VIADDMNMX.S16x2), so the trellis
 * butterfly is a register rename.  Thread t = p*M + j owns window j of pair p.
 * Per-step arrays are window-major: element (step i, thread t) at i*T + t, so a
 * warp's accesses at one step are contiguous, and -- because W divides K and the
 * QPP is contention-free -- DEC2's interleaved accesses at step i all fall in
 * one row (offset Pi(i) mod W) at distinct columns.
 *
 * Exactness: every intermediate provably fits int16 (DESIGN.md "int16 safety",
 * checked by the oracle on adversarial inputs), so wrapping int16x2 arithmetic
 * equals the oracle's int32 arithmetic bit for bit.
 */
#include <cuda_runtime.h>
#include <stdint.h>

#include "crn_internal.h"

typedef uint32_t u32;
typedef uint64_t u64;

namespace {

constexpr int NS = CRN_NSTATE;
constexpr int TMAX = CRN_CTA_THREADS;
constexpr int SUMK = CRN_TASK_SUMK;
constexpr int MAXP = SUMK / 40 + 1;             /* max pairs per task (K = 40) */
constexpr u32 FLOOR2 = 0xE000E000u;             /* (-8192, -8192): state-metric floor  */
constexpr u32 CLIP_HI = 0x10001000u;            /* ( 4096,  4096): channel / extrinsic clamp */
constexpr u32 CLIP_LO = 0xF000F000u;            /* (-4096, -4096) */
constexpr u32 POLY_A = 0x864CFBu, POLY_B = 0x800063u;

/* workspace slot (u32 words) */
constexpr int A_LS = 0, A_LP1 = SUMK, A_LP2 = 2 * SUMK, A_LSI = 3 * SUMK, A_X = 4 * SUMK, A_Y = 5 * SUMK;
constexpr int A_Z = 6 * SUMK;                   /* fast path: Le2 in interleaved order */
constexpr int A_NII = 7 * SUMK;                 /* [c][parity][alpha/beta][s][TMAX] */
constexpr int NII_WORDS = 2 * 2 * 2 * NS * TMAX;
constexpr int A_TAIL = A_NII + NII_WORDS;       /* [pair][12] */
constexpr int SLOT_WORDS = A_TAIL + MAXP * 12;
constexpr size_t WS_HEAD = 256;                 /* task counter */

/* ---- RSC trellis, S = 4 r1 + 2 r2 + r3 (R1), evaluated at compile time */
__host__ __device__ constexpr int nxt(int S, int u) { return (((u ^ (S >> 1) ^ S) & 1) << 2) | (S >> 1); }
__host__ __device__ constexpr int par(int S, int u) { return (u ^ (S >> 1) ^ (S >> 2)) & 1; } /* z = u^r1^r2 */

__device__ __forceinline__ u32 vadd(u32 a, u32 b) { return __vadd2(a, b); }
__device__ __forceinline__ u32 vaddmax(u32 a, u32 b, u32 c) { return __viaddmax_s16x2(a, b, c); } /* max(a+b, c) */

/* gamma(u, z) = u*Lu + z*Lp; the (0,0) branch is never formed */
__device__ __forceinline__ u32 gsel(int u, int z, u32 Lu, u32 Lp, u32 Lup) { return u ? (z ? Lup : Lu) : Lp; }

/* N(v)(s) = max(v(s) - max_s' v(s'), -8192) */
__device__ __forceinline__ void norm8(u32 v[NS]) {
    u32 m0 = __vimax3_s16x2(v[0], v[1], v[2]);
    u32 m1 = __vimax3_s16x2(v[3], v[4], v[5]);
    u32 m = __vimax3_s16x2(v[6], v[7], m0);
    m = __vmaxs2(m, m1);
    u32 neg = __vneg2(m);
#pragma unroll
    for (int s = 0; s < NS; s++) v[s] = vaddmax(v[s], neg, FLOOR2);
}

/* alpha_{k+1}(S') = N(max over the two predecessors S of alpha_k(S) + gamma_k) */
__device__ __forceinline__ void alpha_step(u32 a[NS], u32 Lu, u32 Lp, u32 Lup) {
    u32 an[NS];
#pragma unroll
    for (int Sp = 0; Sp < NS; Sp++) {
        const int S0 = 2 * (Sp & 3), S1 = S0 + 1;
        const int u0 = (nxt(S0, 0) == Sp) ? 0 : 1, u1 = (nxt(S1, 0) == Sp) ? 0 : 1;
        const int z0 = par(S0, u0), z1 = par(S1, u1);
        if (!u0 && !z0) an[Sp] = vaddmax(a[S1], gsel(u1, z1, Lu, Lp, Lup), a[S0]);
        else if (!u1 && !z1) an[Sp] = vaddmax(a[S0], gsel(u0, z0, Lu, Lp, Lup), a[S1]);
        else an[Sp] = vaddmax(a[S1], gsel(u1, z1, Lu, Lp, Lup), vadd(a[S0], gsel(u0, z0, Lu, Lp, Lup)));
    }
    norm8(an);
#pragma unroll
    for (int s = 0; s < NS; s++) a[s] = an[s];
}

/* beta_k(S) = N(max over u of beta_{k+1}(next(S,u)) + gamma_k(u, z(S,u))) */
__device__ __forceinline__ void beta_step(u32 b[NS], u32 Lu, u32 Lp, u32 Lup) {
    u32 v[NS];
#pragma unroll
    for (int S = 0; S < NS; S++) {
        const int n0 = nxt(S, 0), n1 = nxt(S, 1), z0 = par(S, 0), z1 = par(S, 1);
        if (!z0) v[S] = vaddmax(b[n1], gsel(1, z1, Lu, Lp, Lup), b[n0]);
        else v[S] = vaddmax(b[n1], gsel(1, z1, Lu, Lp, Lup), vadd(b[n0], Lp));
    }
    norm8(v);
#pragma unroll
    for (int s = 0; s < NS; s++) b[s] = v[s];
}

/* Le = clamp(Lambda_1 - Lambda_0, +-4096), Lambda_u = max over the 8 transitions
 * with input u of alpha_k(S) + z Lp + beta_{k+1}(S'), grouped by z. */
__device__ __forceinline__ u32 lambda_le(const u32 a[NS], const u32 bn[NS], u32 Lp) {
    u32 lam[2];
#pragma unroll
    for (int u = 0; u < 2; u++) {
        u32 m[2] = {0, 0};
        bool first[2] = {true, true};
#pragma unroll
        for (int S = 0; S < NS; S++) {
            const int z = par(S, u), Sn = nxt(S, u);
            m[z] = first[z] ? vadd(a[S], bn[Sn]) : vaddmax(a[S], bn[Sn], m[z]);
            first[z] = false;
        }
        lam[u] = vaddmax(m[1], Lp, m[0]);
    }
    return __vmins2(__vmaxs2(__vsub2(lam[1], lam[0]), CLIP_LO), CLIP_HI);
}

/* beta_K from the tail: beta_{K+3} = (0, -F x7); three forced steps (R11) */
__device__ __forceinline__ void tail_beta(const u32 *tail, u32 b[NS]) {
    b[0] = 0;
#pragma unroll
    for (int s = 1; s < NS; s++) b[s] = FLOOR2;
#pragma unroll
    for (int tau = 2; tau >= 0; tau--) {
        u32 x = tail[2 * tau], z = tail[2 * tau + 1], xz = vadd(x, z);
        u32 v[NS];
#pragma unroll
        for (int S = 0; S < NS; S++) {
            const int r1 = (S >> 2) & 1, r2 = (S >> 1) & 1, r3 = S & 1;
            const int uS = r2 ^ r3, zS = r1 ^ r3;
            v[S] = (uS | zS) ? vadd(b[S >> 1], gsel(uS, zS, x, z, xz)) : b[S >> 1];
        }
        norm8(v);
#pragma unroll
        for (int s = 0; s < NS; s++) b[s] = v[s];
    }
}

__device__ __forceinline__ u32 clamp_pack(int16_t lo, int16_t hi) {
    u32 v = (u32)(uint16_t)lo | ((u32)(uint16_t)hi << 16);
    return __vmins2(__vmaxs2(v, CLIP_LO), CLIP_HI);
}

__device__ __forceinline__ u32 crc_bit(u32 reg, u32 bit, u32 poly) {
    u32 fb = ((reg >> 23) ^ bit) & 1u;
    return ((reg << 1) & 0xFFFFFFu) ^ (fb ? poly : 0u);
}

/* a(x) * b(x) mod g(x), 24-bit polynomials (Horner over the bits of b) */
__device__ __forceinline__ u32 crc_mulmod(u32 a, u32 b, u32 poly) {
    u32 acc = 0;
    for (int k = 23; k >= 0; k--) {
        acc = ((acc << 1) & 0xFFFFFFu) ^ ((acc & 0x800000u) ? poly : 0u);
        if ((b >> k) & 1u) acc ^= a;
    }
    return acc;
}

struct Ctx {
    int T, t, p, j, M, W, it;
    u32 *slot;
    const u32 *qtab;
    u32 *bst;   /* shared: beta storage (i*NS + s)*T + t */
};

/* One constituent SISO pass (half-iteration) of thread (p, j).  C = 0: DEC1
 * (natural order; La from X, Le to Y); C = 1: DEC2 (interleaved systematic,
 * parity 2, La2 = Le1[Pi(i)] from Y, Le2 scattered to X[Pi(i)] = La1_next). */
template <int C>
__device__ __forceinline__ void siso(const Ctx &c) {
    const int T = c.T, t = c.t, W = c.W;
    const u32 *Ls = c.slot + (C ? A_LSI : A_LS);
    const u32 *Lp = c.slot + (C ? A_LP2 : A_LP1);
    const u32 *La = c.slot + (C ? A_Y : A_X);
    u32 *Le = c.slot + (C ? A_X : A_Y);
    u32 *nii = c.slot + A_NII;
    const int rd = (c.it - 1) & 1, wr = c.it & 1;
    auto nii_at = [&](int ab, int par_, int s, int tt) -> u32 * {
        return nii + ((((C * 2 + par_) * 2 + ab) * NS + s) * TMAX + tt);
    };
    auto addr = [&](int i) -> int {
        if (C == 0) return i * T + t;
        u32 q = c.qtab[i * c.M + c.j];
        return (int)(q >> 16) * T + c.p * c.M + (int)(q & 0xFFFFu);
    };

    /* ---- beta pass (row a5), stores beta_{i+1} for Lambda(i) */
    u32 b[NS];
    if (c.j == c.M - 1) tail_beta(c.slot + A_TAIL + c.p * 12 + C * 6, b);
    else if (c.it == 1) {
#pragma unroll
        for (int s = 0; s < NS; s++) b[s] = 0;
    } else {
#pragma unroll
        for (int s = 0; s < NS; s++) b[s] = *nii_at(1, rd, s, t + 1);
    }
#pragma unroll
    for (int s = 0; s < NS; s++) c.bst[(W * NS + s) * T + t] = b[s];
#pragma unroll 2
    for (int i = W - 1; i >= 0; i--) {
        const int ix = i * T + t;
        u32 lp = Lp[ix], lu = vadd(Ls[ix], La[addr(i)]);
        beta_step(b, lu, lp, vadd(lu, lp));
        if (i > 0) {
#pragma unroll
            for (int s = 0; s < NS; s++) c.bst[(i * NS + s) * T + t] = b[s];
        }
    }
#pragma unroll
    for (int s = 0; s < NS; s++) *nii_at(1, wr, s, t) = b[s];          /* beta_{jW} -> window j-1 */

    /* ---- alpha pass (row a6) + Lambda / extrinsic (row a7) */
    u32 a[NS];
    if (c.j == 0) {
        a[0] = 0;
#pragma unroll
        for (int s = 1; s < NS; s++) a[s] = FLOOR2;
    } else if (c.it == 1) {
#pragma unroll
        for (int s = 0; s < NS; s++) a[s] = 0;
    } else {
#pragma unroll
        for (int s = 0; s < NS; s++) a[s] = *nii_at(0, rd, s, t - 1);
    }
#pragma unroll 2
    for (int i = 0; i < W; i++) {
        const int ix = i * T + t, ax = addr(i);
        u32 lp = Lp[ix], lu = vadd(Ls[ix], La[ax]);
        u32 bn[NS];
#pragma unroll
        for (int s = 0; s < NS; s++) bn[s] = c.bst[((i + 1) * NS + s) * T + t];
        Le[ax] = lambda_le(a, bn, lp);
        alpha_step(a, lu, lp, vadd(lu, lp));
    }
#pragma unroll
    for (int s = 0; s < NS; s++) *nii_at(0, wr, s, t) = a[s];          /* alpha_{(j+1)W} -> window j+1 */
}

/* ======================================================================
 * Fast path: W = 32 (every K that is a multiple of 32: all K >= 1056 and 15
 * of the smaller sizes).  Compile-time window length, so every per-step
 * index is an immediate.  The window's inputs are loaded into registers at
 * the start of each half-iteration (window-major workspace, row stride TS);
 * the alpha and beta recursions run concurrently ("crossing": alpha forward
 * from the window start, beta backward from its end; the first half stores
 * both, the second half pairs each new metric with the stored one of the
 * other sweep and emits two extrinsics per step); stored metrics live in
 * shared memory at (slot*16 + k)*TS + t.  State metrics are kept biased by
 * -1 (a~ = a - 1), which turns the normaliser's negation into one NOT:
 * ~(m - 1) = -m.  Exact: every value stays within int16.
 * ====================================================================== */
constexpr int TS = TMAX;                       /* fast-path row stride (words) */
constexpr u32 M1 = 0xFFFFFFFFu;               /* (-1, -1): biased 0           */
constexpr u32 FLOORB = 0xDFFFDFFFu;           /* (-8193, -8193): biased floor */
constexpr u32 NEG4097 = 0xEFFFEFFFu, ONE2 = 0x00010001u;

__device__ __forceinline__ void norm8b(u32 v[NS]) {
    u32 m0 = __vimax3_s16x2(v[0], v[1], v[2]);
    u32 m1 = __vimax3_s16x2(v[3], v[4], v[5]);
    u32 m = __vimax3_s16x2(v[6], v[7], m0);
    m = __vmaxs2(m, m1);
    const u32 nm = ~m;                         /* biased: ~(m - 1) = -m */
#pragma unroll
    for (int s = 0; s < NS; s++) v[s] = vaddmax(v[s], nm, FLOORB);
}

__device__ __forceinline__ void alpha_step_b(u32 a[NS], u32 Lu, u32 Lp, u32 Lup) {
    u32 an[NS];
#pragma unroll
    for (int Sp = 0; Sp < NS; Sp++) {
        const int S0 = 2 * (Sp & 3), S1 = S0 + 1;
        const int u0 = (nxt(S0, 0) == Sp) ? 0 : 1, u1 = (nxt(S1, 0) == Sp) ? 0 : 1;
        const int z0 = par(S0, u0), z1 = par(S1, u1);
        if (!u0 && !z0) an[Sp] = vaddmax(a[S1], gsel(u1, z1, Lu, Lp, Lup), a[S0]);
        else if (!u1 && !z1) an[Sp] = vaddmax(a[S0], gsel(u0, z0, Lu, Lp, Lup), a[S1]);
        else an[Sp] = vaddmax(a[S1], gsel(u1, z1, Lu, Lp, Lup), vadd(a[S0], gsel(u0, z0, Lu, Lp, Lup)));
    }
    norm8b(an);
#pragma unroll
    for (int s = 0; s < NS; s++) a[s] = an[s];
}

__device__ __forceinline__ void beta_step_b(u32 b[NS], u32 Lu, u32 Lp, u32 Lup) {
    u32 v[NS];
#pragma unroll
    for (int S = 0; S < NS; S++) {
        const int n0 = nxt(S, 0), n1 = nxt(S, 1), z0 = par(S, 0), z1 = par(S, 1);
        if (!z0) v[S] = vaddmax(b[n1], gsel(1, z1, Lu, Lp, Lup), b[n0]);
        else v[S] = vaddmax(b[n1], gsel(1, z1, Lu, Lp, Lup), vadd(b[n0], Lp));
    }
    norm8b(v);
#pragma unroll
    for (int s = 0; s < NS; s++) b[s] = v[s];
}

/* Le = clamp(L1 - L0, +-4096) computed as min(max(L1 + ~L0, -4097) + 1, 4096) */
__device__ __forceinline__ u32 lambda_le_b(const u32 a[NS], const u32 bn[NS], u32 Lp) {
    u32 lam[2];
#pragma unroll
    for (int u = 0; u < 2; u++) {
        u32 m[2] = {0, 0};
        bool first[2] = {true, true};
#pragma unroll
        for (int S = 0; S < NS; S++) {
            const int z = par(S, u), Sn = nxt(S, u);
            m[z] = first[z] ? vadd(a[S], bn[Sn]) : vaddmax(a[S], bn[Sn], m[z]);
            first[z] = false;
        }
        lam[u] = vaddmax(m[1], Lp, m[0]);
    }
    return __viaddmin_s16x2(vaddmax(lam[1], ~lam[0], NEG4097), ONE2, CLIP_HI);
}

__device__ __forceinline__ void tail_beta_b(const u32 *tail, u32 b[NS]) {
    b[0] = M1;
#pragma unroll
    for (int s = 1; s < NS; s++) b[s] = FLOORB;
#pragma unroll
    for (int tau = 2; tau >= 0; tau--) {
        u32 x = tail[2 * tau], z = tail[2 * tau + 1], xz = vadd(x, z);
        u32 v[NS];
#pragma unroll
        for (int S = 0; S < NS; S++) {
            const int r1 = (S >> 2) & 1, r2 = (S >> 1) & 1, r3 = S & 1;
            const int uS = r2 ^ r3, zS = r1 ^ r3;
            v[S] = (uS | zS) ? vadd(b[S >> 1], gsel(uS, zS, x, z, xz)) : b[S >> 1];
        }
        norm8b(v);
#pragma unroll
        for (int s = 0; s < NS; s++) b[s] = v[s];
    }
}

/* One half-iteration of thread t = (pair p, window j) on the W = 32 path.
 * C = 0: DEC1: Ls, Lp1 natural; La1[n] = Le2[Pi^-1(n)] gathered from Z
 *         (zeros in iteration 1); Le1 -> Y, natural order.
 * C = 1: DEC2: Ls[Pi], Lp2 natural-in-interleaved-order; La2[i] = Le1[Pi(i)]
 *         gathered from Y; Le2 -> Z in interleaved order.
 * Both gathers are row-local (contention-free): at step i every window of
 * the pair reads one row of the window-major array. */
template <int C>
__device__ __forceinline__ void siso_w32(u32 *slot, const u32 *qg, u32 *sm, int t, int p, int pM, int j, int M,
                                         int it) {
    constexpr int W = 32, H = 16;
    u32 Lu[W], Lp[W];
    const u32 *Lsrc = slot + (C ? A_LSI : A_LS), *Psrc = slot + (C ? A_LP2 : A_LP1), *Asrc = slot + (C ? A_Y : A_Z);
    if (C == 0 && it == 1) {
#pragma unroll
        for (int i = 0; i < W; i++) {
            Lp[i] = Psrc[i * TS + t];
            Lu[i] = Lsrc[i * TS + t];
        }
    } else {
#pragma unroll
        for (int i = 0; i < W; i++) {
            Lp[i] = Psrc[i * TS + t];
            Lu[i] = vadd(Lsrc[i * TS + t], Asrc[pM + (int)qg[i * M + j]]);
        }
    }

    u32 *nii = slot + A_NII;
    const int rd = (it - 1) & 1, wr = it & 1;
    u32 a[NS], b[NS];
    if (j == 0) {
        a[0] = M1;
#pragma unroll
        for (int s = 1; s < NS; s++) a[s] = FLOORB;
    } else if (it == 1) {
#pragma unroll
        for (int s = 0; s < NS; s++) a[s] = M1;
    } else {
#pragma unroll
        for (int s = 0; s < NS; s++) a[s] = nii[(((C * 2 + rd) * 2 + 0) * NS + s) * TMAX + t - 1];
    }
    if (j == M - 1) tail_beta_b(slot + A_TAIL + p * 12 + C * 6, b);
    else if (it == 1) {
#pragma unroll
        for (int s = 0; s < NS; s++) b[s] = M1;
    } else {
#pragma unroll
        for (int s = 0; s < NS; s++) b[s] = nii[(((C * 2 + rd) * 2 + 1) * NS + s) * TMAX + t + 1];
    }

    u32 *st = sm + t;
    /* first half: store alpha_s and beta_{W-s}, advance both (rows a5, a6) */
#pragma unroll
    for (int s = 0; s < H; s++) {
#pragma unroll
        for (int k = 0; k < NS; k++) {
            st[(s * 16 + k) * TS] = a[k];
            st[(s * 16 + 8 + k) * TS] = b[k];
        }
        const int sl = W - 1 - s;
        alpha_step_b(a, Lu[s], Lp[s], vadd(Lu[s], Lp[s]));
        beta_step_b(b, Lu[sl], Lp[sl], vadd(Lu[sl], Lp[sl]));
    }
    /* second half: alpha_s meets stored beta_{s+1}, beta_{W-s} meets stored
     * alpha_{W-1-s}; two extrinsics per step (row a7) */
    u32 *Le = slot + (C ? A_Z : A_Y) + t;
#pragma unroll
    for (int s = H; s < W; s++) {
        const int sl = W - 1 - s;
        u32 bs[NS], as[NS];
        asm volatile("" ::: "memory");      /* keep the stored-metric loads of one step together:
                                               hoisting all 16 steps' loads costs ~130 registers */
#pragma unroll
        for (int k = 0; k < NS; k++) {
            bs[k] = st[(sl * 16 + 8 + k) * TS];
            as[k] = st[(sl * 16 + k) * TS];
        }
        Le[s * TS] = lambda_le_b(a, bs, Lp[s]);
        Le[sl * TS] = lambda_le_b(as, b, Lp[sl]);
        alpha_step_b(a, Lu[s], Lp[s], vadd(Lu[s], Lp[s]));
        beta_step_b(b, Lu[sl], Lp[sl], vadd(Lu[sl], Lp[sl]));
    }
#pragma unroll
    for (int s = 0; s < NS; s++) {
        nii[(((C * 2 + wr) * 2 + 0) * NS + s) * TMAX + t] = a[s];     /* alpha_{(j+1)W} -> window j+1 */
        nii[(((C * 2 + wr) * 2 + 1) * NS + s) * TMAX + t] = b[s];     /* beta_{jW}      -> window j-1 */
    }
}

struct TaskSh {
    int *cb, *F, *kind;
    uint8_t *done, *fin;
    u32 *crc;
    int *left;
};

__device__ __forceinline__ void run_task_w32(const crn_task &tk, const crn_cb_desc *__restrict__ desc,
                                          const int16_t *__restrict__ l0, const int16_t *__restrict__ l1,
                                          const int16_t *__restrict__ l2, int max_iters, int et,
                                          uint32_t *__restrict__ out_bits, uint8_t *__restrict__ crc_ok,
                                          uint8_t *__restrict__ iters_used, int16_t *__restrict__ ext_out,
                                          const crn_tables &tab, u32 *slot, u32 *sm, TaskSh sh) {
    constexpr int W = 32;
    const int tid = threadIdx.x, nth = blockDim.x;
    const int M = tk.M, NP = tk.n_pairs, T = NP * M;
    const bool active = tid < T;
    const int p = active ? tid / M : 0, j = active ? tid - p * M : 0, pM = p * M;
    const u32 *qts = tab.qpp_ts + tab.qpp_off[tk.kidx];     /* natural pos of Pi(jW+i)   */
    const u32 *qinv = tab.qinv_ts + tab.qpp_off[tk.kidx];   /* interleaved pos of jW+i   */
    const u32 *cpow = tab.crc_pow + tab.crc_off[tk.kidx];

    /* ---- row a2: each thread stages its own window of both CBs of its pair */
    if (active) {
        const int clo = sh.cb[2 * p], chi = sh.cb[2 * p + 1];
        const int Flo = sh.F[2 * p], Fhi = sh.F[2 * p + 1];
        const int64_t olo = clo >= 0 ? desc[clo].llr_off : 0, ohi = chi >= 0 ? desc[chi].llr_off : 0;
#pragma unroll 4
        for (int i = 0; i < W; i++) {
            const int n = j * W + i;
            int16_t vs0 = 0, vs1 = 0, va0 = 0, va1 = 0, vq0 = 0, vq1 = 0;
            if (clo >= 0) { vs0 = l0[olo + n]; va0 = l1[olo + n]; vq0 = l2[olo + n]; }
            if (chi >= 0) { vs1 = l0[ohi + n]; va1 = l1[ohi + n]; vq1 = l2[ohi + n]; }
            if (n < Flo) { vs0 = -4096; va0 = -4096; }            /* known filler 0 */
            if (n < Fhi) { vs1 = -4096; va1 = -4096; }
            slot[A_LS + i * TS + tid] = clamp_pack(vs0, vs1);
            slot[A_LP1 + i * TS + tid] = clamp_pack(va0, va1);
            slot[A_LP2 + i * TS + tid] = clamp_pack(vq0, vq1);
        }
        if (j == M - 1) {
            const int K = tk.K;
#pragma unroll
            for (int m = 0; m < 12; m++) {     /* tails: DESIGN.md R11 column order */
                const int col = K + m / 3;
                const int16_t *src = (m % 3 == 0) ? l0 : (m % 3 == 1) ? l1 : l2;
                const int16_t v0 = clo >= 0 ? src[olo + col] : 0;
                const int16_t v1 = chi >= 0 ? src[ohi + col] : 0;
                slot[A_TAIL + p * 12 + m] = clamp_pack(v0, v1);
            }
        }
    }
    __syncthreads();
    if (active) {       /* interleaved systematic Ls[Pi(jW+i)] for DEC2 */
#pragma unroll 8
        for (int i = 0; i < W; i++) slot[A_LSI + i * TS + tid] = slot[A_LS + pM + (int)qts[i * M + j]];
    }
    __syncthreads();

    for (int it = 1; it <= max_iters; it++) {
        if (active) siso_w32<0>(slot, qinv, sm, tid, p, pM, j, M, it);
        __syncthreads();
        if (active) siso_w32<1>(slot, qts, sm, tid, p, pM, j, M, it);
        __syncthreads();
        if (!et && it != max_iters) continue;     /* fixed mode: decide only at the end */

        /* ---- row a9: one packed word per window and CB lane, windowed CRC */
        u32 wlo = 0, whi = 0;
        if (active) {
#pragma unroll
            for (int i = 0; i < W; i++) {
                const u32 la1n = slot[A_Z + pM + (int)qinv[i * M + j]];     /* La1_next[n] = Le2[Pi^-1(n)] */
                const u32 lapp = vadd(vadd(slot[A_LS + i * TS + tid], slot[A_Y + i * TS + tid]), la1n);
                const u32 ge = __vcmpges2(lapp, 0u);         /* tie -> 1 (R16) */
                wlo |= (ge & 1u) << i;
                whi |= ((ge >> 16) & 1u) << i;
            }
            const int n0 = j * W, Flo = sh.F[2 * p], Fhi = sh.F[2 * p + 1];
            if (Flo > n0) wlo &= (Flo >= n0 + 32) ? 0u : (0xFFFFFFFFu << (Flo - n0));
            if (Fhi > n0) whi &= (Fhi >= n0 + 32) ? 0u : (0xFFFFFFFFu << (Fhi - n0));
#pragma unroll
            for (int l = 0; l < 2; l++) {
                const int kind = sh.kind[2 * p + l];
                if (kind == CRN_CRC_NONE) continue;
                const u32 w = l ? whi : wlo, poly = kind == CRN_CRC24A ? POLY_A : POLY_B;
                u32 r = 0;
#pragma unroll
                for (int i = 0; i < W; i++) r = crc_bit(r, (w >> i) & 1u, poly);
                atomicXor(&sh.crc[2 * p + l], crc_mulmod(r, cpow[(kind == CRN_CRC24A ? 0 : M) + j], poly));
            }
        }
        __syncthreads();
        for (int e = tid; e < 2 * NP; e += nth) {
            if (sh.done[e]) continue;
            const bool pass = sh.kind[e] != CRN_CRC_NONE && sh.crc[e] == 0;
            if ((et && pass) || it == max_iters) {
                sh.fin[e] = 1;
                sh.done[e] = 1;
                crc_ok[sh.cb[e]] = pass;
                if (iters_used) iters_used[sh.cb[e]] = (uint8_t)it;
            }
        }
        __syncthreads();
        if (active) {
#pragma unroll
            for (int l = 0; l < 2; l++) {
                if (!sh.fin[2 * p + l]) continue;
                const crn_cb_desc &d = desc[sh.cb[2 * p + l]];
                out_bits[d.bit_off + j] = l ? whi : wlo;
                if (ext_out) {
#pragma unroll 8
                    for (int i = 0; i < W; i++) {
                        const u32 x = slot[A_Z + pM + (int)qinv[i * M + j]];
                        ext_out[d.ext_off + j * W + i] = (int16_t)(l ? (x >> 16) : (x & 0xFFFFu));
                    }
                }
            }
        }
        if (tid == 0) {
            int left = 0;
            for (int e = 0; e < 2 * NP; e++) left += !sh.done[e];
            *sh.left = left;
        }
        __syncthreads();
        for (int e = tid; e < 2 * NP; e += nth) { sh.fin[e] = 0; sh.crc[e] = 0; }
        const int left = *sh.left;
        __syncthreads();
        if (left == 0) break;
    }
}

__global__ void __launch_bounds__(TMAX, 1)
decode_kernel(const crn_cb_desc *__restrict__ desc, const crn_task *__restrict__ tasks, int n_tasks,
              const crn_pair *__restrict__ pairs, const int16_t *__restrict__ l0,
              const int16_t *__restrict__ l1, const int16_t *__restrict__ l2, int max_iters, int et,
              uint32_t *__restrict__ out_bits, uint8_t *__restrict__ crc_ok, uint8_t *__restrict__ iters_used,
              int16_t *__restrict__ ext_out, crn_tables tab, uint8_t *ws) {
    extern __shared__ u32 bst[];
    __shared__ int s_task, s_left;
    __shared__ u32 s_bits[2 * (SUMK / 32 + MAXP)];
    __shared__ u32 s_crc[2 * MAXP];
    __shared__ int s_cb[2 * MAXP], s_F[2 * MAXP], s_kind[2 * MAXP];
    __shared__ uint8_t s_done[2 * MAXP], s_fin[2 * MAXP];

    int *counter = (int *)ws;
    u32 *slot = (u32 *)(ws + WS_HEAD) + (size_t)blockIdx.x * SLOT_WORDS;
    const int tid = threadIdx.x, nth = blockDim.x;

    for (;;) {
        if (tid == 0) s_task = atomicAdd(counter, 1);
        __syncthreads();
        const int task = s_task;
        if (task >= n_tasks) break;
        const crn_task tk = tasks[task];
        const int K = tk.K, M = tk.M, W = tk.W, NP = tk.n_pairs, T = NP * M;
        const int nw = (K + 31) >> 5;
        const u32 *qtab = tab.qpp_wm + tab.qpp_off[tk.kidx];
        const u32 *cpow = tab.crc_pow + tab.crc_off[tk.kidx];

        for (int e = tid; e < 2 * NP; e += nth) {
            const crn_pair pr = pairs[tk.pair0 + (e >> 1)];
            const int cb = (e & 1) ? pr.hi : pr.lo;
            s_cb[e] = cb;
            s_F[e] = cb >= 0 ? desc[cb].F : 0;
            s_kind[e] = cb >= 0 ? desc[cb].crc_kind : 0;
            s_done[e] = cb < 0;
            s_fin[e] = 0;
            s_crc[e] = 0;
        }
        for (int e = tid; e < 2 * NP * nw; e += nth) s_bits[e] = 0;
        __syncthreads();
        if (W == 32) {
            TaskSh sh{s_cb, s_F, s_kind, s_done, s_fin, s_crc, &s_left};
            run_task_w32(tk, desc, l0, l1, l2, max_iters, et, out_bits, crc_ok, iters_used, ext_out, tab, slot, bst, sh);
            continue;
        }

        /* ===== generic path (W in 33..62, small K only): runtime W, stride T ===== */
        /* ---- row a2: demux, clamp to +-4096, filler override, window-major pair packing */
        for (int e = tid; e < NP * K; e += nth) {
            const int p = e / K, n = e - p * K;
            const int clo = s_cb[2 * p], chi = s_cb[2 * p + 1];
            int16_t s0 = 0, s1 = 0, a0 = 0, a1 = 0, q0 = 0, q1 = 0;
            if (clo >= 0) { const int64_t o = desc[clo].llr_off + n; s0 = l0[o]; a0 = l1[o]; q0 = l2[o]; }
            if (chi >= 0) { const int64_t o = desc[chi].llr_off + n; s1 = l0[o]; a1 = l1[o]; q1 = l2[o]; }
            if (n < s_F[2 * p]) { s0 = -4096; a0 = -4096; }           /* known filler 0 */
            if (n < s_F[2 * p + 1]) { s1 = -4096; a1 = -4096; }
            const int ix = (n % W) * T + p * M + n / W;
            slot[A_LS + ix] = clamp_pack(s0, s1);
            slot[A_LP1 + ix] = clamp_pack(a0, a1);
            slot[A_LP2 + ix] = clamp_pack(q0, q1);
        }
        for (int e = tid; e < NP * 12; e += nth) {
            const int p = e / 12, m = e - p * 12;
            /* DEC1 tail (x_K,z_K,x_K+1,z_K+1,x_K+2,z_K+2) = (d0[K],d1[K],d2[K],d0[K+1],d1[K+1],d2[K+1]);
             * DEC2 tail the same from columns K+2, K+3 (R11) */
            const int col = K + m / 3;
            const int16_t *src = (m % 3 == 0) ? l0 : (m % 3 == 1) ? l1 : l2;
            const int clo = s_cb[2 * p], chi = s_cb[2 * p + 1];
            const int16_t v0 = clo >= 0 ? src[desc[clo].llr_off + col] : 0;
            const int16_t v1 = chi >= 0 ? src[desc[chi].llr_off + col] : 0;
            slot[A_TAIL + p * 12 + m] = clamp_pack(v0, v1);
        }
        __syncthreads();
        /* interleaved systematic Ls[Pi(i)] for DEC2 and La1 = 0 */
        for (int e = tid; e < T * W; e += nth) {
            const int i = e / T, tt = e - i * T, p = tt / M, j = tt - p * M;
            const u32 q = qtab[i * M + j];
            slot[A_LSI + e] = slot[A_LS + (int)(q >> 16) * T + p * M + (int)(q & 0xFFFFu)];
            slot[A_X + e] = 0;
        }
        __syncthreads();

        const bool active = tid < T;
        Ctx c;
        c.T = T; c.t = tid; c.p = active ? tid / M : 0; c.j = active ? tid - c.p * M : 0;
        c.M = M; c.W = W; c.slot = slot; c.qtab = qtab; c.bst = bst;

        for (int it = 1; it <= max_iters; it++) {
            c.it = it;
            if (active) siso<0>(c);
            __syncthreads();
            if (active) siso<1>(c);
            __syncthreads();

            /* ---- row a9: L_APP = Ls + Le1 + La1_next, hard decision (tie -> 1),
             * fillers 0, LSB-first packing, windowed CRC with GF(2) combine */
            if (active) {
                const int p = c.p, j = c.j;
                const int Flo = s_F[2 * p], Fhi = s_F[2 * p + 1];
                const int klo = s_kind[2 * p], khi = s_kind[2 * p + 1];
                const u32 plo = klo == CRN_CRC24A ? POLY_A : POLY_B, phi = khi == CRN_CRC24A ? POLY_A : POLY_B;
                u64 vlo = 0, vhi = 0;
                u32 rlo = 0, rhi = 0;
                for (int i = 0; i < W; i++) {
                    const int ix = i * T + tid, n = j * W + i;
                    const u32 lapp = vadd(vadd(slot[A_LS + ix], slot[A_Y + ix]), slot[A_X + ix]);
                    const u32 ge = __vcmpges2(lapp, 0u);
                    const u32 blo = (n < Flo) ? 0u : (ge & 1u), bhi = (n < Fhi) ? 0u : ((ge >> 16) & 1u);
                    vlo |= (u64)blo << i;
                    vhi |= (u64)bhi << i;
                    rlo = crc_bit(rlo, blo, plo);
                    rhi = crc_bit(rhi, bhi, phi);
                }
                const int start = j * W, w0 = start >> 5, off = start & 31;
                u32 *blo_buf = s_bits + (2 * p) * nw, *bhi_buf = s_bits + (2 * p + 1) * nw;
                u64 vv[2] = {vlo, vhi};
                u32 *bb[2] = {blo_buf, bhi_buf};
#pragma unroll
                for (int l = 0; l < 2; l++) {
                    atomicOr(&bb[l][w0], (u32)(vv[l] << off));
                    if (w0 + 1 < nw) atomicOr(&bb[l][w0 + 1], (u32)(vv[l] >> (32 - off)));
                    if (off && w0 + 2 < nw) atomicOr(&bb[l][w0 + 2], (u32)(vv[l] >> (64 - off)));
                }
                if (klo != CRN_CRC_NONE) atomicXor(&s_crc[2 * p], crc_mulmod(rlo, cpow[(klo == CRN_CRC24A ? 0 : M) + j], plo));
                if (khi != CRN_CRC_NONE) atomicXor(&s_crc[2 * p + 1], crc_mulmod(rhi, cpow[(khi == CRN_CRC24A ? 0 : M) + j], phi));
            }
            __syncthreads();
            /* ---- early termination / completion per CB */
            for (int e = tid; e < 2 * NP; e += nth) {
                if (s_done[e]) continue;
                const bool pass = s_kind[e] != CRN_CRC_NONE && s_crc[e] == 0;
                if ((et && pass) || it == max_iters) {
                    s_fin[e] = 1;
                    s_done[e] = 1;
                    crc_ok[s_cb[e]] = pass;
                    if (iters_used) iters_used[s_cb[e]] = (uint8_t)it;
                }
            }
            __syncthreads();
            for (int e = tid; e < 2 * NP * nw; e += nth) {
                const int pl = e / nw, w = e - pl * nw;
                if (s_fin[pl]) out_bits[desc[s_cb[pl]].bit_off + w] = s_bits[e];
                s_bits[e] = 0;
            }
            if (ext_out) {
                for (int e = tid; e < 2 * NP * K; e += nth) {
                    const int pl = e / K, n = e - pl * K, p = pl >> 1;
                    if (!s_fin[pl]) continue;
                    const u32 x = slot[A_X + (n % W) * T + p * M + n / W];
                    ext_out[desc[s_cb[pl]].ext_off + n] = (int16_t)((pl & 1) ? (x >> 16) : (x & 0xFFFFu));
                }
            }
            if (tid == 0) {
                int left = 0;
                for (int e = 0; e < 2 * NP; e++) left += !s_done[e];
                s_left = left;
            }
            __syncthreads();
            for (int e = tid; e < 2 * NP; e += nth) { s_fin[e] = 0; s_crc[e] = 0; }
            const int left = s_left;
            __syncthreads();
            if (left == 0) break;
        }
    }
}

size_t smem_bytes() { return (size_t)(SUMK + TMAX) * NS * 4; }

}  // namespace

extern "C" size_t crn_decode_ws_bytes(int32_t grid) { return WS_HEAD + (size_t)grid * SLOT_WORDS * 4; }

extern "C" int crn_decode_grid(int device) {
    static int configured = -1;
    if (configured != device) {
        if (cudaFuncSetAttribute(decode_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_bytes()) != cudaSuccess)
            return -1;
        configured = device;
    }
    int sms = 0, occ = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, decode_kernel, TMAX, smem_bytes()) != cudaSuccess || occ < 1)
        return -1;
    return sms * occ;
}

extern "C" int crn_launch_decode(const crn_cb_desc *d_desc, const crn_task *d_tasks, int32_t n_tasks,
                                 const crn_pair *d_pairs, const int16_t *l0, const int16_t *l1, const int16_t *l2,
                                 int32_t max_iters, int32_t et, uint32_t *bits, uint8_t *ok, uint8_t *it,
                                 int16_t *ext, const crn_tables *tab, void *ws, void *stream, int32_t grid) {
    cudaStream_t st = (cudaStream_t)stream;
    if (cudaMemsetAsync(ws, 0, WS_HEAD, st) != cudaSuccess) return CRN_ECUDA;
    int g = grid < n_tasks ? grid : n_tasks;
    decode_kernel<<<g, TMAX, smem_bytes(), st>>>(d_desc, d_tasks, n_tasks, d_pairs, l0, l1, l2, max_iters, et, bits,
                                                 ok, it, ext, *tab, (uint8_t *)ws);
    return cudaGetLastError() == cudaSuccess ? CRN_OK : CRN_ECUDA;
}
