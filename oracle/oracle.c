/*
 * oracle.c -- TEST INFRASTRUCTURE ONLY (see oracle.h for the contract).
 *
 * A plain, slow CPU reference of the decoding function of arxiv 1905.01141
 * (PAPER.md:283-303), written step by step in the paper's order:
 *   demultiplex R(x_i) -> R(b_i), R(b_i)', R(b_i)''
 *   DEC1(R(b_i), R(b_i)') -> extrinsic -> DEC2(interleaved R(b_i), R(b_i)'',
 *   extrinsic) -> de-interleave -> DEC1 ...
 *   until success or the maximum number of iterations; hard decision
 * with the bit-level definition the paper leaves open taken from LTE TS 36.212
 * (the paper's OAI/LTE context) and the readings R1..R19 listed in DESIGN.md.
 *
 * Arithmetic is int32 with explicit clamps; every intermediate value is checked
 * to lie in int16 range, violations are counted.
 * Counted operations (the roofline numerator): every add,
 * sub, max and clamp-side the SISO definition performs, except adds whose
 * operand is the literal-zero branch metric of the (u,z) = (0,0) branch.
 */
#include "oracle.h"
#include <math.h>
#include <pthread.h>
#include <stdatomic.h>
#include <stdlib.h>
#include <string.h>

/* ---------------------------------------------------------------- constants */
#define CLAMP_IN   4096   /* internal channel clamp C   (R12) */
#define CLAMP_EXT  4096   /* extrinsic clamp E          (R12) */
#define FLOOR_SM   8192   /* state-metric floor F_m     (R12) */
#define NSTATE     8

/* ------------------------------------------------ QPP table (36.212 T.5.1.3-3)
 * Recalled values (the 3GPP table is not in the container): the permutation,
 * parity-preservation and contention-free properties are pinned by tests;
 * agreement with 3GPP itself is "parity unpinned" (R25). */
static const int QPP[188][3] = {
    {40, 3, 10}, {48, 7, 12}, {56, 19, 42}, {64, 7, 16},
    {72, 7, 18}, {80, 11, 20}, {88, 5, 22}, {96, 11, 24},
    {104, 7, 26}, {112, 41, 84}, {120, 103, 90}, {128, 15, 32},
    {136, 9, 34}, {144, 17, 108}, {152, 9, 38}, {160, 21, 120},
    {168, 101, 84}, {176, 21, 44}, {184, 57, 46}, {192, 23, 48},
    {200, 13, 50}, {208, 27, 52}, {216, 11, 36}, {224, 27, 56},
    {232, 85, 58}, {240, 29, 60}, {248, 33, 62}, {256, 15, 32},
    {264, 17, 198}, {272, 33, 68}, {280, 103, 210}, {288, 19, 36},
    {296, 19, 74}, {304, 37, 76}, {312, 19, 78}, {320, 21, 120},
    {328, 21, 82}, {336, 115, 84}, {344, 193, 86}, {352, 21, 44},
    {360, 133, 90}, {368, 81, 46}, {376, 45, 94}, {384, 23, 48},
    {392, 243, 98}, {400, 151, 40}, {408, 155, 102}, {416, 25, 52},
    {424, 51, 106}, {432, 47, 72}, {440, 91, 110}, {448, 29, 168},
    {456, 29, 114}, {464, 247, 58}, {472, 29, 118}, {480, 89, 180},
    {488, 91, 122}, {496, 157, 62}, {504, 55, 84}, {512, 31, 64},
    {528, 17, 66}, {544, 35, 68}, {560, 227, 420}, {576, 65, 96},
    {592, 19, 74}, {608, 37, 76}, {624, 41, 234}, {640, 39, 80},
    {656, 185, 82}, {672, 43, 252}, {688, 21, 86}, {704, 155, 44},
    {720, 79, 120}, {736, 139, 92}, {752, 23, 94}, {768, 217, 48},
    {784, 25, 98}, {800, 17, 80}, {816, 127, 102}, {832, 25, 52},
    {848, 239, 106}, {864, 17, 48}, {880, 137, 110}, {896, 215, 112},
    {912, 29, 114}, {928, 15, 58}, {944, 147, 118}, {960, 29, 60},
    {976, 59, 122}, {992, 65, 124}, {1008, 55, 84}, {1024, 31, 64},
    {1056, 17, 66}, {1088, 171, 204}, {1120, 67, 140}, {1152, 35, 72},
    {1184, 19, 74}, {1216, 39, 76}, {1248, 19, 78}, {1280, 199, 240},
    {1312, 21, 82}, {1344, 211, 252}, {1376, 21, 86}, {1408, 43, 88},
    {1440, 149, 60}, {1472, 45, 92}, {1504, 49, 846}, {1536, 71, 48},
    {1568, 13, 28}, {1600, 17, 80}, {1632, 25, 102}, {1664, 183, 104},
    {1696, 55, 954}, {1728, 127, 96}, {1760, 27, 110}, {1792, 29, 112},
    {1824, 29, 114}, {1856, 57, 116}, {1888, 45, 354}, {1920, 31, 120},
    {1952, 59, 610}, {1984, 185, 124}, {2016, 113, 420}, {2048, 31, 64},
    {2112, 17, 66}, {2176, 171, 136}, {2240, 209, 420}, {2304, 253, 216},
    {2368, 367, 444}, {2432, 265, 456}, {2496, 181, 468}, {2560, 39, 80},
    {2624, 27, 164}, {2688, 127, 504}, {2752, 143, 172}, {2816, 43, 88},
    {2880, 29, 300}, {2944, 45, 92}, {3008, 157, 188}, {3072, 47, 96},
    {3136, 13, 28}, {3200, 111, 240}, {3264, 443, 204}, {3328, 51, 104},
    {3392, 51, 212}, {3456, 451, 192}, {3520, 257, 220}, {3584, 57, 336},
    {3648, 313, 228}, {3712, 271, 232}, {3776, 179, 236}, {3840, 331, 120},
    {3904, 363, 244}, {3968, 375, 248}, {4032, 127, 168}, {4096, 31, 64},
    {4160, 33, 130}, {4224, 43, 264}, {4288, 33, 134}, {4352, 477, 408},
    {4416, 35, 138}, {4480, 233, 280}, {4544, 357, 142}, {4608, 337, 480},
    {4672, 37, 146}, {4736, 71, 444}, {4800, 71, 120}, {4864, 37, 152},
    {4928, 39, 462}, {4992, 127, 234}, {5056, 39, 158}, {5120, 39, 80},
    {5184, 31, 96}, {5248, 113, 902}, {5312, 41, 166}, {5376, 251, 336},
    {5440, 43, 170}, {5504, 21, 86}, {5568, 43, 174}, {5632, 45, 176},
    {5696, 45, 178}, {5760, 161, 120}, {5824, 89, 182}, {5888, 323, 184},
    {5952, 47, 186}, {6016, 23, 94}, {6080, 47, 190}, {6144, 263, 480},
};

int oracle_num_k(void) { return 188; }

int oracle_k_at(int i) { return (i >= 0 && i < 188) ? QPP[i][0] : -1; }

static int k_row(int K) {
    for (int i = 0; i < 188; i++)
        if (QPP[i][0] == K) return i;
    return -1;
}

int oracle_qpp_params(int K, int *f1, int *f2) {
    int r = k_row(K);
    if (r < 0) return -1;
    *f1 = QPP[r][1];
    *f2 = QPP[r][2];
    return 0;
}

/* Pi(i) = (f1*i + f2*i^2) mod K -- evaluated literally in 64 bit. */
int oracle_qpp_index(int K, int i) {
    int f1, f2;
    if (oracle_qpp_params(K, &f1, &f2) != 0 || i < 0 || i >= K) return -1;
    int64_t ii = i;
    return (int)((f1 * ii + f2 * ii * ii) % K);
}

/* ---------------------------------------------------------------- CRC24 */
uint32_t oracle_crc24(int kind, const uint8_t *bits, int64_t nbits) {
    /* generator without the D^24 term; bit j of the constant = coeff of D^j */
    uint32_t poly = (kind == ORACLE_CRC24A) ? 0x864CFBu : 0x800063u;
    uint32_t reg = 0;
    for (int64_t n = 0; n < nbits; n++) {
        uint32_t fb = ((reg >> 23) & 1u) ^ (bits[n] & 1u);
        reg = (reg << 1) & 0xFFFFFFu;
        if (fb) reg ^= poly;
    }
    return reg;
}

/* ---------------------------------------------------------------- segmentation
 * 36.212 5.1.2 (R4): Z = 6144, L = 24; CB_MAX_SIZE 6120 = Z - L of
 * PAPER.md:337.  Filler bits F go at the front of CB 0. */
int oracle_segment(int64_t tbs, oracle_seg *o) {
    if (tbs <= 0) return -1;
    const int64_t Z = 6144;
    int64_t B = tbs + 24, Bp, C, L;
    if (B <= Z) { L = 0; C = 1; Bp = B; }
    else { L = 24; C = (B + (Z - L) - 1) / (Z - L); Bp = B + C * L; }
    int kp = -1;
    for (int i = 0; i < 188; i++)
        if (C * QPP[i][0] >= Bp) { kp = i; break; }
    if (kp < 0) return -1;
    int64_t Kp = QPP[kp][0], Km = 0, Cm = 0, Cp = C;
    if (C > 1) {
        Km = (kp > 0) ? QPP[kp - 1][0] : 0;
        int64_t dK = Kp - Km;
        Cm = (C * Kp - Bp) / dK;
        Cp = C - Cm;
    }
    o->C = (int32_t)C; o->Kplus = (int32_t)Kp; o->Kminus = (int32_t)Km;
    o->Cplus = (int32_t)Cp; o->Cminus = (int32_t)Cm;
    o->F = (int32_t)(Cp * Kp + Cm * Km - Bp);
    o->L = (int32_t)L;
    return 0;
}

int oracle_num_windows(int K, int wmin) {
    for (int M = K; M >= 1; M--)
        if (K % M == 0 && K / M >= wmin) return M;
    return 1;
}

/* ---------------------------------------------------------------- encoder
 * RSC constituent (36.212 5.1.3.2.1): registers (r1,r2,r3),
 * feedback g0 = 1 + D^2 + D^3, feed-forward g1 = 1 + D + D^3:
 *   a = u ^ r2 ^ r3 ;  z = a ^ r1 ^ r3 ;  (r1,r2,r3) <- (a,r1,r2).
 * Termination (36.212 5.1.3.2.2): three steps with u = r2 ^ r3 (a = 0),
 * emitting x = u and z = r1 ^ r3. */
static void rsc_encode(const uint8_t *u, int K, uint8_t *z, uint8_t xt[3], uint8_t zt[3]) {
    int r1 = 0, r2 = 0, r3 = 0;
    for (int k = 0; k < K; k++) {
        int a = (u[k] & 1) ^ r2 ^ r3;
        z[k] = (uint8_t)(a ^ r1 ^ r3);
        r3 = r2; r2 = r1; r1 = a;
    }
    for (int t = 0; t < 3; t++) {
        int ut = r2 ^ r3;
        xt[t] = (uint8_t)ut;
        zt[t] = (uint8_t)(r1 ^ r3);
        r3 = r2; r2 = r1; r1 = 0;
    }
}

/* Turbo encoder: b_i systematic, b_i' = RSC(b_i),
 * b_i'' = RSC(interleaved b_i) with c'_i = c_{Pi(i)};
 * the 12 tail bits (x_K,z_K,x_K+1,z_K+1,x_K+2,z_K+2, x'_K,z'_K,...) are
 * written column-wise into d0/d1/d2 at K..K+3 (36.212 5.1.3.2.2, R11). */
int oracle_turbo_encode(const uint8_t *c, int K, uint8_t *d0, uint8_t *d1, uint8_t *d2) {
    if (k_row(K) < 0) return -1;
    uint8_t *ci = (uint8_t *)calloc((size_t)K, 1);
    uint8_t *z2 = (uint8_t *)calloc((size_t)K, 1);
    uint8_t xt1[3], zt1[3], xt2[3], zt2[3];
    for (int i = 0; i < K; i++) ci[i] = c[oracle_qpp_index(K, i)] & 1;
    rsc_encode(c, K, d1, xt1, zt1);
    rsc_encode(ci, K, z2, xt2, zt2);
    for (int k = 0; k < K; k++) { d0[k] = c[k] & 1; d2[k] = z2[k]; }
    uint8_t t[12] = {xt1[0], zt1[0], xt1[1], zt1[1], xt1[2], zt1[2],
                     xt2[0], zt2[0], xt2[1], zt2[1], xt2[2], zt2[2]};
    for (int m = 0; m < 12; m++) {
        uint8_t *d = (m % 3 == 0) ? d0 : (m % 3 == 1) ? d1 : d2;
        d[K + m / 3] = t[m];
    }
    free(ci); free(z2);
    return 0;
}

/* ---------------------------------------------------------------- arithmetic */
typedef struct { uint64_t ops; int64_t viol; int logmap; } ctx_t;

static int32_t chk(ctx_t *c, int32_t v) {
    if (v < -32768 || v > 32767) c->viol++;
    return v;
}
static int32_t ADD(ctx_t *c, int32_t a, int32_t b) { c->ops++; return chk(c, a + b); }
static int32_t SUB(ctx_t *c, int32_t a, int32_t b) { c->ops++; return chk(c, a - b); }
static int32_t MAX(ctx_t *c, int32_t a, int32_t b) { c->ops++; return a > b ? a : b; }

/* Log-MAP (SURVEY.md §8(f) f2 "Log-MAP with a LUT correction", R32):
 * the Jacobian logarithm max*(a, b) = ln(e^a + e^b) = max(a, b) + ln(1 + e^-|a-b|),
 * in the channel quantiser's units (an LLR value v means v/8 nat, R9):
 * max*(a, b) = max(a, b) + c(|a - b|) with c(d) = 8 ln(1 + e^(-d/8)) read from an
 * 8-entry table over buckets of 4 units, entry b = round(c(4b + 1.5)) (the value
 * at the bucket centre), bucket min(d >> 2, 7). */
static int32_t logmap_lut(int b) {
    return (int32_t)floor(8.0 * log(1.0 + exp(-(4.0 * b + 1.5) / 8.0)) + 0.5);
}

int32_t oracle_logmap_correction(int32_t d) {
    if (d < 0) return -1;
    return logmap_lut(d >> 2 < 7 ? d >> 2 : 7);
}

int32_t oracle_max_star(int32_t a, int32_t b) {
    int32_t d = a > b ? a - b : b - a;
    return (a > b ? a : b) + oracle_logmap_correction(d);
}

/* The SISO's two-way selection: max in max-log-MAP, max* in Log-MAP. */
static int32_t SEL(ctx_t *c, int32_t a, int32_t b) {
    c->ops++;
    return c->logmap ? chk(c, oracle_max_star(a, b)) : (a > b ? a : b);
}
static int32_t CLAMP(ctx_t *c, int32_t v, int32_t lim) { /* a max and a min: 2 ops */
    c->ops += 2;
    return v < -lim ? -lim : (v > lim ? lim : v);
}

/* Trellis of the RSC above with S = 4*r1 + 2*r2 + r3 (R1). */
static int next_state(int S, int u) {
    int r1 = (S >> 2) & 1, r2 = (S >> 1) & 1, r3 = S & 1;
    int a = u ^ r2 ^ r3;
    return (a << 2) | (r1 << 1) | r2;
}
static int parity_out(int S, int u) {
    int r1 = (S >> 2) & 1, r2 = (S >> 1) & 1, r3 = S & 1;
    int a = u ^ r2 ^ r3;
    return a ^ r1 ^ r3;
}

/* Branch metric candidate m + gamma(u,z) with gamma = u*Lu + z*Lp:
 * the (0,0) branch adds a literal zero and is not counted. */
static int32_t add_gamma(ctx_t *c, int32_t m, int u, int z, int32_t Lu, int32_t Lp, int32_t Lup) {
    if (!u && !z) return m;
    int32_t g = (u && z) ? Lup : (u ? Lu : Lp);
    return ADD(c, m, g);
}

/* N(v)(s) = max(v(s) - max_s' v(s'), -F_m)  (R12) */
static void normalise(ctx_t *c, int32_t v[NSTATE]) {
    int32_t m = v[0];
    for (int s = 1; s < NSTATE; s++) m = MAX(c, m, v[s]);
    for (int s = 0; s < NSTATE; s++) v[s] = MAX(c, SUB(c, v[s], m), -FLOOR_SM);
}

/* alpha_{k+1}(S') = N( max_{S in pred(S')} alpha_k(S) + gamma_k(u,z) ) */
static void alpha_step(ctx_t *c, const int32_t a[NSTATE], int32_t an[NSTATE],
                       int32_t Lu, int32_t Lp, int32_t Lup) {
    int32_t best[NSTATE];
    int have[NSTATE] = {0};
    for (int S = 0; S < NSTATE; S++)
        for (int u = 0; u < 2; u++) {
            int Sn = next_state(S, u), z = parity_out(S, u);
            int32_t cand = add_gamma(c, a[S], u, z, Lu, Lp, Lup);
            if (!have[Sn]) { best[Sn] = cand; have[Sn] = 1; }
            else best[Sn] = SEL(c, best[Sn], cand);
        }
    normalise(c, best);
    memcpy(an, best, sizeof(best));
}

/* beta_k(S) = N( max_{u} beta_{k+1}(next(S,u)) + gamma_k(u,z) ) */
static void beta_step(ctx_t *c, const int32_t bn[NSTATE], int32_t b[NSTATE],
                      int32_t Lu, int32_t Lp, int32_t Lup) {
    int32_t v[NSTATE];
    for (int S = 0; S < NSTATE; S++) {
        int32_t c0 = add_gamma(c, bn[next_state(S, 0)], 0, parity_out(S, 0), Lu, Lp, Lup);
        int32_t c1 = add_gamma(c, bn[next_state(S, 1)], 1, parity_out(S, 1), Lu, Lp, Lup);
        v[S] = SEL(c, c0, c1);
    }
    normalise(c, v);
    memcpy(b, v, sizeof(v));
}

/* Lambda_u(k) = max over transitions with input u of alpha_k(S) + z*Lp + beta_{k+1}(S');
 * Le = clamp(Lambda_1 - Lambda_0, +-E). */
static int32_t lambda_le(ctx_t *c, const int32_t a[NSTATE], const int32_t bn[NSTATE], int32_t Lp) {
    int32_t lam[2];
    for (int u = 0; u < 2; u++) {
        int first = 1;
        for (int S = 0; S < NSTATE; S++) {
            int32_t t = ADD(c, a[S], bn[next_state(S, u)]);
            if (parity_out(S, u)) t = ADD(c, t, Lp);
            lam[u] = first ? t : SEL(c, lam[u], t);          /* fold over S = 0..7 in order */
            first = 0;
        }
    }
    return CLAMP(c, SUB(c, lam[1], lam[0]), CLAMP_EXT);
}

/* Tail: beta_{K+3} = (0, -F_m x 7); for tau = 2,1,0:
 * beta_{K+tau}(S) = N( gamma^tail_tau(S) + beta_{K+tau+1}(S >> 1) ) with the forced
 * tail input u_S = r2 ^ r3 and output z_S = r1 ^ r3 (R11/R12). */
static void tail_beta(ctx_t *c, const int32_t *tail, int32_t bK[NSTATE]) {
    int32_t b[NSTATE], v[NSTATE];
    b[0] = 0;
    for (int s = 1; s < NSTATE; s++) b[s] = -FLOOR_SM;
    for (int tau = 2; tau >= 0; tau--) {
        int32_t x = tail[2 * tau], z = tail[2 * tau + 1];
        int32_t xz = ADD(c, x, z);            /* gamma of the (1,1) tail branch, once per step */
        for (int S = 0; S < NSTATE; S++) {
            int r1 = (S >> 2) & 1, r2 = (S >> 1) & 1, r3 = S & 1;
            int uS = r2 ^ r3, zS = r1 ^ r3;
            v[S] = add_gamma(c, b[S >> 1], uS, zS, x, z, xz);
        }
        normalise(c, v);
        memcpy(b, v, sizeof(v));
    }
    memcpy(bK, b, sizeof(b));
}

int64_t oracle_siso(const int32_t *lsys, const int32_t *lpar, const int32_t *la,
                    const int32_t *tail, int K, int W,
                    const int32_t *alpha_in, const int32_t *beta_in,
                    int32_t *alpha_out, int32_t *beta_out,
                    int32_t *le, uint64_t *ops) {
    return oracle_siso_v(lsys, lpar, la, tail, K, W, alpha_in, beta_in, alpha_out, beta_out, le, ops,
                         ORACLE_VAR_MAXLOG);
}

int64_t oracle_siso_v(const int32_t *lsys, const int32_t *lpar, const int32_t *la,
                      const int32_t *tail, int K, int W,
                      const int32_t *alpha_in, const int32_t *beta_in,
                      int32_t *alpha_out, int32_t *beta_out,
                      int32_t *le, uint64_t *ops, int variant) {
    ctx_t c = {0, 0, variant == ORACLE_VAR_LOGMAP};
    int M = K / W;
    int32_t *beta = (int32_t *)malloc(sizeof(int32_t) * NSTATE * (size_t)(W + 1));
    int32_t *Lu = (int32_t *)malloc(sizeof(int32_t) * (size_t)K);
    int32_t *Lup = (int32_t *)malloc(sizeof(int32_t) * (size_t)K);
    /* branch metrics: Lu_k = Lsys_k + La_k, gamma_k(u,z) = u*Lu_k + z*Lp_k; the
     * (1,1) value Lu_k + Lp_k is formed once per step */
    for (int k = 0; k < K; k++) {
        Lu[k] = ADD(&c, lsys[k], la[k]);
        Lup[k] = ADD(&c, Lu[k], lpar[k]);
    }
    for (int j = 0; j < M; j++) {
        /* beta init at the window end (k = (j+1)W) */
        int32_t *bw = beta + (size_t)W * NSTATE;
        if (j == M - 1) tail_beta(&c, tail, bw);
        else memcpy(bw, beta_in + (size_t)j * NSTATE, sizeof(int32_t) * NSTATE);
        /* beta recursion k = (j+1)W-1 .. jW ; beta[i] holds beta_{jW+i} */
        for (int i = W - 1; i >= 0; i--) {
            int k = j * W + i;
            beta_step(&c, beta + (size_t)(i + 1) * NSTATE, beta + (size_t)i * NSTATE, Lu[k], lpar[k], Lup[k]);
        }
        if (beta_out) memcpy(beta_out + (size_t)j * NSTATE, beta, sizeof(int32_t) * NSTATE);
        /* alpha init at the window start (k = jW) */
        int32_t a[NSTATE], an[NSTATE];
        if (j == 0) { a[0] = 0; for (int s = 1; s < NSTATE; s++) a[s] = -FLOOR_SM; }
        else memcpy(a, alpha_in + (size_t)j * NSTATE, sizeof(a));
        /* alpha recursion + Lambda, k = jW .. (j+1)W-1 */
        for (int i = 0; i < W; i++) {
            int k = j * W + i;
            le[k] = lambda_le(&c, a, beta + (size_t)(i + 1) * NSTATE, lpar[k]);
            alpha_step(&c, a, an, Lu[k], lpar[k], Lup[k]);
            memcpy(a, an, sizeof(a));
        }
        if (alpha_out) memcpy(alpha_out + (size_t)j * NSTATE, a, sizeof(a));
    }
    free(Lu); free(Lup);
    free(beta);
    if (ops) *ops += c.ops;
    return c.viol;
}

/* ---------------------------------------------------------------- NII
 * Next-iteration initialisation (R13): in iteration t+1 window j
 * starts its alpha recursion from alpha_{jW} that window j-1 produced in
 * iteration t, and its beta recursion from beta_{(j+1)W} that window j+1
 * produced in iteration t. */
void oracle_nii_update(int M, const int32_t *alpha_out, const int32_t *beta_out,
                       int32_t *alpha_in, int32_t *beta_in) {
    for (int j = 0; j < M; j++)
        for (int s = 0; s < NSTATE; s++) {
            alpha_in[(size_t)j * NSTATE + s] = j >= 1 ? alpha_out[(size_t)(j - 1) * NSTATE + s] : 0;
            beta_in[(size_t)j * NSTATE + s] = j + 1 < M ? beta_out[(size_t)(j + 1) * NSTATE + s] : 0;
        }
}

/* ---------------------------------------------------------------- decoder */
static int32_t clamp_in(int32_t v) { return v < -CLAMP_IN ? -CLAMP_IN : (v > CLAMP_IN ? CLAMP_IN : v); }

/* Extrinsic scaling of the scaled max-log-MAP variant (R28):
 * s(x) = floor(3x / 4), written as the floor of a quotient, not as a shift. */
static int32_t scale34(int32_t x) {
    int32_t n = 3 * x;
    return n >= 0 ? n / 4 : -((-n + 3) / 4);
}

int32_t oracle_ext_scale(int32_t x) { return scale34(x); }

/* MI of an LLR of magnitude a/8 (the channel quantiser's scale, R9)
 * under the consistent-Gaussian assumption: I = 1 - Hb(p), p = 1/(1+e^(a/8)),
 * Hb the binary entropy; in Q16, a saturated at 255 (R29). */
int32_t oracle_mi_table(int32_t a) {
    if (a < 0) return -1;
    if (a > 255) a = 255;
    const double L = a / 8.0;
    const double p = 1.0 / (1.0 + exp(L));            /* probability of the less likely value */
    const double q = 1.0 - p;
    const double h = (p > 0 ? -p * log2(p) : 0.0) + (q > 0 ? -q * log2(q) : 0.0);
    return (int32_t)floor(65536.0 * (1.0 - h) + 0.5);
}

int64_t oracle_decode_cb(const int16_t *d0, const int16_t *d1, const int16_t *d2,
                         int K, int F, int crc_kind, int max_iters, int early_term, int wmin,
                         uint8_t *bits, uint8_t *crc_ok, uint8_t *iters_used,
                         int16_t *ext, uint64_t *ops) {
    return oracle_decode_cb_v(d0, d1, d2, K, F, crc_kind, max_iters, early_term, wmin, ORACLE_VAR_MAXLOG,
                              bits, crc_ok, iters_used, ext, ops);
}

int64_t oracle_decode_cb_v(const int16_t *d0, const int16_t *d1, const int16_t *d2,
                           int K, int F, int crc_kind, int max_iters, int early_term, int wmin, int variant,
                           uint8_t *bits, uint8_t *crc_ok, uint8_t *iters_used,
                           int16_t *ext, uint64_t *ops) {
    if (k_row(K) < 0 || F < 0 || F > K - 25 || max_iters < 1 || crc_kind < 0 || crc_kind > 2 ||
        variant < 0 || variant > 2 || early_term < 0 || early_term > 2)
        return -1;
    int64_t viol = 0;
    int W = K / oracle_num_windows(K, wmin), M = K / W;
    size_t nK = (size_t)K;
    int32_t *Ls = malloc(4 * nK), *Lp1 = malloc(4 * nK), *Lp2 = malloc(4 * nK);
    int32_t *La1 = calloc(nK, 4), *Le1 = malloc(4 * nK), *Ls2 = malloc(4 * nK);
    int32_t *La2 = malloc(4 * nK), *Le2 = malloc(4 * nK), *La1n = malloc(4 * nK);
    int *Pi = malloc(sizeof(int) * nK);
    /* NII boundary states per constituent (R13): iteration-1 zeros,
     * afterwards the values produced in the previous iteration only. */
    size_t nb = (size_t)M * NSTATE;
    int32_t *a_prev[2], *b_prev[2], *a_new[2], *b_new[2];
    for (int q = 0; q < 2; q++) {
        a_prev[q] = calloc(nb, 4); b_prev[q] = calloc(nb, 4);
        a_new[q] = calloc(nb, 4); b_new[q] = calloc(nb, 4);
    }
    int32_t tail1[6], tail2[6];

    /* Step 0 -- demultiplex R(x_i) into R(b_i), R(b_i)', R(b_i)'',
     * clamp to +-C, split the tails, override the known filler bits. */
    for (int k = 0; k < K; k++) {
        Ls[k] = clamp_in(d0[k]); Lp1[k] = clamp_in(d1[k]); Lp2[k] = clamp_in(d2[k]);
        if (k < F) { Ls[k] = -CLAMP_IN; Lp1[k] = -CLAMP_IN; }
    }
    int32_t t[12] = {d0[K], d1[K], d2[K], d0[K + 1], d1[K + 1], d2[K + 1],
                     d0[K + 2], d1[K + 2], d2[K + 2], d0[K + 3], d1[K + 3], d2[K + 3]};
    for (int m = 0; m < 6; m++) { tail1[m] = clamp_in(t[m]); tail2[m] = clamp_in(t[6 + m]); }
    for (int i = 0; i < K; i++) Pi[i] = oracle_qpp_index(K, i);
    for (int i = 0; i < K; i++) Ls2[i] = Ls[Pi[i]];

    int t_used = 0, pass = 0;
    int64_t mi_prev = 0;
    for (int it = 1; it <= max_iters; it++) {
        t_used = it;
        /* DEC1: R(b_i), R(b_i)' and the a-priori La1 -> extrinsic Le1 */
        viol += oracle_siso_v(Ls, Lp1, La1, tail1, K, W, a_prev[0], b_prev[0], a_new[0], b_new[0], Le1, ops, variant);
        if (variant == ORACLE_VAR_SCALED)     /* extrinsic handed on = floor(3 Le / 4) (R28) */
            for (int k = 0; k < K; k++) Le1[k] = scale34(Le1[k]);
        /* DEC2: interleaved R(b_i), R(b_i)'' and La2 = interleaved Le1 */
        for (int i = 0; i < K; i++) La2[i] = Le1[Pi[i]];
        viol += oracle_siso_v(Ls2, Lp2, La2, tail2, K, W, a_prev[1], b_prev[1], a_new[1], b_new[1], Le2, ops,
                              variant);
        if (variant == ORACLE_VAR_SCALED)
            for (int i = 0; i < K; i++) Le2[i] = scale34(Le2[i]);
        /* de-interleave back to DEC1 */
        for (int i = 0; i < K; i++) La1n[Pi[i]] = Le2[i];
        for (int q = 0; q < 2; q++) oracle_nii_update(M, a_new[q], b_new[q], a_prev[q], b_prev[q]);
        /* hard decision on L_APP = Ls + Le1 + La1_next; tie -> 1 (R16) */
        int64_t mi = 0;                       /* average-MI statistic of the L_APP (R29) */
        for (int n = 0; n < K; n++) {
            int32_t lapp = Ls[n] + Le1[n] + La1n[n];
            if (lapp < -32768 || lapp > 32767) viol++;
            bits[n] = (uint8_t)(n < F ? 0 : (lapp >= 0 ? 1 : 0));
            if (n >= F) mi += oracle_mi_table(lapp < 0 ? -lapp : lapp);
        }
        pass = (crc_kind != ORACLE_CRC_NONE) && oracle_crc24(crc_kind, bits, K) == 0;
        if (early_term == ORACLE_ET_CRC && pass) break;     /* stopping rule (R3) */
        /* the paper's rule: stop once the average mutual information of
         * the LLRs has converged, |S_t - S_{t-1}| <= (K - F) * eps, from iteration 2 on */
        if (early_term == ORACLE_ET_MI && it >= 2 && llabs(mi - mi_prev) <= (int64_t)(K - F) * ORACLE_MI_EPS) break;
        mi_prev = mi;
        memcpy(La1, La1n, 4 * nK);
    }
    *crc_ok = (uint8_t)pass;
    *iters_used = (uint8_t)t_used;
    if (ext)
        for (int n = 0; n < K; n++) ext[n] = (int16_t)La1n[n];

    free(Ls); free(Lp1); free(Lp2); free(La1); free(Le1); free(Ls2);
    free(La2); free(Le2); free(La1n); free(Pi);
    for (int q = 0; q < 2; q++) { free(a_prev[q]); free(b_prev[q]); free(a_new[q]); free(b_new[q]); }
    return viol;
}

/* ---------------------------------------------------------------- batch (CPU baseline) */
typedef struct {
    int n_cb; const int32_t *K, *F, *crc; const int64_t *lo, *bo;
    const int16_t *d0, *d1, *d2; int I, et, variant;
    uint8_t *bits, *ok, *it; int16_t *ext;
    atomic_int next; atomic_llong viol; atomic_ullong ops;
} batch_t;

static void *batch_worker(void *p) {
    batch_t *b = (batch_t *)p;
    uint64_t ops = 0; int64_t viol = 0;
    for (;;) {
        int i = atomic_fetch_add(&b->next, 1);
        if (i >= b->n_cb) break;
        int64_t lo = b->lo[i], bo = b->bo[i];
        int64_t v = oracle_decode_cb_v(b->d0 + lo, b->d1 + lo, b->d2 + lo, b->K[i], b->F[i], b->crc[i],
                                       b->I, b->et, 32, b->variant, b->bits + bo, b->ok + i, b->it + i,
                                     b->ext ? b->ext + bo : NULL, &ops);
        viol += v < 0 ? 1 : v;
    }
    atomic_fetch_add(&b->viol, viol);
    atomic_fetch_add(&b->ops, ops);
    return NULL;
}

int64_t oracle_decode_batch(int n_cb, const int32_t *K, const int32_t *F, const int32_t *crc_kind,
                            const int64_t *llr_off, const int64_t *bit_off,
                            const int16_t *d0, const int16_t *d1, const int16_t *d2,
                            int max_iters, int early_term, int nthreads,
                            uint8_t *bits, uint8_t *crc_ok, uint8_t *iters_used,
                            int16_t *ext, uint64_t *ops) {
    return oracle_decode_batch_v(n_cb, K, F, crc_kind, llr_off, bit_off, d0, d1, d2, max_iters, early_term,
                                 ORACLE_VAR_MAXLOG, nthreads, bits, crc_ok, iters_used, ext, ops);
}

int64_t oracle_decode_batch_v(int n_cb, const int32_t *K, const int32_t *F, const int32_t *crc_kind,
                              const int64_t *llr_off, const int64_t *bit_off,
                              const int16_t *d0, const int16_t *d1, const int16_t *d2,
                              int max_iters, int early_term, int variant, int nthreads,
                              uint8_t *bits, uint8_t *crc_ok, uint8_t *iters_used,
                              int16_t *ext, uint64_t *ops) {
    batch_t b;
    b.n_cb = n_cb; b.K = K; b.F = F; b.crc = crc_kind; b.lo = llr_off; b.bo = bit_off;
    b.d0 = d0; b.d1 = d1; b.d2 = d2; b.I = max_iters; b.et = early_term; b.variant = variant;
    b.bits = bits; b.ok = crc_ok; b.it = iters_used; b.ext = ext;
    atomic_init(&b.next, 0); atomic_init(&b.viol, 0); atomic_init(&b.ops, 0);
    if (nthreads < 1) nthreads = 1;
    pthread_t *th = malloc(sizeof(pthread_t) * (size_t)nthreads);
    for (int i = 0; i < nthreads; i++) pthread_create(&th[i], NULL, batch_worker, &b);
    for (int i = 0; i < nthreads; i++) pthread_join(th[i], NULL);
    free(th);
    if (ops) *ops += atomic_load(&b.ops);
    return atomic_load(&b.viol);
}

/* ---------------------------------------------------------------- rate matching (row f4)
 * TS 36.212 5.1.4.1 for turbo-coded channels (R30): the received data
 * R(x_i) the paper de-multiplexes are the E rate-matched soft
 * values of a CB.  Sub-block interleaver with 32 columns and the inter-column
 * permutation P; bit collection w = v0 | interlace(v1, v2); bit selection from
 * k0 = R (2 ceil(Ncb / 8R) rv + 2) skipping <NULL>, wrapping modulo Ncb = 3 Kpi
 * (full circular buffer).  De-matching adds every received value to the soft
 * buffer position it was read from (repetition accumulates, punctured positions
 * stay 0) and, for HARQ, onto the previous buffer content, saturating once. */
static const int RM_P[32] = {0, 16, 8, 24, 4, 20, 12, 28, 2, 18, 10, 26, 6, 22, 14, 30,
                             1, 17, 9, 25, 5, 21, 13, 29, 3, 19, 11, 27, 7, 23, 15, 31};

int oracle_rm_perm(int c) { return (c >= 0 && c < 32) ? RM_P[c] : -1; }

int oracle_rm_params(int K, int rv, int *R, int *ND, int *Kpi, int *k0) {
    if (k_row(K) < 0 || rv < 0 || rv > 3) return -1;
    const int D = K + 4, r = (D + 31) / 32, kpi = 32 * r, ncb = 3 * kpi;
    *R = r; *ND = kpi - D; *Kpi = kpi;
    *k0 = r * (2 * ((ncb + 8 * r - 1) / (8 * r)) * rv + 2);
    return 0;
}

/* w position p -> d index of its stream (*s), or -1 for <NULL> */
static int rm_wpos(int K, int p, int *s) {
    const int D = K + 4, R = (D + 31) / 32, kpi = 32 * R, ND = kpi - D;
    int y;
    if (p < kpi) {                                  /* v0: column-wise read of the permuted matrix */
        *s = 0;
        y = (p % R) * 32 + RM_P[p / R];
    } else {
        const int q = p - kpi, k = q / 2;
        if ((q & 1) == 0) { *s = 1; y = (k % R) * 32 + RM_P[k / R]; }
        else { *s = 2; y = (RM_P[k / R] + 32 * (k % R) + 1) % kpi; }
    }
    return y < ND ? -1 : y - ND;
}

int oracle_rate_match(const uint8_t *d0, const uint8_t *d1, const uint8_t *d2, int K, int E, int rv, uint8_t *e) {
    int R, ND, kpi, k0;
    if (E < 1 || oracle_rm_params(K, rv, &R, &ND, &kpi, &k0)) return -1;
    const uint8_t *d[3] = {d0, d1, d2};
    const int ncb = 3 * kpi;
    for (int k = 0, j = 0; k < E; j++) {
        int s;
        const int n = rm_wpos(K, (k0 + j) % ncb, &s);
        if (n >= 0) e[k++] = d[s][n];
    }
    return 0;
}

int oracle_rate_dematch(const int16_t *e, int K, int E, int rv, int combine, int16_t *h0, int16_t *h1,
                        int16_t *h2) {
    int R, ND, kpi, k0;
    if (E < 1 || oracle_rm_params(K, rv, &R, &ND, &kpi, &k0)) return -1;
    const int D = K + 4, ncb = 3 * kpi;
    int32_t *acc = (int32_t *)calloc(3 * (size_t)D, sizeof(int32_t));
    for (int k = 0, j = 0; k < E; j++) {
        int s;
        const int n = rm_wpos(K, (k0 + j) % ncb, &s);
        if (n >= 0) acc[(size_t)s * D + n] += e[k++];
    }
    int16_t *h[3] = {h0, h1, h2};
    for (int s = 0; s < 3; s++)
        for (int n = 0; n < D; n++) {
            int32_t v = acc[(size_t)s * D + n] + (combine ? h[s][n] : 0);
            h[s][n] = (int16_t)(v < -32768 ? -32768 : (v > 32767 ? 32767 : v));
        }
    free(acc);
    return 0;
}
