/* crn_decode.cu -- the hot path of arxiv 1905.01141's uplink channel decoding
 * as one persistent sm_100a kernel: batched LTE turbo
 * decoding, int16 max-log-MAP on the 8-state RSC trellis, QPP interleaver,
 * M_K parallel windows with next-iteration initialisation (NII), fixed or CRC
 * early-terminated iterations, hard decision + CRC (rows a2..a9).
 *
 * Decomposition.  A CTA task holds n_pairs pairs of equal-K code blocks; the
 * two CBs of a pair live in the low / high int16 half of every 32-bit register
 * and word (pair-SIMD: VIADD.16x2, VIMNMX(3).S16x2, VIADDMNMX.S16x2), so the
 * 8-state butterfly is a compile-time register rename.  Window t = p*M + j is
 * window j of pair p.  On the W = 32 path (every K >= 1056) a window is split
 * between a head thread (steps 0..15) and a tail thread (steps 16..31) of a
 * 384-thread CTA (one per SM): 12 warps, three per SM sub-partition.
 *
 * On-chip residency (W = 32): a CB pair never leaves the SM while it is
 * decoded.  Registers hold each thread's static Ls - Lp sums; shared memory
 * holds the parity planes, both extrinsic buffers (Le1 natural, Le2
 * interleaved), the NII boundary states and the per-half-iteration branch-
 * metric chunks; tensor memory (TMEM, otherwise idle in this kernel) holds the
 * alpha/beta metrics each thread stores in its first sweep and reads back in
 * its second.  Element (step i, window t) of a per-step array is at i*192 + t:
 * a warp's access at one step is contiguous, and because W divides K the QPP
 * is contention-free per window, so every interleaved gather at step i hits
 * one row.
 *
 * Exactness.  Every intermediate provably fits int16 (DESIGN.md "int16
 * safety", checked by the oracle on adversarial inputs), so wrapping int16x2
 * arithmetic equals the oracle's int32 arithmetic bit for bit.  State metrics
 * are kept biased by -1 (a~ = a - 1): the normaliser's negation becomes one
 * NOT, ~(m - 1) = -m, and every comparison is unchanged.
 */
#include <cuda_runtime.h>
#include <stdint.h>

#include <type_traits>

#include "crn_internal.h"

typedef uint32_t u32;
typedef uint64_t u64;

namespace {

constexpr int NS = CRN_NSTATE;
constexpr int WMAX = CRN_CTA_THREADS;           /* max windows per task (192) */
constexpr int BLOCK = 2 * CRN_CTA_THREADS;      /* threads per CTA (384): a head and a tail thread per window */
constexpr int SUMK = CRN_TASK_SUMK;
constexpr int TS = WMAX;                        /* fast-path row stride (words) */
constexpr int HW = 16;                          /* trellis steps per half-window thread (W = 32) */
constexpr int MAXP = CRN_MAX_PAIRS;             /* max pairs per task */
constexpr u32 M1 = 0xFFFFFFFFu;                 /* (-1, -1): biased 0 */
constexpr u32 FLOORB = 0xDFFFDFFFu;             /* (-8193, -8193): biased state-metric floor */
constexpr u32 CLIP_HI = 0x10001000u;            /* ( 4096,  4096): channel / extrinsic clamp */
constexpr u32 CLIP_LO = 0xF000F000u;            /* (-4096, -4096) */
constexpr u32 NEG4097 = 0xEFFFEFFFu, ONE2 = 0x00010001u;

constexpr size_t WS_HEAD = 256;                 /* task counter */

/* fast-path shared-memory layout (u32 words).  Y = Le1 (natural order), Z =
 * Le2 (interleaved order), both window-major [step][window]; NII boundary
 * states [c][alpha/beta][s][window]; X = the mid-window hand-over between the
 * head and tail thread of a window [alpha/beta][s][window] (reused for the
 * hard-decision half-words); LP = the static parity LLRs Lp1 (natural) and
 * Lp2 (interleaved order), window-major; CH = per-thread branch-metric chunk
 * [step][thread] of uint2 (Lu+Lp, Lu-Lp); tails [pair][12]. */
constexpr int S_Y = 0, S_Z = SUMK, S_NII = 2 * SUMK;
constexpr int S_NII_WORDS = 2 * 2 * NS * WMAX;
constexpr int S_X = S_NII + S_NII_WORDS;
constexpr int S_LP = S_X + 2 * NS * WMAX;       /* [c][step][window] */
constexpr int S_CH = S_LP + 2 * SUMK;
constexpr int S_TAIL = S_CH + HW * BLOCK * 2;   /* per pair: beta_K of DEC1 (8 words), of DEC2 (8 words) */
constexpr int S_WORDS = S_TAIL + MAXP * 16;
static_assert(S_CH % 2 == 0, "chunk array must be 8-byte aligned");
static_assert(S_WORDS == CRN_SMEM_WORDS, "split-window sizing (crn_internal.h) must see the same shared memory");
/* the window-CRC nibble tables (both CRC kinds) after both paths' layouts: the
 * Y / Z planes stay at the start of the dynamic region, because the fast path
 * packs two of their shared byte addresses into one register (< 64 KiB each) */
constexpr int S_CRCNIB = S_WORDS;
constexpr int S_OFFS = S_CRCNIB + 2 * CRN_CRC_NIB_WORDS;   /* int64 [4][2 MAXP]: bit_off, ext_off (current, next) */
static_assert(S_OFFS % 2 == 0, "8-byte aligned");
constexpr int SMEM_WORDS = S_OFFS + 4 * 2 * MAXP * 2;
/* The CRC-ET and latency kernels keep the nibble tables with every window-
 * distance table shifted by 4 banks (t1: 132-word stride, t2 / t3: 100): the
 * lanes of a warp look up tables of 8 different distances at once, which with
 * 128 / 96-word strides all start on the same bank (3-4 wavefronts per lookup) */
constexpr int NIBP_T1 = 132, NIBP_T23 = 100, NIBP_O2 = 8 * NIBP_T1, NIBP_O3 = NIBP_O2 + 8 * NIBP_T23;
constexpr int NIBP_KIND = NIBP_O3 + 3 * NIBP_T23;
constexpr int S_OFFS_P = S_CRCNIB + 2 * NIBP_KIND;
static_assert(S_OFFS_P % 2 == 0 && CRN_CRC_NIB_WORDS == 1024 + 768 + 288, "padded nibble-table layout");
constexpr int SMEM_WORDS_P = S_OFFS_P + 4 * 2 * MAXP * 2;
static_assert(SMEM_WORDS_P * 4 + 9728 <= 232448, "padded layout over the sm_100 opt-in limit");
constexpr int YZ_END_BYTES = 4 * (S_Z + SUMK);     /* + static shared memory: must stay < 64 KiB */
static_assert(SMEM_WORDS * 4 + 9728 <= 232448, "dynamic + static shared memory over the sm_100 opt-in limit");

/* ---- optional phase profiler (build with -DCRN_PHASE_PROF; never in the product
 * build): lane 0 of warp 0 (a head warp) and of warp 6 (a tail warp) attribute
 * clock64 intervals to the phase that just ended; summed over CTAs. */
enum { P_FETCH, P_STAGE, P_CHUNK, P_PH1, P_BAR1, P_PH2, P_BAR2, P_HD, P_SLD, P_SB1, P_SG, P_HL, P_HB1, P_HC, P_HB2, P_HDEC,
       P_FB, P_N };
#ifdef CRN_PHASE_PROF
__device__ unsigned long long g_prof[2 * P_N];
__shared__ unsigned long long s_pacc[2][P_N];
__shared__ long long s_plast[2];
__device__ __forceinline__ void prof_mark(int ph) {
    const int w = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0 && (w == 0 || w == 6)) {
        const int k = w ? 1 : 0;
        const long long t = clock64();
        s_pacc[k][ph] += (unsigned long long)(t - s_plast[k]);
        s_plast[k] = t;
    }
}
__device__ __forceinline__ void prof_init() {
    const int w = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0 && (w == 0 || w == 6)) {
        const int k = w ? 1 : 0;
        for (int i = 0; i < P_N; i++) s_pacc[k][i] = 0;
        s_plast[k] = clock64();
    }
}
__device__ __forceinline__ void prof_flush() {
    const int w = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0 && (w == 0 || w == 6))
        for (int i = 0; i < P_N; i++) atomicAdd(&g_prof[(w ? 1 : 0) * P_N + i], s_pacc[w ? 1 : 0][i]);
}
#else
__device__ __forceinline__ void prof_mark(int) {}
#endif
/* ---- optional task trace (build with -DCRN_TASK_TRACE; never in the product build):
 * per task its start / end %globaltimer (ns), SM and group, tools/task_trace.py */
#ifdef CRN_TASK_TRACE
constexpr int TRACE_MAX = 1 << 16;
__device__ unsigned long long g_trace[4 * TRACE_MAX];
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ void trace_task(int task, int which, int g) {
    if (task < TRACE_MAX) {
        g_trace[4 * task + which] = gtimer();
        if (which == 0) {
            unsigned sm;
            asm volatile("mov.u32 %0, %smid;" : "=r"(sm));
            g_trace[4 * task + 2] = sm;
            g_trace[4 * task + 3] = (unsigned long long)g;
        }
    }
}
#else
__device__ __forceinline__ void trace_task(int, int, int) {}
#endif
#ifndef CRN_PHASE_PROF
__device__ __forceinline__ void prof_init() {}
__device__ __forceinline__ void prof_flush() {}
#endif

/* ---- RSC trellis, S = 4 r1 + 2 r2 + r3 (R1), evaluated at compile time */
__host__ __device__ constexpr int nxt(int S, int u) { return (((u ^ (S >> 1) ^ S) & 1) << 2) | (S >> 1); }
__host__ __device__ constexpr int par(int S, int u) { return (u ^ (S >> 1) ^ (S >> 2)) & 1; } /* z = u^r1^r2 */

__device__ __forceinline__ u32 vadd(u32 a, u32 b) { return __vadd2(a, b); }
__device__ __forceinline__ u32 vaddmax(u32 a, u32 b, u32 c) { return __viaddmax_s16x2(a, b, c); } /* max(a+b, c) */

/* Log-MAP's max*(a, b) = max(a, b) + LUT[min(|a - b| >> 2, 7)] per int16 half
 * (R32).  |a - b| <= 24576 on every selection (int16 safety), so the
 * difference is exact; the bucket index of each half goes into a PRMT selector
 * that picks the LUT byte (bytes 1 and 3 pick LUT[6] = 0), giving the
 * int16x2 correction in one instruction. */
__device__ __forceinline__ u32 maxs2(u32 a, u32 b, u32 lut_lo, u32 lut_hi) {
    const u32 m = __vmaxs2(a, b), d = __vsub2(m, __vmins2(a, b));
    /* t = min(d, 31) >> 2 per half: bucket_lo in bits 2:0, bucket_hi in 18:16 (and
     * d_hi's low two bits in 15:14); sel = t | t >> 8 | 0x6060 puts the buckets in
     * selector nibbles 0 and 2, and nibbles 1 and 3 select byte 6 (= 0) -- the stray
     * d_hi bits can only set those nibbles' bit 3 (sign-replicate a 0 byte: 0) */
    const u32 t = __vmins2(d, 0x001F001Fu) >> 2;
    return __vadd2(m, __byte_perm(lut_lo, lut_hi, t | (t >> 8) | 0x6060u));
}

struct Lut {                                    /* the LUT's two PRMT source words */
    u32 lo, hi;
};
__constant__ u32 c_logmap[2];                   /* crn_decode_set_logmap */

/* gamma(u, z) = u*Lu + z*Lp; the (0,0) branch is never formed */
__device__ __forceinline__ u32 gsel(int u, int z, u32 Lu, u32 Lp, u32 Lup) { return u ? (z ? Lup : Lu) : Lp; }

/* N(v)(s) = max(v(s) - max_s' v(s'), -8192) on biased values */
__device__ __forceinline__ void norm8(u32 v[NS]) {
    u32 m0 = __vimax3_s16x2(v[0], v[1], v[2]);
    u32 m1 = __vimax3_s16x2(v[3], v[4], v[5]);
    u32 m = __vimax3_s16x2(v[6], v[7], m0);
    m = __vmaxs2(m, m1);
    const u32 nm = ~m;                          /* ~(m - 1) = -m */
#pragma unroll
    for (int s = 0; s < NS; s++) v[s] = vaddmax(v[s], nm, FLOORB);
}

/* ---- Branch-difference form of the recursions (fast path).  The two branches
 * into (alpha) or out of (beta) a state carry complementary (u, z) labels
 * (R1): type A = {(0,0), (1,1)}, type B = {(0,1), (1,0)}.  A type-A
 * candidate pair is max(m0, m1 + Lup); a type-B pair is
 * max(m0 + Lp, m1 + Lu) = Lp + max(m0, m1 + D), D = Lu - Lp, so one fused
 * VIADDMNMX forms every state and the common "+ Lp" of the type-B states is
 * folded into the maximum and into the normaliser's offset.  Exact: every
 * value below is the oracle's integer, and all fit int16. */
__host__ __device__ constexpr int pred_u(int S, int Sp) { return nxt(S, 0) == Sp ? 0 : 1; }
/* alpha: type of state S' (1 = B) and which predecessor carries the unmodified branch */
__host__ __device__ constexpr bool a_isB(int Sp) {
    return !((pred_u(2 * (Sp & 3), Sp) == 0 && par(2 * (Sp & 3), 0) == 0) ||
             (pred_u(2 * (Sp & 3) + 1, Sp) == 0 && par(2 * (Sp & 3) + 1, 0) == 0));
}
/* the predecessor whose branch is (0,0) [type A] or (0,1) [type B] */
__host__ __device__ constexpr int a_base(int Sp) {
    return pred_u(2 * (Sp & 3), Sp) == 0 ? 2 * (Sp & 3) : 2 * (Sp & 3) + 1;
}
__host__ __device__ constexpr bool b_isB(int S) { return par(S, 0) == 1; }
/* group member lists (compile-time): the k-th type-A / type-B state */
__host__ __device__ constexpr int nth_state(bool alpha, bool B, int k) {
    int c = 0;
    for (int s = 0; s < NS; s++)
        if ((alpha ? a_isB(s) : b_isB(s)) == B) {
            if (c == k) return s;
            c++;
        }
    return -1;
}
static_assert(!a_isB(0) && a_isB(1) && a_isB(2) && !a_isB(3) && !a_isB(4) && a_isB(5) && a_isB(6) && !a_isB(7),
              "alpha state types (SURVEY 8c.1: {0,3,4,7} receive (0,0)/(1,1))");
static_assert(nth_state(true, true, 3) >= 0 && nth_state(false, true, 3) >= 0 && nth_state(false, false, 3) >= 0,
              "four states of each type");

/* v[] holds type-A values and type-B differences w (v_B = w + Lp).  Writes
 * N(v) (biased) into out[]: m = max(max_A v, max_B w + Lp); out = max(v - m, F). */
template <bool ALPHA>
__device__ __forceinline__ void norm_ab(const u32 v[NS], u32 Lp, u32 out[NS]) {
    constexpr int a0 = nth_state(ALPHA, false, 0), a1 = nth_state(ALPHA, false, 1), a2 = nth_state(ALPHA, false, 2),
                  a3 = nth_state(ALPHA, false, 3);
    constexpr int b0 = nth_state(ALPHA, true, 0), b1 = nth_state(ALPHA, true, 1), b2 = nth_state(ALPHA, true, 2),
                  b3 = nth_state(ALPHA, true, 3);
    const u32 tA = __vimax3_s16x2(v[a0], v[a1], v[a2]);
    const u32 tB = __vmaxs2(__vimax3_s16x2(v[b0], v[b1], v[b2]), v[b3]);
    const u32 m = __vmaxs2(vaddmax(tB, Lp, tA), v[a3]);
    const u32 nm = ~m;                          /* ~(m - 1) = -m (biased values) */
    const u32 lpm = vadd(Lp, nm);               /* Lp - m */
#pragma unroll
    for (int s = 0; s < NS; s++) out[s] = vaddmax(v[s], (ALPHA ? a_isB(s) : b_isB(s)) ? lpm : nm, FLOORB);
}

/* alpha_{k+1} = N(max over predecessors of alpha_k + gamma_k)  (row a6); with
 * LOG the selection is max* (shift-invariant, so the type-B "+ Lp" still folds
 * into the normaliser exactly) */
template <bool LOG = false>
__device__ __forceinline__ void alpha_step_d(u32 a[NS], u32 Lp, u32 Lup, u32 D, Lut lut = Lut{0, 0}) {
    u32 v[NS];
#pragma unroll
    for (int Sp = 0; Sp < NS; Sp++) {
        const int x = a_base(Sp), y = x ^ 1;    /* y carries (1,1) [A] or (1,0) [B] */
        v[Sp] = LOG ? maxs2(a[x], vadd(a[y], a_isB(Sp) ? D : Lup), lut.lo, lut.hi)
                    : vaddmax(a[y], a_isB(Sp) ? D : Lup, a[x]);
    }
    norm_ab<true>(v, Lp, a);
}

/* beta_k = N(max over successors of beta_{k+1} + gamma_k)  (row a5) */
template <bool LOG = false>
__device__ __forceinline__ void beta_step_d(u32 b[NS], u32 Lp, u32 Lup, u32 D, Lut lut = Lut{0, 0}) {
    u32 v[NS];
#pragma unroll
    for (int S = 0; S < NS; S++)
        v[S] = LOG ? maxs2(b[nxt(S, 0)], vadd(b[nxt(S, 1)], b_isB(S) ? D : Lup), lut.lo, lut.hi)
                   : vaddmax(b[nxt(S, 1)], b_isB(S) ? D : Lup, b[nxt(S, 0)]);
    norm_ab<false>(v, Lp, b);
}

/* Row a7: Lambda_u = max over the 8 transitions with input u of alpha_k(S) +
 * z Lp + beta_{k+1}(S'), grouped by z; Le = clamp(L1 - L0, +-4096) computed as
 * min(max(L1 + ~L0, -4097) + 1, 4096).  The -1 biases of alpha and beta cancel. */
template <bool LOG = false>
__device__ __forceinline__ u32 lambda_le(const u32 a[NS], const u32 bn[NS], u32 Lp, Lut lut = Lut{0, 0}) {
    u32 lam[2];
    if constexpr (LOG) {                        /* max* folded over S = 0..7 in order (R32) */
#pragma unroll
        for (int u = 0; u < 2; u++) {
#pragma unroll
            for (int S = 0; S < NS; S++) {
                u32 t = vadd(a[S], bn[nxt(S, u)]);
                if (par(S, u)) t = vadd(t, Lp);
                lam[u] = S ? maxs2(lam[u], t, lut.lo, lut.hi) : t;
            }
        }
    } else {
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
    }
    return __viaddmin_s16x2(vaddmax(lam[1], ~lam[0], NEG4097), ONE2, CLIP_HI);
}

/* Row f2 variant (R28): the extrinsic handed on is floor(3 Le / 4),
 * per int16 half: 3 Le fits int16 (|Le| <= 4096), then an arithmetic shift by 2
 * (logical shift of the word, each half's low 14 bits kept, its sign copied
 * into its top two bits). */
__device__ __forceinline__ u32 scale34(u32 x) {
    const u32 t = vadd(vadd(x, x), x);
    const u32 s = t & 0x80008000u;
    return ((t >> 2) & 0x3FFF3FFFu) | s | (s >> 1);
}

template <int VAR>
__device__ __forceinline__ u32 ext_out_map(u32 le) { return VAR == CRN_VARIANT_SCALED ? scale34(le) : le; }

/* beta_K from the tail: beta_{K+3} = (0, -F x7), three forced steps (R11) */
__device__ __forceinline__ void tail_beta(const u32 *tail, u32 b[NS]) {
    b[0] = M1;
#pragma unroll
    for (int s = 1; s < NS; s++) b[s] = FLOORB;
#pragma unroll
    for (int tau = 2; tau >= 0; tau--) {
        const u32 x = tail[2 * tau], z = tail[2 * tau + 1], xz = vadd(x, z);
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
    const u32 v = (u32)(uint16_t)lo | ((u32)(uint16_t)hi << 16);
    return __vmins2(__vmaxs2(v, CLIP_LO), CLIP_HI);
}

/* fast path (shared memory, single-buffered): [c][alpha(0)/beta(1)][s][WMAX] */
__device__ __forceinline__ int nii1_ix(int c, int ab, int s, int t) { return ((c * 2 + ab) * NS + s) * WMAX + t; }

/* Q16 MI contribution of the two L_APP halves of a word (fillers excluded by the
 * caller's masks): table[min(|L|, 255)] per half (R29). */
__device__ __forceinline__ int mi_pair(const int *tab, u32 lapp, bool use_lo, bool use_hi) {
    const int lo = (int)(int16_t)(lapp & 0xFFFFu), hi = (int)(int16_t)(lapp >> 16);
    const int alo = min(lo < 0 ? -lo : lo, 255), ahi = min(hi < 0 ? -hi : hi, 255);
    return (use_lo ? tab[alo] : 0) + (use_hi ? tab[ahi] : 0);
}

struct TaskSh {
    const u32 *crcnib;          /* the window-CRC nibble tables (CRN_CRC_NIB_WORDS per CRC kind) */
    int *cb, *F, *kind;
    int *mi, *mip;              /* per CB: average-MI statistic of this / the previous iteration (R29) */
    const int *mitab;           /* Q16 MI of |L_APP| = 0..255 (the tables' mi_tab, staged in smem) */
    uint8_t *done, *fin;
    u32 *crc;
    int *left;
    const int64_t *bo, *eo;     /* per CB: bit_off / ext_off of its descriptor (claimed with the task) */
};

/* Row a9 bookkeeping after the CRC reduction: completion / early termination
 * per CB, CRC flag and iteration count.  Returns after the barrier. */
/* TB purge state (crn_plan_set_purge): per CB of the task its TB id, per TB a
 * "lost" flag in global memory. */
struct Purge {
    const int *tb;
    uint8_t *dead;
};

template <bool PURGE>
__device__ __forceinline__ void decide(TaskSh sh, int NP, int it, int max_iters, int et, int K, uint8_t *crc_ok,
                                       uint8_t *iters_used, Purge pg) {
    for (int e = threadIdx.x; e < 2 * NP; e += BLOCK) {
        if (sh.done[e]) continue;
        const bool pass = sh.kind[e] != CRN_CRC_NONE && sh.crc[e] == 0;
        /* stopping rules: CRC (R3) or the paper's MI convergence (R29) */
        const int dmi = sh.mi[e] - sh.mip[e];
        const bool mi_conv = et == CRN_ET_MI && it >= 2 && (dmi < 0 ? -dmi : dmi) <= (K - sh.F[e]) * CRN_MI_EPS;
        sh.mip[e] = sh.mi[e];
        if ((et == CRN_ET_CRC && pass) || mi_conv || it == max_iters) {
            sh.fin[e] = 1;
            sh.done[e] = 1;
            crc_ok[sh.cb[e]] = pass;
            if (PURGE && !pass && pg.tb[e] >= 0)              /* decoding failure: its TB is lost */
                *(volatile uint8_t *)&pg.dead[pg.tb[e]] = 1;
            if (iters_used) iters_used[sh.cb[e]] = (uint8_t)it;
        }
    }
    __syncthreads();
}

/* Returns the number of CBs still running (one counting barrier: it also
 * orders every use of this iteration's flags before they are cleared) and
 * clears the per-iteration flags; the next use of the flags is separated from
 * the clear by the next half-iteration's barriers. */
__device__ __forceinline__ int finish_iteration(TaskSh sh, int NP) {
    const int e = threadIdx.x;                  /* 2 NP <= 2 MAXP <= BLOCK */
    const int left = __syncthreads_count(e < 2 * NP && !sh.done[e]);
    if (e < 2 * NP) { sh.fin[e] = 0; sh.crc[e] = 0; sh.mi[e] = 0; }
    return left;
}
static_assert(2 * MAXP <= BLOCK, "one thread per CB lane in finish_iteration");

/* ---- tensor memory (tcgen05) helpers.  A warp may touch only the TMEM lanes
 * of its quadrant (warp % 4); warps 4-7 use columns 128-255, warps 8-11 256-383. */
__device__ __forceinline__ u32 smem_addr(const void *p) { return (u32)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void tm_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

/* ---- thread groups (W = 32 path).  G = 1: the whole CTA runs one task of up to
 * 192 windows (tasks with sum K <= 6144).  G = 3: the CTA runs three independent
 * tasks of up to 64 windows (sum K <= 2048), one per group of four warps (two
 * head, two tail warps, one per SM sub-partition), each with its own named
 * barrier.  Group g owns window columns [64 g, 64 g + 64), pair slots
 * [32 g, 32 g + 32) and TMEM column block g, so the shared-memory layout and the
 * TMEM addressing are the G = 1 ones. */
constexpr int G3 = 3;
constexpr int GB3 = BLOCK / G3;                 /* threads per group (128) */
constexpr int GWIN3 = WMAX / G3;                /* windows per group (64) */
constexpr int GPB3 = MAXP / G3;                 /* pair slots per group (32) */
static_assert(G3 == CRN_GROUPS && GWIN3 == CRN_GRP_WIN && GPB3 == CRN_GRP_PAIRS && 32 * CRN_GRP_WIN == CRN_GRP_SUMK,
              "group geometry (crn_internal.h)");

template <int G>
__device__ __forceinline__ void gsync(int g) {
    if constexpr (G == 1) __syncthreads();
    else asm volatile("bar.sync %0, %1;" ::"r"(1 + g), "n"(BLOCK / G) : "memory");
}
/* barrier that also counts the group's threads with pred != 0 */
template <int G>
__device__ __forceinline__ int gsync_count(int g, int pred) {
    if constexpr (G == 1) return __syncthreads_count(pred);
    int r;
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.s32 q, %1, 0;\n\tbar.red.popc.u32 %0, %2, %3, q;\n\t}"
                 : "=r"(r) : "r"(pred), "r"(1 + g), "n"(BLOCK / G) : "memory");
    return r;
}

/* ======================================================================
 * Fast path: W = 32 (every K that is a multiple of 32: all K >= 1056 and 15
 * smaller sizes).  Window t of the task is split between two threads: the
 * head thread (tid = t, warps 0-5) owns steps 0..15, the tail thread (tid =
 * 192 + t, warps 6-11) steps 16..31, so a 192-window CB pair runs on 12 warps,
 * three per SM sub-partition.  Per half-iteration:
 *   phase 0  each thread forms its 16 branch-metric triples (Lp, Lu+Lp, Lu-Lp)
 *            from register-resident static sums and the gathered a-priori LLR;
 *   phase 1  head: alpha forward over steps 0..15, tail: beta backward over
 *            31..16, each storing its metrics in its own TMEM lane;
 *   hand-over  alpha_16 and beta_16 swap through shared memory (one barrier);
 *   phase 2  head: beta backward over 15..0, tail: alpha forward over 16..31;
 *            each step meets the thread's own stored metric of the other
 *            sweep and emits one extrinsic (rows a5-a7);
 *   NII      head: beta_{jW} -> window j-1, tail: alpha_{(j+1)W} -> window
 *            j+1, for the next iteration (row a8).
 * ====================================================================== */
struct SCtx {
    u32 *sm;        /* shared-memory base (fast layout) */
    int g;          /* thread group (G = 3: four warps running their own task; G = 1: the whole CTA) */
    u32 ta;         /* this thread's TMEM metric slots: lane quadrant + 128-column block */
    u32 ts;         /* this thread's TMEM statics: Ls-Lp1 (16 columns), Ls[Pi]-Lp2 (16) */
    int tid, t, p, j, M, pM, k0;
    u32 lut_lo, lut_hi;     /* Log-MAP LUT words (tab.lm_lo / lm_hi) */
    bool wact;              /* the warp holds at least one of the task's windows (warp-uniform) */
};

__device__ __forceinline__ void tm_store8(u32 ta, const u32 v[NS]) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};"
                 :: "r"(ta), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
                 : "memory");
}

__device__ __forceinline__ void tm_load8(u32 ta, u32 v[NS]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                 : "r"(ta)
                 : "memory");
}

/* Waits for outstanding TMEM loads; v is an in/out operand so no use of the
 * loaded registers can be scheduled before the wait. */
__device__ __forceinline__ void tm_wait_ld8(u32 v[NS]) {
    asm volatile("tcgen05.wait::ld.sync.aligned;"
                 : "+r"(v[0]), "+r"(v[1]), "+r"(v[2]), "+r"(v[3]), "+r"(v[4]), "+r"(v[5]), "+r"(v[6]), "+r"(v[7])
                 :: "memory");
}

__device__ __forceinline__ void tm_store16(u32 ta, const u32 v[HW]) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};"
                 :: "r"(ta), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]),
                    "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
                 : "memory");
}

/* Loads 16 columns and waits for them (used outside the recursion loops). */
__device__ __forceinline__ void tm_load16_wait(u32 ta, u32 v[HW]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n\t"
                 "tcgen05.wait::ld.sync.aligned;"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                   "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
                 : "r"(ta)
                 : "memory");
}

/* Loads 4 columns and waits for them (the rolled phase 1's statics, a block at a time). */
__device__ __forceinline__ void tm_load4_wait(u32 ta, u32 v[4]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];\n\t"
                 "tcgen05.wait::ld.sync.aligned;"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3])
                 : "r"(ta)
                 : "memory");
}

/* LLR element idx of a stream: int16, or with sh8 >= 0 (int8 ingest, row f4,
 * crn_plan_set_llr_format) the int8 value x read as the int16 x * 2^sh8. */
template <bool LLR8>
__device__ __forceinline__ int16_t ld_llr(const int16_t *__restrict__ base, int64_t idx, int sh8) {
    if (!LLR8) return __ldg(base + idx);
    return (int16_t)((int)__ldg(reinterpret_cast<const int8_t *>(base) + idx) << sh8);
}

/* int8 bytes (b0, b1) selected by sel (0x9180: bytes 0, 1; 0xB3A2: bytes 2, 3) ->
 * the int16x2 word (b0 2^sh8, b1 2^sh8): prmt sign-replicates into the high bytes */
__device__ __forceinline__ u32 widen8(u32 x, int sh8, bool hi) {
    u32 r;
    if (hi) asm("prmt.b32 %0, %1, 0, 0xB3A2;" : "=r"(r) : "r"(x));
    else asm("prmt.b32 %0, %1, 0, 0x9180;" : "=r"(r) : "r"(x));
    return ((r & 0xFFFF0000u) << sh8) | ((r << sh8) & 0xFFFFu);
}

/* 16 consecutive LLRs of one stream from element idx: 8-byte (int16) or 4-byte
 * (int8) vector loads when aligned.  Returned as 8 words of (element 2i, 2i+1). */
template <bool LLR8>
__device__ __forceinline__ void load16(const int16_t *__restrict__ base, int64_t idx, int sh8, u32 w[HW / 2]) {
    if (!LLR8) {
        const int16_t *src = base + idx;
        if ((reinterpret_cast<uintptr_t>(src) & 7) == 0) {
            const uint2 *v = reinterpret_cast<const uint2 *>(src);
#pragma unroll
            for (int k = 0; k < HW / 4; k++) {
                const uint2 x = __ldg(v + k);
                w[2 * k] = x.x;
                w[2 * k + 1] = x.y;
            }
        } else {
#pragma unroll
            for (int k = 0; k < HW / 2; k++)
                w[k] = (u32)(uint16_t)__ldg(src + 2 * k) | ((u32)(uint16_t)__ldg(src + 2 * k + 1) << 16);
        }
    } else {
        const int8_t *src = reinterpret_cast<const int8_t *>(base) + idx;
        if ((reinterpret_cast<uintptr_t>(src) & 3) == 0) {
            const u32 *v = reinterpret_cast<const u32 *>(src);
#pragma unroll
            for (int k = 0; k < HW / 4; k++) {
                const u32 x = __ldg(v + k);
                w[2 * k] = widen8(x, sh8, false);
                w[2 * k + 1] = widen8(x, sh8, true);
            }
        } else {
#pragma unroll
            for (int k = 0; k < HW / 2; k++)
                w[k] = (u32)(uint16_t)(int16_t)((int)__ldg(src + 2 * k) << sh8) |
                       ((u32)(uint16_t)(int16_t)((int)__ldg(src + 2 * k + 1) << sh8) << 16);
        }
    }
}

/* Shared load at a 32-bit shared-window byte address */
__device__ __forceinline__ u32 lds_at(u32 a) {
    u32 v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
    return v;
}

/* byte offset of nibble q of x in a 16-word table: 4 * ((x >> 4q) & 15) */
__device__ __forceinline__ u32 nib_off(u32 x, int q) { return q ? (x >> (4 * q - 2)) & 60u : (x << 2) & 60u; }

/* Shared load at the packed gather address of constituent c (c = 0: low 16 bits,
 * c = 1: high 16 bits); the halves are split with IMAD-pipe arithmetic so the
 * ALU pipe, the kernel's bottleneck, is not used. */
__device__ __forceinline__ u32 lds_q(u32 qq, int c) {
    const u32 hi = __umulhi(qq, 0x10000u);
    const u32 a = c ? hi : qq - hi * 0x10000u;
    u32 v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
    return v;
}

/* One half-iteration of constituent c (rows a5-a8).  Le -> Y (c = 0, natural
 * order) or Z (c = 1, interleaved order). */
/* ROLL (the latency kernels, crn_launch_decode): phase 1 runs as a loop over
 * blocks of four steps -- the statics come from TMEM a block at a time and the
 * gather addresses move down a register window -- and the caller runs both
 * constituents through one call site, so a lone warp's per-iteration code fits
 * the instruction caches (a step of the fully unrolled phase 1 costs a lone warp
 * ~120 cycles against ~76 when its code stays cached, tools/ubench/step_lat.cu).
 * The arithmetic, and so every output, is the unrolled path's. */
template <int VAR, int G, bool ROLL = false>
__device__ __forceinline__ void siso_split(const SCtx &f, bool tail_thr, int c, int it, const u32 (&qq)[HW],
                                           bool zero_la) {
    constexpr bool LOGV = VAR == CRN_VARIANT_LOGMAP;
    const Lut lut{f.lut_lo, f.lut_hi};
    uint2 *ch = reinterpret_cast<uint2 *>(f.sm + S_CH) + f.tid;
    const u32 *lp = f.sm + S_LP + c * SUMK + f.k0 * TS + f.t;
    u32 *nii = f.sm + S_NII;
    u32 *X = f.sm + S_X;
    u32 *le = f.sm + (c ? S_Z : S_Y) + f.t;
    /* a warp whose windows are all past the task's last one only keeps the barriers */
    if (f.wact) {
    /* row a4 fused into phase 1: this thread's 16 (Lu+Lp, Lu-Lp) pairs are formed
     * step by step from the TMEM static sums, the parity plane and the a-priori
     * LLRs gathered at its QPP indices, used at once and kept in smem for phase 2 */
    if constexpr (ROLL) {
    const u32 lp_s = smem_addr(lp);
    u32 m[NS], w[HW];
#pragma unroll
    for (int k = 0; k < HW; k++) w[k] = qq[k];
    if (!tail_thr) {
        if (f.j == 0) {
            m[0] = M1;
#pragma unroll
            for (int s = 1; s < NS; s++) m[s] = FLOORB;
        } else if (it == 1) {
#pragma unroll
            for (int s = 0; s < NS; s++) m[s] = M1;
        } else {
#pragma unroll
            for (int s = 0; s < NS; s++) m[s] = nii[nii1_ix(c, 0, s, f.t - 1)];
        }
        /* the block's steps use w[0..3]; the next step's loads are issued one step
         * ahead (the last lookahead reads a valid, unused address) */
        u32 avn = zero_la ? 0u : lds_q(w[0], c), pvn;
        asm volatile("ld.shared.u32 %0, [%1];" : "=r"(pvn) : "r"(lp_s));
#pragma unroll 1
        for (int b = 0; b < HW / 4; b++) {
            u32 s4[4];
            tm_load4_wait(f.ts + c * HW + 4 * b, s4);
#pragma unroll
            for (int t = 0; t < 4; t++) {
                const int s = 4 * b + t;
                const u32 av = avn, pv = pvn;
                avn = zero_la ? 0u : lds_q(w[t + 1], c);
                asm volatile("ld.shared.u32 %0, [%1];" : "=r"(pvn) : "r"(lp_s + 4 * (s + 1) * TS));
                const u32 d = vadd(s4[t], av), x = vadd(vadd(d, pv), pv);
                ch[s * BLOCK] = make_uint2(x, d);
                tm_store8(f.ta + s * 8, m);
                alpha_step_d<LOGV>(m, pv, x, d, lut);
            }
#pragma unroll
            for (int k = 0; k < HW - 4; k++) w[k] = w[k + 4];
        }
#pragma unroll
        for (int s = 0; s < NS; s++) X[s * TS + f.t] = m[s];             /* alpha_16 -> tail thread */
    } else {
        if (f.j == f.M - 1) {
#pragma unroll
            for (int s = 0; s < NS; s++) m[s] = f.sm[S_TAIL + f.p * 16 + c * 8 + s];
        } else if (it == 1) {
#pragma unroll
            for (int s = 0; s < NS; s++) m[s] = M1;
        } else {
#pragma unroll
            for (int s = 0; s < NS; s++) m[s] = nii[nii1_ix(c, 1, s, f.t + 1)];
        }
        /* backward: the block's steps use w[12..15] */
        u32 avn = zero_la ? 0u : lds_q(w[HW - 1], c), pvn;
        asm volatile("ld.shared.u32 %0, [%1];" : "=r"(pvn) : "r"(lp_s + 4 * (HW - 1) * TS));
#pragma unroll 1
        for (int b = HW / 4 - 1; b >= 0; b--) {
            u32 s4[4];
            tm_load4_wait(f.ts + c * HW + 4 * b, s4);
#pragma unroll
            for (int t = 3; t >= 0; t--) {
                const int s = 4 * b + t;
                const u32 av = avn, pv = pvn;
                avn = zero_la ? 0u : lds_q(w[HW - 5 + t], c);
                asm volatile("ld.shared.u32 %0, [%1];" : "=r"(pvn) : "r"(lp_s + 4 * (s - 1) * TS));
                const u32 d = vadd(s4[t], av), x = vadd(vadd(d, pv), pv);
                ch[s * BLOCK] = make_uint2(x, d);
                tm_store8(f.ta + s * 8, m);
                beta_step_d<LOGV>(m, pv, x, d, lut);
            }
#pragma unroll
            for (int k = HW - 1; k >= 4; k--) w[k] = w[k - 4];
        }
#pragma unroll
        for (int s = 0; s < NS; s++) X[(NS + s) * TS + f.t] = m[s];      /* beta_16 -> head thread */
    }
    tm_wait_st();
    } else {
    u32 av[HW], pv[HW], sn[HW];
    tm_load16_wait(f.ts + c * HW, sn);
    /* the 32 shared loads are issued LA steps ahead of their use, in processing
     * order (volatile asm keeps that order against the TMEM stores), so the
     * warps do not all queue 32 loads at the phase start */
    constexpr int LA = 1;
    const u32 lp_s = smem_addr(lp);
    auto ld = [&](int s) {
        if (zero_la) av[s] = 0u;
        else av[s] = lds_q(qq[s], c);
        asm volatile("ld.shared.u32 %0, [%1];" : "=r"(pv[s]) : "r"(lp_s + 4 * s * TS));
    };
    u32 m[NS];
    if (!tail_thr) {
        /* alpha_0 of window j: known start state, zero in iteration 1, NII afterwards (R13) */
        if (f.j == 0) {
            m[0] = M1;
#pragma unroll
            for (int s = 1; s < NS; s++) m[s] = FLOORB;
        } else if (it == 1) {
#pragma unroll
            for (int s = 0; s < NS; s++) m[s] = M1;
        } else {
#pragma unroll
            for (int s = 0; s < NS; s++) m[s] = nii[nii1_ix(c, 0, s, f.t - 1)];
        }
#pragma unroll
        for (int s = 0; s < LA; s++) ld(s);
#pragma unroll
        for (int s = 0; s < HW; s++) {          /* store alpha_s, advance to alpha_{s+1} */
            if (s + LA < HW) ld(s + LA);
            const u32 d = vadd(sn[s], av[s]);                /* Lu - Lp */
            const u32 x = vadd(vadd(d, pv[s]), pv[s]);       /* Lu + Lp */
            ch[s * BLOCK] = make_uint2(x, d);
            tm_store8(f.ta + s * 8, m);
            alpha_step_d<LOGV>(m, pv[s], x, d, lut);
        }
#pragma unroll
        for (int s = 0; s < NS; s++) X[s * TS + f.t] = m[s];             /* alpha_16 -> tail thread */
    } else {
        /* beta_32 of window j: tail termination, zero in iteration 1, NII afterwards */
        if (f.j == f.M - 1) {               /* beta_K from the tail, precomputed at staging (static) */
#pragma unroll
            for (int s = 0; s < NS; s++) m[s] = f.sm[S_TAIL + f.p * 16 + c * 8 + s];
        } else if (it == 1) {
#pragma unroll
            for (int s = 0; s < NS; s++) m[s] = M1;
        } else {
#pragma unroll
            for (int s = 0; s < NS; s++) m[s] = nii[nii1_ix(c, 1, s, f.t + 1)];
        }
#pragma unroll
        for (int s = HW - 1; s >= HW - LA; s--) ld(s);
#pragma unroll
        for (int s = HW - 1; s >= 0; s--) {     /* store beta_{17+s}, advance to beta_{16+s} */
            if (s - LA >= 0) ld(s - LA);
            const u32 d = vadd(sn[s], av[s]);
            const u32 x = vadd(vadd(d, pv[s]), pv[s]);
            ch[s * BLOCK] = make_uint2(x, d);
            tm_store8(f.ta + s * 8, m);
            beta_step_d<LOGV>(m, pv[s], x, d, lut);
        }
#pragma unroll
        for (int s = 0; s < NS; s++) X[(NS + s) * TS + f.t] = m[s];      /* beta_16 -> head thread */
    }
    tm_wait_st();
    }   /* ROLL */
    }   /* f.wact */
    prof_mark(P_PH1);
    gsync<G>(f.g);          /* hand-over; also orders this half-iteration's NII reads before its writes */
    prof_mark(P_BAR1);
    if (!f.wact) return;

    u32 bufA[NS], bufB[NS];
    if (!tail_thr) {
        u32 b[NS];
#pragma unroll
        for (int s = 0; s < NS; s++) b[s] = X[(NS + s) * TS + f.t];      /* beta_16 */
        tm_load8(f.ta + (HW - 1) * 8, bufA);
#pragma unroll 2
        for (int s = HW - 1; s >= 0; s -= 2) {
#pragma unroll
            for (int h = 0; h < 2; h++) {
                const int ss = s - h;
                u32 *cur = h ? bufB : bufA, *nx = h ? bufA : bufB;
                const uint2 g = ch[ss * BLOCK];
                const u32 p = lp[ss * TS];
                tm_wait_ld8(cur);
                tm_load8(f.ta + (ss > 0 ? ss - 1 : 0) * 8, nx);      /* unconditional: no branch around the load */
                le[ss * TS] = ext_out_map<VAR>(lambda_le<LOGV>(cur, b, p, lut));   /* alpha_ss (stored) + beta_{ss+1} */
                beta_step_d<LOGV>(b, p, g.x, g.y, lut);
            }
        }
#pragma unroll
        for (int s = 0; s < NS; s++) nii[nii1_ix(c, 1, s, f.t)] = b[s];  /* beta_{jW} -> window j-1 */
    } else {
        u32 a[NS];
#pragma unroll
        for (int s = 0; s < NS; s++) a[s] = X[s * TS + f.t];             /* alpha_16 */
        tm_load8(f.ta, bufA);
#pragma unroll 2
        for (int s = 0; s < HW; s += 2) {
#pragma unroll
            for (int h = 0; h < 2; h++) {
                const int ss = s + h;
                u32 *cur = h ? bufB : bufA, *nx = h ? bufA : bufB;
                const uint2 g = ch[ss * BLOCK];
                const u32 p = lp[ss * TS];
                tm_wait_ld8(cur);
                tm_load8(f.ta + (ss < HW - 1 ? ss + 1 : ss) * 8, nx);
                le[(HW + ss) * TS] = ext_out_map<VAR>(lambda_le<LOGV>(a, cur, p, lut));   /* alpha_{16+ss} + beta_{17+ss} (stored) */
                alpha_step_d<LOGV>(a, p, g.x, g.y, lut);
            }
        }
#pragma unroll
        for (int s = 0; s < NS; s++) nii[nii1_ix(c, 0, s, f.t)] = a[s];  /* alpha_{(j+1)W} -> window j+1 */
    }
}

struct NoHook {
    __device__ __forceinline__ void operator()() const {}
};

/* hook: called by every thread right after its staging loads are issued (the
 * CRC-ET and latency kernels run warp 0's claim of the next task there, so the
 * claim's round trips overlap the staging loads instead of preceding them) */
template <int VAR, bool PURGE, bool LLR8, int G, bool ROLL = false, bool ETC = false, class Hook = NoHook>
__device__ __forceinline__ void run_task_fast(const crn_task &tk, const crn_cb_desc *__restrict__ desc,
                                              const int16_t *__restrict__ l0, const int16_t *__restrict__ l1,
                                              const int16_t *__restrict__ l2, int max_iters, int et,
                                              uint32_t *__restrict__ out_bits, uint8_t *__restrict__ crc_ok,
                                              uint8_t *__restrict__ iters_used, int16_t *__restrict__ ext_out,
                                              const crn_tables &tab, u32 *sm, u32 tmem, TaskSh sh, Purge pg,
                                              int sh8, Hook hook = Hook{}) {
    constexpr int W = 32;
    const int M = tk.M, NP = tk.n_pairs, T = NP * M;
    constexpr int GWIN = WMAX / G;              /* windows of the group's task */
    const int tid = threadIdx.x, warp = tid >> 5;
    const int g = G == 1 ? 0 : tid / (BLOCK / G), ltid = tid - g * (BLOCK / G);
    const bool tail_thr = ltid >= GWIN;         /* warp-uniform: GWIN = 6 or 2 warps */
    const int tl = ltid - (tail_thr ? GWIN : 0);    /* the thread's window in its task */
    SCtx f;
    f.sm = sm;
    f.g = g;
    f.ta = tmem + ((u32)((warp & 3) * 32) << 16) + (u32)((warp >> 2) * 128);
    f.ts = tmem + ((u32)((warp & 3) * 32) << 16) + (u32)(3 * 128 + (warp >> 2) * 2 * HW);
    f.tid = tid;
    f.t = g * GWIN + tl;                        /* its window column in the shared planes */
    const bool active = tl < T;
    f.wact = (tl & ~31) < T;                    /* head / tail warps are 32-window aligned */
    f.M = M;
    const int pl = active ? tl / M : 0;         /* inactive threads run on pair 0 window 0 data; outputs unused */
    f.p = g * (MAXP / G) + pl;                  /* the pair's slot in the per-CB shared arrays */
    f.j = active ? tl - pl * M : 0;
    f.pM = g * GWIN + pl * M;                   /* the pair's first window column */
    f.k0 = tail_thr ? HW : 0;
    if (VAR == CRN_VARIANT_LOGMAP) {
        f.lut_lo = c_logmap[0];
        f.lut_hi = c_logmap[1];
    }
    const u32 *qts = tab.qpp_ts + tab.qpp_off[tk.kidx];     /* natural position of Pi(jW+i)  */
    const u32 *qinv = tab.qinv_ts + tab.qpp_off[tk.kidx];   /* interleaved position of jW+i */

    /* ---- row a2: stage own half-window of both CBs of the pair: Lp1, Lp2 into
     * the shared planes, Ls-Lp1 (natural) and Ls[Pi]-Lp2 (interleaved) into
     * TMEM; the thread's QPP word indices stay in registers for the task */
    u32 q1[HW], q2[HW];     /* pM + position of Pi^-1(jW+k) (DEC1 gather) / Pi(jW+k) (DEC2 gather) */
    u32 qq[HW];             /* for the task: shared byte addresses of the DEC1 gather (Z, low half) and
                               the DEC2 gather (Y, high half); both < 64 KiB */
    {
        const int p = f.p, j = f.j;
        const int clo = sh.cb[2 * p], chi = sh.cb[2 * p + 1];
        const int Flo = sh.F[2 * p], Fhi = sh.F[2 * p + 1];
        u32 *tmp = sm + S_Z;                  /* natural Ls, window-major, for the interleaved gather
                                                 (the Z plane is first written in DEC2 of iteration 1) */
        {
        const int64_t olo = clo >= 0 ? desc[clo].llr_off : 0, ohi = chi >= 0 ? desc[chi].llr_off : 0;
        const int n0 = j * W + f.k0;
        /* every global load of the staging first (one round trip): the thread's 16
         * LLRs of each stream and CB, its QPP word indices and, for the last
         * window's tail thread, the 12 tail columns */
        u32 wl[3][HW / 2], wh[3][HW / 2];
#pragma unroll
        for (int x = 0; x < 3; x++) {
            const int16_t *src = x == 0 ? l0 : x == 1 ? l1 : l2;
            if (clo >= 0) load16<LLR8>(src, olo + n0, sh8, wl[x]);
            else {
#pragma unroll
                for (int k = 0; k < HW / 2; k++) wl[x][k] = 0;
            }
            if (chi >= 0) load16<LLR8>(src, ohi + n0, sh8, wh[x]);
            else {
#pragma unroll
                for (int k = 0; k < HW / 2; k++) wh[x][k] = 0;
            }
        }
#pragma unroll
        for (int s = 0; s < HW; s++) {
            q1[s] = __ldg(qinv + (f.k0 + s) * M + j);
            q2[s] = __ldg(qts + (f.k0 + s) * M + j);
        }
        const bool tail_owner = active && tail_thr && j == M - 1;
        int16_t t0[12], t1[12];
        if (tail_owner) {
#pragma unroll
            for (int mm = 0; mm < 12; mm++) {     /* tails: DESIGN.md R11 column order */
                const int col = tk.K + mm / 3;
                const int16_t *src = (mm % 3 == 0) ? l0 : (mm % 3 == 1) ? l1 : l2;
                t0[mm] = clo >= 0 ? ld_llr<LLR8>(src, olo + col, sh8) : (int16_t)0;
                t1[mm] = chi >= 0 ? ld_llr<LLR8>(src, ohi + col, sh8) : (int16_t)0;
            }
        }
        hook();
        u32 sn[HW];
#pragma unroll
        for (int x = 0; x < 3; x++) {
#pragma unroll
            for (int s = 0; s < HW; s++) {
                u32 v = __byte_perm(wl[x][s / 2], wh[x][s / 2], (s & 1) ? 0x7632 : 0x5410);
                if (x < 2) {                                       /* known filler 0: Ls = Lp1 = -4096 */
                    if (n0 + s < Flo) v = (v & 0xFFFF0000u) | 0xF000u;
                    if (n0 + s < Fhi) v = (v & 0x0000FFFFu) | 0xF0000000u;
                }
                v = __vmins2(__vmaxs2(v, CLIP_LO), CLIP_HI);
                const int ix = (f.k0 + s) * TS + f.t;
                if (x == 0) {
                    sn[s] = v;
                    if (active) tmp[ix] = v;
                } else if (x == 1) {
                    sn[s] = __vsub2(sn[s], v);
                    if (active) sm[S_LP + ix] = v;
                } else if (active) {
                    sm[S_LP + SUMK + ix] = v;
                }
            }
        }
        tm_store16(f.ts, sn);
        if (tail_owner) {
            /* beta_K of both constituents depends on the tail LLRs only: formed once per task */
            u32 tl[12];
#pragma unroll
            for (int mm = 0; mm < 12; mm++) tl[mm] = clamp_pack(t0[mm], t1[mm]);
#pragma unroll
            for (int c = 0; c < 2; c++) {
                u32 b[NS];
                tail_beta(tl + 6 * c, b);
#pragma unroll
                for (int s = 0; s < NS; s++) sm[S_TAIL + p * 16 + c * 8 + s] = b[s];
            }
        }
#pragma unroll
        for (int s = 0; s < HW; s++) {
            q1[s] += f.pM;
            q2[s] += f.pM;
        }
        }
        prof_mark(P_SLD);
        gsync<G>(g);
        prof_mark(P_SB1);
        {
            u32 sn[HW];
#pragma unroll
            for (int s = 0; s < HW; s++)          /* interleaved systematic Ls[Pi(jW+k)] */
                sn[s] = __vsub2(tmp[q2[s]], sm[S_LP + SUMK + (f.k0 + s) * TS + f.t]);
            const u32 base = smem_addr(sm);
#pragma unroll
            for (int s = 0; s < HW; s++) qq[s] = (base + 4 * (S_Z + q1[s])) | ((base + 4 * (S_Y + q2[s])) << 16);
            tm_store16(f.ts + HW, sn);
            tm_wait_st();
        }
        prof_mark(P_SG);
        gsync<G>(g);
        prof_mark(P_STAGE);
    }

    for (int it = 1; it <= max_iters; it++) {
        if constexpr (ROLL) {
            /* both constituents through one call site (one copy of the SISO code) */
#pragma unroll 1
            for (int c = 0; c < 2; c++) {
                prof_mark(P_CHUNK);
                siso_split<VAR, G, true>(f, tail_thr, c, it, qq, it == 1 && c == 0);
                prof_mark(P_PH2);
                gsync<G>(g);
                prof_mark(P_BAR2);
            }
        } else {
        /* DEC1: La1[n] = Le2[Pi^-1(n)] gathered from Z (zero in iteration 1) */
        prof_mark(P_CHUNK);
        siso_split<VAR, G>(f, tail_thr, 0, it, qq, it == 1);
        prof_mark(P_PH2);
        gsync<G>(g);
        prof_mark(P_BAR2);
        /* DEC2: La2[i] = Le1[Pi(i)] gathered from Y */
        prof_mark(P_CHUNK);
        siso_split<VAR, G>(f, tail_thr, 1, it, qq, false);
        prof_mark(P_PH2);
        gsync<G>(g);
        prof_mark(P_BAR2);
        }
        if (!et && it != max_iters) continue;     /* fixed mode: decide only at the end */

        /* ---- row a9: L_APP = Ls + Le1 + La1_next (tie -> 1, R16); 16 bits per
         * thread and CB lane, merged per window; windowed CRC */
        {
            u32 wb = 0;                       /* bit s: lo CB's step k0 + s, bit 16 + s: hi CB's */
            int mlo = 0, mhi = 0;             /* MI statistic of this thread's steps (R29) */
            u32 sn[HW];
            const int n00 = f.j * W + f.k0, Fl = sh.F[2 * f.p], Fh = sh.F[2 * f.p + 1];
            tm_load16_wait(f.ts, sn);
            /* with the stopping-rule test inside the loop every step is its own basic
             * block and its three shared loads cannot be issued ahead (~1.7 k cycles
             * per early-termination iteration) */
            auto lapp_pass = [&](auto mi_rule) {
#pragma unroll
                for (int s = 0; s < HW; s++) {
                    const u32 la1n = lds_q(qq[s], 0);                    /* La1_next[n] = Le2[Pi^-1(n)] */
                    const u32 ls = vadd(sn[s], sm[S_LP + (f.k0 + s) * TS + f.t]);
                    const u32 lapp = vadd(vadd(ls, sm[S_Y + (f.k0 + s) * TS + f.t]), la1n);
                    /* b = (L_APP >= 0) per half enters at bits 15 / 31 and moves down one bit per
                     * later step (w >> 1 as a multiply-high, off the ALU pipe) */
                    wb = __umulhi(wb, 0x80000000u) | (~lapp & 0x80008000u);
                    if (decltype(mi_rule)::value && et == CRN_ET_MI) {
                        mlo += mi_pair(sh.mitab, lapp, n00 + s >= Fl, false);
                        mhi += mi_pair(sh.mitab, lapp, false, n00 + s >= Fh);
                    }
                }
            };
            /* CRC early termination (every iteration): the branch-free copy, in the
             * CRC kernel (ETC) and the latency kernels; fixed iterations (once per
             * task) and the MI rule: the copy with the test (the throughput kernel
             * carries only this one, so its code is unchanged) */
            if constexpr (ETC || ROLL) {
                if (ETC || et == CRN_ET_CRC) lapp_pass(std::false_type{});
                else lapp_pass(std::true_type{});
            } else {
                lapp_pass(std::true_type{});
            }
            u32 *hb = sm + S_X;               /* [half][window] bits of both CBs; [2 + lane][window] window words */
            if (active) {
                hb[(tail_thr ? 1 : 0) * TS + f.t] = wb;
                if (et == CRN_ET_MI) {
                    atomicAdd(&sh.mi[2 * f.p], mlo);
                    atomicAdd(&sh.mi[2 * f.p + 1], mhi);
                }
            }
            prof_mark(P_HL);
            gsync<G>(g);
            prof_mark(P_HB1);
            u32 r3 = 0;                       /* this window's CRC register contribution */
            int kind = CRN_CRC_NONE;
            if (active) {
                /* the window's 32 hard decisions of one CB lane: the head thread takes
                 * the low (first) CB of the pair, the tail thread the high one */
                const int p = f.p, j = f.j, l = tail_thr ? 1 : 0;
                u32 w = __byte_perm(hb[f.t], hb[TS + f.t], l ? 0x7632u : 0x5410u);
                const int n0 = j * W, F = sh.F[2 * p + l];
                if (F > n0) w &= (F >= n0 + 32) ? 0u : (0xFFFFFFFFu << (F - n0));
                hb[(2 + l) * TS + f.t] = w;
                kind = sh.kind[2 * p + l];
                if (kind != CRN_CRC_NONE) {
                    /* CRC register contribution x^(32 d) R(w) mod g, d = M-1-j = 64a + 8b + c, as
                     * three nibble-table maps (crn_internal.h CRN_CRC_NIB_WORDS) */
                    constexpr bool PADNIB = ETC || ROLL;
                    const u32 T = smem_addr(sh.crcnib) +
                                  (kind == CRN_CRC24A ? 0u : 4u * (PADNIB ? NIBP_KIND : CRN_CRC_NIB_WORDS));
                    const u32 d = (u32)(M - 1 - j);
                    const u32 t1 = PADNIB ? T + (d & 7u) * (4u * NIBP_T1) : T + (d & 7u) * 512u,
                              t2 = PADNIB ? T + 4u * NIBP_O2 + ((d >> 3) & 7u) * (4u * NIBP_T23)
                                          : T + 4096u + ((d >> 3) & 7u) * 384u,
                              t3 = PADNIB ? T + 4u * NIBP_O3 + (d >> 6) * (4u * NIBP_T23)
                                          : T + 7168u + (d >> 6) * 384u;   /* byte addresses of the three maps */
                    u32 r = 0, r2 = 0;
#pragma unroll
                    for (int q = 0; q < 8; q++) r ^= lds_at(t1 + 64u * q + nib_off(w, q));
#pragma unroll
                    for (int q = 0; q < 6; q++) r2 ^= lds_at(t2 + 64u * q + nib_off(r, q));
#pragma unroll
                    for (int q = 0; q < 6; q++) r3 ^= lds_at(t3 + 64u * q + nib_off(r2, q));
                }
            }
            /* combine the windows' contributions: one shared atomic per warp when all its
             * lanes hold windows of one CB lane (every K with 32 | M), else one per window */
            {
                const int e = 2 * f.p + (tail_thr ? 1 : 0);
                const int e0 = __shfl_sync(0xFFFFFFFFu, e, 0);      /* every lane: no short-circuit around it */
                const bool uni = __all_sync(0xFFFFFFFFu, active && e == e0);
                if (uni) {
                    r3 = __reduce_xor_sync(0xFFFFFFFFu, r3);
                    if ((threadIdx.x & 31) == 0 && kind != CRN_CRC_NONE) atomicXor(&sh.crc[e], r3);
                } else if (active && kind != CRN_CRC_NONE) {
                    atomicXor(&sh.crc[e], r3);
                }
            }
            prof_mark(P_HC);
            gsync<G>(g);
            prof_mark(P_HB2);
            /* stop decision (row a9; R3 / R29), taken by every thread for both CB lanes of
             * its pair from the complete CRC register and MI sum; the head (tail) thread
             * of window 0 is the low (high) lane's owner: it records crc_ok /
             * iters_used and counts the lane as still running */
            int running = 0;
            if (active) {
                const int p = f.p, j = f.j;
#pragma unroll
                for (int l = 0; l < 2; l++) {
                    const int e = 2 * p + l;
                    if (sh.done[e]) continue;
                    const bool pass = sh.kind[e] != CRN_CRC_NONE && sh.crc[e] == 0;
                    const int dmi = sh.mi[e] - sh.mip[e];
                    const bool mi_conv = et == CRN_ET_MI && it >= 2 && (dmi < 0 ? -dmi : dmi) <= (tk.K - sh.F[e]) * CRN_MI_EPS;
                    const bool fin = (et == CRN_ET_CRC && pass) || mi_conv || it == max_iters;
                    const bool owner = j == 0 && l == (tail_thr ? 1 : 0);
                    if (!fin) {
                        running |= owner;
                        continue;
                    }
                    if (owner) {
                        crc_ok[sh.cb[e]] = pass;
                        if (PURGE && !pass && pg.tb[e] >= 0)      /* decoding failure: its TB is lost */
                            *(volatile uint8_t *)&pg.dead[pg.tb[e]] = 1;
                        if (iters_used) iters_used[sh.cb[e]] = (uint8_t)it;
                    }
                    if (l == (tail_thr ? 1 : 0)) out_bits[sh.bo[e] + j] = hb[(2 + l) * TS + f.t];
                    if (ext_out) {
                        const int64_t oe = sh.eo[e] + j * W + f.k0;
#pragma unroll
                        for (int s = 0; s < HW; s++) {
                            const u32 x = lds_q(qq[s], 0);
                            ext_out[oe + s] = (int16_t)(l ? (x >> 16) : (x & 0xFFFFu));
                        }
                    }
                }
            }
            prof_mark(P_HDEC);
            /* one counting barrier: every read of this iteration's flags is before it */
            const int left = gsync_count<G>(g, running);
            if (active && f.j == 0) {
                const int e = 2 * f.p + (tail_thr ? 1 : 0);
                if (!sh.done[e]) {
                    sh.done[e] = !running;
                    sh.mip[e] = sh.mi[e];
                }
                sh.crc[e] = 0;
                sh.mi[e] = 0;
            }
            prof_mark(P_HD);
            if (left == 0) break;
        }
    }
}

/* ======================================================================
 * Split-window path: W in 33..62 (K <= 1008 that is not a multiple of 32).
 * The W = 32 design with runtime sizes: a window's head thread (tid < Tp)
 * owns steps [0, hw), hw = ceil(W/2), its tail thread (tid = Tp + t) steps
 * [hw, W); everything the CB pairs of the task need stays on chip:
 * extrinsics, parity planes, per-thread QPP word indices and branch-metric
 * pairs, NII states in shared memory (row stride Tp, crn_split_smem_words),
 * stored alpha/beta and the static Ls-Lp sums in TMEM (10*hw columns per
 * thread).  The host sizes n_pairs so both fit (crn_split_fits).  Rolled
 * loops (runtime W); one TMEM column per static sum and step.
 * ====================================================================== */
struct GSplit {
    u32 *Y, *Z, *LP, *Q, *CH, *NII, *X, *TB;
    int W, M, T, Tp, hw_h;     /* geometry */
    int tid2;                  /* position in the per-thread arrays: tid for head, Tp + t for tail */
    int t, p, j, pM, k0, hw;   /* window, pair, window in CB, steps owned */
    u32 ta, ts;                /* TMEM: 8*hw_h stored-metric columns, then 2*hw_h static columns */
    u32 lut_lo, lut_hi;        /* Log-MAP LUT words */
};

__device__ __forceinline__ void tm_store1(u32 ta, u32 v) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(ta), "r"(v) : "memory");
}
__device__ __forceinline__ u32 tm_load1_wait(u32 ta) {
    u32 v;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];\n\ttcgen05.wait::ld.sync.aligned;"
                 : "=r"(v) : "r"(ta) : "memory");
    return v;
}

/* One half-iteration of constituent c on the split-window path (rows a4-a8). */
template <int VAR>
__device__ __forceinline__ void siso_gsplit(const GSplit &g, bool tail_thr, int c, int it) {
    constexpr bool LOGV = VAR == CRN_VARIANT_LOGMAP;
    const Lut lut{g.lut_lo, g.lut_hi};
    const int Tp = g.Tp, W = g.W, hw = g.hw, t = g.t, st2 = 2 * Tp;
    const u32 *lp = g.LP + c * W * Tp + g.k0 * Tp + t;           /* this thread's steps, stride Tp */
    const u32 *Qc = g.Q + c * g.hw_h * st2 + g.tid2;              /* QPP word indices (stride 2Tp) */
    const u32 *la = c ? g.Y : g.Z;
    const bool zero_la = c == 0 && it == 1;
    uint2 *ch = reinterpret_cast<uint2 *>(g.CH) + g.tid2;
    u32 *le = (c ? g.Z : g.Y) + g.k0 * Tp + t;
    const u32 ts = g.ts + c * g.hw_h;
    u32 m[NS];
    /* ---- phase 1: head alpha forward over [0, hw), tail beta backward over [hw_h, W) */
    if (!tail_thr) {
        if (g.j == 0) {
            m[0] = M1;
#pragma unroll
            for (int s = 1; s < NS; s++) m[s] = FLOORB;
        } else if (it == 1) {
#pragma unroll
            for (int s = 0; s < NS; s++) m[s] = M1;
        } else {
#pragma unroll
            for (int s = 0; s < NS; s++) m[s] = g.NII[((c * 2 + 0) * NS + s) * Tp + t - 1];
        }
#pragma unroll 1
        for (int s = 0; s < hw; s++) {
            const u32 av = zero_la ? 0u : la[Qc[s * st2]];
            const u32 pv = lp[s * Tp];
            const u32 sn = tm_load1_wait(ts + s);
            const u32 d = vadd(sn, av), x = vadd(vadd(d, pv), pv);
            ch[s * st2] = make_uint2(x, d);
            tm_store8(g.ta + s * 8, m);
            alpha_step_d<LOGV>(m, pv, x, d, lut);
        }
#pragma unroll
        for (int s = 0; s < NS; s++) g.X[s * Tp + t] = m[s];                 /* alpha_hw -> tail thread */
    } else {
        if (g.j == g.M - 1) {
#pragma unroll
            for (int s = 0; s < NS; s++) m[s] = g.TB[g.p * 16 + c * 8 + s];
        } else if (it == 1) {
#pragma unroll
            for (int s = 0; s < NS; s++) m[s] = M1;
        } else {
#pragma unroll
            for (int s = 0; s < NS; s++) m[s] = g.NII[((c * 2 + 1) * NS + s) * Tp + t + 1];
        }
#pragma unroll 1
        for (int s = hw - 1; s >= 0; s--) {
            const u32 av = zero_la ? 0u : la[Qc[s * st2]];
            const u32 pv = lp[s * Tp];
            const u32 sn = tm_load1_wait(ts + s);
            const u32 d = vadd(sn, av), x = vadd(vadd(d, pv), pv);
            ch[s * st2] = make_uint2(x, d);
            tm_store8(g.ta + s * 8, m);
            beta_step_d<LOGV>(m, pv, x, d, lut);
        }
#pragma unroll
        for (int s = 0; s < NS; s++) g.X[(NS + s) * Tp + t] = m[s];          /* beta_hw_h -> head thread */
    }
    tm_wait_st();
    __syncthreads();        /* hand-over; also orders this half-iteration's NII reads before its writes */
    /* ---- phase 2: head beta backward over [0, hw) + Lambda, tail alpha forward + Lambda */
    u32 nx[NS], cur[NS];
    if (!tail_thr) {
        u32 b[NS];
#pragma unroll
        for (int s = 0; s < NS; s++) b[s] = g.X[(NS + s) * Tp + t];
        tm_load8(g.ta + (hw - 1) * 8, nx);
#pragma unroll 1
        for (int s = hw - 1; s >= 0; s--) {
            const uint2 gg = ch[s * st2];
            const u32 pv = lp[s * Tp];
            tm_wait_ld8(nx);
#pragma unroll
            for (int k = 0; k < NS; k++) cur[k] = nx[k];
            tm_load8(g.ta + (s > 0 ? s - 1 : 0) * 8, nx);
            le[s * Tp] = ext_out_map<VAR>(lambda_le<LOGV>(cur, b, pv, lut));
            beta_step_d<LOGV>(b, pv, gg.x, gg.y, lut);
        }
        tm_wait_ld8(nx);
#pragma unroll
        for (int s = 0; s < NS; s++) g.NII[((c * 2 + 1) * NS + s) * Tp + t] = b[s];   /* beta_{jW} -> window j-1 */
    } else {
        u32 a[NS];
#pragma unroll
        for (int s = 0; s < NS; s++) a[s] = g.X[s * Tp + t];
        tm_load8(g.ta, nx);
#pragma unroll 1
        for (int s = 0; s < hw; s++) {
            const uint2 gg = ch[s * st2];
            const u32 pv = lp[s * Tp];
            tm_wait_ld8(nx);
#pragma unroll
            for (int k = 0; k < NS; k++) cur[k] = nx[k];
            tm_load8(g.ta + (s + 1 < hw ? s + 1 : s) * 8, nx);
            le[s * Tp] = ext_out_map<VAR>(lambda_le<LOGV>(a, cur, pv, lut));
            alpha_step_d<LOGV>(a, pv, gg.x, gg.y, lut);
        }
        tm_wait_ld8(nx);
#pragma unroll
        for (int s = 0; s < NS; s++) g.NII[((c * 2 + 0) * NS + s) * Tp + t] = a[s];   /* alpha_{(j+1)W} -> window j+1 */
    }
}

template <int VAR, bool PURGE, bool LLR8, int TAG = 0>   /* TAG: one copy per kernel family (ROLL 1, ETC 2) */
__device__ __noinline__ void run_task_split(const crn_task &tk, const crn_cb_desc *__restrict__ desc,
                                            const int16_t *__restrict__ l0, const int16_t *__restrict__ l1,
                                            const int16_t *__restrict__ l2, int max_iters, int et,
                                            uint32_t *__restrict__ out_bits, uint8_t *__restrict__ crc_ok,
                                            uint8_t *__restrict__ iters_used, int16_t *__restrict__ ext_out,
                                            const crn_tables &tab, u32 *sm, u32 tmem, TaskSh sh, Purge pg,
                                            int sh8) {
    const int tid = threadIdx.x, warp = tid >> 5;
    GSplit g;
    g.W = tk.W;
    g.M = tk.M;
    g.T = tk.n_pairs * tk.M;
    g.Tp = (g.T + 31) & ~31;
    g.hw_h = (g.W + 1) / 2;
    const int W = g.W, M = g.M, T = g.T, Tp = g.Tp, NP = tk.n_pairs, K = tk.K;
    g.Y = sm;
    g.Z = g.Y + W * Tp;
    g.LP = g.Z + W * Tp;
    g.Q = g.LP + 2 * W * Tp;
    g.CH = g.Q + 2 * g.hw_h * 2 * Tp;
    g.NII = g.CH + 2 * g.hw_h * 2 * Tp;
    g.X = g.NII + 32 * Tp;
    g.TB = g.X + 16 * Tp;
    const bool working = tid < 2 * Tp;          /* whole warps: Tp is a multiple of 32 */
    const bool tail_thr = tid >= Tp;
    g.tid2 = tid;
    g.t = tid - (tail_thr ? Tp : 0);
    const bool active = working && g.t < T;
    g.p = active ? g.t / M : 0;
    g.j = active ? g.t - g.p * M : 0;
    g.pM = g.p * M;
    g.k0 = tail_thr ? g.hw_h : 0;
    g.hw = tail_thr ? W - g.hw_h : g.hw_h;
    if (VAR == CRN_VARIANT_LOGMAP) {
        g.lut_lo = c_logmap[0];
        g.lut_hi = c_logmap[1];
    }
    g.ta = tmem + ((u32)((warp & 3) * 32) << 16) + (u32)((warp >> 2) * 10 * g.hw_h);
    g.ts = g.ta + 8 * g.hw_h;
    const u32 *qw = tab.qpp_wm + tab.qpp_off[tk.kidx];      /* (row << 16) | col of Pi(jW+i) */
    const u32 *qi = tab.qinv_wm + tab.qpp_off[tk.kidx];     /* same for Pi^-1(jW+i) */
    const u32 *cbit = tab.crc_bit + tab.crcb_off[tk.kidx] + g.j;
    const int p = g.p, j = g.j, t = g.t, hw = g.hw, k0 = g.k0, st2 = 2 * Tp;
    const int clo = sh.cb[2 * p], chi = sh.cb[2 * p + 1];
    const int Flo = sh.F[2 * p], Fhi = sh.F[2 * p + 1];

    /* ---- row a2: stage this thread's steps of both CBs of the pair */
    if (working) {
        const int64_t olo = clo >= 0 ? desc[clo].llr_off : 0, ohi = chi >= 0 ? desc[chi].llr_off : 0;
        u32 *tmp = g.CH;                        /* natural Ls, window-major, for the interleaved gather */
#pragma unroll 1
        for (int s = 0; s < hw; s++) {
            const int n = j * W + k0 + s, ix = (k0 + s) * Tp + t;
            u32 v[3];
#pragma unroll
            for (int x = 0; x < 3; x++) {
                const int16_t *src = x == 0 ? l0 : x == 1 ? l1 : l2;
                int16_t a = clo >= 0 ? ld_llr<LLR8>(src, olo + n, sh8) : (int16_t)0;
                int16_t b = chi >= 0 ? ld_llr<LLR8>(src, ohi + n, sh8) : (int16_t)0;
                if (x < 2) {                                   /* known filler 0: Ls = Lp1 = -4096 */
                    if (n < Flo) a = -4096;
                    if (n < Fhi) b = -4096;
                }
                v[x] = clamp_pack(a, b);
            }
            tmp[ix] = v[0];
            g.LP[ix] = v[1];
            g.LP[W * Tp + ix] = v[2];
            tm_store1(g.ts + s, __vsub2(v[0], v[1]));              /* Ls - Lp1 */
            const u32 q1 = __ldg(qi + (k0 + s) * M + j), q2 = __ldg(qw + (k0 + s) * M + j);
            g.Q[s * st2 + tid] = (q1 >> 16) * Tp + g.pM + (q1 & 0xFFFFu);                  /* DEC1 gather: Z */
            g.Q[g.hw_h * st2 + s * st2 + tid] = (q2 >> 16) * Tp + g.pM + (q2 & 0xFFFFu);   /* DEC2 gather: Y */
        }
        if (active && tail_thr && j == M - 1) {      /* beta_K of both constituents from the tails */
            u32 tl[12];
#pragma unroll
            for (int mm = 0; mm < 12; mm++) {
                const int col = K + mm / 3;
                const int16_t *src = (mm % 3 == 0) ? l0 : (mm % 3 == 1) ? l1 : l2;
                tl[mm] = clamp_pack(clo >= 0 ? ld_llr<LLR8>(src, olo + col, sh8) : (int16_t)0,
                                    chi >= 0 ? ld_llr<LLR8>(src, ohi + col, sh8) : (int16_t)0);
            }
#pragma unroll
            for (int c = 0; c < 2; c++) {
                u32 b[NS];
                tail_beta(tl + 6 * c, b);
#pragma unroll
                for (int s = 0; s < NS; s++) g.TB[p * 16 + c * 8 + s] = b[s];
            }
        }
    }
    __syncthreads();
    if (working) {
#pragma unroll 1
        for (int s = 0; s < hw; s++)            /* Ls[Pi(i)] - Lp2 */
            tm_store1(g.ts + g.hw_h + s, __vsub2(g.CH[g.Q[g.hw_h * st2 + s * st2 + tid]], g.LP[W * Tp + (k0 + s) * Tp + t]));
        tm_wait_st();
    }
    __syncthreads();

    const int nw = (K + 31) >> 5;
    for (int it = 1; it <= max_iters; it++) {
        if (working) siso_gsplit<VAR>(g, tail_thr, 0, it);
        else __syncthreads();                   /* the hand-over barrier inside siso_gsplit */
        __syncthreads();
        if (working) siso_gsplit<VAR>(g, tail_thr, 1, it);
        else __syncthreads();
        __syncthreads();
        if (!et && it != max_iters) continue;
        /* ---- row a9: L_APP = Ls + Le1 + La1_next, hard decision (tie -> 1), fillers 0,
         * LSB-first packing into shared words, CRC as the XOR of per-bit constants */
        u32 *bits = g.X;                        /* [pair lane][nw] words, free after the hand-over */
        for (int e = tid; e < 2 * NP * nw; e += BLOCK) bits[e] = 0;
        __syncthreads();
        u32 blo = 0, bhi = 0;
        int mlo = 0, mhi = 0;                   /* MI statistic (R29) */
        if (working) {                          /* TMEM loads are warp-collective: every lane of a working warp */
            int s = 0;
            if constexpr (TAG != 0) {
                /* latency / CRC-ET kernels, CRC rule: eight steps per batch, their TMEM
                 * statics (eight x1 loads, one wait) and shared loads all issued first */
                if (et != CRN_ET_MI) {
                    for (; s + 8 <= hw; s += 8) {
                        u32 st8[8], lpv[8], yv[8], zv[8];
#pragma unroll
                        for (int u = 0; u < 8; u++)
                            asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];"
                                         : "=r"(st8[u]) : "r"(g.ts + s + u) : "memory");
#pragma unroll
                        for (int u = 0; u < 8; u++) {
                            const int ix = (k0 + s + u) * Tp + t;
                            lpv[u] = g.LP[ix];
                            yv[u] = g.Y[ix];
                            zv[u] = g.Z[g.Q[(s + u) * st2 + tid]];
                        }
                        tm_wait_ld8(st8);
#pragma unroll
                        for (int u = 0; u < 8; u++) {
                            const int n = j * W + k0 + s + u;
                            const u32 lapp = vadd(vadd(vadd(st8[u], lpv[u]), yv[u]), zv[u]);
                            const u32 ge = __vcmpges2(lapp, 0u);
                            blo |= (n < Flo ? 0u : (ge & 1u)) << (s + u);
                            bhi |= (n < Fhi ? 0u : ((ge >> 16) & 1u)) << (s + u);
                        }
                    }
                }
            }
#pragma unroll 1
            for (; s < hw; s++) {
                const int ix = (k0 + s) * Tp + t, n = j * W + k0 + s;
                const u32 ls = vadd(tm_load1_wait(g.ts + s), g.LP[ix]);
                const u32 lapp = vadd(vadd(ls, g.Y[ix]), g.Z[g.Q[s * st2 + tid]]);
                const u32 ge = __vcmpges2(lapp, 0u);
                blo |= (n < Flo ? 0u : (ge & 1u)) << s;
                bhi |= (n < Fhi ? 0u : ((ge >> 16) & 1u)) << s;
                if (et == CRN_ET_MI) {
                    mlo += mi_pair(sh.mitab, lapp, n >= Flo, false);
                    mhi += mi_pair(sh.mitab, lapp, false, n >= Fhi);
                }
            }
        }
        if (active && et == CRN_ET_MI) {
            atomicAdd(&sh.mi[2 * p], mlo);
            atomicAdd(&sh.mi[2 * p + 1], mhi);
        }
        if (active) {
            const int n0 = j * W + k0, w0 = n0 >> 5, off = n0 & 31;
#pragma unroll
            for (int l = 0; l < 2; l++) {
                const u32 b = l ? bhi : blo;
                u32 *bb = bits + (2 * p + l) * nw;
                atomicOr(&bb[w0], b << off);
                if (off && w0 + 1 < nw) atomicOr(&bb[w0 + 1], b >> (32 - off));
                const int kind = sh.kind[2 * p + l];
                if (kind == CRN_CRC_NONE) continue;
                const u32 *cb = cbit + (kind == CRN_CRC24A ? 0 : K) + k0 * M;
                u32 acc = 0;
                if constexpr (TAG != 0) {
                    /* the latency / CRC-ET kernels: eight independent constant loads in
                     * flight (one at a time, each waited for, this loop cost a lone task
                     * ~2 x 30 L2 round trips per iteration) */
                    int s = 0;
                    for (; s + 8 <= hw; s += 8) {
                        u32 v[8];
#pragma unroll
                        for (int u = 0; u < 8; u++) v[u] = __ldg(cb + (s + u) * M);
#pragma unroll
                        for (int u = 0; u < 8; u++) acc ^= v[u] & (0u - ((b >> (s + u)) & 1u));
                    }
#pragma unroll 1
                    for (; s < hw; s++) acc ^= __ldg(cb + s * M) & (0u - ((b >> s) & 1u));
                } else {
#pragma unroll 1
                for (int s = 0; s < hw; s++) acc ^= __ldg(cb + s * M) & (0u - ((b >> s) & 1u));
                }
                atomicXor(&sh.crc[2 * p + l], acc);
            }
        }
        __syncthreads();
        decide<PURGE>(sh, NP, it, max_iters, et, K, crc_ok, iters_used, pg);
        for (int e = tid; e < 2 * NP * nw; e += BLOCK) {
            const int pl = e / nw, w = e - pl * nw;
            if (sh.fin[pl]) out_bits[desc[sh.cb[pl]].bit_off + w] = bits[e];
        }
        if (ext_out && active) {
#pragma unroll
            for (int l = 0; l < 2; l++) {
                if (!sh.fin[2 * p + l]) continue;
                const crn_cb_desc &d = desc[sh.cb[2 * p + l]];
                for (int s = 0; s < hw; s++) {
                    const u32 x = g.Z[g.Q[s * st2 + tid]];
                    ext_out[d.ext_off + j * W + k0 + s] = (int16_t)(l ? (x >> 16) : (x & 0xFFFFu));
                }
            }
        }
        if (finish_iteration(sh, NP) == 0) break;
    }
}

/* Claim the CTA's next task (warp 0): its descriptor and CB list go to the
 * shared "next" slots, and its input LLRs (3 streams x K+4 int16 per CB) are
 * bulk-prefetched into L2, so the task starts from on-chip metadata and its
 * staging loads hit L2 instead of waiting on HBM. */
struct NextSh {
    int *task;
    crn_task *tk;
    int *cb, *F, *kind, *tb;
    int64_t *bo, *eo;
};

__device__ __forceinline__ void claim_next(NextSh nx, int *counter, int n_tasks, const crn_task *__restrict__ tasks,
                                           const crn_pair *__restrict__ pairs, const crn_cb_desc *__restrict__ desc,
                                           const int16_t *l0, const int16_t *l1, const int16_t *l2, int lane,
                                           int sh8) {
    int nt = 0;
    if (lane == 0) nt = atomicAdd(counter, 1);
    nt = __shfl_sync(0xFFFFFFFFu, nt, 0);
    if (lane == 0) *nx.task = nt;
    if (nt >= n_tasks) return;
    const crn_task t = tasks[nt];
    if (lane == 0) *nx.tk = t;
    for (int e = lane; e < 2 * t.n_pairs; e += 32) {
        const crn_pair pr = pairs[t.pair0 + (e >> 1)];
        const int cb = (e & 1) ? pr.hi : pr.lo;
        nx.cb[e] = cb;
        if (cb < 0) {
            nx.F[e] = 0;
            nx.kind[e] = 0;
            nx.bo[e] = 0;
            nx.eo[e] = 0;
            if (nx.tb) nx.tb[e] = -1;
            continue;
        }
        const crn_cb_desc &d = desc[cb];
        nx.F[e] = d.F;
        nx.kind[e] = d.crc_kind;
        nx.bo[e] = d.bit_off;
        nx.eo[e] = d.ext_off;
        if (nx.tb) nx.tb[e] = d.reserved;
        const int esz = sh8 < 0 ? 2 : 1;                 /* int16 or int8 LLRs */
        const int64_t off = esz * d.llr_off;
        const uint32_t bytes = (uint32_t)esz * (uint32_t)(t.K + 4);
#pragma unroll
        for (int x = 0; x < 3; x++) {
            const uintptr_t a = reinterpret_cast<uintptr_t>(x == 0 ? l0 : x == 1 ? l1 : l2) + off;
            const uintptr_t a0 = a & ~(uintptr_t)15, a1 = (a + bytes + 15) & ~(uintptr_t)15;
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a0), "r"((uint32_t)(a1 - a0))
                         : "memory");
        }
    }
}

/* One instantiation per (purge?, int8 LLRs?, Log-MAP?): the default
 * <false, false, MAXLOG> (which also runs CRN_VARIANT_SCALED, chosen per launch)
 * has no purge, int8 or Log-MAP code at all. */
template <bool PURGE, bool LLR8, int VAR, bool ROLL = false, bool ETC = false>
__global__ void __launch_bounds__(BLOCK, 1)
decode_kernel(const crn_cb_desc *__restrict__ desc, const crn_task *__restrict__ tasks, int n_tasks,
              const crn_pair *__restrict__ pairs, const int16_t *__restrict__ l0,
              const int16_t *__restrict__ l1, const int16_t *__restrict__ l2, int max_iters, int et,
              uint32_t *__restrict__ out_bits, uint8_t *__restrict__ crc_ok, uint8_t *__restrict__ iters_used,
              int16_t *__restrict__ ext_out, crn_tables tab, uint8_t *ws, int variant, uint8_t *tb_dead_arg) {
    uint8_t *const tb_dead = PURGE ? tb_dead_arg : nullptr;
    const int sh8 = (variant >> 8) - 1;         /* LLR format: -1 int16, else int8 << sh8 (LLR8) */
    extern __shared__ __align__(16) u32 smem[];
    __shared__ int s_ntask[G3], s_left[G3];
    __shared__ crn_task s_ntk[G3];
    __shared__ int s_ncb[2 * MAXP], s_nF[2 * MAXP], s_nkind[2 * MAXP], s_ntb[2 * MAXP];
    __shared__ int s_tb[2 * MAXP];
    __shared__ u32 s_tmem;
    __shared__ u32 s_crc[2 * MAXP];
    __shared__ int s_cb[2 * MAXP], s_F[2 * MAXP], s_kind[2 * MAXP];
    __shared__ uint8_t s_done[2 * MAXP], s_fin[2 * MAXP];
    __shared__ int s_mi[2 * MAXP], s_mip[2 * MAXP], s_mitab[256];

    int *counter = (int *)ws;
    if (n_tasks < 0) n_tasks = ((const volatile int *)ws)[1];   /* built on the device (crn_tasks.cu) */
    const int tid = threadIdx.x;
    u32 *s_crcnib = smem + S_CRCNIB;
    int64_t *s_bo = reinterpret_cast<int64_t *>(smem + ((ETC || ROLL) ? S_OFFS_P : S_OFFS)), *s_eo = s_bo + 2 * MAXP,
            *s_nbo = s_eo + 2 * MAXP,
            *s_neo = s_nbo + 2 * MAXP;
    const TaskSh sh{s_crcnib, s_cb, s_F, s_kind, s_mi, s_mip, s_mitab, s_done, s_fin, s_crc, s_left, s_bo, s_eo};
    const Purge pg{s_tb, tb_dead};
    for (int i = tid; i < 256; i += BLOCK) s_mitab[i] = tab.mi_tab[i];
    if constexpr (ETC || ROLL) {
        for (int i = tid; i < 2 * CRN_CRC_NIB_WORDS; i += BLOCK) {
            const int k = i >= CRN_CRC_NIB_WORDS, r = i - k * CRN_CRC_NIB_WORDS;
            const int dst = r < 1024 ? (r >> 7) * NIBP_T1 + (r & 127)
                          : r < 1792 ? NIBP_O2 + (r - 1024) / 96 * NIBP_T23 + (r - 1024) % 96
                                     : NIBP_O3 + (r - 1792) / 96 * NIBP_T23 + (r - 1792) % 96;
            s_crcnib[k * NIBP_KIND + dst] = tab.crc_nib[i];
        }
    } else {
        for (int i = tid; i < 2 * CRN_CRC_NIB_WORDS; i += BLOCK) s_crcnib[i] = tab.crc_nib[i];
    }

    /* TMEM: the whole 512 columns (one CTA per SM: the shared-memory footprint guarantees it) */
    if ((tid >> 5) == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" :: "r"(smem_addr(&s_tmem)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const u32 tmem = s_tmem;

    /* Tasks are claimed one ahead (claim_next): task t+1's metadata and LLRs
     * move on-chip / into L2 while task t decodes -- while the batch still has
     * more than two tasks per task slot left; near its end a slot claims only
     * when it is free, so no task waits behind a busy one while a slot idles.
     * The host orders whole-CTA tasks (W = 32 with sum K <= 6144, and the split
     * path) before group tasks (crn_task.grp); a CTA that claims a group task
     * switches to three groups of four warps, each claiming its own tasks. */
    const int slots = (int)gridDim.x * G3;
    auto ahead = [&]() { return *(volatile int *)counter + slots < n_tasks; };
    const NextSh nx{&s_ntask[0], &s_ntk[0], s_ncb, s_nF, s_nkind, PURGE ? s_ntb : nullptr, s_nbo, s_neo};
    prof_init();
    if (tid < 32) claim_next(nx, counter, n_tasks, tasks, pairs, desc, l0, l1, l2, tid, sh8);
    bool pend = false;                          /* warp 0: the next task is still to be claimed */
    bool grp_mode = false;
    for (;;) {
        if (pend && tid < 32) claim_next(nx, counter, n_tasks, tasks, pairs, desc, l0, l1, l2, tid, sh8);
        __syncthreads();                        /* next slots filled */
        const int task = s_ntask[0];
        if (task >= n_tasks) break;
        const crn_task tk = s_ntk[0];
        if (tk.grp) {                           /* group tasks from here on: group 0 holds this one */
            grp_mode = true;
            break;
        }
        for (int e = tid; e < 2 * tk.n_pairs; e += BLOCK) {
            const int cb = s_ncb[e];
            s_cb[e] = cb;
            s_F[e] = s_nF[e];
            s_kind[e] = s_nkind[e];
            s_bo[e] = s_nbo[e];
            s_eo[e] = s_neo[e];
            s_done[e] = cb < 0;
            s_fin[e] = 0;
            s_crc[e] = 0;
            s_mi[e] = 0;
            s_mip[e] = 0;
            if (PURGE) s_tb[e] = s_ntb[e];
            /* purge ("purge waiting CCDU of the same TB"): a waiting CB
             * whose TB already lost a CB is not decoded: crc_ok = 0, iters_used = 0 */
            if (PURGE && cb >= 0 && s_ntb[e] >= 0 && *(volatile uint8_t *)&tb_dead[s_ntb[e]]) {
                s_done[e] = 1;
                crc_ok[cb] = 0;
                if (iters_used) iters_used[cb] = 0;
            }
        }
        __syncthreads();                        /* next slots consumed */
        prof_mark(P_FB);
        auto claim_ahead = [&]() {
            if (tid < 32) {
                pend = !ahead();
                if (!pend) claim_next(nx, counter, n_tasks, tasks, pairs, desc, l0, l1, l2, tid, sh8);
            }
        };
        if constexpr (!(ETC || ROLL)) claim_ahead();
        if (PURGE) {                            /* a fully purged task is skipped */
            if (tid == 0) {
                int left = 0;
                for (int e = 0; e < 2 * tk.n_pairs; e++) left += !s_done[e];
                s_left[0] = left;
            }
            __syncthreads();
            if (s_left[0] == 0) continue;
        }
        prof_mark(P_FETCH);
        if (tid == 0) trace_task(task, 0, 0);
        /* VAR = LOGMAP: its own kernels; otherwise MAXLOG / SCALED chosen per launch */
#define CRN_RUN(V)                                                                                                \
        do {                                                                                                      \
            if constexpr (ETC || ROLL) {                                                                          \
                if (tk.W == 32) {                                                                                 \
                    run_task_fast<V, PURGE, LLR8, 1, ROLL, ETC>(tk, desc, l0, l1, l2, max_iters, et, out_bits,    \
                                                                crc_ok, iters_used, ext_out, tab, smem, tmem, sh, \
                                                                pg, sh8, claim_ahead);                            \
                } else {                                                                                          \
                    claim_ahead();                                                                                \
                    run_task_split<V, PURGE, LLR8, ROLL ? 1 : 2>(tk, desc, l0, l1, l2, max_iters, et, out_bits,   \
                                                                 crc_ok, iters_used, ext_out, tab, smem, tmem,    \
                                                                 sh, pg, sh8);                                    \
                }                                                                                                 \
            } else if (tk.W == 32) {                                                                              \
                run_task_fast<V, PURGE, LLR8, 1>(tk, desc, l0, l1, l2, max_iters, et, out_bits, crc_ok,           \
                                                 iters_used, ext_out, tab, smem, tmem, sh, pg, sh8);              \
            } else {                                                                                              \
                run_task_split<V, PURGE, LLR8, 0>(tk, desc, l0, l1, l2, max_iters, et, out_bits, crc_ok,          \
                                                  iters_used, ext_out, tab, smem, tmem, sh, pg, sh8);             \
            }                                                                                                     \
        } while (0)
        if constexpr (VAR == CRN_VARIANT_LOGMAP) CRN_RUN(CRN_VARIANT_LOGMAP);
        else if ((variant & 0xFF) == CRN_VARIANT_SCALED) CRN_RUN(CRN_VARIANT_SCALED);
        else CRN_RUN(CRN_VARIANT_MAXLOG);
#undef CRN_RUN
        if (tid == 0) trace_task(task, 1, 0);
    }
    if (grp_mode) {                             /* CTA-uniform */
        const int g = tid / GB3, ltid = tid - g * GB3, eb = 2 * GPB3 * g;
        const NextSh ng{&s_ntask[g], &s_ntk[g], s_ncb + eb, s_nF + eb, s_nkind + eb, PURGE ? s_ntb + eb : nullptr,
                        s_nbo + eb, s_neo + eb};
        bool gpend = g > 0;                     /* group 0 starts with the task the CTA claimed */
        /* groups 1 and 2 claim only after every CTA has claimed its first task: a
         * small batch (one task per CTA, crn_launch_tasks) then stays spread over the SMs */
        if (g > 0 && ltid < 32)
            while (*(volatile int *)counter < (int)gridDim.x) __nanosleep(128);
        for (;;) {
            if (gpend && ltid < 32) claim_next(ng, counter, n_tasks, tasks, pairs, desc, l0, l1, l2, ltid, sh8);
            gsync<G3>(g);                       /* next slots filled */
            const int task = s_ntask[g];
            if (task >= n_tasks) break;
            const crn_task tk = s_ntk[g];
            if (!tk.grp) __trap();              /* host invariant: group tasks are the batch's last */
            for (int e = eb + ltid; e < eb + 2 * tk.n_pairs; e += GB3) {
                const int cb = s_ncb[e];
                s_cb[e] = cb;
                s_F[e] = s_nF[e];
                s_kind[e] = s_nkind[e];
                s_bo[e] = s_nbo[e];
                s_eo[e] = s_neo[e];
                s_done[e] = cb < 0;
                s_fin[e] = 0;
                s_crc[e] = 0;
                s_mi[e] = 0;
                s_mip[e] = 0;
                if (PURGE) s_tb[e] = s_ntb[e];
                if (PURGE && cb >= 0 && s_ntb[e] >= 0 && *(volatile uint8_t *)&tb_dead[s_ntb[e]]) {
                    s_done[e] = 1;
                    crc_ok[cb] = 0;
                    if (iters_used) iters_used[cb] = 0;
                }
            }
            gsync<G3>(g);                       /* next slots consumed */
            if (ltid < 32) {
                gpend = !ahead();
                if (!gpend) claim_next(ng, counter, n_tasks, tasks, pairs, desc, l0, l1, l2, ltid, sh8);
            }
            if (PURGE) {
                if (ltid == 0) {
                    int left = 0;
                    for (int e = eb; e < eb + 2 * tk.n_pairs; e++) left += !s_done[e];
                    s_left[g] = left;
                }
                gsync<G3>(g);
                if (s_left[g] == 0) continue;
            }
            if (ltid == 0) trace_task(task, 0, 1 + g);
            if constexpr (VAR == CRN_VARIANT_LOGMAP)
                run_task_fast<CRN_VARIANT_LOGMAP, PURGE, LLR8, G3, ROLL, ETC>(tk, desc, l0, l1, l2, max_iters, et, out_bits,
                                                                   crc_ok, iters_used, ext_out, tab, smem, tmem, sh,
                                                                   pg, sh8);
            else if ((variant & 0xFF) == CRN_VARIANT_SCALED)
                run_task_fast<CRN_VARIANT_SCALED, PURGE, LLR8, G3, ROLL, ETC>(tk, desc, l0, l1, l2, max_iters, et, out_bits,
                                                                   crc_ok, iters_used, ext_out, tab, smem, tmem, sh,
                                                                   pg, sh8);
            else
                run_task_fast<CRN_VARIANT_MAXLOG, PURGE, LLR8, G3, ROLL, ETC>(tk, desc, l0, l1, l2, max_iters, et, out_bits,
                                                                   crc_ok, iters_used, ext_out, tab, smem, tmem, sh,
                                                                   pg, sh8);
            if (ltid == 0) trace_task(task, 1, 1 + g);
        }
    }
    prof_flush();
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if ((tid >> 5) == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" :: "r"(tmem));
}

size_t smem_bytes() { return (size_t)SMEM_WORDS * 4; }
size_t smem_bytes_p() { return (size_t)SMEM_WORDS_P * 4; }   /* CRC-ET and latency kernels */

}  // namespace

extern "C" size_t crn_decode_ws_bytes(int32_t) { return WS_HEAD; }

extern "C" int crn_decode_set_logmap(uint32_t lo, uint32_t hi) {
    const u32 w[2] = {lo, hi};
    return cudaMemcpyToSymbol(c_logmap, w, sizeof(w)) == cudaSuccess ? CRN_OK : CRN_ECUDA;
}   /* the task counter; all decode state is on chip */

/* the instantiations: <purge?, int8 LLRs?, variant> and the two latency (ROLL) kernels */
template <class F>
cudaError_t for_each_kernel(F &&f) {
    const void *k[] = {
        (const void *)decode_kernel<false, false, CRN_VARIANT_MAXLOG>, (const void *)decode_kernel<true, false, CRN_VARIANT_MAXLOG>,
        (const void *)decode_kernel<false, true, CRN_VARIANT_MAXLOG>, (const void *)decode_kernel<true, true, CRN_VARIANT_MAXLOG>,
        (const void *)decode_kernel<false, false, CRN_VARIANT_LOGMAP>, (const void *)decode_kernel<true, false, CRN_VARIANT_LOGMAP>,
        (const void *)decode_kernel<false, true, CRN_VARIANT_LOGMAP>, (const void *)decode_kernel<true, true, CRN_VARIANT_LOGMAP>,
        (const void *)decode_kernel<false, false, CRN_VARIANT_MAXLOG, true>,
        (const void *)decode_kernel<false, true, CRN_VARIANT_MAXLOG, true>,
        (const void *)decode_kernel<false, false, CRN_VARIANT_MAXLOG, false, true>};
    cudaError_t e = cudaSuccess;
    for (const void *x : k)
        if (e == cudaSuccess) e = f(x);
    return e;
}

extern "C" int crn_decode_grid(int device) {
    /* returns the persistent grid (one CTA per SM), or a negative code:
     * -100 - cudaError of the smem attribute, -200 - cudaError of the occupancy
     * query, -300 - occupancy (must be exactly 1: the CTA owns all TMEM columns),
     * -400: static shared memory pushes the Y / Z planes past 64 KiB */
    static int configured = -1;
    if (configured != device) {
        cudaError_t e = for_each_kernel([](const void *k) {
            return cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_bytes_p());
        });
        if (e != cudaSuccess) return -100 - (int)e;
        configured = device;
    }
    int sms = 0, bad = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    /* the fast path's packed gather addresses: static + Y / Z planes below 64 KiB */
    cudaError_t e = for_each_kernel([&](const void *k) {
        cudaFuncAttributes a;
        cudaError_t r = cudaFuncGetAttributes(&a, k);
        if (r == cudaSuccess && a.sharedSizeBytes + YZ_END_BYTES > 65536) bad = -1;
        return r;
    });
    if (e != cudaSuccess) return -200 - (int)e;
    if (bad) return -400;
    e = for_each_kernel([&](const void *k) {
        int occ = 0;
        cudaError_t r = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, BLOCK, smem_bytes_p());
        if (r == cudaSuccess && occ != 1) bad = occ ? occ : -1;
        return r;
    });
    if (e != cudaSuccess) return -200 - (int)e;
    if (bad) return -300 - (bad > 0 ? bad : 0);
    return sms;
}

extern "C" int crn_decode_kernel_info(int32_t *static_smem, int32_t *dyn_smem, int32_t *max_dyn, int32_t *regs) {
    cudaFuncAttributes a;
    if (cudaFuncGetAttributes(&a, decode_kernel<false, false, CRN_VARIANT_MAXLOG>) != cudaSuccess) return CRN_ECUDA;
    *static_smem = (int32_t)a.sharedSizeBytes;
    *dyn_smem = (int32_t)smem_bytes();
    *max_dyn = a.maxDynamicSharedSizeBytes;
    *regs = a.numRegs;
    return CRN_OK;
}

extern "C" int crn_launch_decode(const crn_cb_desc *d_desc, const crn_task *d_tasks, int32_t n_tasks,
                                 const crn_pair *d_pairs, const int16_t *l0, const int16_t *l1, const int16_t *l2,
                                 int32_t max_iters, int32_t et, uint32_t *bits, uint8_t *ok, uint8_t *it,
                                 int16_t *ext, const crn_tables *tab, void *ws, void *stream, int32_t grid,
                                 int32_t variant, uint8_t *tb_dead, int32_t ws_zeroed) {
    cudaStream_t st = (cudaStream_t)stream;
    if (!ws_zeroed && cudaMemsetAsync(ws, 0, WS_HEAD, st) != cudaSuccess) return CRN_ECUDA;
    const int g = (n_tasks >= 0 && n_tasks < grid) ? n_tasks : grid;   /* n_tasks < 0: the count is in ws[1] */
    const bool llr8 = (variant >> 8) != 0;      /* crn_plan_set_llr_format: int8 LLRs */
    const int var = variant & 0xFF;
#define CRN_LAUNCH(PG, L8, V)                                                                                      \
    decode_kernel<PG, L8, V><<<g, BLOCK, smem_bytes(), st>>>(d_desc, d_tasks, n_tasks, d_pairs, l0, l1, l2,         \
                                                             max_iters, et, bits, ok, it, ext, *tab, (uint8_t *)ws, \
                                                             variant, PG ? tb_dead : nullptr)
#define CRN_LAUNCH_V(PG, L8)                                                                                       \
    do {                                                                                                           \
        if (var == CRN_VARIANT_LOGMAP) CRN_LAUNCH(PG, L8, CRN_VARIANT_LOGMAP);                                     \
        else CRN_LAUNCH(PG, L8, CRN_VARIANT_MAXLOG);   /* MAXLOG or SCALED, chosen inside */                       \
    } while (0)
    /* a batch that fits one wave (every task its own CTA) runs the latency kernel:
     * rolled phase 1, one SISO call site (CRN_ROLL=0 / 1 forces it off / on) */
    static const int roll_env = [] {
        const char *e = getenv("CRN_ROLL");
        return e ? (e[0] == '1' ? 1 : 0) : -1;
    }();
    const bool roll = !tb_dead && var != CRN_VARIANT_LOGMAP &&
                      (roll_env >= 0 ? roll_env == 1 : (n_tasks > 0 && n_tasks <= grid));
    if (roll) {
        if (llr8) decode_kernel<false, true, CRN_VARIANT_MAXLOG, true><<<g, BLOCK, smem_bytes_p(), st>>>(
            d_desc, d_tasks, n_tasks, d_pairs, l0, l1, l2, max_iters, et, bits, ok, it, ext, *tab, (uint8_t *)ws,
            variant, nullptr);
        else decode_kernel<false, false, CRN_VARIANT_MAXLOG, true><<<g, BLOCK, smem_bytes_p(), st>>>(
            d_desc, d_tasks, n_tasks, d_pairs, l0, l1, l2, max_iters, et, bits, ok, it, ext, *tab, (uint8_t *)ws,
            variant, nullptr);
    } else if (!tb_dead && !llr8 && var != CRN_VARIANT_LOGMAP && et == CRN_ET_CRC) {
        /* CRC early termination, int16 LLRs: the kernel with the branch-free hard decision */
        decode_kernel<false, false, CRN_VARIANT_MAXLOG, false, true><<<g, BLOCK, smem_bytes_p(), st>>>(
            d_desc, d_tasks, n_tasks, d_pairs, l0, l1, l2, max_iters, et, bits, ok, it, ext, *tab, (uint8_t *)ws,
            variant, nullptr);
    } else if (tb_dead) {
        if (llr8) CRN_LAUNCH_V(true, true);
        else CRN_LAUNCH_V(true, false);
    } else {
        if (llr8) CRN_LAUNCH_V(false, true);
        else CRN_LAUNCH_V(false, false);
    }
#undef CRN_LAUNCH_V
#undef CRN_LAUNCH
    return cudaGetLastError() == cudaSuccess ? CRN_OK : CRN_ECUDA;
}

#ifdef CRN_PHASE_PROF
/* phase profiler readout (profiling builds only): 2 x P_N cycle sums, then reset */
extern "C" int crn_prof_read(unsigned long long *out) {
    if (cudaMemcpyFromSymbol(out, g_prof, sizeof(unsigned long long) * 2 * P_N) != cudaSuccess) return CRN_ECUDA;
    static const unsigned long long z[2 * P_N] = {};
    cudaMemcpyToSymbol(g_prof, z, sizeof(z));
    return CRN_OK;
}
#endif

#ifdef CRN_TASK_TRACE
/* task trace readout (tracing builds only): 4 words per task (start ns, end ns, SM, group), then reset */
extern "C" int crn_trace_read(unsigned long long *out, int32_t n_tasks) {
    const size_t n = (size_t)(n_tasks < TRACE_MAX ? n_tasks : TRACE_MAX) * 4;
    if (cudaMemcpyFromSymbol(out, g_trace, n * sizeof(unsigned long long)) != cudaSuccess) return CRN_ECUDA;
    return CRN_OK;
}
#endif
