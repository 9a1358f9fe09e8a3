/*
 * oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, obviously-correct CPU reference for the hot path of
 * arxiv 1905.01141 (uplink channel decoding of a pooled C-RAN BBU):
 * LTE turbo decoding, int16-range fixed-point max-log-MAP, QPP interleaver,
 * windowed recursions with next-iteration initialisation (NII), CRC24
 * early termination, hard decision.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load this library.  The product (paper_1905_01141_b200/, libcrn) never
 * links, imports or calls it, and shares no code, table or header with it.
 *
 * Citations: "PAPER.md:<line>" is /root/reference/PAPER.md (the paper text),
 * "SPEC.md:<line>" the CPU-program spec written from it, "DESIGN.md R<n>" a
 * reading of a passage where the paper is silent (listed in DESIGN.md).
 *
 * Parity pins: every function is pinned by tests/test_oracle_*.py EXCEPT the
 * exact 3GPP (f1,f2) QPP values, which are recalled (TS 36.212 Table 5.1.3-3
 * is not in the container): "parity unpinned" for 3GPP interop of those
 * values; their permutation / contention-free properties are pinned.
 */
#ifndef CRN_ORACLE_H
#define CRN_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { ORACLE_CRC_NONE = 0, ORACLE_CRC24A = 1, ORACLE_CRC24B = 2 };
/* Decoder variants: plain max-log-MAP (the product definition, R2) and
 * the scaled-extrinsic max-log-MAP of SURVEY.md §8(f) f2 (R28): each
 * SISO's extrinsic Le = clamp(L1 - L0, +-4096) is handed on as floor(3 Le / 4). */
/* and Log-MAP (f2, R32): every two-way selection of the recursions and
 * of Lambda is max*(a, b) = max(a, b) + c(|a - b|) (oracle_max_star). */
enum { ORACLE_VAR_MAXLOG = 0, ORACLE_VAR_SCALED = 1, ORACLE_VAR_LOGMAP = 2 };
/* Log-MAP correction c(d) = LUT[min(d >> 2, 7)], LUT[b] = round(8 ln(1 + e^(-(4b+1.5)/8)));
 * -1 for d < 0.  max*(a, b) = max(a, b) + c(|a - b|). */
int32_t oracle_logmap_correction(int32_t d);
int32_t oracle_max_star(int32_t a, int32_t b);
/* Stopping rules (early_term): none (fixed iterations), CRC (R3), or
 * the paper's average-MI convergence (R29). */
enum { ORACLE_ET_NONE = 0, ORACLE_ET_CRC = 1, ORACLE_ET_MI = 2 };
#define ORACLE_MI_EPS 66   /* per-bit MI change threshold in Q16 (about 0.001) */
/* Q16 MI of an LLR of magnitude a/8, a saturated at 255 (R29); -1 for a < 0. */
int32_t oracle_mi_table(int32_t a);

/* Number of supported interleaver sizes (188 sizes 40..6144). */
int oracle_num_k(void);
/* i-th supported K (ascending); -1 if out of range. */
int oracle_k_at(int i);
/* (f1, f2) for K; returns 0, or -1 if K is not a supported size. */
int oracle_qpp_params(int K, int *f1, int *f2);
/* Pi(i) = (f1*i + f2*i^2) mod K; -1 if K unsupported. */
int oracle_qpp_index(int K, int i);

/* CRC register after feeding nbits bits (one bit per byte, MSB-first order,
 * zero initial register, no reflection, no final xor) through generator
 * CRC24A (D^24+D^23+D^18+D^17+D^14+D^11+D^10+D^7+D^6+D^5+D^4+D^3+D+1) or
 * CRC24B (D^24+D^23+D^6+D^5+D+1).  A block is valid iff the register is 0
 * after all its bits, parity included.  DESIGN.md R7. */
uint32_t oracle_crc24(int kind, const uint8_t *bits, int64_t nbits);

/* TB -> CB segmentation (36.212 5.1.2; Algorithm 1 with
 * CB_MAX_SIZE = 6120 = 6144 - 24; R4). B = tbs + 24. */
typedef struct { int32_t C, Kplus, Kminus, Cplus, Cminus, F, L; } oracle_seg;
int oracle_segment(int64_t tbs_bits, oracle_seg *out);

/* Window split: M = max{M : M | K, K/M >= wmin}; returns M (W = K/M). */
int oracle_num_windows(int K, int wmin);

/* Rate-1/3 turbo encoder: c[0..K) -> d0,d1,d2[0..K+4)
 * (36.212 5.1.3.2 stream layout incl. 12 tail bits; R11).
 * Returns 0, -1 if K unsupported. */
int oracle_turbo_encode(const uint8_t *c, int K, uint8_t *d0, uint8_t *d1, uint8_t *d2);

/* One constituent SISO pass (one half-iteration) over a block of K steps
 * split into M = K/W windows (R12/R13).
 *   lsys, lpar, la : int16-range values for k in [0,K) (already clamped)
 *   tail[6]        : (x_K, z_K, x_K+1, z_K+1, x_K+2, z_K+2)
 *   alpha_in [M][8]: alpha_{jW} used by window j >= 1 (row 0 ignored: known start state)
 *   beta_in  [M][8]: beta_{(j+1)W} used by window j <= M-2 (row M-1 ignored: tail)
 *   alpha_out[M][8]: alpha_{(j+1)W} produced by window j   (may be NULL)
 *   beta_out [M][8]: beta_{jW} produced by window j        (may be NULL)
 *   le[K]          : extrinsic output
 *   ops            : counted-operation accumulator (may be NULL)
 * Returns the number of int16-range violations observed (0 expected). */
int64_t oracle_siso(const int32_t *lsys, const int32_t *lpar, const int32_t *la,
                    const int32_t *tail, int K, int W,
                    const int32_t *alpha_in, const int32_t *beta_in,
                    int32_t *alpha_out, int32_t *beta_out,
                    int32_t *le, uint64_t *ops);

/* Same with a decoder variant (ORACLE_VAR_LOGMAP: max* selections; the others
 * are plain max-log-MAP SISOs). */
int64_t oracle_siso_v(const int32_t *lsys, const int32_t *lpar, const int32_t *la,
                      const int32_t *tail, int K, int W,
                      const int32_t *alpha_in, const int32_t *beta_in,
                      int32_t *alpha_out, int32_t *beta_out,
                      int32_t *le, uint64_t *ops, int variant);

/* NII hand-over between iterations (R13): alpha_in[j] <- alpha_out[j-1]
 * (j >= 1), beta_in[j] <- beta_out[j+1] (j <= M-2); the unused rows are zeroed. */
void oracle_nii_update(int M, const int32_t *alpha_out, const int32_t *beta_out,
                       int32_t *alpha_in, int32_t *beta_in);

/* Full iterative decode of one CB (R1-R19).
 *   d0,d1,d2 : the K+4 received int16 LLRs of each stream (positive => bit 1)
 *   F        : number of leading filler bits (known 0)
 *   crc_kind : ORACLE_CRC_NONE / 24A / 24B (the check used for ET and crc_ok)
 *   max_iters: I >= 1;  early_term: ORACLE_ET_CRC stops after the first full
 *              iteration whose hard decision passes the CRC; ORACLE_ET_MI after the
 *              first iteration t >= 2 whose MI statistic sum_{n>=F} mi_table(|L_APP_n|)
 *              moved by at most (K-F)*ORACLE_MI_EPS from iteration t-1
 *   wmin     : minimum window length (32 in the product definition; K forces M = 1)
 * Outputs: bits[K] (0/1 per byte), *crc_ok, *iters_used, ext[K] (La1_next of
 * the last iteration, natural order), *ops (counted ops, accumulated).
 * Returns the number of int16-range violations (0 expected), or -1 if the
 * arguments are invalid. */
int64_t oracle_decode_cb(const int16_t *d0, const int16_t *d1, const int16_t *d2,
                         int K, int F, int crc_kind, int max_iters, int early_term, int wmin,
                         uint8_t *bits, uint8_t *crc_ok, uint8_t *iters_used,
                         int16_t *ext, uint64_t *ops);

/* The variant's extrinsic scaling s(x) = floor(3x / 4) (R28). */
int32_t oracle_ext_scale(int32_t x);

/* Same with a decoder variant (ORACLE_VAR_*): with ORACLE_VAR_SCALED, Le1 and
 * Le2 are replaced by floor(3 Le / 4) right after each SISO, so the a-priori
 * inputs, L_APP and ext all use the scaled values.  -1 for an unknown variant. */
int64_t oracle_decode_cb_v(const int16_t *d0, const int16_t *d1, const int16_t *d2,
                           int K, int F, int crc_kind, int max_iters, int early_term, int wmin, int variant,
                           uint8_t *bits, uint8_t *crc_ok, uint8_t *iters_used,
                           int16_t *ext, uint64_t *ops);

/* Batch helper for the CPU baseline: CB i uses K[i], F[i], crc_kind[i]; its
 * LLRs start at llr_off[i] in each of d0/d1/d2, its K bits at bit_off[i] in
 * bits (one per byte), its ext at bit_off[i] in ext (may be NULL).
 * Runs nthreads POSIX threads, one CB per task.  Returns total violations. */
int64_t oracle_decode_batch(int n_cb, const int32_t *K, const int32_t *F, const int32_t *crc_kind,
                            const int64_t *llr_off, const int64_t *bit_off,
                            const int16_t *d0, const int16_t *d1, const int16_t *d2,
                            int max_iters, int early_term, int nthreads,
                            uint8_t *bits, uint8_t *crc_ok, uint8_t *iters_used,
                            int16_t *ext, uint64_t *ops);
int64_t oracle_decode_batch_v(int n_cb, const int32_t *K, const int32_t *F, const int32_t *crc_kind,
                              const int64_t *llr_off, const int64_t *bit_off,
                              const int16_t *d0, const int16_t *d1, const int16_t *d2,
                              int max_iters, int early_term, int variant, int nthreads,
                              uint8_t *bits, uint8_t *crc_ok, uint8_t *iters_used,
                              int16_t *ext, uint64_t *ops);

/* Rate matching for turbo-coded channels, TS 36.212 5.1.4.1 (row f4, DESIGN.md
 * R30): full circular buffer Ncb = 3*Kpi, Kpi = 32*ceil((K+4)/32).
 *   oracle_rm_perm(c): the sub-block inter-column permutation P(c), c in [0,32)
 *   oracle_rm_params: R rows, ND dummy bits, Kpi, and k0 for redundancy version rv
 *   oracle_rate_match: d0/d1/d2 coded bits (K+4 each) -> e[E] selected bits
 *   oracle_rate_dematch: e[E] soft values -> soft buffers h0/h1/h2 (K+4 each):
 *     h = sat16((combine ? h : 0) + sum of the values read from each position).
 * All return 0, or -1 for an unsupported K, rv outside [0,3] or E < 1. */
int oracle_rm_perm(int c);
int oracle_rm_params(int K, int rv, int *R, int *ND, int *Kpi, int *k0);
int oracle_rate_match(const uint8_t *d0, const uint8_t *d1, const uint8_t *d2, int K, int E, int rv, uint8_t *e);
int oracle_rate_dematch(const int16_t *e, int K, int E, int rv, int combine, int16_t *h0, int16_t *h1,
                        int16_t *h2);

#ifdef __cplusplus
}
#endif
#endif
