/* crn_internal.h -- structures shared by libcrn's host code and its kernels.
 * Not part of the ABI (see include/crn.h). */
#pragma once
#include <stddef.h>
#include <stdint.h>

#include "../../include/crn.h"

#define CRN_NSTATE 8
#ifndef CRN_NUM_K
#define CRN_NUM_K 188      /* the LTE interleaver sizes (qpp_table.h) */
#endif
#define CRN_MI_EPS 66      /* MI stopping rule: per-bit change threshold in Q16 (R29) */
/* Decode work unit: one CTA task = n_pairs pairs of CBs with the same K; the
 * two CBs of a pair share every int16x2 register (lo half / hi half), so all
 * trellis arithmetic is pair-SIMD and the 8-state butterfly is a register
 * rename.  Thread t = p*M + j owns window j of pair p.  Sum of K over a task
 * is <= CRN_TASK_SUMK, hence T = n_pairs*M <= CRN_TASK_SUMK/32 = CRN_CTA_THREADS. */
#define CRN_TASK_SUMK 6144
#define CRN_CTA_THREADS 192
/* At most this many CB pairs per task (bounds the per-task shared arrays). */
#define CRN_MAX_PAIRS 96

typedef struct {
    int32_t K, M, W, n_pairs;
    int32_t pair0;   /* first pair index of the task */
    int32_t kidx;    /* index of K in the size table */
    int32_t grp;     /* 1: a group task (W = 32, n_pairs*M <= CRN_GRP_WIN), run by four warps while the
                        CTA's other eight run two more; group tasks follow every whole-CTA task */
} crn_task;

/* Group tasks (W = 32 path, crn_decode.cu): a CTA runs three tasks of up to
 * CRN_GRP_WIN windows (sum K <= CRN_GRP_SUMK, <= CRN_GRP_PAIRS pairs) at once. */
#define CRN_GROUPS 3
#define CRN_GRP_SUMK 2048
#define CRN_GRP_WIN 64
#define CRN_GRP_PAIRS 32

typedef struct {
    int32_t lo, hi;  /* CB indices; hi = -1 for the dummy partner of an odd bucket */
} crn_pair;

/* Split-window path for W in 33..62 (crn_decode.cu run_task_split): a task of
 * n_pairs pairs has T = n_pairs*M windows, Tp = T rounded up to 32; the head
 * thread of a window owns steps [0, hw) with hw = ceil(W/2), the tail thread
 * [hw, W).  Shared-memory words of its layout (row stride Tp):
 *   Y, Z (extrinsics) W*Tp each | Lp1, Lp2 W*Tp each | Q1, Q2 (per-thread QPP
 *   word indices) hw*2Tp each | CH (branch-metric pairs) 2*hw*2Tp |
 *   NII 32*Tp | X (hand-over / hard-decision bits) 16*Tp | tail beta 16*n_pairs
 * and TMEM columns per thread 10*hw (8 per stored step + 2 static sums), one
 * 10*hw block per group of 4 warps.  The host sizes n_pairs so both fit. */
#define CRN_SMEM_WORDS 47616
#define CRN_TMEM_COLS 512
static inline int crn_split_tp(int T) { return (T + 31) & ~31; }
static inline int crn_split_smem_words(int W, int M, int n_pairs) {
    const int T = n_pairs * M, Tp = crn_split_tp(T), hw = (W + 1) / 2;
    return 4 * W * Tp + 8 * hw * Tp + 48 * Tp + 16 * n_pairs;
}
static inline int crn_split_tmem_cols(int W, int M, int n_pairs) {
    const int Tp = crn_split_tp(n_pairs * M), hw = (W + 1) / 2;
    return ((2 * Tp + 127) / 128) * 10 * hw;
}
static inline int crn_split_fits(int W, int M, int n_pairs) {
    return n_pairs * M <= CRN_CTA_THREADS && crn_split_smem_words(W, M, n_pairs) <= CRN_SMEM_WORDS &&
           crn_split_tmem_cols(W, M, n_pairs) <= CRN_TMEM_COLS;
}

/* Window CRC of the W = 32 decode path (row a9).  With K = 32 M, window j's
 * packed hard decisions w (bit i = message bit 32 j + i, MSB-first order)
 * contribute x^(32 d) * R(w) mod g to the CRC register, d = M - 1 - j, R(w) =
 * sum_i w_i x^(55 - i) mod g; d = 64 a + 8 b + c (a <= 2) is applied as three
 * fixed linear maps, each an XOR of nibble-table lookups (bank-conflict-free
 * 16-word tables):
 *   [0, 1024)     TRC[c][q][v] = (sum over bits k of v of x^(55 - 4q - k)) x^(32 c) mod g, q = 0..7
 *   [1024, 1792)  TB[b][q][v]  = (v x^(4q)) x^(256 b) mod g, q = 0..5
 *   [1792, 2080)  TA[a][q][v]  = (v x^(4q)) x^(2048 a) mod g, q = 0..5          */
#define CRN_CRC_NIB_WORDS 2080

/* Device record of one TB for crn_tb_build_cbs_batch (crn_tbseg.cu). */
typedef struct {
    int64_t tbs, payload_off, cb_bit0;     /* payload bits; bit 0's byte in payload; CB 0's first byte in cb_bits */
    int32_t C, Kplus, Kminus, Cminus, F, L;
} crn_tbseg;

/* Max CBs per TB accepted by crn_tb_verdict_batch (LTE needs <= 64). */
#define CRN_TB_MAX_CB 128

/* Per-device constant tables (built once on the host, uploaded once). */
typedef struct {
    const uint32_t *qpp_wm;   /* per K at qpp_off[kidx]: [i*M + j] = (Pi(jW+i) % W) << 16 | Pi(jW+i) / W */
    const uint32_t *qpp_ts;   /* same index: (Pi(jW+i) % W) * CRN_CTA_THREADS + Pi(jW+i) / W (fast path) */
    const uint32_t *qinv_ts;  /* same index, inverse permutation: m = Pi^-1(jW+i) -> (m % W) * CRN_CTA_THREADS + m / W */
    const uint32_t *qinv_wm;  /* same index, inverse permutation in the qpp_wm format: (m % W) << 16 | m / W */
    const uint32_t *crc_bit;  /* per K at crcb_off[kidx]: [kind(0=A,1=B)*K + i*M + j] = x^(K-1-n+24) mod g, n = jW+i:
                                 the CRC register contribution of a 1 at bit n (register = XOR over the set bits) */
    const int32_t *mi_tab;    /* [256] Q16 MI of an LLR of magnitude a/8 (crn_mi_table, R29) */
    const uint32_t *crc_nib;  /* [2][CRN_CRC_NIB_WORDS] (CRC24A, CRC24B): nibble tables of the W = 32 path's
                                 window CRC, see CRN_CRC_NIB_WORDS */
    const int32_t *qpp_off;
    const int32_t *crcb_off;
} crn_tables;

#ifdef __cplusplus
extern "C" {
#endif
/* crn_decode.cu */
int crn_launch_decode(const crn_cb_desc *d_desc, const crn_task *d_tasks, int32_t n_tasks,
                      const crn_pair *d_pairs, const int16_t *l0, const int16_t *l1,
                      const int16_t *l2, int32_t max_iters, int32_t early_term,
                      uint32_t *out_bits, uint8_t *crc_ok, uint8_t *iters_used, int16_t *ext_out,
                      const crn_tables *tab, void *ws, void *stream, int32_t grid, int32_t variant,
                      uint8_t *tb_dead, int32_t ws_zeroed);
size_t crn_decode_ws_bytes(int32_t grid);
/* Log-MAP correction LUT[0..7] as two byte-packed words into the decode kernel's
 * constant bank (crn_logmap_lut, R32); once per device. */
int crn_decode_set_logmap(uint32_t lo, uint32_t hi);
int crn_decode_grid(int device);
/* crn_tasks.cu: row a1 on the device for descriptors in device memory.  bucket[4 k ..] = K, M, W,
 * pairs per task | group flag << 16 of size index k; border[q] = the size index issued q-th.
 * scratch >= crn_tasks_dev_bytes(n_cb); hdr[0] = 0 (task counter), hdr[1] = task count. */
size_t crn_tasks_dev_bytes(int32_t n_cb);
int crn_launch_tasks_dev(const crn_cb_desc *d_desc, int32_t n_cb, int32_t want_ext, int32_t purge,
                         const int32_t *bucket, const int32_t *border, void *scratch, int32_t *hdr,
                         crn_task **tasks, crn_pair **pairs, uint8_t **dead, uint8_t *crc_ok,
                         uint8_t *iters_used, void *stream);
/* crn_encode.cu */
int crn_launch_encode(const crn_cb_desc *d_desc, int32_t n_cb, const void *info, int32_t attach_crc,
                      void *d0, void *d1, void *d2, int32_t packed, const crn_tables *tab, void *stream);
/* crn_tb.cu */
int crn_launch_tb(const crn_tb_desc *d_tbs, int32_t n_tb, const crn_cb_desc *d_desc, const uint32_t *cb_words,
                  const uint8_t *crc_ok, uint8_t *tb_ok, uint32_t *tb_words, void *stream);
/* crn_ratematch.cu */
int crn_launch_dematch(const crn_rm_desc *d_desc, int32_t n_cb, const int16_t *e, int32_t combine, int16_t *h0,
                       int16_t *h1, int16_t *h2, void *stream);
int crn_launch_match(const crn_rm_desc *d_desc, int32_t n_cb, const uint8_t *d0, const uint8_t *d1,
                     const uint8_t *d2, uint8_t *e, void *stream);
/* packed-bit matching: stream bits at bit offset llr_off, e bits at bit offset e_off */
int crn_launch_match_packed(const crn_rm_desc *d_desc, int32_t n_cb, const uint32_t *d0, const uint32_t *d1,
                            const uint32_t *d2, uint32_t *e, void *stream);
/* crn_tbseg.cu */
int crn_launch_tbseg(const crn_tbseg *d_tbs, int32_t n_tb, int64_t max_tbs, const uint8_t *payload, uint8_t *cb_bits,
                     void *stream);
/* crn_ubench.cu */
int crn_launch_ubench(int32_t op, int64_t *lane_instr, float *ms, int64_t *cycles_per_block);
/* crn_host.cpp */
int crn_k_index(int32_t K);
#ifdef __cplusplus
}
#endif
