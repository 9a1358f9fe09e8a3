/*
 * crn.h -- C ABI of libcrn: B200-native batched LTE turbo decoding for a pooled
 * C-RAN BBU (the uplink channel-decoding function of arxiv 1905.01141).
 *
 * All functions are extern "C", take plain pointers and sizes, and return a
 * status (0 = CRN_OK, < 0 = error) unless stated otherwise.  No torch types.
 *
 * Citations: PAPER.md:<line> (the paper), SPEC.md:<line> (the CPU-program spec
 * written from it, used here for interface shapes), DESIGN.md R<n> (a reading
 * where the paper is silent).  The operation every decode entry point computes
 * is DESIGN.md "decoder definition": per code block (CB), demultiplex the
 * received streams, run DEC1 -> DEC2 -> de-interleave for
 * fixed or CRC-early-terminated iterations, take the hard
 * decision and check the CRC; int16 max-log-MAP on the 8-state
 * LTE RSC trellis with the QPP interleaver and M_K parallel windows (R1-R19).
 *
 * Ownership: the caller owns every buffer.  libcrn allocates only (a) a cached
 * per-device workspace + interleaver tables (guarded by a mutex) and (b) the
 * device copies held by a plan.  Decode calls are asynchronous on the given
 * CUDA stream (NULL = legacy default stream); launch errors return at once,
 * kernel faults surface as CRN_ECUDA on a later call or at the caller's sync.
 * Determinism: each CB's outputs depend only on that CB's inputs and
 * descriptor -- never on batch order, composition, stream or GPU count.
 * There is NO CPU fallback: without a usable sm_100 device every decode
 * entry point returns CRN_ENODEV.
 */
#ifndef CRN_H
#define CRN_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { CRN_OK = 0, CRN_EINVAL = -1, CRN_ECUDA = -2, CRN_ENOMEM = -3, CRN_ENODEV = -4 };
enum { CRN_CRC_NONE = 0, CRN_CRC24A = 1, CRN_CRC24B = 2 };
enum { CRN_DESC_ON_DEVICE = 1 };           /* flag bit 0 of crn_decode_batch_ex */
enum { CRN_EXT_SCALED = 2 };               /* flag bit 1: scaled-extrinsic variant (below) */
enum { CRN_PURGE = 4 };                    /* flag bit 2: purge waiting CBs of failed TBs (below) */
/* Decoder variants: CRN_VARIANT_MAXLOG is the definition
 * every entry point computes by default (R2); CRN_VARIANT_SCALED
 * hands on floor(3 Le / 4) instead of each SISO's extrinsic Le, so the
 * a-priori inputs, L_APP and ext_out all use the scaled value (R28);
 * CRN_VARIANT_LOGMAP replaces every two-way selection of the alpha / beta
 * recursions and of the Lambda fold (over the 8 transitions in state order) by
 * max*(a, b) = max(a, b) + LUT[min(|a - b| >> 2, 7)], LUT[b] = round(8 ln(1 +
 * e^(-(4b + 1.5)/8))): Log-MAP with the Jacobian correction in the LLR
 * quantiser's 1/8-nat units (R32; normalisation, clamps and NII as
 * in max-log-MAP).  Selected per plan (crn_plan_set_variant). */
enum { CRN_VARIANT_MAXLOG = 0, CRN_VARIANT_SCALED = 1, CRN_VARIANT_LOGMAP = 2 };
enum { CRN_MAX_ITERS = 32, CRN_KMIN = 40, CRN_KMAX = 6144 };
/* Stopping rules (the early_term argument of every decode entry point):
 * CRN_ET_NONE runs max_iters iterations; CRN_ET_CRC stops a CB after the first
 * full iteration whose hard decision passes its CRC (R3, R18);
 * CRN_ET_MI is the paper's rule ("the average mutual information
 * of LLR, if it converges the decoding process may terminate earlier"): after
 * each full iteration t the CB's statistic S_t = sum over non-filler n of
 * crn_mi_table[min(|L_APP(n)|, 255)] is formed, and the CB stops at the first
 * t >= 2 with |S_t - S_{t-1}| <= (K - F) * 66 (a per-bit MI change of about
 * 0.001 in Q16; R29). */
enum { CRN_ET_NONE = 0, CRN_ET_CRC = 1, CRN_ET_MI = 2 };

/* Per-CB descriptor (the paper's CCDU at CB granularity).
 *   K        interleaver size, one of the 188 LTE sizes 40..6144
 *   F        leading filler bits (known 0), 0 <= F <= K-25 (36.212 5.1.2; R6)
 *   crc_kind CRN_CRC24A (TB with C=1), CRN_CRC24B (CB of a segmented TB), or
 *            CRN_CRC_NONE (never passes; runs max iterations)          (R7)
 *   llr_off  element offset of the CB's K+4 LLRs in each of llr_sys/p1/p2
 *   bit_off  uint32-WORD offset of the CB's ceil(K/32) packed output words
 *   ext_off  element offset of the CB's K extrinsic outputs in ext_out
 *   reserved the CB's TB id (0, 1, ...; -1 = none) when purging (CRN_PURGE /
 *            crn_plan_set_purge), otherwise ignored                       */
typedef struct {
    int32_t K, F, crc_kind, reserved;
    int64_t llr_off, bit_off, ext_off;
} crn_cb_desc;

/* 36.212 5.1.2 segmentation result (Algorithm 1; R4). */
typedef struct { int32_t C, Kplus, Kminus, Cplus, Cminus, F, L; } crn_seg;

/* ------------------------------------------------------------------ decode */

/* BASELINE.json form.  iters > 0: that many fixed iterations; iters < 0:
 * CRC early termination with at most -iters iterations (R3).
 * CRC24B per CB, F = 0, dense layout: CB i's K_i+4 LLRs (positive => bit 1,
 * PAPER.md:285) start at sum_{j<i}(K_j+4) in each stream (sys = d0, p1 = d1,
 * p2 = d2 of 36.212 incl. the tail columns, R11); its hard-decision bits are
 * packed LSB-first (bit n -> word n/32, bit n%32; R19) from word
 * sum_{j<i} ceil(K_j/32) of out_bits; crc_ok[i] = 1 iff the final hard
 * decision passes CRC24B.  K[] is HOST memory, every other pointer DEVICE
 * memory.  Enqueues on the legacy default stream.  Errors: CRN_EINVAL for a K
 * outside the table, n_cb < 0, |iters| outside [1,32] or a NULL pointer. */
int crn_decode_batch(const int16_t *llr_sys, const int16_t *llr_p1, const int16_t *llr_p2,
                     const int32_t *K, int32_t n_cb, int32_t iters,
                     uint32_t *out_bits, uint8_t *crc_ok);

/* General form.  desc: n_cb descriptors in HOST memory (copied during the
 * call; the last few distinct descriptor sets are kept validated, bucketed and
 * uploaded, so a repeated layout costs one comparison), or in DEVICE memory if
 * flags & CRN_DESC_ON_DEVICE: then they are bucketed and validated on the
 * device by a task-builder kernel enqueued before the decode (nothing is copied
 * back, the call does not wait on the stream); an invalid one (K, F, crc_kind,
 * negative offsets, with CRN_PURGE a TB id outside [-1, n_cb)) yields crc_ok =
 * 0, iters_used = 0; overlapping ranges are not detected on the device.
 * max_iters in [1,32]; early_term one of CRN_ET_NONE / CRN_ET_CRC / CRN_ET_MI
 * (above; CRN_EINVAL otherwise).
 * Outputs (device memory): out_bits (required), crc_ok[n_cb] (required),
 * iters_used[n_cb] (may be NULL; full iterations executed, R17), ext_out
 * (may be NULL; int16 La1_next of the last iteration in natural order, R15).
 * workspace: NULL -> the cached per-(device, stream) workspace; else >=
 * crn_workspace_bytes(desc, n_cb) bytes of device memory owned by the caller,
 * used by this call only (stream-ordered: reusable by the next call on the
 * same stream).
 * cuda_stream: a cudaStream_t (NULL = legacy default stream).
 * Host-side validation (descriptors in host memory) returns CRN_EINVAL for a
 * K outside the table, F < 0 or F > K-25, an unknown crc_kind, overlapping
 * LLR or output ranges, or unknown flag bits.  flags & CRN_EXT_SCALED selects
 * CRN_VARIANT_SCALED.  n_cb == 0 is a no-op.  Input
 * LLRs of any int16 value are accepted (clamped to +-4096, R12). */
int crn_decode_batch_ex(const crn_cb_desc *desc, int32_t n_cb,
                        const int16_t *llr_sys, const int16_t *llr_p1, const int16_t *llr_p2,
                        int32_t max_iters, int32_t early_term, int32_t flags,
                        uint32_t *out_bits, uint8_t *crc_ok, uint8_t *iters_used, int16_t *ext_out,
                        void *workspace, size_t workspace_bytes, void *cuda_stream);

/* Bytes of caller-provided workspace crn_decode_batch_ex needs on the current
 * device for a batch of n_cb CBs: 256 bytes for the
 * persistent decoder's task counter (it keeps every CB's state on chip) plus,
 * used only with CRN_DESC_ON_DEVICE, the device task builder's arrays (tasks,
 * pairs, per-CB bucket index, purge flags: O(n_cb)).  desc may be NULL: the
 * size depends on n_cb only.  0 without a device or for n_cb < 0. */
size_t crn_workspace_bytes(const crn_cb_desc *desc, int32_t n_cb);

/* Plans: validate + bucket + upload a descriptor set once, decode many times
 * (the per-TTI pattern of a BBU, "CCDUs arrive in batches every
 * millisecond").  *plan receives an opaque handle. */
int crn_plan_create(const crn_cb_desc *desc_host, int32_t n_cb, void **plan);
int crn_plan_decode(void *plan, const int16_t *llr_sys, const int16_t *llr_p1,
                    const int16_t *llr_p2, int32_t max_iters, int32_t early_term,
                    uint32_t *out_bits, uint8_t *crc_ok, uint8_t *iters_used, int16_t *ext_out,
                    void *cuda_stream);
/* Decoder variant of later crn_plan_decode / crn_plan_decode_host calls of this
 * plan (CRN_VARIANT_MAXLOG / _SCALED / _LOGMAP; default CRN_VARIANT_MAXLOG).
 * CRN_EINVAL otherwise. */
int crn_plan_set_variant(void *plan, int32_t variant);
/* TB purge ("In case of decoding failure, the
 * scheduler purges all CCDUs belonging to the same UE (TB)" -- Algorithm 2
 * "purge waiting CCDU of the same TB"): with on = 1, a CB whose decoding fails
 * (crc_ok = 0 at its stop) marks its TB (descriptor field reserved) lost, and
 * a CB of a lost TB that has not started decoding yet is not decoded at all:
 * crc_ok = 0, iters_used = 0, its out_bits / ext_out left untouched; CBs that
 * do get decoded have exactly the outputs they have without purging, and
 * every TB verdict is unchanged (a TB with a failed CB is lost either way).
 * Which CBs get purged depends on timing.  CRN_EINVAL if a reserved field is
 * < -1.  Applies to crn_plan_decode (crn_decode_batch_ex: flag CRN_PURGE). */
int crn_plan_set_purge(void *plan, int32_t on);
/* At most max_ctas persistent CTAs for this plan's decodes (0 = one per SM):
 * shares the GPU with other work; with 1 the tasks run strictly in order. */
int crn_plan_set_grid(void *plan, int32_t max_ctas);
/* LLR input format of later crn_plan_decode / crn_plan_decode_host calls of
 * this plan (SURVEY.md §8(f) row f4 "int8 LLR ingest": half the host->device
 * and HBM bytes).  bits = 16, shift = 0: int16 LLRs (the default).  bits = 8,
 * shift in [0, 8]: the three LLR arrays hold int8 values x at the same element
 * offsets (desc.llr_off) -- pass them cast to const int16_t * -- and each is
 * read as the int16 LLR x * 2^shift, after which decoding is exactly that of
 * the int16 input (clamp to +-4096, filler override, R31).
 * crn_stream_run stays int16.  CRN_EINVAL for any other (bits, shift). */
int crn_plan_set_llr_format(void *plan, int32_t bits, int32_t shift);
/* Bytes per LLR element of the plan's current format (2 or 1). */
int crn_plan_llr_bytes(void *plan);
/* The Log-MAP correction table of CRN_VARIANT_LOGMAP: out[0..7] = LUT[b]. */
int crn_logmap_lut(int32_t *out);
/* Diagnostic: task_of_cb[i] = the CTA task (row a1: bucket by K, pair equal-K
 * CBs, group pairs) CB i is decoded in, in issue order; n_cb must equal the
 * plan's.  Returns the number of tasks, or CRN_EINVAL. */
int crn_plan_layout(void *plan, int32_t *task_of_cb, int32_t n_cb);
/* Host-only diagnostic of row a1 (no device needed): buckets, pairs and tasks
 * n_cb HOST descriptors the way a plan does (spread_to > 0: a batch that fills
 * fewer CTAs is cut into more, smaller tasks, up to spread_to CTAs).  Per CB:
 * task_of_cb[i] = its task in issue order.  Per task (arrays of >= n_cb + 1
 * entries, may be NULL): task_info[4 t .. 4 t + 3] = K, n_pairs, windows
 * (n_pairs * M), group flag (1: a four-warp group task, three per CTA).
 * *units = the CTAs the tasks keep busy at once (whole-CTA tasks + ceil(group
 * tasks / 3)).  Returns the number of tasks, or CRN_EINVAL (invalid descriptors). */
int crn_task_layout(const crn_cb_desc *desc, int32_t n_cb, int32_t spread_to, int32_t *task_of_cb,
                    int32_t *task_info, int32_t *units);
/* Number of decode-kernel launches one crn_plan_decode performs (for gpu_launches). */
int crn_plan_launches(void *plan);
void crn_plan_destroy(void *plan);

/* Host-buffer decode (the end-to-end path: LLRs arrive in host memory from the
 * fronthaul).  h_llr_* are HOST arrays laid out exactly as
 * the plan's descriptors say (llr_off), h_out_bits / h_crc_ok / h_iters_used
 * (may be NULL) HOST outputs (bit_off, CB index).  Pinned (page-locked) host
 * memory is required for the copies to overlap the decode; pageable memory
 * works but serialises.  The plan's CBs are cut into n_chunks chunks of
 * consecutive CB indices (0 = automatic: about 4 waves of the persistent grid
 * per chunk, at most 16); chunk c's upload, chunk c-1's decode and chunk c-2's
 * download run concurrently on two internal copy streams and cuda_stream.
 * Asynchronous: every step is ordered after prior work on cuda_stream and
 * cuda_stream waits for the last download, so synchronising cuda_stream makes
 * the host outputs valid.  The plan owns the device staging buffers (sized
 * once, on the first call).  Output contract: each chunk's words come back as
 * one span [min bit_off, max bit_off + ceil(K/32)) of its CBs, so host words in
 * gaps between CBs' ranges inside a span are overwritten with 0 (crn_plan_decode
 * writes only each CB's own words).  Errors as crn_plan_decode, CRN_EINVAL for
 * n_chunks outside [0, 64]; ext_out is not offered on this path. */
int crn_plan_decode_host(void *plan, const int16_t *h_llr_sys, const int16_t *h_llr_p1,
                         const int16_t *h_llr_p2, int32_t max_iters, int32_t early_term,
                         uint32_t *h_out_bits, uint8_t *h_crc_ok, uint8_t *h_iters_used,
                         int32_t n_chunks, void *cuda_stream);
/* Chunks the last crn_plan_decode_host of this plan used (0 if none yet). */
int crn_plan_chunks(void *plan);

/* ------------------------------------------------------------------ streaming TTIs */

/* One cell group's share of one TTI (the CCDUs of PAPER.md:326 that arrive
 * together every millisecond).  All pointers are HOST memory (pinned for
 * overlap): desc[n_cb] as in crn_decode_batch_ex (llr_off / bit_off relative
 * to this group's own arrays), llr_* of n_llr elements each, out_bits of
 * n_words words, crc_ok[n_cb], iters_used[n_cb] (may be NULL).  n_cb may be 0. */
typedef struct {
    const crn_cb_desc *desc;
    int32_t n_cb, reserved;
    const int16_t *llr_sys, *llr_p1, *llr_p2;
    int64_t n_llr;
    uint32_t *out_bits;
    int64_t n_words;
    uint8_t *crc_ok, *iters_used;
} crn_tti_group;

/* Per-TTI timestamps in microseconds from the run's start (steady clock):
 * release (the pacer's release instant), submitted (all groups enqueued),
 * complete (the last group's downloads observed done by the completion
 * thread), latency = complete - release, device = span of the TTI's GPU work
 * (first upload start .. last download end, CUDA events).  The stage split of
 * the device span (the paper's captor KPIs: pre-processing,
 * channel coding, post-processing), CUDA events relative to the TTI's first
 * upload start: upload_us = when the last group's inputs are on the device,
 * decode_start_us / decode_end_us = first decode launch start / last end. */
typedef struct {
    double release_us, submitted_us, complete_us, latency_us, device_us;
    double upload_us, decode_start_us, decode_end_us;
} crn_tti_timing;

/* Paced streaming decode (Algorithm 2 as a GPU executor;
 * the timestamps play the paper's performance captor, :398-411).  groups[t *
 * n_groups + g] is group g of TTI t.  TTI t is released at t0 + t * period_us
 * (period_us = 0: back to back); at release the host buckets each group's CBs
 * into tasks (row a1) and enqueues upload -> decode -> download on the
 * group's own CUDA stream (created by the call).  A completion thread records
 * when each group's downloads finish.  Blocks until every TTI is done and
 * fills timing[n_tti].  Every group is validated before the first release
 * (CRN_EINVAL as crn_decode_batch_ex, or n_llr / n_words too small). */
int crn_stream_run(const crn_tti_group *groups, int32_t n_tti, int32_t n_groups, double period_us,
                   int32_t max_iters, int32_t early_term, crn_tti_timing *timing);
/* Same with flags: CRN_STREAM_MERGED keeps one CUDA stream per cell group for
 * the uploads and downloads but decodes each TTI with ONE launch over all
 * groups' CBs (on an internal decode stream that waits for every group's
 * upload; each group's download waits for the decode): the groups' persistent
 * kernels no longer split the SMs between them.  CRN_STREAM_STAGES records
 * the stage split of crn_tti_timing (three more events per group and TTI;
 * otherwise those fields are -1; always recorded in merged mode).  Other flag
 * bits: CRN_EINVAL.  When a group's out_bits, crc_ok and iters_used are one
 * host block (crc_ok right after the n_words words, iters_used right after
 * crc_ok) they come back in a single copy; likewise llr_sys/p1/p2 laid out
 * back to back go up in one copy.  CRN_STREAM_ZEROCOPY (not with MERGED):
 * the decode kernel reads each group's descriptors, tasks and LLRs straight
 * from pinned host memory and writes its bits / crc_ok / iters_used straight
 * into the host buffers (over PCIe, no copy stage; one launch per group and
 * TTI); every host buffer must be pinned (CRN_EINVAL otherwise).
 * CRN_STREAM_LLR8 | CRN_STREAM_LLR8_SHIFT(s), s in [0, 8] (not with MERGED or
 * ZEROCOPY): the groups' llr_sys / p1 / p2 hold int8 LLRs (n_llr elements of 1
 * byte), read as x * 2^s exactly as crn_plan_set_llr_format does -- half the
 * upload bytes. */
enum { CRN_STREAM_MERGED = 1, CRN_STREAM_STAGES = 2, CRN_STREAM_ZEROCOPY = 4, CRN_STREAM_LLR8 = 8 };
#define CRN_STREAM_LLR8_SHIFT(s) ((s) << 8)
int crn_stream_run_ex(const crn_tti_group *groups, int32_t n_tti, int32_t n_groups, double period_us,
                      int32_t max_iters, int32_t early_term, int32_t flags, crn_tti_timing *timing);

/* Counted operations of one decode (the roofline numerator, DESIGN.md "op
 * count"): sum over CBs and executed iterations of 2 x (129 K + 90).  For a
 * fixed-iteration batch pass iters_used = NULL and it uses max_iters. */
int64_t crn_counted_ops(const int32_t *K_host, int32_t n_cb, const uint8_t *iters_used_host,
                        int32_t max_iters);

/* The paper's iteration KPI ("Performance captor": the captor
 * records "the number of iterations carried out by the decoder per CB", and
 * "decoding failures are detected when a value greater than the maximum
 * number of allowed iterations is registered"): out[i] = iters_used[i] if
 * crc_ok[i], else max_iters + 1 (R17).  HOST arrays of n entries;
 * CRN_EINVAL for n < 0, a NULL array or max_iters outside [1, 32]. */
int crn_kpi_iterations(const uint8_t *iters_used, const uint8_t *crc_ok, int32_t n, int32_t max_iters,
                       uint8_t *out);

/* ------------------------------------------------------------------ encode (DL) */

/* Rate-1/3 turbo encoding of n_cb CBs on the device.  info: one bit per byte,
 * CB i's K_i bits at desc[i].ext_off (the whole CB content incl. fillers and
 * CRC).  If attach_crc != 0 the last 24 bits are (re)computed as the CRC of
 * desc[i].crc_kind over the first K-24 bits (fillers counted as 0) before
 * encoding.  Output d0/d1/d2: one bit per byte, CB i's K_i+4 coded bits at
 * desc[i].llr_off (36.212 5.1.3.2 layout incl. the 12 tail bits, R11).
 * desc is HOST memory; info/d0/d1/d2 device memory. */
int crn_encode_batch(const crn_cb_desc *desc, int32_t n_cb, const uint8_t *info, int32_t attach_crc,
                     uint8_t *d0, uint8_t *d1, uint8_t *d2, void *cuda_stream);
/* The same with packed bits (bit b of a stream is bit b % 32 of word b / 32,
 * LSB first; one eighth of the bytes of the form above): CB i's K_i content bits
 * are bits [ext_off, ext_off + K_i) of info, its K_i + 4 coded bits of stream x
 * are written to bits [llr_off, llr_off + K_i + 4) of dx.  Offsets need no
 * alignment: CBs may share a word (such words are merged atomically, bits
 * outside every CB's range are left as they were).  Errors as crn_encode_batch. */
int crn_encode_batch_packed(const crn_cb_desc *desc, int32_t n_cb, const uint32_t *info, int32_t attach_crc,
                            uint32_t *d0, uint32_t *d1, uint32_t *d2, void *cuda_stream);

/* ------------------------------------------------------------------ rate matching */

/* One CB's rate-matching parameters (TS 36.212 5.1.4.1, R30):
 *   K       interleaver size (the 188 LTE sizes); the CB has 3 (K+4) coded bits
 *   E       rate-matched length (>= 1; E > 3(K+4) repeats, E < 3(K+4) punctures)
 *   rv      redundancy version 0..3 (start k0 = R (24 rv + 2) of the circular buffer)
 *   e_off   element offset of the CB's E values in e
 *   llr_off element offset of the CB's K+4 values in each of the three streams */
typedef struct {
    int32_t K, E, rv, reserved;
    int64_t e_off, llr_off;
} crn_rm_desc;

/* De-matching on the DEVICE (the input side of the decoder):
 * for every CB, each of the E received int16 soft values e[e_off + k] is added
 * to the coded-bit position it was selected from (repetitions accumulate,
 * punctured positions receive nothing); the int32 sums are written to
 * h_sys / h_p1 / h_p2 [llr_off .. llr_off + K+4) saturated to int16 -- onto the
 * previous content (HARQ soft combining) if combine != 0, else replacing it.
 * The three output streams are exactly the decoder's llr_sys / llr_p1 /
 * llr_p2 inputs (dense or any layout).  desc: HOST array (copied); e, h_*:
 * DEVICE memory.  Asynchronous on cuda_stream.  CRN_EINVAL for a bad K, rv, E,
 * negative offsets.  Results do not depend on order (exact integer sums). */
int crn_rate_dematch_batch(const crn_rm_desc *desc, int32_t n_cb, const int16_t *e, int32_t combine,
                           int16_t *h_sys, int16_t *h_p1, int16_t *h_p2, void *cuda_stream);
/* Rate matching on the DEVICE (DL direction): CB i's coded
 * bits d0/d1/d2 [llr_off .. +K+4) (one bit per byte, as crn_encode_batch writes
 * them) -> its E selected bits e[e_off ..) (one bit per byte). */
int crn_rate_match_batch(const crn_rm_desc *desc, int32_t n_cb, const uint8_t *d0, const uint8_t *d1,
                         const uint8_t *d2, uint8_t *e, void *cuda_stream);
/* The same with packed bits (LSB-first words, as crn_encode_batch_packed writes
 * them): CB i's stream x is bits [llr_off, llr_off + K + 4) of dx, its E selected
 * bits go to bits [e_off, e_off + E) of e (e_off, llr_off in BITS; no alignment
 * needed: words shared with neighbouring CBs are merged atomically, bits outside
 * every CB's range are left as they were).  Errors as crn_rate_match_batch. */
int crn_rate_match_batch_packed(const crn_rm_desc *desc, int32_t n_cb, const uint32_t *d0, const uint32_t *d1,
                                const uint32_t *d2, uint32_t *e, void *cuda_stream);

/* ------------------------------------------------------------------ host helpers */

/* TB of tbs_bits payload bits -> 36.212 5.1.2 code-block segmentation (B = tbs+24). */
int crn_segment_tb(int64_t tbs_bits, crn_seg *out);
/* Build the CBs of one TB (36.212 5.1.1-5.1.2; Algorithm 1 and
 * the CB/TB relation of PAPER.md:369): CRC24A is attached to the tbs_bits
 * payload bits (one per byte, HOST memory), the result is segmented, CB 0 gets
 * the F leading filler zeros and, if C > 1, every CB gets its CRC24B.
 * cb_bits receives sum K_r bits (one per byte); desc[r] gets K, F, crc_kind
 * (CRC24A if C == 1 else CRC24B), ext_off = bit offset inside cb_bits (plus
 * base_bit), llr_off = sum_{s<r}(K_s+4) (plus base_llr), bit_off = word offset
 * sum_{s<r} ceil(K_s/32) (plus base_word).  *n_cb receives C; max_cb bounds it. */
int crn_tb_build_cbs(const uint8_t *tb_bits, int64_t tbs_bits, int32_t max_cb, int64_t base_bit,
                     int64_t base_llr, int64_t base_word, uint8_t *cb_bits, crn_cb_desc *desc,
                     int32_t *n_cb);
/* The same for a whole batch of TBs on the DEVICE (DL direction: the "code
 * block creation, segmentation" the paper times before its encoder,
 * PAPER.md:270-272, :404-406).  TB t has tbs_bits[t]
 * payload bits, one per byte, at payload[payload_off[t] ..] (DEVICE memory).
 * The CBs of all TBs are laid out densely in TB order: desc (HOST, capacity
 * max_cb) receives K, F, crc_kind, reserved = t (the CB's TB index, as
 * crn_plan_set_purge expects), ext_off = sum of the preceding K (the CB's first
 * byte in cb_bits), llr_off = sum of the preceding K+4, bit_off = sum of the
 * preceding ceil(K/32); cb_bits (DEVICE, sum K bytes) receives every CB's
 * complete content exactly as crn_tb_build_cbs builds it: F filler zeros in CB
 * 0, the bits of payload || CRC24A, and each CB's CRC24B when C > 1.  *n_cb
 * receives the CB count.  The segmentation arithmetic (O(1) per TB) runs on
 * the host; CRC24A, the bit placement and CRC24B run in one kernel (a CTA per
 * TB), asynchronously on cuda_stream (the first call on a device builds the
 * kernel's CRC tables and waits for them once).  The kernel writes cb_bits
 * eight bytes at a time when cb_bits is 8-byte aligned, byte by byte otherwise
 * (same result).  Like every one-shot batch call here (decode, encode, rate
 * (de)matching) the descriptor upload comes from the device's default
 * stream-ordered memory pool; the library raises that pool's release threshold
 * to 256 MiB once per device (unless it is already higher) so that a
 * synchronisation between calls does not return the blocks to the driver.
 * CRN_EINVAL for n_tb < 0, tbs < 1, a
 * negative offset, more than max_cb CBs in total or a TB of more than
 * CRN_TB_MAX_CB CBs. */
int crn_tb_build_cbs_batch(const int64_t *tbs_bits, const int64_t *payload_off, int32_t n_tb, const uint8_t *payload,
                           int32_t max_cb, uint8_t *cb_bits, crn_cb_desc *desc, int32_t *n_cb, void *cuda_stream);
/* TB post-processing ("a TB can be successfully decoded only when
 * all CBs have been individually decoded", :408 "combination of CBs"): given the
 * C decoded CBs of one TB (packed words as written by the decoder, HOST memory,
 * CB r at desc[r].bit_off) strip fillers and CB CRCs, concatenate, check the TB
 * CRC24A.  Returns 1 if every crc_ok[r] is set and the TB CRC passes (payload
 * written to tb_out, one bit per byte, if non-NULL), 0 otherwise, <0 on error. */
int crn_tb_reassemble(const uint32_t *cb_words, const crn_cb_desc *desc, const uint8_t *crc_ok,
                      int32_t n_cb, int64_t tbs_bits, uint8_t *tb_out);
/* Transport block of a decoded batch: its C = n_cb code blocks are
 * desc[cb0 .. cb0+n_cb) in segment order (as crn_tb_build_cbs emits them),
 * tbs payload bits; its payload words go to tb_words[word_off ..]. */
typedef struct {
    int32_t cb0, n_cb;
    int64_t tbs, word_off;
} crn_tb_desc;

/* TB post-processing on the DEVICE for a whole batch (PAPER.md:408
 * "combination of CBs", :369 TB success rule): for each TB
 * strip fillers and CB CRC24Bs, concatenate, check the TB CRC24A;
 * tb_ok[i] = 1 iff every CB's crc_ok is set and the TB CRC passes.  tb_words
 * (may be NULL) receives the ceil(tbs/32) payload words LSB-first from
 * word_off (written whatever the verdict).  tb and desc are HOST arrays
 * (copied; n_cb = the length of desc, TBs index into it); cb_words
 * (the decoder's out_bits), crc_ok, tb_ok, tb_words are DEVICE memory.
 * Asynchronous on cuda_stream.  CRN_EINVAL if a TB's CB range is outside desc,
 * its CBs do not match the 36.212 segmentation of tbs (C, K+/K-, F, crc_kind)
 * or C > 128. */
int crn_tb_verdict_batch(const crn_tb_desc *tb, int32_t n_tb, const crn_cb_desc *desc, int32_t n_cb,
                         const uint32_t *cb_words, const uint8_t *crc_ok, uint8_t *tb_ok,
                         uint32_t *tb_words, void *cuda_stream);
/* QPP parameters of TS 36.212 Table 5.1.3-3 for K; CRN_EINVAL if K is not a size. */
int crn_qpp_params(int32_t K, int32_t *f1, int32_t *f2);
/* Window split of the decoder: M = max{M : M | K, K/M >= 32}, W = K/M (R13). */
int crn_windows(int32_t K, int32_t *M, int32_t *W);
/* CRC register after nbits bits (one per byte, MSB-first; zero init; 0 <=> valid). */
uint32_t crn_crc24a(const uint8_t *bits, int64_t nbits);
uint32_t crn_crc24b(const uint8_t *bits, int64_t nbits);
const char *crn_strerror(int code);
/* Text of the last CUDA failure seen by this thread inside libcrn ("" if none). */
const char *crn_last_error(void);

/* The MI stopping rule's table (host computation, no device needed): out[a] =
 * round(65536 * (1 - Hb(1 / (1 + e^(a/8))))) for a = 0..255, the mutual
 * information of a consistent LLR of magnitude a/8 (R29). */
int crn_mi_table(int32_t *out);

/* ------------------------------------------------------------------ device facts / microbench */

/* SM count, SM max clock (kHz) and sm major/minor of the current device. */
int crn_device_info(int32_t *num_sms, int32_t *clock_khz, int32_t *cc_major, int32_t *cc_minor);
/* Decode kernel resources: static / dynamic shared memory (bytes), the kernel's
 * current max dynamic shared memory attribute, registers per thread. */
int crn_decode_kernel_info(int32_t *static_smem, int32_t *dyn_smem, int32_t *max_dyn, int32_t *regs);
/* int16x2 ALU microbenchmark: op 0 VIADD.16x2, 1 VIMNMX.S16x2,
 * 2 VIMNMX3.S16x2, 3 VIADDMNMX.S16x2.  Runs independent chains at full
 * occupancy (8 CTAs x 256 threads per SM); *lane_instr = warp-instructions x 32
 * of the opcode executed, *ms = kernel time, *max_block_cycles = the longest
 * CTA's clock64 span (all CTAs are co-resident, so SM throughput in lane-instr
 * per cycle = lane_instr / (num_sms x max_block_cycles)). */
int crn_ubench_int16x2(int32_t op, int64_t *lane_instr, float *ms, int64_t *max_block_cycles);

#ifdef __cplusplus
}
#endif
#endif
