/* crn_plan.h -- host-side internals shared by crn_host.cpp (plans, tables,
 * validation, task building) and crn_runtime.cpp (host-buffer pipeline, TTI
 * stream runner).  Not part of the ABI (see include/crn.h). */
#pragma once
#include <cuda_runtime.h>

#include <vector>

#include "crn_internal.h"

struct DevTables {
    uint32_t *qpp_wm = nullptr, *qpp_ts = nullptr, *qinv_ts = nullptr, *crc_bit = nullptr,
             *qinv_wm = nullptr;
    int32_t *qpp_off = nullptr, *crcb_off = nullptr, *mi_tab = nullptr;
    uint32_t *crc_nib = nullptr;
    int32_t *bucket = nullptr, *border = nullptr;   /* device task builder (crn_tasks.cu) */
    crn_tables tab{};
    int grid = 0;
};

struct HostPipe;      /* crn_runtime.cpp: staging buffers + streams of crn_plan_decode_host */

/* the kernel's variant word: decoder variant | (LLR format + 1) << 8 */
struct Plan;
int crn_plan_kernel_variant(const Plan *P);
/* The Log-MAP LUT as the decode kernel's two PRMT source words (crn_host.cpp). */
void crn_logmap_words(uint32_t *lo, uint32_t *hi);

struct Plan {
    int dev = -1;
    int n_cb = 0, n_tasks = 0;
    int units = 0;                     /* CTAs the tasks fill (crn_build_tasks) */
    crn_cb_desc *d_desc = nullptr;
    crn_task *d_tasks = nullptr;
    crn_pair *d_pairs = nullptr;
    void *mem = nullptr;          /* one allocation holding the three arrays */
    std::vector<crn_cb_desc> h_desc;   /* host copy (kept for the host-buffer pipeline) */
    int variant = CRN_VARIANT_MAXLOG;  /* decoder variant (crn_plan_set_variant) */
    int purge = 0;                     /* TB purge (crn_plan_set_purge) */
    int grid_cap = 0;                  /* persistent-grid limit (crn_plan_set_grid), 0 = one CTA per SM */
    int llr8 = -1;                     /* LLR format (crn_plan_set_llr_format): -1 int16, else int8 << llr8 */
    int n_tb = 0;                      /* TB ids in the descriptors' reserved field: 0..n_tb-1 */
    int spread = 0;                    /* the spread_to its tasks were built with (crn_build_tasks) */
    uint8_t *d_tb_dead = nullptr;      /* per TB: a CB of it failed (purge) */
    HostPipe *pipe = nullptr;
};

/* Per-size task parameters shared by the host and device task builders: windows
 * (M, W), pairs per task before spreading, group flag (crn_internal.h CRN_GROUPS),
 * and the LPT issue key (larger first; group tasks after every whole-CTA task). */
void crn_bucket_params(int K, int *M, int *W, int *per, int *grp);
int crn_bucket_issue_key(int K);
/* Device context: checks for an sm_100 device and builds the per-device tables once. */
int crn_get_ctx(int *dev, DevTables **t);
/* Cached per-(device, stream) decode workspace. */
int crn_get_ws(int dev, void *stream, size_t bytes, void **ws);
/* Descriptor validation (include/crn.h CRN_EINVAL rules). */
int crn_validate(const crn_cb_desc *d, int n, bool want_ext);
/* Bucket by K (largest first), pair equal-K CBs, group pairs into CTA tasks.
 * Only the CBs idx[0..n_idx) take part; pair0 of the tasks indexes `pairs`.
 * spread_to > 0: a batch of fewer tasks is cut into smaller tasks, up to
 * spread_to of them (the persistent grid), so a small batch spreads over the SMs. */
int crn_build_tasks(const crn_cb_desc *d, const int *idx, int n_idx, std::vector<crn_task> &tasks,
                    std::vector<crn_pair> &pairs, int spread_to = 0);   /* returns the CTAs the tasks fill */
/* Launch the decode kernel over n_tasks tasks (device arrays), workspace from the cache if ws == NULL. */
int crn_launch_tasks(int dev, DevTables *t, const crn_cb_desc *d_desc, const crn_task *d_tasks, int n_tasks,
                     const crn_pair *d_pairs, const int16_t *l0, const int16_t *l1, const int16_t *l2,
                     int32_t max_iters, int32_t et, uint32_t *bits, uint8_t *ok, uint8_t *it, int16_t *ext,
                     void *ws, size_t ws_bytes, cudaStream_t st, int variant = CRN_VARIANT_MAXLOG,
                     uint8_t *tb_dead = nullptr, int grid_cap = 0,
                     bool ws_zeroed = false,    /* the task counter in ws is already 0 (uploaded with a blob) */
                     int units = 0);            /* CTAs the tasks can fill (crn_build_tasks), 0: n_tasks */
/* Records the CUDA error behind a CRN_ECUDA / CRN_ENOMEM for crn_last_error(). */
int crn_cuda_fail(cudaError_t e, const char *where, int code);
/* Frees the host pipeline of a plan (crn_runtime.cpp). */
void crn_pipe_destroy(HostPipe *p);
