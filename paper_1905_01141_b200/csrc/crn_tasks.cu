/* crn_tasks.cu -- row a1 on the device: bucket, pair and task CB descriptors
 * that live in device memory (crn_decode_batch_ex with CRN_DESC_ON_DEVICE), so
 * the call never copies them back to the host or waits on the stream.
 *
 * The same decomposition as the host builder (crn_host.cpp crn_build_tasks,
 * without its small-batch spreading): CBs are bucketed by K (the paper's
 * unit of parallel work is the CB), two CBs of one K share a
 * pair (int16x2 lanes), floor(6144/K) pairs form a whole-CTA task or
 * floor(2048/K) pairs a group task; whole-CTA tasks are issued longest first,
 * group tasks last.  The per-size parameters (M, W, pairs per task, group
 * flag) and the issue order of the 188 buckets are host-built tables, so both
 * builders follow one definition.  Which two CBs of a bucket share a pair is
 * the order the atomic slot counter hands out: every CB's outputs depend only
 * on its own inputs (the two lanes of a pair never mix), so any pairing gives
 * the same results.
 *
 * Descriptors are validated here (crn.h rules except range overlaps, which
 * would need a sort): an invalid CB is not decoded, crc_ok = 0 and
 * iters_used = 0.  One CTA of 1024 threads; the header words hdr[0] (the
 * decode kernel's task counter) and hdr[1] (the task count it reads) are
 * written for the decode launch that follows on the stream. */
#include <cuda_runtime.h>
#include <stdint.h>

#include "crn_internal.h"

namespace {

constexpr int NB = CRN_NUM_K;
constexpr int THREADS = 1024;

/* closed-form index of an LTE interleaver size (36.212 Table 5.1.3-3), -1 if none */
__device__ __forceinline__ int k_index(int K) {
    if (K >= 40 && K <= 512) return (K - 40) % 8 ? -1 : (K - 40) / 8;
    if (K > 512 && K <= 1024) return (K - 528) % 16 ? -1 : 60 + (K - 528) / 16;
    if (K > 1024 && K <= 2048) return (K - 1056) % 32 ? -1 : 92 + (K - 1056) / 32;
    if (K > 2048 && K <= 6144) return (K - 2112) % 64 ? -1 : 124 + (K - 2112) / 64;
    return -1;
}

__global__ void __launch_bounds__(THREADS, 1)
build_tasks_kernel(const crn_cb_desc *__restrict__ d, int n, int want_ext, int purge,
                   const int32_t *__restrict__ bucket, const int32_t *__restrict__ border, int32_t *hdr,
                   crn_task *__restrict__ tasks, crn_pair *__restrict__ pairs, int32_t *__restrict__ kx,
                   uint8_t *__restrict__ dead, uint8_t *__restrict__ crc_ok, uint8_t *__restrict__ iters_used) {
    __shared__ int cnt[NB], cur[NB], poff[NB];
    __shared__ int tstart[NB + 1];             /* first task of the bucket at issue position q */
    __shared__ int s_np;
    const int tid = threadIdx.x;
    for (int k = tid; k < NB; k += THREADS) cnt[k] = cur[k] = 0;
    if (purge)
        for (int i = tid; i < n; i += THREADS) dead[i] = 0;
    __syncthreads();
    for (int i = tid; i < n; i += THREADS) {
        const crn_cb_desc c = d[i];
        int k = k_index(c.K);
        if (k >= 0 && bucket[4 * k] != c.K) k = -1;
        const bool ok = k >= 0 && c.F >= 0 && c.F <= c.K - 25 && c.crc_kind >= 0 && c.crc_kind <= 2 &&
                        c.llr_off >= 0 && c.bit_off >= 0 && (!want_ext || c.ext_off >= 0) &&
                        (!purge || (c.reserved >= -1 && c.reserved < n));
        kx[i] = ok ? k : -1;
        if (ok) atomicAdd(&cnt[k], 1);
        else {
            crc_ok[i] = 0;
            if (iters_used) iters_used[i] = 0;
        }
    }
    __syncthreads();
    if (tid == 0) {                            /* 188 buckets in issue order: pair and task offsets */
        int P = 0, T = 0;
        for (int q = 0; q < NB; q++) {
            const int k = border[q], np = (cnt[k] + 1) / 2, per = bucket[4 * k + 3] & 0xFFFF;
            poff[k] = P;
            tstart[q] = T;
            P += np;
            T += (np + per - 1) / per;
        }
        tstart[NB] = T;
        s_np = P;
        hdr[0] = 0;                            /* the decode kernel's task counter */
        hdr[1] = T;                            /* its task count */
    }
    __syncthreads();
    const int n_tasks = tstart[NB];
    for (int t = tid; t < n_tasks; t += THREADS) {
        int lo = 0, hi = NB - 1;               /* the issue position q with tstart[q] <= t < tstart[q + 1] */
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (tstart[mid] <= t) lo = mid;
            else hi = mid - 1;
        }
        const int k = border[lo], np = (cnt[k] + 1) / 2, pw = bucket[4 * k + 3];
        const int per = pw & 0xFFFF, x = t - tstart[lo];
        crn_task tk;
        tk.K = bucket[4 * k];
        tk.M = bucket[4 * k + 1];
        tk.W = bucket[4 * k + 2];
        tk.n_pairs = min(per, np - x * per);
        tk.pair0 = poff[k] + x * per;
        tk.kidx = k;
        tk.grp = pw >> 16;
        tasks[t] = tk;
    }
    for (int p = tid; p < s_np; p += THREADS) pairs[p].hi = -1;     /* the dummy partner of an odd bucket */
    __syncthreads();
    for (int i = tid; i < n; i += THREADS) {
        const int k = kx[i];
        if (k < 0) continue;
        const int s = atomicAdd(&cur[k], 1);
        crn_pair *pr = pairs + poff[k] + (s >> 1);
        if (s & 1) pr->hi = i;
        else pr->lo = i;
    }
}

}  // namespace

extern "C" size_t crn_tasks_dev_bytes(int32_t n_cb) {
    /* pairs <= sum over buckets of ceil(c/2) <= n/2 + 188; tasks <= pairs */
    const size_t np = (size_t)n_cb / 2 + NB + 1;
    auto a = [](size_t x) { return (x + 255) & ~(size_t)255; };
    return a(sizeof(crn_task) * np) + a(sizeof(crn_pair) * np) + a(sizeof(int32_t) * (size_t)n_cb) +
           a((size_t)n_cb);
}

extern "C" int crn_launch_tasks_dev(const crn_cb_desc *d_desc, int32_t n_cb, int32_t want_ext, int32_t purge,
                                    const int32_t *bucket, const int32_t *border, void *scratch, int32_t *hdr,
                                    crn_task **tasks, crn_pair **pairs, uint8_t **dead, uint8_t *crc_ok,
                                    uint8_t *iters_used, void *stream) {
    const size_t np = (size_t)n_cb / 2 + NB + 1;
    auto a = [](size_t x) { return (x + 255) & ~(size_t)255; };
    uint8_t *m = (uint8_t *)scratch;
    *tasks = (crn_task *)m;
    m += a(sizeof(crn_task) * np);
    *pairs = (crn_pair *)m;
    m += a(sizeof(crn_pair) * np);
    int32_t *kx = (int32_t *)m;
    m += a(sizeof(int32_t) * (size_t)n_cb);
    *dead = purge ? m : nullptr;
    build_tasks_kernel<<<1, THREADS, 0, (cudaStream_t)stream>>>(d_desc, n_cb, want_ext, purge, bucket, border, hdr,
                                                                *tasks, *pairs, kx, *dead, crc_ok, iters_used);
    return cudaGetLastError() == cudaSuccess ? CRN_OK : CRN_ECUDA;
}
