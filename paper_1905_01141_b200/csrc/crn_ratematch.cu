/* crn_ratematch.cu -- TS 36.212 5.1.4.1 rate matching / de-matching for
 * turbo-coded channels on the device (R30):
 * the input side of the decoder -- the received data R(x_i) of PAPER.md:289
 * are the E rate-matched soft values of a CB.
 *
 * Geometry per CB: D = K + 4 bits per stream, R = ceil(D/32) rows, Kpi = 32 R,
 * ND = Kpi - D dummy bits, circular buffer w of Ncb = 3 Kpi positions (v0, then
 * v1/v2 interlaced), k0 = R (2 ceil(Ncb / 8R) rv + 2).  The dummy positions are
 * few (<= 97: the first row of each sub-block, plus one wrapped position of
 * v2), so each CTA lists them in shared memory and both directions become
 * gathers:
 *   de-matching: for every output (stream s, bit n) find its w position p by
 *     inverting the sub-block interleaver (the column permutation is the 5-bit
 *     bit reversal, its own inverse), its rank r among non-dummy positions
 *     counted circularly from k0, and sum the received values e[r + m 3D],
 *     m >= 0 (repetition); punctured positions get nothing.  The sum is exact
 *     int32 and is saturated once (onto the previous HARQ buffer when
 *     combining), so the result does not depend on any order.
 *   matching: for every output e[k] find the (k mod 3D)-th non-dummy position
 *     after k0 and copy its coded bit.
 * One CTA per CB, a thread per output element.
 */
#include <cuda_runtime.h>
#include <stdint.h>

#include "crn_internal.h"

namespace {

constexpr int RM_THREADS = 256;
constexpr int MAX_NULL = 128;

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

/* Sorted w positions of the dummy bits, written by warp 0; returns the count. */
__device__ int list_nulls(const Geo &g, int *nul, int *s_n) {
    if (threadIdx.x == 0) {
        int n = 0;
        /* v0: row 0 of column c holds y = P(c), a dummy if P(c) < ND */
        for (int c = 0; c < 32; c++)
            if (bitrev5(c) < g.ND) nul[n++] = c * g.R;
        const int n0 = n;
        /* v1 (even w offsets after Kpi) repeats v0's pattern; v2 (odd offsets):
         * y = (P(c) + 32 row + 1) mod Kpi, a dummy at row 0 if P(c) + 1 < ND and at
         * the wrap k = Kpi - 1 (y = 0) if ND > 0; merge the two in w order */
        int i1 = 0;
        for (int c = 0; c < 32; c++) {
            const int k = c * g.R;
            const bool d2 = bitrev5(c) + 1 < g.ND;
            while (i1 < n0 && nul[i1] < k) { nul[n++] = g.Kpi + 2 * nul[i1]; i1++; }
            if (i1 < n0 && nul[i1] == k) { nul[n++] = g.Kpi + 2 * k; i1++; }
            if (d2) nul[n++] = g.Kpi + 2 * k + 1;
        }
        while (i1 < n0) { nul[n++] = g.Kpi + 2 * nul[i1]; i1++; }
        if (g.ND > 0) nul[n++] = g.Kpi + 2 * (g.Kpi - 1) + 1;
        *s_n = n;
    }
    __syncthreads();
    return *s_n;
}

/* number of dummy positions < x */
__device__ __forceinline__ int nulls_below(const int *nul, int n, int x) {
    int lo = 0, hi = n;
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (nul[mid] < x) lo = mid + 1; else hi = mid;
    }
    return lo;
}

/* w position of bit n of stream s (inverse sub-block interleaving) */
__device__ __forceinline__ int w_of(const Geo &g, int s, int n) {
    const int y = n + g.ND;
    if (s < 2) {
        const int k = bitrev5(y & 31) * g.R + (y >> 5);
        return s == 0 ? k : g.Kpi + 2 * k;
    }
    const int y1 = (y - 1 + g.Kpi) % g.Kpi;      /* y = (P(col) + 32 row + 1) mod Kpi */
    const int k = bitrev5(y1 & 31) * g.R + (y1 >> 5);
    return g.Kpi + 2 * k + 1;
}

__global__ void __launch_bounds__(RM_THREADS)
dematch_kernel(const crn_rm_desc *__restrict__ desc, const int16_t *__restrict__ e, int combine,
               int16_t *__restrict__ h0, int16_t *__restrict__ h1, int16_t *__restrict__ h2) {
    __shared__ int nul[MAX_NULL];
    __shared__ int s_n;
    const crn_rm_desc d = desc[blockIdx.x];
    const Geo g = geo(d.K, d.rv);
    const int n_null = list_nulls(g, nul, &s_n);
    const int base = g.k0 - nulls_below(nul, n_null, g.k0);      /* non-dummy positions before k0 */
    const int16_t *ec = e + d.e_off;
    for (int x = threadIdx.x; x < 3 * g.D; x += RM_THREADS) {
        const int s = x / g.D, n = x - s * g.D;
        const int p = w_of(g, s, n);
        int r = p - nulls_below(nul, n_null, p) - base;              /* rank counted from k0 */
        if (r < 0) r += g.nn;
        int32_t acc = 0;
        for (int k = r; k < d.E; k += g.nn) acc += ec[k];
        int16_t *h = (s == 0 ? h0 : s == 1 ? h1 : h2) + d.llr_off + n;
        if (combine) acc += *h;
        *h = (int16_t)(acc < -32768 ? -32768 : (acc > 32767 ? 32767 : acc));
    }
}

__global__ void __launch_bounds__(RM_THREADS)
match_kernel(const crn_rm_desc *__restrict__ desc, const uint8_t *__restrict__ d0, const uint8_t *__restrict__ d1,
             const uint8_t *__restrict__ d2, uint8_t *__restrict__ e) {
    __shared__ int nul[MAX_NULL];
    __shared__ int s_n;
    const crn_rm_desc d = desc[blockIdx.x];
    const Geo g = geo(d.K, d.rv);
    const int n_null = list_nulls(g, nul, &s_n);
    const int base = g.k0 - nulls_below(nul, n_null, g.k0);
    for (int k = threadIdx.x; k < d.E; k += RM_THREADS) {
        int j = base + k % g.nn;                                      /* j-th non-dummy position overall */
        if (j >= g.nn) j -= g.nn;
        /* the j-th non-dummy position is p = j + c, c = #dummies before it: the number of
         * dummies i with nul[i] - i <= j (nul[i] - i is nondecreasing) -- binary search */
        int lo = 0, hi = n_null;
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (nul[mid] - mid <= j) lo = mid + 1; else hi = mid;
        }
        const int p = j + lo;
        int s, n, y;
        if (p < g.Kpi) { s = 0; y = (p % g.R) * 32 + bitrev5(p / g.R); }
        else {
            const int q = p - g.Kpi, kk = q >> 1;
            if ((q & 1) == 0) { s = 1; y = (kk % g.R) * 32 + bitrev5(kk / g.R); }
            else { s = 2; y = (bitrev5(kk / g.R) + 32 * (kk % g.R) + 1) % g.Kpi; }
        }
        n = y - g.ND;
        const uint8_t *src = s == 0 ? d0 : s == 1 ? d1 : d2;
        e[d.e_off + k] = src[d.llr_off + n];
    }
}

}  // namespace

extern "C" int crn_launch_dematch(const crn_rm_desc *d_desc, int32_t n_cb, const int16_t *e, int32_t combine,
                                  int16_t *h0, int16_t *h1, int16_t *h2, void *stream) {
    dematch_kernel<<<n_cb, RM_THREADS, 0, (cudaStream_t)stream>>>(d_desc, e, combine, h0, h1, h2);
    return cudaGetLastError() == cudaSuccess ? CRN_OK : CRN_ECUDA;
}

extern "C" int crn_launch_match(const crn_rm_desc *d_desc, int32_t n_cb, const uint8_t *d0, const uint8_t *d1,
                                const uint8_t *d2, uint8_t *e, void *stream) {
    match_kernel<<<n_cb, RM_THREADS, 0, (cudaStream_t)stream>>>(d_desc, d0, d1, d2, e);
    return cudaGetLastError() == cudaSuccess ? CRN_OK : CRN_ECUDA;
}
