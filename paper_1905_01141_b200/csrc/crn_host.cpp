/* crn_host.cpp -- libcrn host side: the C ABI of include/crn.h.
 *
 * Row a1 of the hot path (CB packing): validation of
 * the per-CB descriptors, bucketing by K, pairing two CBs of equal K into one
 * int16x2 lane pair, grouping pairs into CTA tasks, plus the 36.212 helpers
 * (segmentation, CRC24A/B) and the per-device tables (QPP window-major
 * addresses, CRC combine powers).  Everything that decodes runs in the CUDA
 * kernels of crn_decode.cu; nothing here computes the method on the CPU.
 */
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cmath>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <utility>
#include <vector>

#include "crn_internal.h"
#include "crn_plan.h"
#include "qpp_table.h"

/* ------------------------------------------------------------------ size table */
static int k_at(int i) {
    if (i < 60) return 40 + 8 * i;              /* 40..512 step 8     */
    if (i < 92) return 528 + 16 * (i - 60);     /* 528..1024 step 16  */
    if (i < 124) return 1056 + 32 * (i - 92);   /* 1056..2048 step 32 */
    return 2112 + 64 * (i - 124);               /* 2112..6144 step 64 */
}

extern "C" int crn_k_index(int32_t K) {            /* closed-form inverse of k_at; -1 if K is not a size */
    int i;
    if (K >= 40 && K <= 512) i = (K - 40) % 8 ? -1 : (K - 40) / 8;
    else if (K > 512 && K <= 1024) i = (K - 528) % 16 ? -1 : 60 + (K - 528) / 16;
    else if (K > 1024 && K <= 2048) i = (K - 1056) % 32 ? -1 : 92 + (K - 1056) / 32;
    else if (K > 2048 && K <= 6144) i = (K - 2112) % 64 ? -1 : 124 + (K - 2112) / 64;
    else i = -1;
    return i >= 0 && k_at(i) == K ? i : -1;
}

extern "C" int crn_qpp_params(int32_t K, int32_t *f1, int32_t *f2) {
    int i = crn_k_index(K);
    if (i < 0 || !f1 || !f2) return CRN_EINVAL;
    *f1 = crn_qpp_f1[i];
    *f2 = crn_qpp_f2[i];
    return CRN_OK;
}

extern "C" int crn_windows(int32_t K, int32_t *M, int32_t *W) {
    if (crn_k_index(K) < 0 || !M || !W) return CRN_EINVAL;
    for (int m = K / 32; m >= 1; m--)
        if (K % m == 0) { *M = m; *W = K / m; return CRN_OK; }
    *M = 1; *W = K;
    return CRN_OK;
}

/* ------------------------------------------------------------------ CRC24 (36.212 5.1.1) */
static const uint32_t POLY_A = 0x864CFBu, POLY_B = 0x800063u;

static uint32_t crc_table[2][256];
static std::once_flag crc_once;
static void crc_init() {
    for (int k = 0; k < 2; k++) {
        uint32_t poly = k ? POLY_B : POLY_A;
        for (uint32_t b = 0; b < 256; b++) {
            uint32_t r = b << 16;
            for (int i = 0; i < 8; i++) r = ((r << 1) ^ ((r & 0x800000u) ? poly : 0)) & 0xFFFFFFu;
            crc_table[k][b] = r;
        }
    }
}

static uint32_t crc24(int k, const uint8_t *bits, int64_t n) {
    std::call_once(crc_once, crc_init);
    uint32_t reg = 0;
    int64_t i = 0;
    for (; i + 8 <= n; i += 8) {            /* byte-at-a-time table form */
        uint32_t byte = 0;
        for (int b = 0; b < 8; b++) byte = (byte << 1) | (bits[i + b] & 1u);
        reg = ((reg << 8) & 0xFFFFFFu) ^ crc_table[k][((reg >> 16) ^ byte) & 0xFFu];
    }
    uint32_t poly = k ? POLY_B : POLY_A;
    for (; i < n; i++) {
        uint32_t fb = ((reg >> 23) ^ bits[i]) & 1u;
        reg = ((reg << 1) & 0xFFFFFFu) ^ (fb ? poly : 0u);
    }
    return reg;
}

extern "C" uint32_t crn_crc24a(const uint8_t *bits, int64_t nbits) { return bits ? crc24(0, bits, nbits) : 0; }
extern "C" uint32_t crn_crc24b(const uint8_t *bits, int64_t nbits) { return bits ? crc24(1, bits, nbits) : 0; }

/* ------------------------------------------------------------------ segmentation (36.212 5.1.2) */
extern "C" int crn_segment_tb(int64_t tbs, crn_seg *o) {
    if (!o || tbs <= 0) return CRN_EINVAL;
    const int64_t Z = 6144;
    int64_t B = tbs + 24, C, L, Bp;
    if (B <= Z) { L = 0; C = 1; Bp = B; }
    else { L = 24; C = (B + Z - L - 1) / (Z - L); Bp = B + C * L; }
    /* K+ = the smallest table size with C K >= B': the table is every multiple of
     * 8 / 16 / 32 / 64 in its four ranges, so round ceil(B'/C) up in its range */
    const int64_t x = (Bp + C - 1) / C;
    int64_t kp;
    if (x <= 40) kp = 40;
    else if (x <= 512) kp = (x + 7) / 8 * 8;
    else if (x <= 1024) kp = (x + 15) / 16 * 16;
    else if (x <= 2048) kp = (x + 31) / 32 * 32;
    else if (x <= 6144) kp = (x + 63) / 64 * 64;
    else return CRN_EINVAL;
    const int ip = crn_k_index((int32_t)kp);
    if (ip < 0) return CRN_EINVAL;
    int64_t Kp = k_at(ip), Km = 0, Cm = 0;
    if (C > 1) {
        Km = ip > 0 ? k_at(ip - 1) : 0;
        Cm = (C * Kp - Bp) / (Kp - Km);
    }
    o->C = (int32_t)C; o->Kplus = (int32_t)Kp; o->Kminus = (int32_t)Km;
    o->Cminus = (int32_t)Cm; o->Cplus = (int32_t)(C - Cm);
    o->F = (int32_t)((C - Cm) * Kp + Cm * Km - Bp);
    o->L = (int32_t)L;
    return CRN_OK;
}

extern "C" const char *crn_strerror(int code) {
    switch (code) {
        case CRN_OK: return "ok";
        case CRN_EINVAL: return "invalid argument";
        case CRN_ECUDA: return "CUDA error";
        case CRN_ENOMEM: return "out of device memory";
        case CRN_ENODEV: return "no usable sm_100 CUDA device";
        default: return "unknown error";
    }
}

extern "C" int64_t crn_counted_ops(const int32_t *K, int32_t n_cb, const uint8_t *iters, int32_t max_iters) {
    /* 129 counted ops per trellis step per SISO + 90 for the three tail steps;
     * two SISOs per iteration (pinned against the oracle's counter) */
    int64_t s = 0;
    for (int i = 0; i < n_cb; i++)
        s += 2LL * (iters ? iters[i] : max_iters) * (129LL * K[i] + 90);
    return s;
}

extern "C" int crn_kpi_iterations(const uint8_t *it, const uint8_t *ok, int32_t n, int32_t max_iters, uint8_t *out) {
    /* a failure registers a value greater than the maximum (R17) */
    if (n < 0 || max_iters < 1 || max_iters > CRN_MAX_ITERS || (n > 0 && (!it || !ok || !out))) return CRN_EINVAL;
    for (int i = 0; i < n; i++) out[i] = ok[i] ? it[i] : (uint8_t)(max_iters + 1);
    return CRN_OK;
}

/* ------------------------------------------------------------------ MI stopping rule */
/* Log-MAP correction (R32): LUT[b] = round(8 ln(1 + e^(-(4b+1.5)/8))),
 * b = min(|a-b| >> 2, 7), packed as the eight bytes the kernel's PRMT selects
 * from (bytes 6 and 7 are 0 and double as its zero filler). */
extern "C" int crn_logmap_lut(int32_t *out) {
    if (!out) return CRN_EINVAL;
    for (int b = 0; b < 8; b++) out[b] = (int32_t)std::floor(8.0 * std::log(1.0 + std::exp(-(4.0 * b + 1.5) / 8.0)) + 0.5);
    return CRN_OK;
}

void crn_logmap_words(uint32_t *lo, uint32_t *hi) {
    int32_t l[8];
    crn_logmap_lut(l);
    *lo = (uint32_t)l[0] | (uint32_t)l[1] << 8 | (uint32_t)l[2] << 16 | (uint32_t)l[3] << 24;
    *hi = (uint32_t)l[4] | (uint32_t)l[5] << 8 | (uint32_t)l[6] << 16 | (uint32_t)l[7] << 24;
}

extern "C" int crn_mi_table(int32_t *out) {
    /* I(L) = 1 - Hb(p), p = 1/(1 + e^L), L = a/8 (the channel quantiser's LLR scale), in
     * Q16 rounded to nearest; the MI of a consistent Gaussian LLR of magnitude L
     * ("average mutual information of LLR", R29) */
    if (!out) return CRN_EINVAL;
    for (int a = 0; a < 256; a++) {
        const double L = a / 8.0;
        const double p = 1.0 / (1.0 + std::exp(L)), q = 1.0 - p;
        const double h = (p > 0 ? -p * std::log2(p) : 0.0) + (q > 0 ? -q * std::log2(q) : 0.0);
        out[a] = (int32_t)std::floor(65536.0 * (1.0 - h) + 0.5);
    }
    return CRN_OK;
}

/* ------------------------------------------------------------------ device context */
static bool check_device(int *dev) {
    if (cudaGetDevice(dev) != cudaSuccess) return false;
    int major = 0;
    if (cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, *dev) != cudaSuccess) return false;
    return major == 10;
}

extern "C" int crn_device_info(int32_t *num_sms, int32_t *clock_khz, int32_t *cc_major, int32_t *cc_minor) {
    int dev;
    if (cudaGetDevice(&dev) != cudaSuccess) { cudaGetLastError(); return CRN_ENODEV; }
    int v;
    if (num_sms) { cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev); *num_sms = v; }
    if (clock_khz) { cudaDeviceGetAttribute(&v, cudaDevAttrClockRate, dev); *clock_khz = v; }
    if (cc_major) { cudaDeviceGetAttribute(&v, cudaDevAttrComputeCapabilityMajor, dev); *cc_major = v; }
    if (cc_minor) { cudaDeviceGetAttribute(&v, cudaDevAttrComputeCapabilityMinor, dev); *cc_minor = v; }
    return CRN_OK;
}

static std::mutex g_mu;
static thread_local char g_err[256] = "";

int crn_cuda_fail(cudaError_t e, const char *where, int code) {
    snprintf(g_err, sizeof(g_err), "%s: %s", where, cudaGetErrorString(e));
    cudaGetLastError();
    return code;
}

extern "C" const char *crn_last_error(void) { return g_err; }
static std::map<int, DevTables> g_tables;
static std::map<std::pair<int, void *>, std::pair<void *, size_t>> g_ws;

/* x^e mod g with the register convention of crc24 (low 24 bits of g = poly). */
static uint32_t mulx_mod(uint32_t a, uint32_t poly) { return ((a << 1) ^ ((a & 0x800000u) ? poly : 0u)) & 0xFFFFFFu; }

static int build_tables(int dev, DevTables **out) {
    auto it = g_tables.find(dev);
    if (it != g_tables.end()) { *out = &it->second; return CRN_OK; }
    {   /* The one-shot batch calls take their descriptor uploads from the device's
         * default stream-ordered pool (cudaMallocAsync).  With the pool's default
         * release threshold of 0 every synchronisation hands the freed blocks back
         * to the driver and the next call pays a fresh allocation (~0.2 ms); keep up
         * to 256 MiB cached unless the application already asked for more. */
        cudaMemPool_t mp;
        uint64_t cur = 0;
        const uint64_t want = 256ull << 20;
        if (cudaDeviceGetDefaultMemPool(&mp, dev) == cudaSuccess &&
            cudaMemPoolGetAttribute(mp, cudaMemPoolAttrReleaseThreshold, &cur) == cudaSuccess && cur < want) {
            uint64_t v = want;
            cudaMemPoolSetAttribute(mp, cudaMemPoolAttrReleaseThreshold, &v);
        }
        cudaGetLastError();
    }
    std::vector<uint32_t> qpp, qts, qin, qiw, cb;
    std::vector<int32_t> qoff(CRN_NUM_K), cboff(CRN_NUM_K);
    for (int ki = 0; ki < CRN_NUM_K; ki++) {
        int K = k_at(ki), M, W;
        crn_windows(K, &M, &W);
        int64_t f1 = crn_qpp_f1[ki], f2 = crn_qpp_f2[ki];
        qoff[ki] = (int32_t)qpp.size();
        qpp.resize(qpp.size() + (size_t)K);
        qts.resize(qpp.size());
        qin.resize(qpp.size());
        qiw.resize(qpp.size());
        for (int j = 0; j < M; j++)
            for (int i = 0; i < W; i++) {
                int64_t x = (int64_t)j * W + i;
                uint32_t n = (uint32_t)((f1 * x + f2 * x % K * x) % K);
                qpp[qoff[ki] + (size_t)i * M + j] = ((n % W) << 16) | (n / W);
                qts[qoff[ki] + (size_t)i * M + j] = (n % W) * CRN_CTA_THREADS + n / W;
                /* inverse: natural position n = Pi(x) is read back from interleaved position x */
                qin[qoff[ki] + (size_t)(n % W) * M + n / W] = (uint32_t)((x % W) * CRN_CTA_THREADS + x / W);
                qiw[qoff[ki] + (size_t)(n % W) * M + n / W] = (uint32_t)(((x % W) << 16) | (x / W));
            }
        cboff[ki] = (int32_t)cb.size();            /* per-bit CRC constants, window-major */
        cb.resize(cb.size() + 2 * (size_t)K);
        for (int k = 0; k < 2; k++) {
            uint32_t poly = k ? POLY_B : POLY_A, c = poly;        /* x^24 mod g for n = K-1 */
            for (int n = K - 1; n >= 0; n--) {
                cb[cboff[ki] + (size_t)k * K + (size_t)(n % W) * M + n / W] = c;
                c = mulx_mod(c, poly);
            }
        }
    }
    /* nibble tables of the W = 32 path's window CRC (crn_internal.h CRN_CRC_NIB_WORDS) */
    std::vector<uint32_t> nib(2 * (size_t)CRN_CRC_NIB_WORDS);
    for (int k = 0; k < 2; k++) {
        const uint32_t poly = k ? POLY_B : POLY_A;
        auto mulxn = [&](uint32_t r, int n) { for (int i = 0; i < n; i++) r = mulx_mod(r, poly); return r; };
        auto xpow = [&](int e) { return mulxn(1u, e); };            /* x^e mod g */
        uint32_t *T = nib.data() + (size_t)k * CRN_CRC_NIB_WORDS;
        for (int c = 0; c < 8; c++)
            for (int q = 0; q < 8; q++)
                for (int v = 0; v < 16; v++) {
                    uint32_t r = 0;
                    for (int b = 0; b < 4; b++)
                        if ((v >> b) & 1) r ^= xpow(55 - 4 * q - b);
                    T[c * 128 + q * 16 + v] = mulxn(r, 32 * c);
                }
        for (int l = 0; l < 2; l++)                                    /* TB (x^256 b), TA (x^2048 a) */
            for (int m = 0; m < (l ? 3 : 8); m++)
                for (int q = 0; q < 6; q++)
                    for (int v = 0; v < 16; v++)
                        T[(l ? 1792 : 1024) + m * 96 + q * 16 + v] = mulxn((uint32_t)v << (4 * q), (l ? 2048 : 256) * m);
    }
    DevTables t;
    if (cudaMalloc(&t.crc_nib, nib.size() * 4) != cudaSuccess ||
        cudaMalloc(&t.qpp_wm, qpp.size() * 4) != cudaSuccess ||
        cudaMalloc(&t.qpp_ts, qts.size() * 4) != cudaSuccess ||
        cudaMalloc(&t.qinv_ts, qin.size() * 4) != cudaSuccess ||
        cudaMalloc(&t.qinv_wm, qiw.size() * 4) != cudaSuccess ||
        cudaMalloc(&t.qpp_off, CRN_NUM_K * 4) != cudaSuccess ||
        cudaMalloc(&t.crc_bit, cb.size() * 4) != cudaSuccess ||
        cudaMalloc(&t.crcb_off, CRN_NUM_K * 4) != cudaSuccess ||
        cudaMalloc(&t.mi_tab, 256 * 4) != cudaSuccess) {
        cudaGetLastError();
        return CRN_ENOMEM;
    }
    cudaMemcpy(t.qpp_wm, qpp.data(), qpp.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(t.qpp_ts, qts.data(), qts.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(t.qinv_ts, qin.data(), qin.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(t.qinv_wm, qiw.data(), qiw.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(t.qpp_off, qoff.data(), CRN_NUM_K * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(t.crc_bit, cb.data(), cb.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(t.crcb_off, cboff.data(), CRN_NUM_K * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(t.crc_nib, nib.data(), nib.size() * 4, cudaMemcpyHostToDevice);
    int32_t mt[256];
    crn_mi_table(mt);
    cudaMemcpy(t.mi_tab, mt, sizeof(mt), cudaMemcpyHostToDevice);
    if (cudaError_t e = cudaGetLastError()) return crn_cuda_fail(e, "table upload", CRN_ECUDA);
    t.tab.qpp_wm = t.qpp_wm; t.tab.qpp_ts = t.qpp_ts; t.tab.qinv_ts = t.qinv_ts;
    t.tab.qpp_off = t.qpp_off;
    t.tab.crc_bit = t.crc_bit; t.tab.crcb_off = t.crcb_off; t.tab.mi_tab = t.mi_tab; t.tab.crc_nib = t.crc_nib;
    {
        uint32_t lo, hi;
        crn_logmap_words(&lo, &hi);
        crn_decode_set_logmap(lo, hi);
    }
    t.tab.qinv_wm = t.qinv_wm;
    {   /* the device task builder's per-size parameters and bucket issue order */
        std::vector<int32_t> bk(4 * CRN_NUM_K), ord(CRN_NUM_K);
        for (int ki = 0; ki < CRN_NUM_K; ki++) {
            int M, W, per, grp;
            crn_bucket_params(k_at(ki), &M, &W, &per, &grp);
            bk[4 * ki] = k_at(ki); bk[4 * ki + 1] = M; bk[4 * ki + 2] = W; bk[4 * ki + 3] = per | (grp << 16);
            ord[ki] = ki;
        }
        std::stable_sort(ord.begin(), ord.end(), [](int a, int b) {   /* K descending within one key */
            const int ka = crn_bucket_issue_key(k_at(a)), kb = crn_bucket_issue_key(k_at(b));
            return ka != kb ? ka > kb : k_at(a) > k_at(b);
        });
        if (cudaMalloc(&t.bucket, bk.size() * 4) != cudaSuccess || cudaMalloc(&t.border, ord.size() * 4) != cudaSuccess) {
            cudaGetLastError();
            return CRN_ENOMEM;
        }
        cudaMemcpy(t.bucket, bk.data(), bk.size() * 4, cudaMemcpyHostToDevice);
        cudaMemcpy(t.border, ord.data(), ord.size() * 4, cudaMemcpyHostToDevice);
    }
    t.grid = crn_decode_grid(dev);
    if (t.grid <= 0) {
        char where[96];
        snprintf(where, sizeof(where), "decode kernel configuration (code %d; needs exactly 1 CTA/SM)", t.grid);
        return crn_cuda_fail(cudaGetLastError(), where, CRN_ECUDA);
    }
    auto r = g_tables.emplace(dev, t);
    *out = &r.first->second;
    return CRN_OK;
}

int crn_get_ctx(int *dev, DevTables **t) {
    if (!check_device(dev)) { cudaGetLastError(); return CRN_ENODEV; }
    std::lock_guard<std::mutex> lk(g_mu);
    return build_tables(*dev, t);
}

int crn_get_ws(int dev, void *stream, size_t bytes, void **ws) {
    std::lock_guard<std::mutex> lk(g_mu);
    /* cudaStreamPerThread names a different stream on every host thread: key its
     * workspace by the calling thread, so two threads' concurrently running
     * persistent kernels never share a task counter (the legacy default stream is
     * one stream shared by all threads, whose launches serialise: one key) */
    static thread_local char per_thread_tag;
    if (stream == (void *)cudaStreamPerThread) stream = (void *)&per_thread_tag;
    auto key = std::make_pair(dev, stream);
    auto it = g_ws.find(key);
    if (it != g_ws.end() && it->second.second >= bytes) { *ws = it->second.first; return CRN_OK; }
    if (it != g_ws.end()) { cudaFree(it->second.first); g_ws.erase(it); }
    void *p = nullptr;
    if (cudaMalloc(&p, bytes) != cudaSuccess) { cudaGetLastError(); return CRN_ENOMEM; }
    g_ws[key] = std::make_pair(p, bytes);
    *ws = p;
    return CRN_OK;
}

extern "C" size_t crn_workspace_bytes(const crn_cb_desc *desc, int32_t n_cb) {
    (void)desc;                  /* the size depends on n_cb only */
    int dev;
    DevTables *t;
    if (n_cb < 0 || crn_get_ctx(&dev, &t) != CRN_OK) return 0;
    return crn_decode_ws_bytes(t->grid) + crn_tasks_dev_bytes(n_cb);
}

/* ------------------------------------------------------------------ plans (row a1) */
static bool ranges_overlap(std::vector<std::pair<int64_t, int64_t>> &r) {
    std::sort(r.begin(), r.end());
    for (size_t i = 1; i < r.size(); i++)
        if (r[i].first < r[i - 1].second) return true;
    return false;
}

/* Validate descriptors (crn.h: CRN_EINVAL rules). */
int crn_validate(const crn_cb_desc *d, int n, bool want_ext) {
    std::vector<std::pair<int64_t, int64_t>> lr, br, er;
    lr.reserve(n); br.reserve(n);
    for (int i = 0; i < n; i++) {
        const crn_cb_desc &c = d[i];
        if (crn_k_index(c.K) < 0 || c.F < 0 || c.F > c.K - 25 || c.crc_kind < 0 || c.crc_kind > 2 ||
            c.llr_off < 0 || c.bit_off < 0 || (want_ext && c.ext_off < 0))
            return CRN_EINVAL;
        lr.emplace_back(c.llr_off, c.llr_off + c.K + 4);
        br.emplace_back(c.bit_off, c.bit_off + (c.K + 31) / 32);
        if (want_ext) er.emplace_back(c.ext_off, c.ext_off + c.K);
    }
    if (ranges_overlap(lr) || ranges_overlap(br) || (want_ext && ranges_overlap(er))) return CRN_EINVAL;
    return CRN_OK;
}


/* Group tasks on or off (CRN_GROUPS=0 in the environment turns them off, for A/B runs). */
static bool groups_on() {
    static const int on = [] {
        const char *e = getenv("CRN_GROUPS");
        return (e && e[0] == '0') ? 0 : 1;
    }();
    return on != 0;
}

void crn_bucket_params(int K, int *M, int *W, int *per, int *grp) {
    crn_windows(K, M, W);
    *grp = *W == 32 && K <= CRN_GRP_SUMK && groups_on();
    *per = *grp ? std::max(1, std::min(CRN_GRP_SUMK / K, CRN_GRP_PAIRS))
                : std::max(1, std::min(CRN_TASK_SUMK / K, CRN_MAX_PAIRS));
    if (*W != 32)                      /* split-window path: shared memory and TMEM bound the task */
        while (*per > 1 && !crn_split_fits(*W, *M, *per)) (*per)--;
}

/* LPT issue key of a task of size K: a task's critical path is the trellis steps
 * one thread runs per half-iteration -- 16 on the W = 32 path (split windows),
 * ceil(W/2) on the split path; group tasks (key 0) after every whole-CTA task */
int crn_bucket_issue_key(int K) {
    int M, W, per, grp;
    crn_bucket_params(K, &M, &W, &per, &grp);
    return grp ? 0 : (W == 32 ? 16 : (W + 1) / 2);
}

/* Bucket by K (largest first: longest tasks start first), pair equal-K CBs in
 * index order, group floor(6144/K) pairs per whole-CTA task, or floor(2048/K)
 * pairs per group task for W = 32 and K <= 2048 (three such tasks share a CTA,
 * crn_internal.h CRN_GROUPS).  Whole-CTA tasks come first (LPT order), group
 * tasks last.  Returns the CTAs the appended tasks can keep busy at once:
 * whole-CTA tasks + ceil(group tasks / 3). */
int crn_build_tasks(const crn_cb_desc *d, const int *sel, int n, std::vector<crn_task> &tasks,
                    std::vector<crn_pair> &pairs, int spread_to) {
    const size_t t0 = tasks.size();
    std::vector<int> idx(sel, sel + n);
    std::stable_sort(idx.begin(), idx.end(), [&](int a, int b) { return d[a].K > d[b].K; });
    struct Bucket {
        int K, M, W, per, np, grp;
        size_t s, e;
        int64_t tasks() const { return (np + per - 1) / per; }
        int64_t thirds() const { return (grp ? 1 : CRN_GROUPS) * tasks(); }   /* CTA share x 3 */
    };
    std::vector<Bucket> bk;
    int64_t thirds = 0;
    size_t s = 0;
    while (s < idx.size()) {
        int K = d[idx[s]].K;
        size_t e = s;
        while (e < idx.size() && d[idx[e]].K == K) e++;
        Bucket b;
        b.K = K; b.s = s; b.e = e;
        crn_bucket_params(K, &b.M, &b.W, &b.per, &b.grp);
        b.np = (int)((e - s + 1) / 2);
        thirds += b.thirds();
        bk.push_back(b);
        s = e;
    }
    /* a small batch (fewer tasks than CTAs) is spread over more CTAs: the bucket
     * whose tasks hold the most windows gives up one pair per task while the
     * batch still fits in spread_to CTAs -- fewer windows per SM mean fewer
     * busy warps sharing its ALU pipe, so each task's dependent chain runs faster */
    const int64_t cap3 = (int64_t)CRN_GROUPS * spread_to;
    while (spread_to > 0 && thirds < cap3) {
        int best = -1;
        for (int i = 0; i < (int)bk.size(); i++)
            if (bk[i].per > 1 && bk[i].np > 1 && (best < 0 || bk[i].per * bk[i].M > bk[best].per * bk[best].M))
                best = i;
        if (best < 0) break;
        Bucket &b = bk[best];
        const int64_t before = b.thirds();
        const int cur = (int)b.tasks();                           /* one more, balanced, task */
        const int per_old = b.per;
        /* per strictly decreases, so the loop ends (floor((np + cur) / (cur + 1)) alone can
         * equal per, e.g. np = 16, per = 4) */
        b.per = std::min(b.per - 1, (b.np + cur) / (cur + 1));
        const int64_t grow = b.thirds() - before;
        if (thirds + grow > cap3) { b.per = per_old; break; }
        thirds += grow;
    }
    int64_t n_big = 0, n_grp = 0;
    for (const Bucket &b : bk) {
        int32_t first_pair = (int32_t)pairs.size();
        for (size_t i = b.s; i < b.e; i += 2) pairs.push_back({idx[i], i + 1 < b.e ? idx[i + 1] : -1});
        int32_t np = (int32_t)pairs.size() - first_pair;
        for (int32_t p = 0; p < np; p += b.per) {
            crn_task t;
            t.K = b.K; t.M = b.M; t.W = b.W; t.n_pairs = std::min(b.per, np - p);
            t.pair0 = first_pair + p; t.kidx = crn_k_index(b.K);
            t.grp = b.grp;
            tasks.push_back(t);
            (b.grp ? n_grp : n_big)++;
        }
    }
    /* whole-CTA tasks first, longest first (LPT order for the persistent grid), then
     * the group tasks (crn_bucket_issue_key) */
    std::stable_sort(tasks.begin() + (std::ptrdiff_t)t0, tasks.end(), [&](const crn_task &a, const crn_task &b) {
        return crn_bucket_issue_key(a.K) > crn_bucket_issue_key(b.K);
    });
    return (int)(n_big + (n_grp + CRN_GROUPS - 1) / CRN_GROUPS);
}

static int plan_build(const crn_cb_desc *desc, int n, bool want_ext, cudaStream_t st, bool async, Plan *P,
                      int spread_to) {
    int rc = crn_validate(desc, n, want_ext);
    if (rc) return rc;
    std::vector<crn_task> tasks;
    std::vector<crn_pair> pairs;
    std::vector<int> all(n);
    for (int i = 0; i < n; i++) all[i] = i;
    P->units = crn_build_tasks(desc, all.data(), n, tasks, pairs, spread_to);
    P->spread = spread_to;
    size_t b0 = sizeof(crn_cb_desc) * (size_t)n, b1 = sizeof(crn_task) * tasks.size(),
           b2 = sizeof(crn_pair) * pairs.size();
    size_t o1 = (b0 + 255) & ~(size_t)255, o2 = (o1 + b1 + 255) & ~(size_t)255, tot = o2 + b2 + 256;
    std::vector<uint8_t> host(tot);
    memcpy(host.data(), desc, b0);
    memcpy(host.data() + o1, tasks.data(), b1);
    memcpy(host.data() + o2, pairs.data(), b2);
    cudaError_t e = async ? cudaMallocAsync(&P->mem, tot, st) : cudaMalloc(&P->mem, tot);
    if (e != cudaSuccess) { cudaGetLastError(); return CRN_ENOMEM; }
    if (cudaMemcpyAsync(P->mem, host.data(), tot, cudaMemcpyHostToDevice, st) != cudaSuccess) {
        cudaGetLastError();
        return CRN_ECUDA;
    }
    if (!async && cudaStreamSynchronize(st) != cudaSuccess) return CRN_ECUDA;
    P->n_cb = n;
    P->n_tasks = (int)tasks.size();
    P->d_desc = (crn_cb_desc *)P->mem;
    P->d_tasks = (crn_task *)((uint8_t *)P->mem + o1);
    P->d_pairs = (crn_pair *)((uint8_t *)P->mem + o2);
    return CRN_OK;
}

int crn_launch_tasks(int dev, DevTables *t, const crn_cb_desc *d_desc, const crn_task *d_tasks, int n_tasks,
                     const crn_pair *d_pairs, const int16_t *l0, const int16_t *l1, const int16_t *l2,
                     int32_t max_iters, int32_t et, uint32_t *bits, uint8_t *ok, uint8_t *it, int16_t *ext,
                     void *ws, size_t ws_bytes, cudaStream_t st, int variant, uint8_t *tb_dead, int grid_cap,
                     bool ws_zeroed, int units) {
    if (n_tasks == 0) return CRN_OK;
    if (!ws) {
        int rc = crn_get_ws(dev, (void *)st, crn_decode_ws_bytes(t->grid), &ws);
        if (rc) return rc;
    } else if (ws_bytes < crn_decode_ws_bytes(t->grid)) {
        return CRN_EINVAL;
    }
    /* A batch whose tasks fit in one wave gets one CTA per task: group tasks then
     * run alone on their SM (one warp per sub-partition) instead of three to a
     * CTA -- cfg1 70 -> 52 us; larger batches keep the packed grid (CTA units).
     * CRN_GRID_PACK=1 keeps the packed grid always (A/B runs). */
    static const bool pack = [] {
        const char *e = getenv("CRN_GRID_PACK");
        return e && e[0] == '1';
    }();
    const int cap = grid_cap > 0 && grid_cap < t->grid ? grid_cap : t->grid;
    int g = units > 0 ? units : n_tasks;
    if (!pack && n_tasks > 0 && n_tasks <= cap) g = n_tasks;
    return crn_launch_decode(d_desc, d_tasks, n_tasks, d_pairs, l0, l1, l2, max_iters, et, bits, ok, it, ext,
                             &t->tab, ws, (void *)st, std::min(cap, g),
                             variant, tb_dead, ws_zeroed ? 1 : 0);
}

static int launch(Plan *P, DevTables *t, const int16_t *l0, const int16_t *l1, const int16_t *l2,
                  int32_t max_iters, int32_t et, uint32_t *bits, uint8_t *ok, uint8_t *it, int16_t *ext,
                  void *ws, size_t ws_bytes, cudaStream_t st) {
    if (P->n_cb == 0) return CRN_OK;
    uint8_t *dead = nullptr;
    if (P->purge && P->n_tb > 0) {
        if (!P->d_tb_dead && cudaMalloc(&P->d_tb_dead, (size_t)P->n_tb) != cudaSuccess) {
            cudaGetLastError();
            return CRN_ENOMEM;
        }
        dead = P->d_tb_dead;
        if (cudaMemsetAsync(dead, 0, (size_t)P->n_tb, st) != cudaSuccess) return CRN_ECUDA;
    }
    return crn_launch_tasks(P->dev, t, P->d_desc, P->d_tasks, P->n_tasks, P->d_pairs, l0, l1, l2, max_iters, et,
                            bits, ok, it, ext, ws, ws_bytes, st, crn_plan_kernel_variant(P), dead, P->grid_cap,
                            false, P->units);
}

extern "C" int crn_plan_create(const crn_cb_desc *desc, int32_t n_cb, void **plan) {
    if (!plan || n_cb < 0 || (n_cb > 0 && !desc)) return CRN_EINVAL;
    int dev;
    DevTables *t;
    int rc = crn_get_ctx(&dev, &t);
    if (rc) return rc;
    Plan *P = new Plan();
    P->dev = dev;
    rc = plan_build(desc, n_cb, true, 0, false, P, t->grid);
    if (rc) { delete P; return rc; }
    P->h_desc.assign(desc, desc + n_cb);
    *plan = P;
    return CRN_OK;
}

extern "C" int crn_plan_decode(void *plan, const int16_t *l0, const int16_t *l1, const int16_t *l2,
                               int32_t max_iters, int32_t et, uint32_t *bits, uint8_t *ok, uint8_t *it,
                               int16_t *ext, void *stream) {
    Plan *P = (Plan *)plan;
    if (!P || max_iters < 1 || max_iters > CRN_MAX_ITERS || et < 0 || et > CRN_ET_MI) return CRN_EINVAL;
    if (P->n_cb && (!l0 || !l1 || !l2 || !bits || !ok)) return CRN_EINVAL;
    int dev;
    DevTables *t;
    int rc = crn_get_ctx(&dev, &t);
    if (rc) return rc;
    if (dev != P->dev) return CRN_EINVAL;
    return launch(P, t, l0, l1, l2, max_iters, et, bits, ok, it, ext, nullptr, 0, (cudaStream_t)stream);
}

extern "C" int crn_plan_set_variant(void *plan, int32_t variant) {
    Plan *P = (Plan *)plan;
    if (!P || (variant != CRN_VARIANT_MAXLOG && variant != CRN_VARIANT_SCALED && variant != CRN_VARIANT_LOGMAP))
        return CRN_EINVAL;
    P->variant = variant;
    return CRN_OK;
}

extern "C" int crn_plan_set_purge(void *plan, int32_t on) {
    Plan *P = (Plan *)plan;
    if (!P || on < 0 || on > 1) return CRN_EINVAL;
    if (on) {                                   /* TB ids: reserved >= -1, n_tb = max + 1 */
        int n_tb = 0;
        for (const crn_cb_desc &d : P->h_desc) {
            if (d.reserved < -1) return CRN_EINVAL;
            n_tb = std::max(n_tb, d.reserved + 1);
        }
        P->n_tb = n_tb;
    }
    P->purge = on;
    return CRN_OK;
}

int crn_plan_kernel_variant(const Plan *P) { return P->variant | ((P->llr8 + 1) << 8); }

extern "C" int crn_plan_set_llr_format(void *plan, int32_t bits, int32_t shift) {
    Plan *P = (Plan *)plan;
    if (!P) return CRN_EINVAL;
    if (bits == 16 && shift == 0) { P->llr8 = -1; return CRN_OK; }
    if (bits == 8 && shift >= 0 && shift <= 8) { P->llr8 = shift; return CRN_OK; }
    return CRN_EINVAL;
}

extern "C" int crn_plan_llr_bytes(void *plan) {
    const Plan *P = (const Plan *)plan;
    return P ? (P->llr8 < 0 ? 2 : 1) : CRN_EINVAL;
}

extern "C" int crn_plan_set_grid(void *plan, int32_t max_ctas) {
    Plan *P = (Plan *)plan;
    if (!P || max_ctas < 0) return CRN_EINVAL;
    P->grid_cap = max_ctas;
    return CRN_OK;
}

extern "C" int crn_plan_layout(void *plan, int32_t *task_of_cb, int32_t n_cb) {
    /* diagnostic: the CTA task each CB was bucketed into (row a1), -1 if none */
    Plan *P = (Plan *)plan;
    if (!P || !task_of_cb || n_cb != P->n_cb) return CRN_EINVAL;
    std::vector<crn_task> tasks;
    std::vector<crn_pair> pairs;
    std::vector<int> all(P->n_cb);
    for (int i = 0; i < P->n_cb; i++) all[i] = i;
    crn_build_tasks(P->h_desc.data(), all.data(), P->n_cb, tasks, pairs, P->spread);
    for (int i = 0; i < n_cb; i++) task_of_cb[i] = -1;
    for (size_t t = 0; t < tasks.size(); t++)
        for (int p = 0; p < tasks[t].n_pairs; p++) {
            const crn_pair &q = pairs[(size_t)tasks[t].pair0 + p];
            task_of_cb[q.lo] = (int32_t)t;
            if (q.hi >= 0) task_of_cb[q.hi] = (int32_t)t;
        }
    return (int)tasks.size();
}

extern "C" int crn_task_layout(const crn_cb_desc *desc, int32_t n_cb, int32_t spread_to, int32_t *task_of_cb,
                               int32_t *task_info, int32_t *units) {
    if (n_cb < 0 || spread_to < 0 || (n_cb > 0 && (!desc || !task_of_cb))) return CRN_EINVAL;
    if (crn_validate(desc, n_cb, false)) return CRN_EINVAL;
    std::vector<crn_task> tasks;
    std::vector<crn_pair> pairs;
    std::vector<int> all(n_cb);
    for (int i = 0; i < n_cb; i++) all[i] = i;
    const int u = crn_build_tasks(desc, all.data(), n_cb, tasks, pairs, spread_to);
    if (units) *units = u;
    for (int i = 0; i < n_cb; i++) task_of_cb[i] = -1;
    for (size_t t = 0; t < tasks.size(); t++) {
        for (int p = 0; p < tasks[t].n_pairs; p++) {
            const crn_pair &q = pairs[(size_t)tasks[t].pair0 + p];
            task_of_cb[q.lo] = (int32_t)t;
            if (q.hi >= 0) task_of_cb[q.hi] = (int32_t)t;
        }
        if (task_info) {
            task_info[4 * t] = tasks[t].K;
            task_info[4 * t + 1] = tasks[t].n_pairs;
            task_info[4 * t + 2] = tasks[t].n_pairs * tasks[t].M;
            task_info[4 * t + 3] = tasks[t].grp;
        }
    }
    return (int)tasks.size();
}

extern "C" int crn_plan_launches(void *plan) {
    Plan *P = (Plan *)plan;
    return (P && P->n_cb) ? 1 : 0;
}

extern "C" void crn_plan_destroy(void *plan) {
    Plan *P = (Plan *)plan;
    if (!P) return;
    if (P->pipe) crn_pipe_destroy(P->pipe);
    if (P->d_tb_dead) cudaFree(P->d_tb_dead);
    if (P->mem) cudaFree(P->mem);
    delete P;
}

/* Plans behind the one-shot calls (crn_decode_batch / _ex with HOST descriptors):
 * a BBU decodes the same CB layout TTI after TTI, so the last few
 * validated + bucketed + uploaded descriptor sets are kept, keyed by the exact
 * descriptor bytes (and device, n_cb, ext_out use).  A hit costs one memcmp; a
 * miss builds the plan and uploads it on a private stream (never waiting on the
 * caller's).  Entries are shared_ptrs: a plan evicted while another thread still
 * launches from it lives until that launch is enqueued; its device memory is
 * released by cudaFree, which waits for the device. */
namespace {
struct CachedPlan {
    int dev = -1;
    bool want_ext = false;
    int n_tb = 0;                             /* TB ids in the reserved field (purge) */
    std::vector<crn_cb_desc> key;
    Plan P;
    ~CachedPlan() {
        if (P.mem) cudaFree(P.mem);
    }
};
constexpr size_t PLAN_CACHE = 4;
std::mutex g_pc_mu;
std::vector<std::shared_ptr<CachedPlan>> g_pc;   /* most recently used first */
std::map<int, cudaStream_t> g_upload_stream;      /* per device, non-blocking */

int cached_plan(int dev, DevTables *t, const crn_cb_desc *desc, int n, bool want_ext,
                std::shared_ptr<CachedPlan> *out) {
    {
        std::lock_guard<std::mutex> lk(g_pc_mu);
        for (size_t i = 0; i < g_pc.size(); i++) {
            const auto &c = g_pc[i];
            if (c->dev == dev && c->want_ext == want_ext && c->key.size() == (size_t)n &&
                memcmp(c->key.data(), desc, sizeof(crn_cb_desc) * (size_t)n) == 0) {
                *out = c;
                std::rotate(g_pc.begin(), g_pc.begin() + (std::ptrdiff_t)i, g_pc.begin() + (std::ptrdiff_t)i + 1);
                return CRN_OK;
            }
        }
    }
    auto c = std::make_shared<CachedPlan>();
    c->dev = dev;
    c->want_ext = want_ext;
    c->key.assign(desc, desc + n);
    for (int i = 0; i < n; i++) {
        if (desc[i].reserved < -1) c->n_tb = -1;
        else if (c->n_tb >= 0) c->n_tb = std::max(c->n_tb, desc[i].reserved + 1);
    }
    cudaStream_t up;
    {
        std::lock_guard<std::mutex> lk(g_pc_mu);
        auto it = g_upload_stream.find(dev);
        if (it == g_upload_stream.end()) {
            if (cudaStreamCreateWithFlags(&up, cudaStreamNonBlocking) != cudaSuccess) {
                cudaGetLastError();
                return CRN_ECUDA;
            }
            g_upload_stream[dev] = up;
        } else {
            up = it->second;
        }
    }
    c->P.dev = dev;
    int rc = plan_build(desc, n, want_ext, up, false, &c->P, t->grid);   /* cudaMalloc + upload + sync of `up` */
    if (rc) return rc;
    std::lock_guard<std::mutex> lk(g_pc_mu);
    g_pc.insert(g_pc.begin(), c);
    if (g_pc.size() > PLAN_CACHE) g_pc.pop_back();
    *out = c;
    return CRN_OK;
}
}  // namespace

extern "C" int crn_decode_batch_ex(const crn_cb_desc *desc, int32_t n_cb, const int16_t *l0,
                                   const int16_t *l1, const int16_t *l2, int32_t max_iters,
                                   int32_t et, int32_t flags, uint32_t *bits, uint8_t *ok,
                                   uint8_t *it, int16_t *ext, void *ws, size_t ws_bytes, void *stream) {
    if (n_cb < 0 || (flags & ~(CRN_DESC_ON_DEVICE | CRN_EXT_SCALED | CRN_PURGE)) || max_iters < 1 ||
        max_iters > CRN_MAX_ITERS ||
        et < 0 || et > CRN_ET_MI)
        return CRN_EINVAL;
    if (n_cb == 0) return CRN_OK;
    if (!desc || !l0 || !l1 || !l2 || !bits || !ok) return CRN_EINVAL;
    int dev;
    DevTables *t;
    int rc = crn_get_ctx(&dev, &t);
    if (rc) return rc;
    cudaStream_t st = (cudaStream_t)stream;
    const int variant = (flags & CRN_EXT_SCALED) ? CRN_VARIANT_SCALED : CRN_VARIANT_MAXLOG;
    if (flags & CRN_DESC_ON_DEVICE) {
        /* row a1 on the device (crn_tasks.cu): nothing returns to the host, nothing waits */
        const size_t head = crn_decode_ws_bytes(t->grid), need = head + crn_tasks_dev_bytes(n_cb);
        if (!ws) {
            rc = crn_get_ws(dev, (void *)st, need, &ws);
            if (rc) return rc;
        } else if (ws_bytes < need) {
            return CRN_EINVAL;
        }
        crn_task *dt;
        crn_pair *dp;
        uint8_t *dead;
        rc = crn_launch_tasks_dev(desc, n_cb, ext != nullptr, (flags & CRN_PURGE) != 0, t->bucket, t->border,
                                  (uint8_t *)ws + head, (int32_t *)ws, &dt, &dp, &dead, ok, it, (void *)st);
        if (rc) return crn_cuda_fail(cudaGetLastError(), "device task builder launch", rc);
        return crn_launch_decode(desc, dt, -1, dp, l0, l1, l2, max_iters, et, bits, ok, it, ext, &t->tab, ws,
                                 (void *)st, t->grid, variant, dead, 1);
    }
    std::shared_ptr<CachedPlan> c;
    rc = cached_plan(dev, t, desc, n_cb, ext != nullptr, &c);
    if (rc) return rc;
    uint8_t *dead = nullptr;
    if (flags & CRN_PURGE) {
        if (c->n_tb < 0) return CRN_EINVAL;
        if (c->n_tb > 0) {
            if (cudaMallocAsync((void **)&dead, (size_t)c->n_tb, st) != cudaSuccess) {
                cudaGetLastError();
                return CRN_ENOMEM;
            }
            cudaMemsetAsync(dead, 0, (size_t)c->n_tb, st);
        }
    }
    const Plan &P = c->P;
    rc = crn_launch_tasks(P.dev, t, P.d_desc, P.d_tasks, P.n_tasks, P.d_pairs, l0, l1, l2, max_iters, et, bits, ok,
                          it, ext, ws, ws_bytes, st, variant, dead, 0, false, P.units);
    if (dead) cudaFreeAsync(dead, st);
    return rc;
}

extern "C" int crn_decode_batch(const int16_t *l0, const int16_t *l1, const int16_t *l2, const int32_t *K,
                                int32_t n_cb, int32_t iters, uint32_t *bits, uint8_t *ok) {
    if (n_cb < 0 || iters == 0 || iters > CRN_MAX_ITERS || iters < -CRN_MAX_ITERS) return CRN_EINVAL;
    if (n_cb == 0) return CRN_OK;
    if (!K) return CRN_EINVAL;
    std::vector<crn_cb_desc> d(n_cb);
    int64_t lo = 0, bo = 0;
    for (int i = 0; i < n_cb; i++) {
        d[i].K = K[i]; d[i].F = 0; d[i].crc_kind = CRN_CRC24B; d[i].reserved = 0;
        d[i].llr_off = lo; d[i].bit_off = bo; d[i].ext_off = 0;
        lo += (int64_t)K[i] + 4;
        bo += ((int64_t)K[i] + 31) / 32;
    }
    return crn_decode_batch_ex(d.data(), n_cb, l0, l1, l2, iters > 0 ? iters : -iters, iters < 0, 0, bits,
                               ok, nullptr, nullptr, nullptr, 0, nullptr);
}

/* ------------------------------------------------------------------ encode / ubench wrappers */
/* ------------------------------------------------------------------ descriptor uploads */
/* Stream-ordered upload of a host descriptor array for the one-shot batch calls
 * (encode, rate matching, TB verdicts): a memcpy into a pinned staging buffer
 * kept per (host thread, device) and an asynchronous DMA from it, so the call
 * does not wait on a pageable copy (which waits for the stream).  Four staging
 * buffers rotate; one is reused once its previous copy has completed (event).
 * *d_out is stream-ordered device memory (cudaFreeAsync it on the same stream). */
namespace {
struct UploadStage {
    void *pin = nullptr;
    size_t cap = 0;
    cudaEvent_t ev = nullptr;
    bool pending = false;
};
constexpr int UPLOAD_RING = 4;
struct UploadRing {
    UploadStage slot[UPLOAD_RING];
    int next = 0;
};
struct UploadStages {
    std::map<int, UploadRing> by_dev;
    ~UploadStages() {                        /* thread exit: best effort */
        for (auto &kv : by_dev)
            for (UploadStage &u : kv.second.slot) {
                if (u.ev) cudaEventDestroy(u.ev);
                if (u.pin) cudaFreeHost(u.pin);
            }
    }
};
thread_local UploadStages g_upload;
}  // namespace

static int crn_upload(const void *const *parts, const size_t *sizes, const size_t *offs, int n_parts, size_t total,
                      int dev, cudaStream_t st, void **d_out) {
    UploadRing &ring = g_upload.by_dev[dev];
    UploadStage &u = ring.slot[ring.next];
    ring.next = (ring.next + 1) % UPLOAD_RING;
    if (!u.ev && cudaEventCreateWithFlags(&u.ev, cudaEventDisableTiming) != cudaSuccess) {
        cudaGetLastError();
        return CRN_ECUDA;
    }
    if (u.pending) cudaEventSynchronize(u.ev);        /* the previous copy out of the staging buffer */
    u.pending = false;
    if (u.cap < total) {
        if (u.pin) cudaFreeHost(u.pin);
        u.pin = nullptr;
        u.cap = 0;
        const size_t cap = std::max(total, (size_t)1 << 16) * 2;
        if (cudaMallocHost(&u.pin, cap) != cudaSuccess) { cudaGetLastError(); return CRN_ENOMEM; }
        u.cap = cap;
    }
    for (int i = 0; i < n_parts; i++) memcpy((uint8_t *)u.pin + offs[i], parts[i], sizes[i]);
    if (cudaMallocAsync(d_out, total, st) != cudaSuccess) { cudaGetLastError(); return CRN_ENOMEM; }
    if (cudaMemcpyAsync(*d_out, u.pin, total, cudaMemcpyHostToDevice, st) != cudaSuccess ||
        cudaEventRecord(u.ev, st) != cudaSuccess) {
        cudaGetLastError();
        cudaFreeAsync(*d_out, st);
        return CRN_ECUDA;
    }
    u.pending = true;
    return CRN_OK;
}

static int crn_upload1(const void *h, size_t bytes, int dev, cudaStream_t st, void **d_out) {
    const size_t off = 0;
    return crn_upload(&h, &bytes, &off, 1, bytes, dev, st, d_out);
}

static int encode_common(const crn_cb_desc *desc, int32_t n_cb, const void *info, int32_t attach_crc, void *d0,
                         void *d1, void *d2, int32_t packed, void *stream) {
    if (n_cb < 0) return CRN_EINVAL;
    if (n_cb == 0) return CRN_OK;
    if (!desc || !info || !d0 || !d1 || !d2) return CRN_EINVAL;
    for (int i = 0; i < n_cb; i++)
        if (crn_k_index(desc[i].K) < 0 || desc[i].F < 0 || desc[i].F > desc[i].K - 25 ||
            desc[i].crc_kind < 0 || desc[i].crc_kind > 2 || desc[i].llr_off < 0 || desc[i].ext_off < 0)
            return CRN_EINVAL;
    int dev;
    DevTables *t;
    int rc = crn_get_ctx(&dev, &t);
    if (rc) return rc;
    cudaStream_t st = (cudaStream_t)stream;
    void *dd = nullptr;
    if ((rc = crn_upload1(desc, sizeof(crn_cb_desc) * (size_t)n_cb, dev, st, &dd))) return rc;
    rc = crn_launch_encode((const crn_cb_desc *)dd, n_cb, info, attach_crc, d0, d1, d2, packed, &t->tab, (void *)st);
    cudaFreeAsync(dd, st);
    return rc;
}

extern "C" int crn_encode_batch(const crn_cb_desc *desc, int32_t n_cb, const uint8_t *info, int32_t attach_crc,
                                uint8_t *d0, uint8_t *d1, uint8_t *d2, void *stream) {
    return encode_common(desc, n_cb, info, attach_crc, d0, d1, d2, 0, stream);
}

extern "C" int crn_encode_batch_packed(const crn_cb_desc *desc, int32_t n_cb, const uint32_t *info,
                                       int32_t attach_crc, uint32_t *d0, uint32_t *d1, uint32_t *d2, void *stream) {
    return encode_common(desc, n_cb, info, attach_crc, d0, d1, d2, 1, stream);
}

extern "C" int crn_ubench_int16x2(int32_t op, int64_t *lane_instr, float *ms, int64_t *cycles) {
    int dev;
    if (!check_device(&dev)) { cudaGetLastError(); return CRN_ENODEV; }
    if (op < 0 || op > 3 || !lane_instr || !ms || !cycles) return CRN_EINVAL;
    return crn_launch_ubench(op, lane_instr, ms, cycles);
}

/* ------------------------------------------------------------------ TB <-> CB (row a1, host) */
extern "C" int crn_tb_build_cbs(const uint8_t *tb, int64_t tbs, int32_t max_cb, int64_t base_bit,
                                int64_t base_llr, int64_t base_word, uint8_t *cb_bits, crn_cb_desc *desc,
                                int32_t *n_cb) {
    if (!tb || !cb_bits || !desc || !n_cb) return CRN_EINVAL;
    crn_seg s;
    if (crn_segment_tb(tbs, &s) != CRN_OK || s.C > max_cb) return CRN_EINVAL;
    std::vector<uint8_t> b((size_t)tbs + 24);
    for (int64_t i = 0; i < tbs; i++) b[i] = tb[i] & 1u;
    uint32_t r = crc24(0, b.data(), tbs);
    for (int i = 0; i < 24; i++) b[tbs + i] = (uint8_t)((r >> (23 - i)) & 1u);
    int64_t src = 0, bit = 0, llr = 0, word = 0;
    for (int c = 0; c < s.C; c++) {
        int K = c < s.Cminus ? s.Kminus : s.Kplus, F = c == 0 ? s.F : 0;
        uint8_t *o = cb_bits + bit;
        for (int k = 0; k < F; k++) o[k] = 0;
        for (int k = F; k < K - s.L; k++) o[k] = b[src++];
        if (s.C > 1) {
            uint32_t rb = crc24(1, o, K - 24);
            for (int i = 0; i < 24; i++) o[K - 24 + i] = (uint8_t)((rb >> (23 - i)) & 1u);
        }
        crn_cb_desc &d = desc[c];
        d.K = K; d.F = F; d.crc_kind = s.C > 1 ? CRN_CRC24B : CRN_CRC24A; d.reserved = 0;
        d.ext_off = base_bit + bit; d.llr_off = base_llr + llr; d.bit_off = base_word + word;
        bit += K; llr += K + 4; word += (K + 31) / 32;
    }
    *n_cb = s.C;
    return src == tbs + 24 ? CRN_OK : CRN_EINVAL;
}

extern "C" int crn_tb_build_cbs_batch(const int64_t *tbs_bits, const int64_t *payload_off, int32_t n_tb,
                                      const uint8_t *payload, int32_t max_cb, uint8_t *cb_bits, crn_cb_desc *desc,
                                      int32_t *n_cb, void *stream) {
    if (n_tb < 0 || max_cb < 0 || !n_cb) return CRN_EINVAL;
    *n_cb = 0;
    if (n_tb == 0) return CRN_OK;
    if (!tbs_bits || !payload_off || !payload || !cb_bits || !desc) return CRN_EINVAL;
    std::vector<crn_tbseg> rec((size_t)n_tb);
    int32_t n = 0;
    int64_t bit = 0, llr = 0, word = 0, max_tbs = 0;
    for (int t = 0; t < n_tb; t++) {
        crn_seg g;
        if (payload_off[t] < 0 || crn_segment_tb(tbs_bits[t], &g) != CRN_OK || g.C > CRN_TB_MAX_CB ||
            (int64_t)n + g.C > max_cb)
            return CRN_EINVAL;
        crn_tbseg &r = rec[(size_t)t];
        r.tbs = tbs_bits[t]; r.payload_off = payload_off[t]; r.cb_bit0 = bit;
        r.C = g.C; r.Kplus = g.Kplus; r.Kminus = g.Kminus; r.Cminus = g.Cminus; r.F = g.F; r.L = g.L;
        max_tbs = std::max(max_tbs, tbs_bits[t]);
        for (int c = 0; c < g.C; c++) {           /* 36.212 5.1.2: the C- smaller CBs first, fillers in CB 0 */
            crn_cb_desc &d = desc[n++];
            d.K = c < g.Cminus ? g.Kminus : g.Kplus;
            d.F = c == 0 ? g.F : 0;
            d.crc_kind = g.C > 1 ? CRN_CRC24B : CRN_CRC24A;
            d.reserved = t;
            d.ext_off = bit; d.llr_off = llr; d.bit_off = word;
            bit += d.K; llr += d.K + 4; word += (d.K + 31) / 32;
        }
    }
    int dev;
    DevTables *tt;
    int rc = crn_get_ctx(&dev, &tt);
    if (rc) return rc;
    cudaStream_t st = (cudaStream_t)stream;
    void *dd = nullptr;
    if ((rc = crn_upload1(rec.data(), sizeof(crn_tbseg) * rec.size(), dev, st, &dd))) return rc;
    rc = crn_launch_tbseg((const crn_tbseg *)dd, n_tb, max_tbs, payload, cb_bits, (void *)st);
    cudaFreeAsync(dd, st);
    if (rc == CRN_OK) *n_cb = n;
    return rc;
}

extern "C" int crn_tb_reassemble(const uint32_t *w, const crn_cb_desc *desc, const uint8_t *ok, int32_t n_cb,
                                 int64_t tbs, uint8_t *out) {
    if (!w || !desc || !ok || n_cb < 1) return CRN_EINVAL;
    crn_seg s;
    if (crn_segment_tb(tbs, &s) != CRN_OK || s.C != n_cb) return CRN_EINVAL;
    std::vector<uint8_t> b;
    b.reserve((size_t)tbs + 24);
    bool all = true;
    for (int c = 0; c < n_cb; c++) {
        const crn_cb_desc &d = desc[c];
        all = all && ok[c];
        for (int k = d.F; k < d.K - s.L; k++) b.push_back((uint8_t)((w[d.bit_off + k / 32] >> (k % 32)) & 1u));
    }
    if ((int64_t)b.size() != tbs + 24) return CRN_EINVAL;
    if (!all || crc24(0, b.data(), tbs + 24) != 0) return 0;
    if (out) memcpy(out, b.data(), (size_t)tbs);
    return 1;
}

extern "C" int crn_tb_verdict_batch(const crn_tb_desc *tb, int32_t n_tb, const crn_cb_desc *desc, int32_t n_cb,
                                    const uint32_t *cb_words, const uint8_t *crc_ok, uint8_t *tb_ok,
                                    uint32_t *tb_words, void *stream) {
    if (n_tb < 0 || n_cb < 0) return CRN_EINVAL;
    if (n_tb == 0) return CRN_OK;
    if (!tb || !desc || !cb_words || !crc_ok || !tb_ok) return CRN_EINVAL;
    for (int i = 0; i < n_tb; i++) {
        const crn_tb_desc &t = tb[i];
        crn_seg s;
        if (t.cb0 < 0 || t.n_cb < 1 || t.n_cb > CRN_TB_MAX_CB || (int64_t)t.cb0 + t.n_cb > n_cb ||
            t.word_off < 0 || crn_segment_tb(t.tbs, &s) != CRN_OK || s.C != t.n_cb)
            return CRN_EINVAL;
        for (int r = 0; r < t.n_cb; r++) {
            const crn_cb_desc &d = desc[t.cb0 + r];
            if (d.K != (r < s.Cminus ? s.Kminus : s.Kplus) || d.F != (r == 0 ? s.F : 0) ||
                d.crc_kind != (s.C > 1 ? CRN_CRC24B : CRN_CRC24A) || d.bit_off < 0)
                return CRN_EINVAL;
        }
    }
    int dev;
    DevTables *t;
    int rc = crn_get_ctx(&dev, &t);
    if (rc) return rc;
    cudaStream_t st = (cudaStream_t)stream;
    const size_t b0 = sizeof(crn_tb_desc) * (size_t)n_tb, o1 = (b0 + 255) & ~(size_t)255;
    const size_t tot = o1 + sizeof(crn_cb_desc) * (size_t)n_cb;
    void *dm = nullptr;
    const void *parts[2] = {tb, desc};
    const size_t sizes[2] = {b0, sizeof(crn_cb_desc) * (size_t)n_cb}, offs[2] = {0, o1};
    if ((rc = crn_upload(parts, sizes, offs, 2, tot, dev, st, &dm))) return rc;
    rc = crn_launch_tb((const crn_tb_desc *)dm, n_tb, (const crn_cb_desc *)((uint8_t *)dm + o1), cb_words, crc_ok,
                       tb_ok, tb_words, (void *)st);
    cudaFreeAsync(dm, st);
    if (cudaError_t e = cudaGetLastError()) return crn_cuda_fail(e, "crn_tb_verdict_batch", CRN_ECUDA);
    return rc;
}

/* ------------------------------------------------------------------ rate matching (row f4) */
static int rm_validate(const crn_rm_desc *desc, int32_t n_cb) {
    for (int i = 0; i < n_cb; i++) {
        const crn_rm_desc &d = desc[i];
        if (crn_k_index(d.K) < 0 || d.E < 1 || d.rv < 0 || d.rv > 3 || d.e_off < 0 || d.llr_off < 0)
            return CRN_EINVAL;
    }
    return CRN_OK;
}

static int rm_upload(const crn_rm_desc *desc, int32_t n_cb, int dev, cudaStream_t st, void **dd) {
    return crn_upload1(desc, sizeof(crn_rm_desc) * (size_t)n_cb, dev, st, dd);
}

extern "C" int crn_rate_dematch_batch(const crn_rm_desc *desc, int32_t n_cb, const int16_t *e, int32_t combine,
                                      int16_t *h0, int16_t *h1, int16_t *h2, void *stream) {
    if (n_cb < 0) return CRN_EINVAL;
    if (n_cb == 0) return CRN_OK;
    if (!desc || !e || !h0 || !h1 || !h2 || rm_validate(desc, n_cb)) return CRN_EINVAL;
    int dev;
    DevTables *t;
    int rc = crn_get_ctx(&dev, &t);
    if (rc) return rc;
    cudaStream_t st = (cudaStream_t)stream;
    void *dd = nullptr;
    if ((rc = rm_upload(desc, n_cb, dev, st, &dd))) return rc;
    rc = crn_launch_dematch((const crn_rm_desc *)dd, n_cb, e, combine, h0, h1, h2, (void *)st);
    cudaFreeAsync(dd, st);
    return rc;
}

extern "C" int crn_rate_match_batch(const crn_rm_desc *desc, int32_t n_cb, const uint8_t *d0, const uint8_t *d1,
                                    const uint8_t *d2, uint8_t *e, void *stream) {
    if (n_cb < 0) return CRN_EINVAL;
    if (n_cb == 0) return CRN_OK;
    if (!desc || !d0 || !d1 || !d2 || !e || rm_validate(desc, n_cb)) return CRN_EINVAL;
    int dev;
    DevTables *t;
    int rc = crn_get_ctx(&dev, &t);
    if (rc) return rc;
    cudaStream_t st = (cudaStream_t)stream;
    void *dd = nullptr;
    if ((rc = rm_upload(desc, n_cb, dev, st, &dd))) return rc;
    rc = crn_launch_match((const crn_rm_desc *)dd, n_cb, d0, d1, d2, e, (void *)st);
    cudaFreeAsync(dd, st);
    return rc;
}

extern "C" int crn_rate_match_batch_packed(const crn_rm_desc *desc, int32_t n_cb, const uint32_t *d0,
                                           const uint32_t *d1, const uint32_t *d2, uint32_t *e, void *stream) {
    if (n_cb < 0) return CRN_EINVAL;
    if (n_cb == 0) return CRN_OK;
    if (!desc || !d0 || !d1 || !d2 || !e || rm_validate(desc, n_cb)) return CRN_EINVAL;
    int dev;
    DevTables *t;
    int rc = crn_get_ctx(&dev, &t);
    if (rc) return rc;
    cudaStream_t st = (cudaStream_t)stream;
    void *dd = nullptr;
    if ((rc = rm_upload(desc, n_cb, dev, st, &dd))) return rc;
    rc = crn_launch_match_packed((const crn_rm_desc *)dd, n_cb, d0, d1, d2, e, (void *)st);
    cudaFreeAsync(dd, st);
    return rc;
}
