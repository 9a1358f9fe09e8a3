/* crn_runtime.cpp -- libcrn's host runtime around the decode kernel:
 *
 *  (1) crn_plan_decode_host: decode from HOST buffers.  The plan's CBs are cut
 *      into chunks of consecutive CB indices; chunk c's LLRs are copied in on a
 *      copy stream while chunk c-1 decodes on the caller's stream and chunk
 *      c-2's results are copied out on a third stream, so the PCIe transfers
 *      overlap the decode (the end-to-end path of a BBU whose LLRs arrive from
 *      the fronthaul into host memory).
 *
 *  (2) crn_stream_run: the paper's per-TTI operation ("CCDUs
 *      arrive in batches every millisecond"; Algorithm 2, :372-393) as a paced
 *      streaming executor: TTI i is released at t0 + i * period; each cell
 *      group has its own CUDA stream (H2D -> decode -> D2H); a completion
 *      thread time-stamps every (TTI, group) the moment its last copy lands,
 *      like the paper's performance captor which records
 *      the stage timestamps outside the real-time path.
 *
 * Nothing here computes the method: all decoding runs in crn_decode.cu.
 */
#include <cuda.h>            /* types of the one driver entry point used (cuStreamWriteValue32) */
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstring>
#include <thread>
#include <vector>

#include "crn_internal.h"
#include "crn_plan.h"

namespace {

using Clock = std::chrono::steady_clock;

double us_since(Clock::time_point t0, Clock::time_point t) {
    return std::chrono::duration<double, std::micro>(t - t0).count();
}

struct Chunk {
    int32_t cb0 = 0, cb1 = 0;             /* CB index range [cb0, cb1) */
    int64_t llr0 = 0, llr1 = 0;           /* element range of the chunk's LLRs */
    int64_t w0 = 0, w1 = 0;               /* output word range */
    int32_t task0 = 0, n_tasks = 0;       /* slice of the pipe's task array */
    int32_t units = 0;                    /* CTAs its tasks fill (crn_build_tasks) */
};

}  // namespace

struct HostPipe {
    int requested = 0;                    /* chunk count asked for (n_chunks may be smaller) */
    int n_chunks = 0;
    std::vector<Chunk> ch;
    void *mem = nullptr;                  /* device: tasks, pairs, LLR staging, outputs */
    crn_task *d_tasks = nullptr;
    crn_pair *d_pairs = nullptr;
    int16_t *d_l[3] = {nullptr, nullptr, nullptr};
    uint32_t *d_bits = nullptr;
    uint8_t *d_ok = nullptr, *d_it = nullptr;
    int64_t n_llr = 0, n_words = 0;
    cudaStream_t s_in = nullptr, s_out = nullptr;
    std::vector<cudaEvent_t> ev_in, ev_comp;
    cudaEvent_t ev_start = nullptr, ev_end = nullptr;
};

void crn_pipe_destroy(HostPipe *p) {
    if (!p) return;
    if (p->s_in) cudaStreamSynchronize(p->s_in);
    if (p->s_out) cudaStreamSynchronize(p->s_out);
    for (auto e : p->ev_in) cudaEventDestroy(e);
    for (auto e : p->ev_comp) cudaEventDestroy(e);
    if (p->ev_start) cudaEventDestroy(p->ev_start);
    if (p->ev_end) cudaEventDestroy(p->ev_end);
    if (p->s_in) cudaStreamDestroy(p->s_in);
    if (p->s_out) cudaStreamDestroy(p->s_out);
    if (p->mem) cudaFree(p->mem);
    delete p;
}

/* cuStreamWriteValue32 through the runtime's driver entry point (no -lcuda):
 * the stream runner's completion flags (nullptr when unavailable) */
typedef CUresult (*WriteValue32Fn)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
static WriteValue32Fn write_value32() {
    static WriteValue32Fn fn = [] {
        void *f = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuStreamWriteValue32", &f, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess) {
            cudaGetLastError();
            f = nullptr;
        }
        return (WriteValue32Fn)f;
    }();
    return fn;
}

static size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

/* Cut the plan into n chunks of consecutive CB indices with about equal sum K,
 * build each chunk's tasks, allocate staging + outputs, create streams/events. */
static int pipe_build(Plan *P, int n_chunks, HostPipe **out) {
    const crn_cb_desc *d = P->h_desc.data();
    const int n = P->n_cb;
    HostPipe *p = new HostPipe();
    int64_t sumk = 0;
    for (int i = 0; i < n; i++) sumk += d[i].K;
    std::vector<crn_task> tasks;
    std::vector<crn_pair> pairs;
    int64_t acc = 0;
    int cb0 = 0;
    for (int c = 0; c < n_chunks && cb0 < n; c++) {
        int cb1 = cb0;
        const int64_t target = (sumk * (c + 1) + n_chunks - 1) / n_chunks;
        while (cb1 < n && (acc < target || cb1 == cb0)) acc += d[cb1++].K;
        if (c == n_chunks - 1) while (cb1 < n) acc += d[cb1++].K;
        Chunk k;
        k.cb0 = cb0; k.cb1 = cb1;
        k.llr0 = INT64_MAX; k.w0 = INT64_MAX;
        for (int i = cb0; i < cb1; i++) {
            k.llr0 = std::min(k.llr0, d[i].llr_off);
            k.llr1 = std::max(k.llr1, d[i].llr_off + d[i].K + 4);
            k.w0 = std::min(k.w0, d[i].bit_off);
            k.w1 = std::max(k.w1, d[i].bit_off + (d[i].K + 31) / 32);
        }
        std::vector<int> sel(cb1 - cb0);
        for (int i = cb0; i < cb1; i++) sel[i - cb0] = i;
        k.task0 = (int32_t)tasks.size();
        k.units = crn_build_tasks(d, sel.data(), (int)sel.size(), tasks, pairs);
        k.n_tasks = (int32_t)tasks.size() - k.task0;
        p->n_llr = std::max(p->n_llr, k.llr1);
        p->n_words = std::max(p->n_words, k.w1);
        p->ch.push_back(k);
        cb0 = cb1;
    }
    p->n_chunks = (int)p->ch.size();
    p->requested = n_chunks;
    const size_t bt = sizeof(crn_task) * tasks.size(), bp = sizeof(crn_pair) * pairs.size();
    const size_t o_p = align256(bt), o_l = o_p + align256(bp), bl = align256(sizeof(int16_t) * p->n_llr);
    const size_t o_b = o_l + 3 * bl, o_ok = o_b + align256(4 * p->n_words), o_it = o_ok + align256(n);
    const size_t tot = o_it + align256(n);
    if (cudaMalloc(&p->mem, tot) != cudaSuccess) {
        cudaGetLastError();
        delete p;
        return CRN_ENOMEM;
    }
    uint8_t *m = (uint8_t *)p->mem;
    p->d_tasks = (crn_task *)m;
    p->d_pairs = (crn_pair *)(m + o_p);
    for (int s = 0; s < 3; s++) p->d_l[s] = (int16_t *)(m + o_l + s * bl);
    p->d_bits = (uint32_t *)(m + o_b);
    p->d_ok = m + o_ok;
    p->d_it = m + o_it;
    /* output staging starts zeroed: the chunks' downloads copy whole word spans,
     * so host words in gaps between CBs' bit_off ranges come back as 0 (crn.h) */
    cudaMemset(p->d_bits, 0, 4 * (size_t)p->n_words);
    cudaMemcpy(p->d_tasks, tasks.data(), bt, cudaMemcpyHostToDevice);
    cudaMemcpy(p->d_pairs, pairs.data(), bp, cudaMemcpyHostToDevice);
    cudaStreamCreateWithFlags(&p->s_in, cudaStreamNonBlocking);
    cudaStreamCreateWithFlags(&p->s_out, cudaStreamNonBlocking);
    p->ev_in.resize(p->n_chunks);
    p->ev_comp.resize(p->n_chunks);
    for (int c = 0; c < p->n_chunks; c++) {
        cudaEventCreateWithFlags(&p->ev_in[c], cudaEventDisableTiming);
        cudaEventCreateWithFlags(&p->ev_comp[c], cudaEventDisableTiming);
    }
    cudaEventCreateWithFlags(&p->ev_start, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&p->ev_end, cudaEventDisableTiming);
    if (cudaError_t e = cudaGetLastError()) {
        crn_pipe_destroy(p);
        return crn_cuda_fail(e, "host pipeline setup", CRN_ECUDA);
    }
    *out = p;
    return CRN_OK;
}

extern "C" int crn_plan_decode_host(void *plan, const int16_t *h0, const int16_t *h1, const int16_t *h2,
                                    int32_t max_iters, int32_t et, uint32_t *h_bits, uint8_t *h_ok,
                                    uint8_t *h_it, int32_t n_chunks, void *stream) {
    Plan *P = (Plan *)plan;
    if (!P || max_iters < 1 || max_iters > CRN_MAX_ITERS || n_chunks < 0 || n_chunks > 64 || et < 0 || et > CRN_ET_MI)
        return CRN_EINVAL;
    if (P->n_cb == 0) return CRN_OK;
    if (!h0 || !h1 || !h2 || !h_bits || !h_ok) return CRN_EINVAL;
    int dev;
    DevTables *t;
    int rc = crn_get_ctx(&dev, &t);
    if (rc) return rc;
    if (dev != P->dev) return CRN_EINVAL;
    if (n_chunks == 0) /* auto: >= 4 waves of the persistent grid per chunk, at most 16 chunks */
        n_chunks = std::max(1, std::min(16, P->n_tasks / (4 * t->grid)));
    if (!P->pipe || P->pipe->requested != n_chunks) {
        if (P->pipe) crn_pipe_destroy(P->pipe);
        P->pipe = nullptr;
        rc = pipe_build(P, n_chunks, &P->pipe);
        if (rc) return rc;
    }
    HostPipe *p = P->pipe;
    cudaStream_t st = (cudaStream_t)stream;
    cudaEventRecord(p->ev_start, st);
    cudaStreamWaitEvent(p->s_in, p->ev_start, 0);
    cudaStreamWaitEvent(p->s_out, p->ev_start, 0);
    const uint8_t *hs[3] = {(const uint8_t *)h0, (const uint8_t *)h1, (const uint8_t *)h2};
    const size_t esz = P->llr8 < 0 ? sizeof(int16_t) : sizeof(int8_t);    /* crn_plan_set_llr_format */
    for (int c = 0; c < p->n_chunks; c++) {
        const Chunk &k = p->ch[c];
        const size_t nb = esz * (size_t)(k.llr1 - k.llr0);
        for (int s = 0; s < 3; s++)
            cudaMemcpyAsync((uint8_t *)p->d_l[s] + esz * k.llr0, hs[s] + esz * k.llr0, nb, cudaMemcpyHostToDevice,
                            p->s_in);
        cudaEventRecord(p->ev_in[c], p->s_in);
        cudaStreamWaitEvent(st, p->ev_in[c], 0);
        rc = crn_launch_tasks(dev, t, P->d_desc, p->d_tasks + k.task0, k.n_tasks, p->d_pairs, p->d_l[0], p->d_l[1],
                              p->d_l[2], max_iters, et, p->d_bits, p->d_ok, h_it ? p->d_it : nullptr, nullptr,
                              nullptr, 0, st, crn_plan_kernel_variant(P), nullptr, P->grid_cap, false, k.units);
        if (rc) return rc;
        cudaEventRecord(p->ev_comp[c], st);
        cudaStreamWaitEvent(p->s_out, p->ev_comp[c], 0);
        cudaMemcpyAsync(h_bits + k.w0, p->d_bits + k.w0, 4 * (size_t)(k.w1 - k.w0), cudaMemcpyDeviceToHost, p->s_out);
        cudaMemcpyAsync(h_ok + k.cb0, p->d_ok + k.cb0, (size_t)(k.cb1 - k.cb0), cudaMemcpyDeviceToHost, p->s_out);
        if (h_it)
            cudaMemcpyAsync(h_it + k.cb0, p->d_it + k.cb0, (size_t)(k.cb1 - k.cb0), cudaMemcpyDeviceToHost,
                            p->s_out);
    }
    cudaEventRecord(p->ev_end, p->s_out);
    cudaStreamWaitEvent(st, p->ev_end, 0);
    cudaStreamWaitEvent(p->s_in, p->ev_end, 0);    /* the next call's uploads follow this call's downloads */
    if (cudaError_t e = cudaGetLastError()) return crn_cuda_fail(e, "crn_plan_decode_host", CRN_ECUDA);
    return CRN_OK;
}

extern "C" int crn_plan_chunks(void *plan) {
    Plan *P = (Plan *)plan;
    return (P && P->pipe) ? P->pipe->n_chunks : 0;
}

/* ------------------------------------------------------------------ TTI stream runner */
namespace {

struct GroupRes {
    cudaStream_t st = nullptr;
    int *ctr = nullptr;            /* zero copy: one zeroed task counter per TTI (no per-TTI memset) */
    void *dmem = nullptr;          /* device: plan blob + LLRs + outputs */
    size_t dbytes = 0;
    void *hblob[2] = {nullptr, nullptr};  /* pinned host plan blobs, double-buffered by TTI parity */
    size_t hbytes = 0;
    cudaEvent_t ev_blob[2] = {nullptr, nullptr};
    void *ws = nullptr;
};

struct Layout {
    size_t o_desc, o_tasks, o_pairs, o_l, bl, o_bits, o_ok, o_it, tot;
};

/* [task counter (zeroed in the host blob, used as the decode workspace) | desc |
 * tasks | pairs] = the uploaded blob; then the three LLR streams; then bits, crc_ok
 * and iters_used back to back (one download when the host buffers are too). */
Layout layout(int n_cb, int n_tasks, int n_pairs, int64_t n_llr, int64_t n_words, int esz = 2) {
    Layout L;
    L.o_desc = 256;
    L.o_tasks = L.o_desc + align256(sizeof(crn_cb_desc) * n_cb);
    L.o_pairs = L.o_tasks + align256(sizeof(crn_task) * n_tasks);
    L.o_l = L.o_pairs + align256(sizeof(crn_pair) * n_pairs);
    /* int16: 256-byte aligned streams; int8 (CRN_STREAM_LLR8): back to back, so a
     * host block [sys | p1 | p2] goes up in one copy */
    L.bl = esz == 2 ? align256(sizeof(int16_t) * n_llr) : (size_t)n_llr;
    L.o_bits = (L.o_l + 3 * L.bl + 255) & ~(size_t)255;
    L.o_ok = L.o_bits + 4 * n_words;
    L.o_it = L.o_ok + n_cb;
    L.tot = L.o_it + align256(n_cb);
    return L;
}

}  // namespace

extern "C" int crn_stream_run_ex(const crn_tti_group *g, int32_t n_tti, int32_t n_groups, double period_us,
                                 int32_t max_iters, int32_t et, int32_t flags, crn_tti_timing *timing) {
    if (!g || !timing || n_tti < 1 || n_groups < 1 || n_groups > 64 || period_us < 0 || max_iters < 1 ||
        max_iters > CRN_MAX_ITERS || et < 0 || et > CRN_ET_MI ||
        (flags & ~(CRN_STREAM_MERGED | CRN_STREAM_STAGES | CRN_STREAM_ZEROCOPY | CRN_STREAM_LLR8 | (0xF << 8))) ||
        ((flags & CRN_STREAM_MERGED) && (flags & CRN_STREAM_ZEROCOPY)))
        return CRN_EINVAL;
    const bool llr8 = flags & CRN_STREAM_LLR8;
    const int sh8 = (flags >> 8) & 0xF;
    if ((!llr8 && sh8) || (llr8 && (sh8 > 8 || (flags & (CRN_STREAM_MERGED | CRN_STREAM_ZEROCOPY)))))
        return CRN_EINVAL;
    const int esz = llr8 ? 1 : 2;
    const int kvariant = CRN_VARIANT_MAXLOG | (llr8 ? (sh8 + 1) << 8 : 0);   /* the decode kernel's variant word */
    const bool merged = flags & CRN_STREAM_MERGED, stages = merged || (flags & CRN_STREAM_STAGES);
    const bool zc = flags & CRN_STREAM_ZEROCOPY;
    int dev;
    DevTables *t;
    int rc = crn_get_ctx(&dev, &t);
    if (rc) return rc;
    const int64_t NG = (int64_t)n_tti * n_groups;
    /* validate every group up front (host); per group its LLR / word extent */
    std::vector<int64_t> g_llr(NG, 0), g_words(NG, 0);
    std::vector<size_t> need(n_groups, 0), hneed(n_groups, 0);
    size_t m_need = 0, m_hneed = 0;                 /* merged mode: one buffer set for the whole TTI */
    for (int ti = 0; ti < n_tti; ti++) {
        int m_cb = 0;
        int64_t m_llr = 0, m_words = 0;
        for (int gi = 0; gi < n_groups; gi++) {
            const int64_t x = (int64_t)ti * n_groups + gi;
            const crn_tti_group &q = g[x];
            if (q.n_cb < 0 || (q.n_cb > 0 && (!q.desc || !q.llr_sys || !q.llr_p1 || !q.llr_p2 || !q.out_bits ||
                                              !q.crc_ok)))
                return CRN_EINVAL;
            if ((rc = crn_validate(q.desc, q.n_cb, false))) return rc;
            for (int i = 0; i < q.n_cb; i++) {
                g_llr[x] = std::max(g_llr[x], q.desc[i].llr_off + q.desc[i].K + 4);
                g_words[x] = std::max(g_words[x], q.desc[i].bit_off + (q.desc[i].K + 31) / 32);
            }
            if (g_llr[x] > q.n_llr || g_words[x] > q.n_words) return CRN_EINVAL;
            if (zc && q.n_cb > 0) {                     /* the kernel reads / writes these directly */
                const void *ptrs[6] = {q.llr_sys, q.llr_p1, q.llr_p2, q.out_bits, q.crc_ok, q.iters_used};
                for (const void *pp : ptrs) {
                    if (!pp) continue;
                    cudaPointerAttributes at;
                    if (cudaPointerGetAttributes(&at, pp) != cudaSuccess || at.type != cudaMemoryTypeHost) {
                        cudaGetLastError();
                        return CRN_EINVAL;
                    }
                }
            }
            const Layout L = layout(q.n_cb, q.n_cb, q.n_cb, g_llr[x], g_words[x], esz);   /* tasks, pairs <= CBs */
            need[gi] = std::max(need[gi], L.tot);
            hneed[gi] = std::max(hneed[gi], L.o_l);
            m_cb += q.n_cb;
            m_llr += g_llr[x];
            m_words += g_words[x];
        }
        const Layout L = layout(m_cb, m_cb, m_cb, m_llr, m_words);
        m_need = std::max(m_need, L.tot);
        m_hneed = std::max(m_hneed, L.o_l);
    }
    std::vector<GroupRes> G(n_groups + (merged ? 1 : 0));   /* merged: G[n_groups] = the shared decode set */
    auto cleanup = [&]() {
        for (auto &r : G) {
            if (r.st) cudaStreamSynchronize(r.st);
            for (int b = 0; b < 2; b++) {
                if (r.hblob[b]) cudaFreeHost(r.hblob[b]);
                if (r.ev_blob[b]) cudaEventDestroy(r.ev_blob[b]);
            }
            if (r.dmem) cudaFree(r.dmem);
            if (r.ws) cudaFree(r.ws);
            if (r.ctr) cudaFree(r.ctr);
            if (r.st) cudaStreamDestroy(r.st);
        }
    };
    for (int gi = 0; gi < (int)G.size(); gi++) {
        GroupRes &r = G[gi];
        const bool dec = merged && gi == n_groups;
        const size_t dn = merged ? (dec ? m_need : 0) : need[gi], hn = merged ? (dec ? m_hneed : 0) : hneed[gi];
        if (cudaStreamCreateWithFlags(&r.st, cudaStreamNonBlocking) != cudaSuccess ||
            (dn && cudaMalloc(&r.dmem, std::max<size_t>(dn, 256)) != cudaSuccess) ||
            (hn && cudaMallocHost(&r.hblob[0], std::max<size_t>(hn, 256)) != cudaSuccess) ||
            (hn && cudaMallocHost(&r.hblob[1], std::max<size_t>(hn, 256)) != cudaSuccess) ||
            cudaEventCreateWithFlags(&r.ev_blob[0], cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&r.ev_blob[1], cudaEventDisableTiming) != cudaSuccess ||
            ((!merged || dec) && cudaMalloc(&r.ws, crn_decode_ws_bytes(t->grid)) != cudaSuccess) ||
            (zc && (cudaMalloc(&r.ctr, sizeof(int) * 64 * (size_t)n_tti) != cudaSuccess ||
                    cudaMemset(r.ctr, 0, sizeof(int) * 64 * (size_t)n_tti) != cudaSuccess))) {
            cudaGetLastError();
            cleanup();
            return CRN_ENOMEM;
        }
    }
    /* per (TTI, group): timing events (start before the uploads, end after the downloads) */
    std::vector<cudaEvent_t> ev0(NG), ev1(NG), ev_in(merged ? n_groups : 0);
    std::vector<cudaEvent_t> evu(NG), evk0(NG), evk1(NG);   /* stage split: upload done, decode start / end */
    for (int64_t x = 0; x < NG; x++) {
        cudaEventCreate(&ev0[x]);
        cudaEventCreate(&ev1[x]);
        cudaEventCreate(&evu[x]);
        cudaEventCreate(&evk0[x]);
        cudaEventCreate(&evk1[x]);
    }
    for (auto &e : ev_in) cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
    cudaEvent_t ev_dec = nullptr;
    if (merged) cudaEventCreateWithFlags(&ev_dec, cudaEventDisableTiming);
    /* completion flags in pinned host memory, one per (TTI, group), written by the
     * group's stream after its download (cuStreamWriteValue32): the completion
     * thread spins on host memory instead of cudaEventQuery, whose driver lock the
     * group threads' submissions would otherwise wait on.  Without the entry point
     * (or CRN_STREAM_EVQ=1) the thread polls the events as before. */
    static const bool evq_env = [] {
        const char *e = getenv("CRN_STREAM_EVQ");
        return e && e[0] == '1';
    }();
    WriteValue32Fn wv32 = evq_env || NG == 0 ? nullptr : write_value32();
    uint32_t *hflag_mem = nullptr;
    if (wv32 && cudaHostAlloc((void **)&hflag_mem, sizeof(uint32_t) * (size_t)(NG + 1), cudaHostAllocMapped) !=
                    cudaSuccess) {
        cudaGetLastError();
        hflag_mem = nullptr;
    }
    if (hflag_mem) {                                /* probe once: stream memory operations usable? */
        memset(hflag_mem, 0, sizeof(uint32_t) * (size_t)(NG + 1));
        if (wv32((CUstream)G[0].st, (CUdeviceptr)(uintptr_t)(hflag_mem + NG), 1u, 0) != CUDA_SUCCESS ||
            cudaStreamSynchronize(G[0].st) != cudaSuccess || ((volatile uint32_t *)hflag_mem)[NG] != 1u) {
            cudaGetLastError();
            cudaFreeHost(hflag_mem);
            hflag_mem = nullptr;
        }
    }
    volatile uint32_t *const hflag = hflag_mem;
    auto signal_done = [&](int64_t x, cudaStream_t st) {      /* after the download, before ev1[x] */
        if (hflag) wv32((CUstream)st, (CUdeviceptr)(uintptr_t)(hflag + x), 1u, 0);
    };
    std::vector<double> done_us(NG, 0.0), rel_us(n_tti, 0.0), sub_us(n_tti, 0.0), gsub_us(NG, 0.0);
    std::vector<std::atomic<int>> submitted(n_groups);       /* per group: TTIs enqueued so far */
    for (auto &a : submitted) a.store(0);
    std::atomic<bool> abort_flag{false};
    const Clock::time_point t0 = Clock::now() + std::chrono::milliseconds(2);
    for (int ti = 0; ti < n_tti; ti++) rel_us[ti] = period_us * ti;

    /* completion thread (the "captor"): time-stamps each (TTI, group) when its end event fires */
    std::thread watcher;
    try {
    watcher = std::thread([&]() {
        for (int64_t x = 0; x < NG; x++) {
            const int ti = (int)(x / n_groups), gi = (int)(x % n_groups);
            while (submitted[gi].load(std::memory_order_acquire) <= ti) {
                if (abort_flag.load()) return;
                std::this_thread::yield();
            }
            if (hflag) {
                /* spin on host memory; an event query only every 64 k spins (a failed
                 * stream never writes its flag) */
                for (uint32_t n = 1; hflag[x] == 0u; n++) {
                    if ((n & 0xFFFFu) == 0u) {
                        cudaError_t q = cudaEventQuery(ev1[x]);
                        if (q == cudaSuccess && hflag[x] == 0u) break;
                        if ((q != cudaSuccess && q != cudaErrorNotReady) || abort_flag.load()) return;
                    }
                }
            } else {
                for (;;) {
                    cudaError_t q = cudaEventQuery(ev1[x]);
                    if (q == cudaSuccess) break;
                    if (q != cudaErrorNotReady || abort_flag.load()) return;
                }
            }
            done_us[x] = us_since(t0, Clock::now());
        }
    });
    } catch (const std::exception &) {           /* no thread: give everything back */
        for (int64_t x = 0; x < NG; x++) {
            cudaEventDestroy(ev0[x]);
            cudaEventDestroy(ev1[x]);
            cudaEventDestroy(evu[x]);
            cudaEventDestroy(evk0[x]);
            cudaEventDestroy(evk1[x]);
        }
        for (auto &ev : ev_in) cudaEventDestroy(ev);
        if (ev_dec) cudaEventDestroy(ev_dec);
        cleanup();
        if (hflag_mem) cudaFreeHost(hflag_mem);
        return CRN_ENOMEM;
    }

    auto release = [&](int ti) {                /* pacer: TTI ti is released at t0 + ti * period */
        const Clock::time_point rel = t0 + std::chrono::duration_cast<Clock::duration>(
                                               std::chrono::duration<double, std::micro>(period_us * ti));
        while (Clock::now() < rel) {
        }
    };
    /* one cell group's share of one TTI on its own stream: row a1 on the host
     * (bucket / pair / task its CBs), then upload -> decode -> download */
    auto submit_group = [&](int ti, int gi) -> int {
        const int64_t x = (int64_t)ti * n_groups + gi;
        const crn_tti_group &q = g[x];
        GroupRes &r = G[gi];
        int src = CRN_OK;
        cudaEventRecord(ev0[x], r.st);
        if (q.n_cb > 0) {
            const int64_t n_llr = g_llr[x], n_words = g_words[x];
            /* Offsets from the upper bound tasks, pairs <= CBs (the buffers are sized
             * for it): known before the tasks are built, so the LLR upload -- most of
             * the bytes -- is enqueued first and the host-side task building and blob
             * assembly below overlap its DMA. */
            const Layout L = layout(q.n_cb, q.n_cb, q.n_cb, n_llr, n_words, esz);
            uint8_t *dm = (uint8_t *)r.dmem;
            int16_t *dl[3];
            for (int s = 0; s < 3; s++) dl[s] = (int16_t *)(dm + L.o_l + s * L.bl);
            if (!zc) {
                const uint8_t *hs[3] = {(const uint8_t *)q.llr_sys, (const uint8_t *)q.llr_p1,
                                        (const uint8_t *)q.llr_p2};
                const size_t sb = (size_t)esz * (size_t)n_llr;             /* bytes per stream */
                if (hs[1] == hs[0] + sb && hs[2] == hs[1] + sb && L.bl == sb)
                    cudaMemcpyAsync(dl[0], hs[0], 3 * sb, cudaMemcpyHostToDevice, r.st);
                else                                            /* the three streams: one copy if contiguous */
                    for (int s = 0; s < 3; s++) cudaMemcpyAsync(dl[s], hs[s], sb, cudaMemcpyHostToDevice, r.st);
            }
            std::vector<crn_task> tasks;
            std::vector<crn_pair> pairs;
            std::vector<int> sel(q.n_cb);
            for (int i = 0; i < q.n_cb; i++) sel[i] = i;
            /* the groups' kernels run concurrently: each spreads over its share of the SMs */
            const int units = crn_build_tasks(q.desc, sel.data(), q.n_cb, tasks, pairs,
                                              std::max(1, t->grid / n_groups));
            const int b = ti & 1;
            if (ti >= 2) {                              /* blob slot b was last uploaded by TTI ti-2 */
                const cudaEvent_t prev = ev1[x - 2 * (int64_t)n_groups];
                while (cudaEventQuery(prev) == cudaErrorNotReady) {
                }
            }
            uint8_t *hb = (uint8_t *)r.hblob[b];
            memset(hb, 0, L.o_desc);                    /* the decode's task counter */
            memcpy(hb + L.o_desc, q.desc, sizeof(crn_cb_desc) * q.n_cb);
            memcpy(hb + L.o_tasks, tasks.data(), sizeof(crn_task) * tasks.size());
            memcpy(hb + L.o_pairs, pairs.data(), sizeof(crn_pair) * pairs.size());
            if (zc) {
                /* zero copy: the kernel reads the pinned blob and LLRs and writes the
                 * results over PCIe itself -- one launch per group and TTI, no copy stage */
                if (stages) {
                    cudaEventRecord(evu[x], r.st);
                    cudaEventRecord(evk0[x], r.st);
                }
                src = crn_launch_tasks(dev, t, (const crn_cb_desc *)(hb + L.o_desc), (const crn_task *)(hb + L.o_tasks),
                                       (int)tasks.size(), (const crn_pair *)(hb + L.o_pairs), q.llr_sys, q.llr_p1,
                                       q.llr_p2, max_iters, et, q.out_bits, q.crc_ok, q.iters_used, nullptr,
                                       r.ctr + 64 * (size_t)ti, crn_decode_ws_bytes(t->grid), r.st, CRN_VARIANT_MAXLOG,
                                       nullptr, 0, true, units);
                if (stages) cudaEventRecord(evk1[x], r.st);
                signal_done(x, r.st);
                cudaEventRecord(ev1[x], r.st);
                gsub_us[x] = us_since(t0, Clock::now());
                submitted[gi].store(ti + 1, std::memory_order_release);
                return src;
            }
            /* the blob: counter | descriptors | tasks | pairs, up to the last pair */
            cudaMemcpyAsync(dm, hb, L.o_pairs + sizeof(crn_pair) * pairs.size(), cudaMemcpyHostToDevice, r.st);
            uint32_t *dbits = (uint32_t *)(dm + L.o_bits);
            uint8_t *dok = dm + L.o_ok, *dit = dm + L.o_it;
            if (stages) {
                cudaEventRecord(evu[x], r.st);
                cudaEventRecord(evk0[x], r.st);
            }
            src = crn_launch_tasks(dev, t, (const crn_cb_desc *)(dm + L.o_desc), (const crn_task *)(dm + L.o_tasks),
                                   (int)tasks.size(), (const crn_pair *)(dm + L.o_pairs), dl[0], dl[1], dl[2],
                                   max_iters, et, dbits, dok, q.iters_used ? dit : nullptr, nullptr, dm,
                                   crn_decode_ws_bytes(t->grid), r.st, kvariant, nullptr, 0, true, units);
            if (stages) cudaEventRecord(evk1[x], r.st);
            const bool packed = (const uint8_t *)q.crc_ok == (const uint8_t *)(q.out_bits + n_words) &&
                                (!q.iters_used || q.iters_used == q.crc_ok + q.n_cb);
            if (packed)                                     /* bits | crc_ok | iters_used in one download */
                cudaMemcpyAsync(q.out_bits, dbits, 4 * (size_t)n_words + (size_t)q.n_cb * (q.iters_used ? 2 : 1),
                                cudaMemcpyDeviceToHost, r.st);
            else {
                cudaMemcpyAsync(q.out_bits, dbits, 4 * (size_t)n_words, cudaMemcpyDeviceToHost, r.st);
                cudaMemcpyAsync(q.crc_ok, dok, (size_t)q.n_cb, cudaMemcpyDeviceToHost, r.st);
                if (q.iters_used)
                    cudaMemcpyAsync(q.iters_used, dit, (size_t)q.n_cb, cudaMemcpyDeviceToHost, r.st);
            }
        } else if (stages) {
            cudaEventRecord(evu[x], r.st);
            cudaEventRecord(evk0[x], r.st);
            cudaEventRecord(evk1[x], r.st);
        }
        signal_done(x, r.st);
                cudaEventRecord(ev1[x], r.st);
        gsub_us[x] = us_since(t0, Clock::now());
        submitted[gi].store(ti + 1, std::memory_order_release);
        return src;
    };
    if (!merged) {
        /* one host thread per cell group (the paper's dedicated channel-coding
         * threads): each waits for the release of
         * TTI ti itself and enqueues its group, so the groups submit in parallel */
        std::vector<std::thread> workers;
        std::vector<int> grc(n_groups, CRN_OK);
        try {
            for (int gi = 0; gi < n_groups; gi++)
                workers.emplace_back([&, gi]() {
                    cudaSetDevice(dev);
                    for (int ti = 0; ti < n_tti && !abort_flag.load(); ti++) {
                        release(ti);
                        if ((grc[gi] = submit_group(ti, gi)) != CRN_OK) abort_flag.store(true);
                    }
                });
        } catch (const std::exception &) {       /* could not start every group thread */
            abort_flag.store(true);
            rc = CRN_ENOMEM;
        }
        for (auto &w : workers) w.join();
        for (int gi = 0; gi < n_groups; gi++)
            if (grc[gi] != CRN_OK && rc == CRN_OK) rc = grc[gi];
        for (int ti = 0; ti < n_tti; ti++)
            for (int gi = 0; gi < n_groups; gi++)
                sub_us[ti] = std::max(sub_us[ti], gsub_us[(int64_t)ti * n_groups + gi]);
    }
    std::vector<crn_cb_desc> mdesc;
    std::vector<int64_t> lbase(n_groups), wbase(n_groups);
    std::vector<int> cbase(n_groups);
    for (int ti = 0; merged && ti < n_tti && rc == CRN_OK; ti++) {
        release(ti);
        const int64_t x0 = (int64_t)ti * n_groups;
        {
            /* merged: every group uploads its slice of one TTI-wide buffer set on its own
             * stream; one decode launch over all groups' tasks waits for every upload;
             * each group downloads its slice on its own stream after the decode */
            GroupRes &dr = G[n_groups];
            int m_cb = 0;
            int64_t m_llr = 0, m_words = 0;
            for (int gi = 0; gi < n_groups; gi++) {
                cbase[gi] = m_cb;
                lbase[gi] = m_llr;
                wbase[gi] = m_words;
                m_cb += g[x0 + gi].n_cb;
                m_llr += g_llr[x0 + gi];
                m_words += g_words[x0 + gi];
            }
            mdesc.resize(m_cb);
            for (int gi = 0; gi < n_groups; gi++) {
                const crn_tti_group &q = g[x0 + gi];
                for (int i = 0; i < q.n_cb; i++) {
                    crn_cb_desc d = q.desc[i];
                    d.llr_off += lbase[gi];
                    d.bit_off += wbase[gi];
                    mdesc[cbase[gi] + i] = d;
                }
            }
            std::vector<crn_task> tasks;
            std::vector<crn_pair> pairs;
            std::vector<int> sel(m_cb);
            for (int i = 0; i < m_cb; i++) sel[i] = i;
            const int units = crn_build_tasks(mdesc.data(), sel.data(), m_cb, tasks, pairs, t->grid);
            const Layout L = layout(m_cb, (int)tasks.size(), (int)pairs.size(), m_llr, m_words);
            uint8_t *dm = (uint8_t *)dr.dmem;
            int16_t *dl[3];
            for (int s = 0; s < 3; s++) dl[s] = (int16_t *)(dm + L.o_l + s * L.bl);
            uint32_t *dbits = (uint32_t *)(dm + L.o_bits);
            uint8_t *dok = dm + L.o_ok, *dit = dm + L.o_it;
            for (int gi = 0; gi < n_groups; gi++) {
                const int64_t x = x0 + gi;
                const crn_tti_group &q = g[x];
                GroupRes &r = G[gi];
                cudaEventRecord(ev0[x], r.st);
                const int16_t *hs[3] = {q.llr_sys, q.llr_p1, q.llr_p2};
                for (int s = 0; s < 3; s++)
                    if (g_llr[x])
                        cudaMemcpyAsync(dl[s] + lbase[gi], hs[s], sizeof(int16_t) * g_llr[x], cudaMemcpyHostToDevice,
                                        r.st);
                cudaEventRecord(ev_in[gi], r.st);
                cudaEventRecord(evu[x], r.st);
                cudaStreamWaitEvent(dr.st, ev_in[gi], 0);
            }
            const int b = ti & 1;
            cudaEventSynchronize(dr.ev_blob[b]);
            uint8_t *hb = (uint8_t *)dr.hblob[b];
            memcpy(hb + L.o_desc, mdesc.data(), sizeof(crn_cb_desc) * m_cb);
            memcpy(hb + L.o_tasks, tasks.data(), sizeof(crn_task) * tasks.size());
            memcpy(hb + L.o_pairs, pairs.data(), sizeof(crn_pair) * pairs.size());
            cudaMemcpyAsync(dm, hb, L.o_l, cudaMemcpyHostToDevice, dr.st);
            cudaEventRecord(dr.ev_blob[b], dr.st);
            cudaEventRecord(evk0[x0], dr.st);
            if (m_cb > 0)
                rc = crn_launch_tasks(dev, t, (const crn_cb_desc *)(dm + L.o_desc), (const crn_task *)(dm + L.o_tasks),
                                      (int)tasks.size(), (const crn_pair *)(dm + L.o_pairs), dl[0], dl[1], dl[2],
                                      max_iters, et, dbits, dok, dit, nullptr, dr.ws, crn_decode_ws_bytes(t->grid),
                                      dr.st, CRN_VARIANT_MAXLOG, nullptr, 0, false, units);
            cudaEventRecord(ev_dec, dr.st);
            cudaEventRecord(evk1[x0], dr.st);
            for (int gi = 1; gi < n_groups; gi++) {          /* one decode for all groups */
                cudaEventRecord(evk0[x0 + gi], dr.st);
                cudaEventRecord(evk1[x0 + gi], dr.st);
            }
            for (int gi = 0; gi < n_groups; gi++) {
                const int64_t x = x0 + gi;
                const crn_tti_group &q = g[x];
                GroupRes &r = G[gi];
                cudaStreamWaitEvent(r.st, ev_dec, 0);
                if (q.n_cb > 0) {
                    cudaMemcpyAsync(q.out_bits, dbits + wbase[gi], 4 * (size_t)g_words[x], cudaMemcpyDeviceToHost,
                                    r.st);
                    cudaMemcpyAsync(q.crc_ok, dok + cbase[gi], (size_t)q.n_cb, cudaMemcpyDeviceToHost, r.st);
                    if (q.iters_used)
                        cudaMemcpyAsync(q.iters_used, dit + cbase[gi], (size_t)q.n_cb, cudaMemcpyDeviceToHost, r.st);
                }
                signal_done(x, r.st);
                cudaEventRecord(ev1[x], r.st);
            }
            for (int gi = 0; gi < n_groups; gi++) submitted[gi].store(ti + 1, std::memory_order_release);
        }
        sub_us[ti] = us_since(t0, Clock::now());
    }
    if (rc != CRN_OK) abort_flag.store(true);
    watcher.join();
    cudaError_t e = cudaSuccess;
    for (auto &r : G)
        if (cudaStreamSynchronize(r.st) != cudaSuccess) e = cudaGetLastError();
    if (rc == CRN_OK && e != cudaSuccess) rc = crn_cuda_fail(e, "crn_stream_run", CRN_ECUDA);
    if (rc == CRN_OK) {
        for (int ti = 0; ti < n_tti; ti++) {
            crn_tti_timing &o = timing[ti];
            o.release_us = rel_us[ti];                  /* the pacer's release instant (t0 + ti * period) */
            o.submitted_us = sub_us[ti];
            o.complete_us = 0;
            float smin = 0, emax = 0;
            for (int gi = 0; gi < n_groups; gi++) {
                const int64_t x = (int64_t)ti * n_groups + gi;
                o.complete_us = std::max(o.complete_us, done_us[x]);
                float s = 0, en = 0;
                cudaEventElapsedTime(&s, ev0[(int64_t)ti * n_groups], ev0[x]);
                cudaEventElapsedTime(&en, ev0[(int64_t)ti * n_groups], ev1[x]);
                smin = std::min(smin, s);
                emax = std::max(emax, en);
            }
            o.latency_us = o.complete_us - o.release_us;
            o.device_us = 1e3 * (double)(emax - smin);
            float up = 0, k0 = 1e30f, k1 = 0;
            for (int gi = 0; stages && gi < n_groups; gi++) {
                const int64_t x = (int64_t)ti * n_groups + gi;
                float a = 0, b0 = 0, b1 = 0;
                cudaEventElapsedTime(&a, ev0[(int64_t)ti * n_groups], evu[x]);
                cudaEventElapsedTime(&b0, ev0[(int64_t)ti * n_groups], evk0[x]);
                cudaEventElapsedTime(&b1, ev0[(int64_t)ti * n_groups], evk1[x]);
                up = std::max(up, a);
                k0 = std::min(k0, b0);
                k1 = std::max(k1, b1);
            }
            o.upload_us = stages ? 1e3 * (double)(up - smin) : -1.0;
            o.decode_start_us = stages ? 1e3 * (double)(k0 - smin) : -1.0;
            o.decode_end_us = stages ? 1e3 * (double)(k1 - smin) : -1.0;
        }
    }
    for (int64_t x = 0; x < NG; x++) {
        cudaEventDestroy(ev0[x]);
        cudaEventDestroy(ev1[x]);
        cudaEventDestroy(evu[x]);
        cudaEventDestroy(evk0[x]);
        cudaEventDestroy(evk1[x]);
    }
    for (auto &ev : ev_in) cudaEventDestroy(ev);
    if (ev_dec) cudaEventDestroy(ev_dec);
    cleanup();
    if (hflag_mem) cudaFreeHost(hflag_mem);
    return rc;
}

extern "C" int crn_stream_run(const crn_tti_group *g, int32_t n_tti, int32_t n_groups, double period_us,
                              int32_t max_iters, int32_t et, crn_tti_timing *timing) {
    return crn_stream_run_ex(g, n_tti, n_groups, period_us, max_iters, et, 0, timing);
}
