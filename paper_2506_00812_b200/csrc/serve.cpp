// f1 -- persistent-kernel serving (E13 P:L733-L738): a kernel stays resident
// on the GPU; the host publishes queries into a job ring in pinned, device-mapped memory and reads
// the answers back from it. No kernel launch, no stream synchronisation and no host API call per
// query: submit = a few stores into the ring + a release store of the head counter; wait = a spin on
// the slot's done word. The device side is k_serve (small.cu), the same per-query body as k_small.
#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <cstring>
#include <immintrin.h>
#include <mutex>

#include "host_internal.h"
#include "small.h"

struct vf_server {
    vf_index *ix = nullptr;
    int device = 0;
    vf::SearchArgs a{};
    bool two_views = false;
    int64_t cap = 0;
    int raw_bytes = 0, raw_stride = 0, k = 0, n_ctas = 0;
    // host-mapped ring (one pinned allocation) and its device view
    uint8_t *host = nullptr;
    uint8_t *hq = nullptr;
    int32_t *hlab = nullptr, *hnlab = nullptr, *hids = nullptr, *hstop = nullptr;
    float *hd = nullptr;
    long long *hdone = nullptr, *hhead = nullptr;
    vf::ServeRing ring{};
    vf::DevBuf next, gtab, ctr, partials, part_done, dring;
    int nparts = 1;
    cudaStream_t stream = nullptr;
    std::atomic<int64_t> submitted{0};   // written under mu, read by vf_serve_wait / info without it
    std::mutex mu;
    bool running = false;
};

namespace vf {
// visited-set geometry of one beam search (the same sizing as plan_search)
void beam_sizes(int itopk, int w, int R, int n_init, int max_iter, int *hash_slots, uint64_t *gslots,
                int warp_bytes);
}

using namespace vf;

static void free_server(vf_server *sv) {
    if (sv->stream) cudaStreamDestroy(sv->stream);
    if (sv->host) cudaFreeHost(sv->host);
    delete sv;
}

extern "C" vf_status vf_serve_start(vf_index *ix, const vf_search_params *p, int32_t capacity, int32_t n_workers,
                                    vf_server **out) {
    if (!ix || !p || !out) return fail(VF_ERR_INVALID_ARG, "NULL argument");
    *out = nullptr;
    if (ix->world > 1) return fail(VF_ERR_INVALID_ARG, "serving runs on a single-GPU index");
    if (capacity < 1 || capacity > (1 << 20)) return fail(VF_ERR_INVALID_ARG, "capacity must be in [1, 2^20]");
    if (p->k < 1 || p->k > kSmallMaxK) return fail(VF_ERR_INVALID_ARG, "serving supports 1 <= k <= 32");
    if (p->itopk < p->k || p->itopk > kMaxItopk) return fail(VF_ERR_INVALID_ARG, "itopk must be in [k, 1024]");
    const int w = p->search_width < 1 ? 1 : p->search_width;
    if (w * ix->dev.R > 64) return fail(VF_ERR_INVALID_ARG, "search_width * R must be <= 64");
    if (p->op < 0 || p->op > 2 || p->recall_mode < 0 || p->recall_mode > 1)
        return fail(VF_ERR_INVALID_ARG, "bad op / recall_mode");
    const DevIndex &F = ix->enc8 ? ix->dev8 : ix->dev;
    if (!small_supported(F, ix->dev, ix->enc8, p->k)) return fail(VF_ERR_INVALID_ARG, "row size not served");
    VF_CUDA(cudaSetDevice(ix->device));

    vf_server *sv = new vf_server();
    sv->ix = ix;
    sv->device = ix->device;
    sv->cap = capacity;
    sv->k = p->k;
    sv->raw_bytes = ix->dev.dim * (ix->dev.dtype == VF_U8 ? 1 : 4);
    sv->raw_stride = (sv->raw_bytes + 15) & ~15;
    sv->two_views = ix->enc8;
    SearchArgs &a = sv->a;
    a.ix = F;
    a.k = p->k;
    a.itopk = p->itopk;
    a.w = w;
    a.n_init = p->n_init > 0 ? p->n_init : ix->dev.R * w;
    a.max_iter = p->max_iterations > 0 ? p->max_iterations : 2 * ((p->itopk + w - 1) / w) + 16;
    a.seed = p->seed;
    a.knobs = vf::kDefaultKnobs;
    a.op = p->op;
    a.recall_mode = p->recall_mode;
    a.exact = p->exact ? 1 : 0;
    a.and_scan_thr = p->and_scan_threshold;
    a.scan_thr = std::max(ix->dev.T, p->scan_threshold);
    uint64_t gslots = 0;
    beam_sizes(p->itopk, w, ix->dev.R, a.n_init, a.max_iter, &a.hash_slots, &gslots, 7168);
    a.gtab_slots = (int64_t)gslots;
    a.chk_lo = ix->chk_lo;
    a.chk_hi = ix->chk_hi;
    a.q8_row_bytes = ix->enc8 ? ix->dev8.row_bytes : 0;
    auto bail = [&](vf_status st) { free_server(sv); return st; };

    int n = serve_max_ctas(a, ix->dev, sv->two_views) - 1;         // one slot for the dispatcher CTA
    if (n <= 0)
        return bail(fail(VF_ERR_INTERNAL, "serving kernel does not fit (" +
                                              std::string(n < 0 ? cudaGetErrorString((cudaError_t)-n) : "0 CTAs/SM") + ")"));
    if (n_workers > 0) n = std::min(n, (int)n_workers);
    sv->n_ctas = n;
    const size_t warps = (size_t)n * kSmallWarps;
    cudaError_t e;
    if ((e = sv->gtab.ensure(warps * gslots * 8 + warps * 4)) != cudaSuccess ||
        (e = cudaMemset(sv->gtab.p, 0, warps * gslots * 8 + warps * 4)) != cudaSuccess ||
        (e = sv->ctr.ensure(sizeof(Counters))) != cudaSuccess ||
        (e = cudaMemset(sv->ctr.p, 0, sizeof(Counters))) != cudaSuccess ||
        (e = sv->next.ensure(128)) != cudaSuccess || (e = cudaMemset(sv->next.p, 0, 128)) != cudaSuccess)
        return bail(fail(VF_ERR_OUT_OF_MEMORY, std::string("serve buffers: ") + cudaGetErrorString(e)));
    // a job is answered by nparts CTAs together (VF_SERVE_PARTS, default 2): scan items split by
    // rows, graph items spread over the CTAs' warps, the last CTA merges and publishes
    {
        const char *e = getenv("VF_SERVE_PARTS");
        sv->nparts = std::max(1, std::min(8, e ? atoi(e) : 2));   // see DESIGN.md §6 (k_serve)
    }
    const size_t pbytes = (size_t)capacity * sv->nparts * kServeLabels * kSmallMaxK * 8;
    if ((e = sv->partials.ensure(pbytes)) != cudaSuccess || (e = sv->part_done.ensure((size_t)capacity * 4)) != cudaSuccess ||
        (e = cudaMemset(sv->part_done.p, 0, (size_t)capacity * 4)) != cudaSuccess)
        return bail(fail(VF_ERR_OUT_OF_MEMORY, std::string("serve partials: ") + cudaGetErrorString(e)));
    a.gtab = sv->gtab.as<unsigned long long>();
    a.n_warp_slots = (int32_t)warps;
    a.ctr = sv->ctr.as<Counters>();

    // the ring: one pinned, device-mapped allocation
    const size_t C = (size_t)capacity;
    size_t o = 0;
    const size_t o_q = o; o += C * sv->raw_stride;
    const size_t o_lab = o; o += C * kServeLabels * 4;
    const size_t o_nlab = o; o += C * 4;
    o = (o + 15) & ~(size_t)15;
    const size_t o_ids = o; o += C * p->k * 4;
    const size_t o_d = o; o += C * p->k * 4;
    o = (o + 63) & ~(size_t)63;
    const size_t o_done = o; o += C * 8;
    o = (o + 63) & ~(size_t)63;
    const size_t o_head = o; o += 64;
    const size_t o_stop = o; o += 64;
    if ((e = cudaHostAlloc((void **)&sv->host, o, cudaHostAllocMapped | cudaHostAllocPortable)) != cudaSuccess)
        return bail(fail(VF_ERR_OUT_OF_MEMORY, std::string("cudaHostAlloc: ") + cudaGetErrorString(e)));
    std::memset(sv->host, 0, o);
    uint8_t *dev = nullptr;
    if ((e = cudaHostGetDevicePointer((void **)&dev, sv->host, 0)) != cudaSuccess)
        return bail(fail(VF_ERR_CUDA, std::string("cudaHostGetDevicePointer: ") + cudaGetErrorString(e)));
    sv->hq = sv->host + o_q;
    sv->hlab = reinterpret_cast<int32_t *>(sv->host + o_lab);
    sv->hnlab = reinterpret_cast<int32_t *>(sv->host + o_nlab);
    sv->hids = reinterpret_cast<int32_t *>(sv->host + o_ids);
    sv->hd = reinterpret_cast<float *>(sv->host + o_d);
    sv->hdone = reinterpret_cast<long long *>(sv->host + o_done);
    sv->hhead = reinterpret_cast<long long *>(sv->host + o_head);
    sv->hstop = reinterpret_cast<int32_t *>(sv->host + o_stop);
    ServeRing &r = sv->ring;
    r.cap = capacity;
    r.raw_stride = sv->raw_stride;
    r.queries = dev + o_q;
    r.labels = reinterpret_cast<const int32_t *>(dev + o_lab);
    r.nlab = reinterpret_cast<const int32_t *>(dev + o_nlab);
    r.out_ids = reinterpret_cast<int32_t *>(dev + o_ids);
    r.out_dists = reinterpret_cast<float *>(dev + o_d);
    r.done = reinterpret_cast<long long *>(dev + o_done);
    r.head = reinterpret_cast<const long long *>(dev + o_head);
    r.stop = reinterpret_cast<const int32_t *>(dev + o_stop);
    r.next = sv->next.as<unsigned long long>();
    {
        const size_t dq = (size_t)capacity * sv->raw_stride, dl = (size_t)capacity * kServeLabels * 4;
        if ((e = sv->dring.ensure(dq + dl + (size_t)capacity * 4)) != cudaSuccess)
            return bail(fail(VF_ERR_OUT_OF_MEMORY, std::string("serve ring: ") + cudaGetErrorString(e)));
        r.dq = sv->dring.as<uint8_t>();
        r.dlab = reinterpret_cast<int32_t *>(sv->dring.as<uint8_t>() + dq);
        r.dnlab = reinterpret_cast<int32_t *>(sv->dring.as<uint8_t>() + dq + dl);
    }
    r.nparts = sv->nparts;
    r.stats = reinterpret_cast<unsigned long long *>(sv->next.as<uint8_t>() + 64);
    r.partials = sv->partials.as<unsigned long long>();
    r.part_done = sv->part_done.as<int32_t>();
    r.dev_head = reinterpret_cast<long long *>(sv->next.as<uint8_t>() + 16);
    r.dev_stop = reinterpret_cast<int32_t *>(sv->next.as<uint8_t>() + 32);
    // VF_SERVE_IDLE_MS > 0: the resident kernel exits after that long without a new job (then
    // vf_serve_wait reports VF_ERR_CUDA "serving kernel ended"); default: it runs until stopped
    {
        const char *e = getenv("VF_SERVE_IDLE_MS");
        const long long ms = e ? atoll(e) : 0;
        r.idle_ns = ms > 0 ? (unsigned long long)ms * 1000000ull : 0ull;
    }

    if ((e = cudaStreamCreateWithFlags(&sv->stream, cudaStreamNonBlocking)) != cudaSuccess)
        return bail(fail(VF_ERR_CUDA, std::string("stream: ") + cudaGetErrorString(e)));
    if (launch_serve(a, ix->dev, sv->two_views, sv->raw_bytes, n, r, sv->stream) < 0)
        return bail(fail(VF_ERR_INTERNAL, "serving kernel dispatch failed"));
    if ((e = cudaGetLastError()) != cudaSuccess)
        return bail(fail(VF_ERR_CUDA, std::string("serving kernel launch: ") + cudaGetErrorString(e)));
    sv->running = true;
    *out = sv;
    return VF_OK;
}

extern "C" vf_status vf_serve_submit(vf_server *sv, const void *query, const int32_t *labels, int32_t n_labels,
                                     int64_t *ticket) {
    if (!sv || !query || !ticket || (n_labels > 0 && !labels)) return fail(VF_ERR_INVALID_ARG, "NULL argument");
    if (n_labels < 0 || n_labels > kServeLabels) return fail(VF_ERR_INVALID_ARG, "n_labels must be in [0, 16]");
    if (!sv->running) return fail(VF_ERR_INVALID_ARG, "server stopped");
    std::lock_guard<std::mutex> g(sv->mu);
    const int64_t j = sv->submitted.load(std::memory_order_relaxed);
    const int64_t slot = j % sv->cap;
    // the slot's previous job (j - cap) must have been answered before it is overwritten
    if (j >= sv->cap) {
        volatile long long *dn = sv->hdone + slot;
        while (*dn < j - sv->cap + 1) _mm_pause();
    }
    std::memcpy(sv->hq + slot * sv->raw_stride, query, (size_t)sv->raw_bytes);
    if (n_labels > 0) std::memcpy(sv->hlab + slot * kServeLabels, labels, (size_t)n_labels * 4);
    sv->hnlab[slot] = n_labels;
    std::atomic_thread_fence(std::memory_order_release);
    *(volatile long long *)sv->hhead = j + 1;                    // publish job j
    sv->submitted.store(j + 1, std::memory_order_release);
    *ticket = j;
    return VF_OK;
}

extern "C" vf_status vf_serve_wait(vf_server *sv, int64_t ticket, int32_t *out_ids, float *out_dists) {
    if (!sv || !out_ids || !out_dists) return fail(VF_ERR_INVALID_ARG, "NULL argument");
    if (ticket < 0 || ticket >= sv->submitted.load(std::memory_order_acquire))
        return fail(VF_ERR_INVALID_ARG, "unknown ticket");
    const int64_t slot = ticket % sv->cap;
    volatile long long *dn = sv->hdone + slot;
    long long v;
    int spins = 0;
    while ((v = *dn) < ticket + 1) {
        _mm_pause();
        if (++spins == (1 << 22)) {            // ~1 s without progress: check the kernel is alive
            spins = 0;
            const cudaError_t e = cudaStreamQuery(sv->stream);
            if (e != cudaErrorNotReady) return fail(VF_ERR_CUDA, std::string("serving kernel ended: ") +
                                                                     cudaGetErrorString(e));
        }
    }
    if (v != ticket + 1) return fail(VF_ERR_INVALID_ARG, "ticket's results were overwritten (capacity exceeded)");
    std::atomic_thread_fence(std::memory_order_acquire);
    std::memcpy(out_ids, sv->hids + slot * sv->k, (size_t)sv->k * 4);
    std::memcpy(out_dists, sv->hd + slot * sv->k, (size_t)sv->k * 4);
    if (*dn != ticket + 1) return fail(VF_ERR_INVALID_ARG, "ticket's results were overwritten (capacity exceeded)");
    return VF_OK;
}

extern "C" vf_status vf_serve_run(vf_server *sv, int64_t n, const void *queries, const int64_t *qlabel_offsets,
                                  const int32_t *qlabels, int32_t max_in_flight, int32_t *out_ids, float *out_dists) {
    if (!sv || n < 0 || (n > 0 && (!queries || !qlabel_offsets || !out_ids || !out_dists)))
        return fail(VF_ERR_INVALID_ARG, "NULL argument");
    if (max_in_flight < 1 || max_in_flight > sv->cap) return fail(VF_ERR_INVALID_ARG, "max_in_flight must be in [1, capacity]");
    const uint8_t *q = static_cast<const uint8_t *>(queries);
    int64_t first = -1, waited = 0;
    for (int64_t i = 0; i < n; i++) {
        if (i - waited == max_in_flight) {
            vf_status st = vf_serve_wait(sv, first + waited, out_ids + waited * sv->k, out_dists + waited * sv->k);
            if (st != VF_OK) return st;
            waited++;
        }
        int64_t t = 0;
        const int64_t lo = qlabel_offsets[i];
        vf_status st = vf_serve_submit(sv, q + i * sv->raw_bytes, qlabels + lo, (int32_t)(qlabel_offsets[i + 1] - lo), &t);
        if (st != VF_OK) return st;
        if (first < 0) first = t;
        else if (t != first + i) return fail(VF_ERR_INVALID_ARG, "vf_serve_run needs the server to itself");
    }
    for (; waited < n; waited++) {
        vf_status st = vf_serve_wait(sv, first + waited, out_ids + waited * sv->k, out_dists + waited * sv->k);
        if (st != VF_OK) return st;
    }
    return VF_OK;
}

extern "C" vf_status vf_serve_stop(vf_server *sv) {
    if (!sv) return VF_OK;
    cudaSetDevice(sv->device);
    vf_status st = VF_OK;
    if (sv->running) {
        *(volatile int32_t *)sv->hstop = 1;
        std::atomic_thread_fence(std::memory_order_seq_cst);
        const cudaError_t e = cudaStreamSynchronize(sv->stream);
        if (e != cudaSuccess) st = fail(VF_ERR_CUDA, std::string("serving kernel: ") + cudaGetErrorString(e));
        sv->running = false;
    }
    free_server(sv);
    return st;
}

extern "C" vf_status vf_serve_stats(vf_server *sv, double *wait_us, double *copy_us, double *search_us,
                                    int64_t *parts_done) {
    if (!sv) return fail(VF_ERR_INVALID_ARG, "NULL server");
    unsigned long long h[4] = {0, 0, 0, 0};
    // a copy on a side stream: the serving stream never completes while the kernel runs
    cudaStream_t st;
    VF_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    cudaError_t e = cudaMemcpyAsync(h, sv->ring.stats, sizeof(h), cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    cudaStreamDestroy(st);
    if (e != cudaSuccess) return fail(VF_ERR_CUDA, std::string("serve stats: ") + cudaGetErrorString(e));
    const double n = h[3] ? (double)h[3] : 1.0;
    if (wait_us) *wait_us = h[0] / n / 1e3;
    if (copy_us) *copy_us = h[1] / n / 1e3;
    if (search_us) *search_us = h[2] / n / 1e3;
    if (parts_done) *parts_done = (int64_t)h[3];
    return VF_OK;
}

extern "C" vf_status vf_serve_info(const vf_server *sv, int32_t *n_workers, int64_t *submitted) {
    if (!sv) return fail(VF_ERR_INVALID_ARG, "NULL server");
    if (n_workers) *n_workers = sv->n_ctas;
    if (submitted) *submitted = sv->submitted.load();
    return VF_OK;
}
