// C-ABI of libvecflow (include/vf.h): validation, index build (Alg. 1) into the HBM
// layout of DESIGN.md §5, and the per-batch orchestration of the search path (Alg. 2): copies,
// route/bucket (a1), scan (a2), graph (a3), merge (a5). Host code only plans and launches;
// every step of the search runs in the CUDA kernels of this directory.
#include "vf.h"

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <unordered_map>
#include <vector>

#include "vf_internal.h"

namespace vf {
int scan_qg(int row_bytes, int k);
}

using namespace vf;

static thread_local std::string g_err;

static vf_status fail(vf_status s, const std::string &m) {
    g_err = m;
    return s;
}

#define VF_CUDA(x)                                                                              \
    do {                                                                                        \
        cudaError_t e_ = (x);                                                                   \
        if (e_ != cudaSuccess) {                                                                \
            vf_status st_ = e_ == cudaErrorMemoryAllocation ? VF_ERR_OUT_OF_MEMORY : VF_ERR_CUDA;\
            return fail(st_, std::string(#x) + ": " + cudaGetErrorString(e_));                  \
        }                                                                                       \
    } while (0)

// ------------------------------------------------------------------ device buffers
struct DevBuf {
    void *p = nullptr;
    size_t n = 0;
    DevBuf() = default;
    DevBuf(const DevBuf &) = delete;
    DevBuf &operator=(const DevBuf &) = delete;
    ~DevBuf() { release(); }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        n = 0;
    }
    // grow to at least `bytes` (contents not preserved); returns true if reallocated
    cudaError_t ensure(size_t bytes, bool *fresh = nullptr) {
        if (fresh) *fresh = false;
        if (bytes <= n && p) return cudaSuccess;
        release();
        size_t want = bytes < 256 ? 256 : bytes;
        cudaError_t e = cudaMalloc(&p, want);
        if (e != cudaSuccess) { p = nullptr; return e; }
        n = want;
        if (fresh) *fresh = true;
        return cudaSuccess;
    }
    template <class T> T *as() const { return reinterpret_cast<T *>(p); }
};

struct Scratch {
    DevBuf raw, Qp, qoff, qlab, qinfo, items, item_ctr, graph_list, scan_slots, scan_q, segs, tiles, item_seg,
        item_res, partials, ctr, out_ids, out_dists, ls_count, ls_segbase, ls_itembase, gtab;
    size_t gtab_slots = 0, gtab_warps = 0;
    cudaEvent_t ev[8];
    bool ev_ok = false;
    bool profiled = false;
    SearchArgs last{};
    int64_t last_slots = 0;
    int last_launches = 0;
    bool has_last = false;
    ~Scratch() {
        if (ev_ok)
            for (auto &e : ev) cudaEventDestroy(e);
    }
};

struct vf_index {
    DevIndex dev{};
    int device = 0;
    DevBuf X, dir, G, M_hs, Xls, M_ls, pt_off, pt_lab;
    vf_index_info info{};
    int32_t max_ls_size = 0, max_label_size = 0;
    std::mutex mu;
    std::unordered_map<cudaStream_t, Scratch *> scratch;
    bool profiling = false;
    ~vf_index() {
        for (auto &kv : scratch) delete kv.second;
    }
};

// ------------------------------------------------------------------ helpers
static bool is_device_ptr(const void *p) {
    if (!p) return false;
    cudaPointerAttributes at;
    cudaError_t e = cudaPointerGetAttributes(&at, p);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged;
}

static int elem_size(int dtype) { return dtype == VF_U8 ? 1 : 4; }

static uint64_t pow2ceil(uint64_t x) {
    uint64_t p = 1;
    while (p < x) p <<= 1;
    return p;
}

extern "C" const char *vf_last_error(void) { return g_err.c_str(); }

extern "C" void vf_free(vf_index *index) {
    if (!index) return;
    cudaSetDevice(index->device);
    delete index;
}

// ------------------------------------------------------------------ build (Alg. 1)
extern "C" vf_status vf_build_index(const vf_build_desc *d, vf_index **out) {
    if (!out) return fail(VF_ERR_INVALID_ARG, "out is NULL");
    *out = nullptr;
    if (!d) return fail(VF_ERR_INVALID_ARG, "desc is NULL");
    if (d->dtype != VF_U8 && d->dtype != VF_F32) return fail(VF_ERR_INVALID_ARG, "dtype must be VF_U8 or VF_F32");
    if (d->dim < 1 || (int64_t)d->dim * elem_size(d->dtype) > 4096)
        return fail(VF_ERR_INVALID_ARG, "dim must satisfy 1 <= dim*sizeof(elem) <= 4096");
    if (d->n_points < 0 || d->n_points >= (1ll << 31)) return fail(VF_ERR_INVALID_ARG, "n_points out of range");
    if (d->n_points > 0 && !d->vectors) return fail(VF_ERR_INVALID_ARG, "vectors is NULL");
    if (d->n_labels < 0) return fail(VF_ERR_INVALID_ARG, "n_labels < 0");
    if (!d->posting_offsets || (d->n_labels > 0 && !d->posting_ids && d->posting_offsets[d->n_labels] > 0))
        return fail(VF_ERR_INVALID_ARG, "posting lists are NULL");
    if (d->threshold_T < 1) return fail(VF_ERR_INVALID_ARG, "threshold_T must be >= 1");
    if (d->degree_R < 1 || d->degree_R > 64) return fail(VF_ERR_INVALID_ARG, "degree_R must be in [1, 64]");
    if (d->world_size != 1 && d->world_size != 0)
        return fail(VF_ERR_INVALID_ARG, "world_size > 1: use the sharded build (vf_shard.cpp)");

    const int64_t N = d->n_points;
    const int L = d->n_labels, R = d->degree_R, T = d->threshold_T;
    const int es = elem_size(d->dtype);
    const int raw_bytes = d->dim * es;
    const int row_bytes = (raw_bytes + 15) & ~15;
    const int64_t *po = d->posting_offsets;
    const int32_t *pi = d->posting_ids;

    // -- validate posting lists (ascending global ids) and graphs
    if (po[0] != 0) return fail(VF_ERR_INVALID_ARG, "posting_offsets[0] must be 0");
    int64_t hs_rows = 0, ls_rows = 0, ls_rows_pad = 0, n_hs = 0, n_ls = 0;
    int32_t max_ls = 0, max_any = 0;
    for (int l = 0; l < L; l++) {
        const int64_t a = po[l], b = po[l + 1];
        if (b < a) return fail(VF_ERR_INVALID_ARG, "posting_offsets not non-decreasing at label " + std::to_string(l));
        if (b - a >= (1ll << 31)) return fail(VF_ERR_INVALID_ARG, "posting list too long");
        for (int64_t e = a; e < b; e++) {
            if (pi[e] < 0 || pi[e] >= N)
                return fail(VF_ERR_INVALID_ARG, "posting id out of range in label " + std::to_string(l));
            if (e > a && pi[e] <= pi[e - 1])
                return fail(VF_ERR_INVALID_ARG, "posting list of label " + std::to_string(l) + " not strictly ascending");
        }
        const int64_t S = b - a;
        if (S == 0) continue;
        max_any = std::max<int32_t>(max_any, (int32_t)S);
        const int64_t rows = d->graph_row_offsets ? d->graph_row_offsets[l + 1] - d->graph_row_offsets[l] : 0;
        if (S >= T) {
            if (rows != S)
                return fail(VF_ERR_INVALID_ARG, "HS label " + std::to_string(l) + " (|C_l| >= T) needs |C_l| graph rows");
            const int32_t *g = d->graph_local_ids + d->graph_row_offsets[l] * R;
            for (int64_t e = 0; e < S * R; e++)
                if (g[e] < -1 || g[e] >= S)
                    return fail(VF_ERR_INVALID_ARG, "graph entry outside [-1, |C_l|) in label " + std::to_string(l));
            hs_rows += S;
            n_hs++;
        } else {
            if (rows != 0 && rows != S)
                return fail(VF_ERR_INVALID_ARG, "graph rows of label " + std::to_string(l) + " must be 0 or |C_l|");
            ls_rows += S;
            ls_rows_pad += (S + 3) & ~3ll;        // label bases 4-row aligned (16-byte id slices)
            n_ls++;
            max_ls = std::max<int32_t>(max_ls, (int32_t)S);
        }
    }
    if (d->graph_row_offsets && d->graph_row_offsets[0] != 0)
        return fail(VF_ERR_INVALID_ARG, "graph_row_offsets[0] must be 0");

    VF_CUDA(cudaSetDevice(d->device));
    vf_index *ix = new vf_index();
    ix->device = d->device;
    auto bail = [&](vf_status s) { delete ix; return s; };
#define VF_B(x)                                                                                  \
    do {                                                                                         \
        cudaError_t e_ = (x);                                                                    \
        if (e_ != cudaSuccess)                                                                   \
            return bail(fail(e_ == cudaErrorMemoryAllocation ? VF_ERR_OUT_OF_MEMORY : VF_ERR_CUDA, \
                             std::string(#x) + ": " + cudaGetErrorString(e_)));                 \
    } while (0)

    cudaStream_t s = 0;
    // -- X: one shared copy of the vectors, rows padded to 16 bytes
    VF_B(ix->X.ensure((size_t)std::max<int64_t>(N, 1) * row_bytes));
    if (N > 0) {
        if (raw_bytes == row_bytes) {
            VF_B(cudaMemcpy(ix->X.p, d->vectors, (size_t)N * raw_bytes, cudaMemcpyHostToDevice));
        } else {
            DevBuf tmp;
            VF_B(tmp.ensure((size_t)N * raw_bytes));
            VF_B(cudaMemcpy(tmp.p, d->vectors, (size_t)N * raw_bytes, cudaMemcpyHostToDevice));
            launch_pad_rows(tmp.as<uint8_t>(), raw_bytes, N, row_bytes, ix->X.as<uint8_t>(), s);
            VF_B(cudaGetLastError());
            VF_B(cudaDeviceSynchronize());
        }
    }
    // -- directory + M_HS / G_HS (compacted, ordered by label) + M_LS
    std::vector<LabelDir> dir(std::max(L, 1));
    std::vector<int32_t> m_hs((size_t)std::max<int64_t>(hs_rows, 1)), m_ls((size_t)ls_rows_pad + 4, -1);   // + slack: the last id slice is read 16 B-rounded
    std::vector<int2> g_hs((size_t)std::max<int64_t>(hs_rows * R, 1));
    int64_t hb = 0, lb = 0;
    int32_t bslot = 0;
    for (int l = 0; l < L; l++) {
        const int64_t a = po[l], S = po[l + 1] - po[l];
        dir[l].size = (int32_t)S;
        dir[l].bslot = -1;
        dir[l].base = 0;
        if (S == 0) continue;
        dir[l].bslot = bslot++;
        if (S >= T) {
            dir[l].base = hb;
            std::memcpy(&m_hs[hb], pi + a, S * sizeof(int32_t));
            const int32_t *src = d->graph_local_ids + d->graph_row_offsets[l] * R;
            for (int64_t e = 0; e < S * R; e++) {
                const int32_t c = src[e];
                g_hs[hb * R + e] = c >= 0 ? make_int2(c, pi[a + c]) : make_int2(-1, -1);
            }
            hb += S;
        } else {
            dir[l].base = lb;
            std::memcpy(&m_ls[lb], pi + a, S * sizeof(int32_t));
            lb += (S + 3) & ~3ll;
        }
    }
    VF_B(ix->dir.ensure(dir.size() * sizeof(LabelDir)));
    VF_B(cudaMemcpy(ix->dir.p, dir.data(), dir.size() * sizeof(LabelDir), cudaMemcpyHostToDevice));
    VF_B(ix->M_hs.ensure(m_hs.size() * 4));
    VF_B(cudaMemcpy(ix->M_hs.p, m_hs.data(), m_hs.size() * 4, cudaMemcpyHostToDevice));
    VF_B(ix->G.ensure(g_hs.size() * 8));
    VF_B(cudaMemcpy(ix->G.p, g_hs.data(), g_hs.size() * 8, cudaMemcpyHostToDevice));
    VF_B(ix->M_ls.ensure(m_ls.size() * 4));
    VF_B(cudaMemcpy(ix->M_ls.p, m_ls.data(), m_ls.size() * 4, cudaMemcpyHostToDevice));
    // -- X_LS: label-contiguous row copies of the LS lists, gathered on the device
    VF_B(ix->Xls.ensure((size_t)std::max<int64_t>(ls_rows_pad, 1) * row_bytes));
    launch_gather_rows(ix->X.as<uint8_t>(), row_bytes, ix->M_ls.as<int32_t>(), ls_rows_pad, ix->Xls.as<uint8_t>(), s);
    VF_B(cudaGetLastError());
    // -- predicate table: point -> sorted labels, transposed from the posting lists
    std::vector<int64_t> poff((size_t)N + 1, 0);
    for (int l = 0; l < L; l++)
        for (int64_t e = po[l]; e < po[l + 1]; e++) poff[(size_t)pi[e] + 1]++;
    for (int64_t i = 0; i < N; i++) poff[i + 1] += poff[i];
    const int64_t n_entries = poff[N];
    std::vector<int32_t> plab((size_t)std::max<int64_t>(n_entries, 1));
    {
        std::vector<int64_t> fill(poff.begin(), poff.end() - 1);
        for (int l = 0; l < L; l++)
            for (int64_t e = po[l]; e < po[l + 1]; e++) plab[fill[pi[e]]++] = l;
    }
    VF_B(ix->pt_off.ensure(poff.size() * 8));
    VF_B(cudaMemcpy(ix->pt_off.p, poff.data(), poff.size() * 8, cudaMemcpyHostToDevice));
    VF_B(ix->pt_lab.ensure(plab.size() * 4));
    VF_B(cudaMemcpy(ix->pt_lab.p, plab.data(), plab.size() * 4, cudaMemcpyHostToDevice));
    VF_B(cudaDeviceSynchronize());

    DevIndex &D = ix->dev;
    D.dtype = d->dtype;
    D.dim = d->dim;
    D.row_bytes = row_bytes;
    D.chunks = row_bytes / 16;
    D.n_points = N;
    D.n_labels = L;
    D.T = T;
    D.R = R;
    D.n_bslots = bslot;
    D.X = ix->X.as<uint8_t>();
    D.dir = ix->dir.as<LabelDir>();
    D.G = ix->G.as<int2>();
    D.M_hs = ix->M_hs.as<int32_t>();
    D.Xls = ix->Xls.as<uint8_t>();
    D.M_ls = ix->M_ls.as<int32_t>();
    D.pt_off = ix->pt_off.as<int64_t>();
    D.pt_lab = ix->pt_lab.as<int32_t>();
    ix->max_ls_size = max_ls;
    ix->max_label_size = max_any;

    vf_index_info &I = ix->info;
    I.n_points = N;
    I.n_labels = L;
    I.n_hs_labels = n_hs;
    I.n_ls_labels = n_ls;
    I.hs_rows = hs_rows;
    I.ls_rows = ls_rows;
    I.row_bytes = row_bytes;
    I.degree_R = R;
    I.bytes_vectors = N * row_bytes;
    I.bytes_graph = hs_rows * R * 8;
    I.bytes_map_hs = hs_rows * 4;
    I.bytes_ls_vectors = ls_rows_pad * row_bytes;
    I.bytes_map_ls = (ls_rows_pad + 4) * 4;
    I.bytes_predicate = (N + 1) * 8 + n_entries * 4;
    I.bytes_directory = (int64_t)L * sizeof(LabelDir);
    I.bytes_total = I.bytes_vectors + I.bytes_graph + I.bytes_map_hs + I.bytes_ls_vectors + I.bytes_map_ls +
                    I.bytes_predicate + I.bytes_directory;
    I.world_size = 1;
    I.rank = 0;
    I.owned_labels = n_hs + n_ls;
    *out = ix;
    return VF_OK;
#undef VF_B
}

extern "C" vf_status vf_get_index_info(const vf_index *index, vf_index_info *info) {
    if (!index || !info) return fail(VF_ERR_INVALID_ARG, "NULL argument");
    *info = index->info;
    return VF_OK;
}

extern "C" vf_status vf_set_profiling(vf_index *index, int32_t enable) {
    if (!index) return fail(VF_ERR_INVALID_ARG, "NULL index");
    index->profiling = enable != 0;
    return VF_OK;
}

// ------------------------------------------------------------------ search (Alg. 2)
static Scratch *get_scratch(vf_index *ix, cudaStream_t s) {
    std::lock_guard<std::mutex> g(ix->mu);
    auto it = ix->scratch.find(s);
    if (it != ix->scratch.end()) return it->second;
    Scratch *sc = new Scratch();
    ix->scratch[s] = sc;
    return sc;
}

extern "C" vf_status vf_search(vf_index *ix, const void *queries, int64_t n, const int64_t *qoff,
                               const int32_t *qlab, const vf_search_params *p, int32_t *out_ids,
                               float *out_dists, void *cuda_stream) {
    if (!ix) return fail(VF_ERR_INVALID_ARG, "index is NULL");
    if (!p) return fail(VF_ERR_INVALID_ARG, "params is NULL");
    if (n < 0) return fail(VF_ERR_INVALID_ARG, "n_queries < 0");
    if (p->k < 1 || p->k > kMaxK) return fail(VF_ERR_INVALID_ARG, "k must be in [1, 256]");
    if (p->itopk < p->k || p->itopk > kMaxItopk) return fail(VF_ERR_INVALID_ARG, "itopk must be in [k, 1024]");
    const int R = ix->dev.R;
    const int w = p->search_width < 1 ? 1 : p->search_width;
    if (w * R > 64) return fail(VF_ERR_INVALID_ARG, "search_width * R must be <= 64");
    if (p->op < 0 || p->op > 2) return fail(VF_ERR_INVALID_ARG, "op must be VF_SINGLE, VF_OR or VF_AND");
    if (p->recall_mode < 0 || p->recall_mode > 1) return fail(VF_ERR_INVALID_ARG, "bad recall_mode");
    if (n > 0 && (!queries || !qoff || !out_ids || !out_dists))
        return fail(VF_ERR_INVALID_ARG, "NULL queries / offsets / outputs");
    if (n == 0) return VF_OK;
    VF_CUDA(cudaSetDevice(ix->device));
    cudaStream_t s = (cudaStream_t)cuda_stream;
    Scratch *sc = get_scratch(ix, s);
    const DevIndex &D = ix->dev;
    const int k = p->k;

    const bool q_dev = is_device_ptr(queries);
    const bool off_dev = is_device_ptr(qoff);
    const bool lab_dev = is_device_ptr(qlab);
    const bool out_dev = is_device_ptr(out_ids);
    if (out_dev != is_device_ptr(out_dists))
        return fail(VF_ERR_INVALID_ARG, "out_ids and out_dists must both be host or both be device");

    int64_t n_slots = 0;
    if (!off_dev) {
        if (qoff[0] != 0) return fail(VF_ERR_INVALID_ARG, "qlabel_offsets[0] must be 0");
        n_slots = qoff[n];
        for (int64_t i = 0; i < n; i++) {
            const int64_t c = qoff[i + 1] - qoff[i];
            if (c < 0 || c > kMaxQueryLabels)
                return fail(VF_ERR_INVALID_ARG, "query " + std::to_string(i) + " has a bad label count (max 64)");
            if (p->op == VF_SINGLE && c > 1 && !lab_dev) {
                for (int64_t e = qoff[i] + 1; e < qoff[i + 1]; e++)
                    if (qlab[e] != qlab[qoff[i]])
                        return fail(VF_ERR_INVALID_ARG, "VF_SINGLE query " + std::to_string(i) + " has more than one label");
            }
        }
    } else {
        VF_CUDA(cudaMemcpyAsync(&n_slots, qoff + n, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
        VF_CUDA(cudaStreamSynchronize(s));
    }
    if (n_slots > 0 && !qlab) return fail(VF_ERR_INVALID_ARG, "qlabels is NULL");
    if (n_slots >= (1ll << 31)) return fail(VF_ERR_INVALID_ARG, "too many query labels");

    // -- plan
    const int scan_max = p->exact ? ix->max_label_size : ix->max_ls_size;
    // row tiles: small in the normal path (load balance across SMs; a label split over several
    // tiles is finalised in-kernel), large in exact mode (<= 256 tiles per label)
    int tile_rows = p->exact ? 4096 : 512;
    if (!p->exact) {
        static const int env_tile = [] { const char *e = getenv("VF_TILE_ROWS"); return e ? atoi(e) : 0; }();
        if (env_tile >= 64) tile_rows = env_tile & ~63;   // experiment knob (scripts/ab.py)
    }
    if ((scan_max + 255) / 256 > tile_rows) tile_rows = (((scan_max + 255) / 256) + 63) & ~63;  // x64 rows
    const int mtpl = std::max(1, (scan_max + tile_rows - 1) / tile_rows);
    const bool multi = mtpl > 1;
    const int qg = scan_qg(D.row_bytes, k);
    const int64_t slots = std::max<int64_t>(n_slots, 1);
    const int64_t max_tiles = slots * mtpl;
    const int n_init = p->n_init > 0 ? p->n_init : R * w;
    const int max_iter = p->max_iterations > 0 ? p->max_iterations : 2 * ((p->itopk + w - 1) / w) + 16;
    // visited sets: shared-memory table sized for ~16 warps/SM, exact global overflow table
    // ~32 itopk-sized expansions' worth of ids in shared memory, within ~7 KB per warp
    int hs = 1024;
    {
        const int64_t budget = 7168 - 16ll * p->itopk - 1024;
        while (hs < 64 * p->itopk && hs < 8192 && (int64_t)hs * 2 * 4 <= budget) hs <<= 1;
    }
    const int64_t v_bound = (int64_t)n_init + (int64_t)max_iter * w * R + 32;
    const uint64_t gslots = pow2ceil((uint64_t)(2 * v_bound + 64));

    SearchArgs a{};
    a.ix = D;
    a.n_q = n;
    a.k = k;
    a.itopk = p->itopk;
    a.w = w;
    a.n_init = n_init;
    a.max_iter = max_iter;
    a.seed = p->seed;
    a.op = p->op;
    a.recall_mode = p->recall_mode;
    a.exact = p->exact ? 1 : 0;
    a.tile_rows = tile_rows;
    a.max_tiles_per_label = mtpl;
    a.max_tiles = (int32_t)std::min<int64_t>(max_tiles, INT32_MAX);
    a.hash_slots = hs;
    a.gtab_slots = (int64_t)gslots;

    const int graph_ctas = graph_max_ctas(a);
    if (graph_ctas <= 0) return fail(VF_ERR_INTERNAL, "no graph kernel for this row size");
    const size_t nwarp = (size_t)graph_ctas * kWarpsPerGraphCta;
    a.n_warp_slots = (int32_t)nwarp;

    // -- scratch
    const int raw_bytes = D.dim * elem_size(D.dtype);
    bool fresh = false;
    if (!q_dev) VF_CUDA(sc->raw.ensure((size_t)n * raw_bytes));
    VF_CUDA(sc->Qp.ensure((size_t)n * D.row_bytes));
    if (!off_dev) VF_CUDA(sc->qoff.ensure((size_t)(n + 1) * 8));
    VF_CUDA(sc->qlab.ensure((size_t)slots * 4));
    VF_CUDA(sc->qinfo.ensure((size_t)n * sizeof(QueryInfo)));
    VF_CUDA(sc->items.ensure((size_t)slots * sizeof(Item)));
    VF_CUDA(sc->item_ctr.ensure((size_t)slots * 12));
    VF_CUDA(sc->graph_list.ensure((size_t)slots * 4));
    VF_CUDA(sc->scan_slots.ensure((size_t)slots * 4));
    VF_CUDA(sc->scan_q.ensure((size_t)slots * sizeof(ScanQuery)));
    VF_CUDA(sc->segs.ensure((size_t)slots * sizeof(Segment)));
    VF_CUDA(sc->tiles.ensure((size_t)max_tiles * sizeof(Tile)));
    VF_CUDA(sc->item_seg.ensure((size_t)slots * 4));
    VF_CUDA(sc->item_res.ensure((size_t)slots * k * 8));
    if (multi) VF_CUDA(sc->partials.ensure((size_t)slots * mtpl * k * 8));
    VF_CUDA(sc->ctr.ensure(sizeof(Counters)));
    const size_t nls = (size_t)std::max(D.n_bslots, 1);
    VF_CUDA(sc->ls_count.ensure(nls * 4, &fresh));
    if (fresh) VF_CUDA(cudaMemsetAsync(sc->ls_count.p, 0, nls * 4, s));
    VF_CUDA(sc->ls_segbase.ensure(nls * 4));
    VF_CUDA(sc->ls_itembase.ensure(nls * 4));
    if (sc->gtab_slots < gslots || sc->gtab_warps < nwarp) {
        sc->gtab.release();
        const size_t gs = std::max<size_t>(sc->gtab_slots, gslots), gw = std::max(sc->gtab_warps, nwarp);
        VF_CUDA(sc->gtab.ensure(gw * gs * 8 + gw * 4));
        VF_CUDA(cudaMemsetAsync(sc->gtab.p, 0, gw * gs * 8 + gw * 4, s));
        sc->gtab_slots = gs;
        sc->gtab_warps = gw;
    }
    // the kernels index the tables with the allocated geometry
    a.gtab_slots = (int64_t)sc->gtab_slots;
    a.n_warp_slots = (int32_t)sc->gtab_warps;
    if (!out_dev) {
        VF_CUDA(sc->out_ids.ensure((size_t)n * k * 4));
        VF_CUDA(sc->out_dists.ensure((size_t)n * k * 4));
    }
    if (!sc->ev_ok) {
        for (auto &e : sc->ev) VF_CUDA(cudaEventCreate(&e));
        sc->ev_ok = true;
    }
    const bool prof = ix->profiling;
    if (prof) VF_CUDA(cudaEventRecord(sc->ev[0], s));

    // -- inputs to the device
    if (!q_dev) VF_CUDA(cudaMemcpyAsync(sc->raw.p, queries, (size_t)n * raw_bytes, cudaMemcpyHostToDevice, s));
    if (!off_dev) VF_CUDA(cudaMemcpyAsync(sc->qoff.p, qoff, (size_t)(n + 1) * 8, cudaMemcpyHostToDevice, s));
    if (n_slots > 0)
        VF_CUDA(cudaMemcpyAsync(sc->qlab.p, qlab, (size_t)n_slots * 4,
                                lab_dev ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, s));
    VF_CUDA(cudaMemsetAsync(sc->ctr.p, 0, sizeof(Counters), s));
    if (prof) VF_CUDA(cudaEventRecord(sc->ev[1], s));

    a.Qraw = q_dev ? reinterpret_cast<const uint8_t *>(queries) : sc->raw.as<uint8_t>();
    a.Qp = sc->Qp.as<uint8_t>();
    a.q_off = off_dev ? qoff : sc->qoff.as<int64_t>();
    a.qlab = sc->qlab.as<int32_t>();
    a.qinfo = sc->qinfo.as<QueryInfo>();
    a.items = sc->items.as<Item>();
    a.item_ctr = sc->item_ctr.as<int32_t>();
    a.ls_count = sc->ls_count.as<int32_t>();
    a.ls_segbase = sc->ls_segbase.as<int32_t>();
    a.ls_itembase = sc->ls_itembase.as<int32_t>();
    a.graph_list = sc->graph_list.as<int32_t>();
    a.scan_slots = sc->scan_slots.as<int32_t>();
    a.scan_q = sc->scan_q.as<ScanQuery>();
    a.segs = sc->segs.as<Segment>();
    a.tiles = sc->tiles.as<Tile>();
    a.item_seg = sc->item_seg.as<int32_t>();
    a.item_res = sc->item_res.as<unsigned long long>();
    a.partials = multi ? sc->partials.as<unsigned long long>() : nullptr;
    a.ctr = sc->ctr.as<Counters>();
    a.out_ids = out_dev ? out_ids : sc->out_ids.as<int32_t>();
    a.out_dists = out_dev ? out_dists : sc->out_dists.as<float>();
    a.gtab = sc->gtab.as<unsigned long long>();

    int launches = 0;
    launches += launch_prepare(a, s);
    launches += launch_bucket(a, s, n_slots, qg);
    if (prof) VF_CUDA(cudaEventRecord(sc->ev[2], s));
    const int sl = launch_scan(a, s, (int)std::min<int64_t>(max_tiles, INT32_MAX));
    if (sl < 0) return fail(VF_ERR_INTERNAL, "scan kernel dispatch failed");
    launches += sl;
    if (prof) VF_CUDA(cudaEventRecord(sc->ev[3], s));
    const int gl = launch_graph(a, s, (int)std::min<int64_t>(n_slots, INT32_MAX), graph_ctas);
    if (gl < 0) return fail(VF_ERR_INTERNAL, "graph kernel dispatch failed");
    launches += gl;
    if (prof) VF_CUDA(cudaEventRecord(sc->ev[4], s));
    const bool need_merge = p->op == VF_OR || (p->op == VF_AND && p->recall_mode == VF_RECALL_PARALLEL);
    if (need_merge) launches += launch_merge(a, s);
    if (prof) VF_CUDA(cudaEventRecord(sc->ev[5], s));
    VF_CUDA(cudaGetLastError());
    if (!out_dev) {
        VF_CUDA(cudaMemcpyAsync(out_ids, sc->out_ids.p, (size_t)n * k * 4, cudaMemcpyDeviceToHost, s));
        VF_CUDA(cudaMemcpyAsync(out_dists, sc->out_dists.p, (size_t)n * k * 4, cudaMemcpyDeviceToHost, s));
    }
    if (prof) VF_CUDA(cudaEventRecord(sc->ev[6], s));
    sc->last = a;
    sc->last_slots = n_slots;
    sc->last_launches = launches;
    sc->profiled = prof;
    sc->has_last = true;
    if (!out_dev) VF_CUDA(cudaStreamSynchronize(s));
    return VF_OK;
}

extern "C" vf_status vf_get_last_stats(vf_index *ix, void *cuda_stream, vf_search_stats *st) {
    if (!ix || !st) return fail(VF_ERR_INVALID_ARG, "NULL argument");
    VF_CUDA(cudaSetDevice(ix->device));
    cudaStream_t s = (cudaStream_t)cuda_stream;
    Scratch *sc = get_scratch(ix, s);
    std::memset(st, 0, sizeof(*st));
    if (!sc->has_last) return fail(VF_ERR_INVALID_ARG, "no search on this stream yet");
    VF_CUDA(cudaStreamSynchronize(s));
    Counters c;
    VF_CUDA(cudaMemcpy(&c, sc->ctr.p, sizeof(c), cudaMemcpyDeviceToHost));
    st->n_queries = sc->last.n_q;
    st->n_items = (int64_t)c.n_graph + c.n_scan_items;
    st->n_graph_items = c.n_graph;
    st->n_scan_items = c.n_scan_items;
    st->n_segments = c.n_segs;
    st->n_tiles = c.n_tiles;
    st->scan_rows = (int64_t)c.scan_rows;
    st->scan_query_rows = (int64_t)c.scan_qrows;
    st->graph_V = (int64_t)c.graph_V;
    st->graph_E = (int64_t)c.graph_E;
    st->graph_iterations = (int64_t)c.graph_iters;
    st->graph_V_max = (int64_t)c.graph_V_max;
    st->kernel_launches = sc->last_launches;
    st->row_bytes = ix->dev.row_bytes;
    if (sc->profiled) {
        float t;
        cudaEventElapsedTime(&t, sc->ev[1], sc->ev[2]); st->ms_route = t;
        cudaEventElapsedTime(&t, sc->ev[2], sc->ev[3]); st->ms_scan = t;
        cudaEventElapsedTime(&t, sc->ev[3], sc->ev[4]); st->ms_graph = t;
        cudaEventElapsedTime(&t, sc->ev[4], sc->ev[5]); st->ms_merge = t;
        float c0, c1;
        cudaEventElapsedTime(&c0, sc->ev[0], sc->ev[1]);
        cudaEventElapsedTime(&c1, sc->ev[5], sc->ev[6]);
        st->ms_copy = c0 + c1;
        cudaEventElapsedTime(&t, sc->ev[0], sc->ev[6]); st->ms_total = t;
    }
    return VF_OK;
}

extern "C" vf_status vf_get_last_items(vf_index *ix, void *cuda_stream, int64_t max_items, int32_t *rec,
                                       int64_t *n_items) {
    if (!ix || !n_items) return fail(VF_ERR_INVALID_ARG, "NULL argument");
    VF_CUDA(cudaSetDevice(ix->device));
    cudaStream_t s = (cudaStream_t)cuda_stream;
    Scratch *sc = get_scratch(ix, s);
    if (!sc->has_last) return fail(VF_ERR_INVALID_ARG, "no search on this stream yet");
    VF_CUDA(cudaStreamSynchronize(s));
    const int64_t ns = sc->last_slots;
    std::vector<Item> items((size_t)std::max<int64_t>(ns, 1));
    std::vector<int32_t> ctr((size_t)std::max<int64_t>(ns, 1) * 3);
    if (ns > 0) {
        VF_CUDA(cudaMemcpy(items.data(), sc->items.p, ns * sizeof(Item), cudaMemcpyDeviceToHost));
        VF_CUDA(cudaMemcpy(ctr.data(), sc->item_ctr.p, ns * 12, cudaMemcpyDeviceToHost));
    }
    int64_t m = 0;
    for (int64_t i = 0; i < ns; i++) {
        const uint32_t path = items[i].meta & 3u;
        if (path == PATH_NONE) continue;
        if (rec && m < max_items) {
            int32_t *r = rec + m * 6;
            r[0] = items[i].qid;
            r[1] = items[i].label;
            r[2] = (int32_t)path;
            const bool g = path == PATH_GRAPH;
            r[3] = g ? ctr[i * 3 + 0] : 0;
            r[4] = g ? ctr[i * 3 + 1] : 0;
            r[5] = g ? ctr[i * 3 + 2] : 0;
        }
        m++;
    }
    *n_items = m;
    return VF_OK;
}
