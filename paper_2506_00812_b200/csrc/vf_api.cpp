// C-ABI of libvecflow (include/vf.h): validation, index build (Alg. 1) into the HBM
// layout of DESIGN.md §5, and the per-batch orchestration of the search path (Alg. 2): copies,
// route/bucket (a1), scan (a2), graph (a3), merge (a5). Host code only plans and launches; every
// step of the search runs in the CUDA kernels of this directory. Label sharding (§8(e)) is in
// shard.cpp.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "host_internal.h"
#include "small.h"

namespace vf {
int scan_qg(int row_bytes, int k);

static thread_local std::string g_err;

vf_status fail(vf_status s, const std::string &m) {
    g_err = m;
    return s;
}

bool is_device_ptr(const void *p) {
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

Scratch *get_scratch(vf_index *ix, cudaStream_t s, int role) {
    std::lock_guard<std::mutex> g(ix->mu);
    const uint64_t key = (uint64_t)(uintptr_t)s * 4 + (uint64_t)role;
    auto it = ix->scratch.find(key);
    if (it != ix->scratch.end()) return it->second;
    Scratch *sc = new Scratch();
    ix->scratch[key] = sc;
    return sc;
}

}  // namespace vf

using namespace vf;

vf_index::~vf_index() {
    for (auto &kv : scratch) delete kv.second;
    for (vf_index *s : vshards) delete s;
    if (transport) transport_destroy(transport);
}

extern "C" const char *vf_last_error(void) { return vf::g_err.c_str(); }

extern "C" void vf_free(vf_index *index) {
    if (!index) return;
    cudaSetDevice(index->device);
    delete index;
}

// ------------------------------------------------------------------ build (Alg. 1)
static vf_status validate_desc(const vf_build_desc *d) {
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
    const int64_t N = d->n_points;
    const int L = d->n_labels, R = d->degree_R, T = d->threshold_T;
    const int64_t *po = d->posting_offsets;
    const int32_t *pi = d->posting_ids;
    if (po[0] != 0) return fail(VF_ERR_INVALID_ARG, "posting_offsets[0] must be 0");
    if (d->graph_row_offsets && d->graph_row_offsets[0] != 0)
        return fail(VF_ERR_INVALID_ARG, "graph_row_offsets[0] must be 0");
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
        const int64_t rows = d->graph_row_offsets ? d->graph_row_offsets[l + 1] - d->graph_row_offsets[l] : 0;
        if (S >= T) {
            if (rows != S)
                return fail(VF_ERR_INVALID_ARG, "HS label " + std::to_string(l) + " (|C_l| >= T) needs |C_l| graph rows");
            const int32_t *g = d->graph_local_ids + d->graph_row_offsets[l] * R;
            for (int64_t e = 0; e < S * R; e++)
                if (g[e] < -1 || g[e] >= S)
                    return fail(VF_ERR_INVALID_ARG, "graph entry outside [-1, |C_l|) in label " + std::to_string(l));
        } else if (rows != 0 && rows != S) {
            return fail(VF_ERR_INVALID_ARG, "graph rows of label " + std::to_string(l) + " must be 0 or |C_l|");
        }
    }
    return VF_OK;
}

// One rank's index: X and the predicate table replicated, graphs / LS rows only of the labels
// this rank owns (all labels when owner is empty). The directory keeps |C_l| of every label so
// routing decisions (path, greedy l*) are the same on every rank.
static vf_status build_one(const vf_build_desc *d, int world, int rank, const std::vector<int32_t> &owner,
                           vf_index **out) {
    const int64_t N = d->n_points;
    const int L = d->n_labels, R = d->degree_R, T = d->threshold_T;
    const int raw_bytes = d->dim * elem_size(d->dtype);
    const int row_bytes = (raw_bytes + 15) & ~15;
    const int64_t *po = d->posting_offsets;
    const int32_t *pi = d->posting_ids;
    auto mine = [&](int l) { return owner.empty() || owner[l] == rank; };

    int64_t hs_rows = 0, ls_rows = 0, ls_rows_pad = 0, n_hs = 0, n_ls = 0;
    int32_t max_ls = 0, max_any = 0;
    for (int l = 0; l < L; l++) {
        const int64_t S = po[l + 1] - po[l];
        if (S == 0 || !mine(l)) continue;
        max_any = std::max<int32_t>(max_any, (int32_t)S);
        if (S >= T) {
            hs_rows += S;
            n_hs++;
        } else {
            ls_rows += S;
            ls_rows_pad += (S + 3) & ~3ll;        // label bases 4-row aligned (16-byte id slices)
            n_ls++;
            max_ls = std::max<int32_t>(max_ls, (int32_t)S);
        }
    }

    VF_CUDA(cudaSetDevice(d->device));
    vf_index *ix = new vf_index();
    ix->device = d->device;
    ix->world = world;
    ix->rank = rank;
    ix->owner = owner;
    auto bail = [&](vf_status st) {
        delete ix;
        return st;
    };
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
    // -- directory + G_HS (fat rows, compacted by label) + M_HS + M_LS
    std::vector<LabelDir> dir(std::max(L, 1));
    std::vector<int32_t> m_hs((size_t)std::max<int64_t>(hs_rows, 1));
    std::vector<int32_t> m_ls((size_t)ls_rows_pad + 4, -1);   // + slack: the last id slice is read 16 B-rounded
    std::vector<int2> g_hs((size_t)std::max<int64_t>(hs_rows * R, 1));
    int64_t hb = 0, lb = 0;
    int32_t bslot = 0;
    for (int l = 0; l < L; l++) {
        const int64_t a = po[l], S = po[l + 1] - po[l];
        dir[l].size = (int32_t)S;          // every label's size: routing is identical on all ranks
        dir[l].bslot = -1;
        dir[l].base = -1;
        if (S == 0 || !mine(l)) continue;
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
    // -- integer-valued fp32 fast paths, both exact:
    //    (a) every value an integer in [0, 255]: a lossless u8 row store (X8, X_LS8) is the copy the
    //        kernels read -- 4x fewer bytes, identical distances; the fp32 rows stay for batches
    //        holding a query outside that range (gated fallback on the device);
    //    (b) else every value an integer in the tf32-exact range: the scan runs on kind::tf32.
    // Row norms feed the tensor-core scan's ||x||^2 + ||q||^2 - 2 q.x expansion (exact int32).
    static const bool tc_off = [] { const char *e = getenv("VF_SCAN_TC"); return e && atoi(e) == 0; }();
    static const bool u8_off = [] { const char *e = getenv("VF_U8_STORE"); return e && atoi(e) == 0; }();
    const bool enc8 = d->dtype == VF_F32 && !u8_off && rows_int_in_range(ix->X.as<uint8_t>(), N, row_bytes, d->dim,
                                                                          0.f, 255.f, s);
    const float vmax = tf32_exact_vmax(d->dim);
    const bool tc_rows = !tc_off && (d->dtype == VF_U8 || enc8 ||
                                     rows_int_in_range(ix->X.as<uint8_t>(), N, row_bytes, d->dim, -vmax, vmax, s));
    const int row_bytes8 = (d->dim + 15) & ~15;
    if (enc8) {
        VF_B(ix->X8.ensure((size_t)std::max<int64_t>(N, 1) * row_bytes8));
        launch_f32_to_u8(ix->X.as<uint8_t>(), row_bytes, N, d->dim, ix->X8.as<uint8_t>(), row_bytes8, s);
        VF_B(ix->Xls8.ensure((size_t)std::max<int64_t>(ls_rows_pad, 1) * row_bytes8));
        launch_gather_rows(ix->X8.as<uint8_t>(), row_bytes8, ix->M_ls.as<int32_t>(), ls_rows_pad,
                           ix->Xls8.as<uint8_t>(), s);
        VF_B(cudaGetLastError());
    }
    const int fast_dt = enc8 ? VF_U8 : d->dtype;
    const int fast_rb = enc8 ? row_bytes8 : row_bytes;
    const uint8_t *fast_X = enc8 ? ix->X8.as<uint8_t>() : ix->X.as<uint8_t>();
    if (tc_rows) {
        VF_B(ix->xn.ensure((size_t)std::max<int64_t>(N, 1) * 4));
        VF_B(ix->xn_ls.ensure(m_ls.size() * 4));
        launch_row_norms(fast_dt, fast_X, fast_rb, nullptr, N, ix->xn.as<uint32_t>(), s);
        launch_row_norms(fast_dt, fast_X, fast_rb, ix->M_ls.as<int32_t>(), (int64_t)m_ls.size(),
                         ix->xn_ls.as<uint32_t>(), s);
        VF_B(cudaGetLastError());
    }
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
    {
        // per-point label signatures (the predicate's negative fast path, DevIndex::lsig)
        std::vector<unsigned long long> sig((size_t)std::max<int64_t>(N, 1), 0ull);
        for (int64_t i = 0; i < N; i++)
            for (int64_t e = poff[i]; e < poff[i + 1]; e++) sig[(size_t)i] |= label_sig_bits(plab[e]);
        VF_B(ix->lsig.ensure(sig.size() * 8));
        VF_B(cudaMemcpy(ix->lsig.p, sig.data(), sig.size() * 8, cudaMemcpyHostToDevice));
    }
    // -- membership bitmaps of the largest labels (predicate fast path): labels with
    // |C_l| >= N / VF_BITMAP_DENSITY (default 1024: a bitmap is at most 32x its posting list), at most
    // kMaxBitmaps of them, largest first. 0 disables them. HBM is plentiful (YFCC-shaped: ~860
    // bitmaps, 1.1 GB); each turns a predicate check into one bit read (k_and_filter, verify_pred).
    int64_t n_bitmaps = 0, lbit_words = (N + 31) / 32;
    {
        const char *e = getenv("VF_BITMAP_DENSITY");
        const int64_t dens = e ? atoll(e) : 1024;
        std::vector<int32_t> cand;
        if (dens > 0 && N > 0)
            for (int l = 0; l < L; l++)
                if ((po[l + 1] - po[l]) * dens >= N && po[l + 1] > po[l]) cand.push_back(l);
        std::stable_sort(cand.begin(), cand.end(),
                         [&](int32_t x, int32_t y) { return po[x + 1] - po[x] > po[y + 1] - po[y]; });
        if ((int64_t)cand.size() > kMaxBitmaps) cand.resize(kMaxBitmaps);
        n_bitmaps = (int64_t)cand.size();
        if (n_bitmaps > 0) {
            std::vector<int16_t> slot((size_t)L, (int16_t)-1);
            std::vector<uint32_t> bits((size_t)(n_bitmaps * lbit_words), 0u);
            for (int64_t b = 0; b < n_bitmaps; b++) {
                const int32_t l = cand[(size_t)b];
                slot[(size_t)l] = (int16_t)b;
                uint32_t *w = bits.data() + b * lbit_words;
                for (int64_t e2 = po[l]; e2 < po[l + 1]; e2++) w[pi[e2] >> 5] |= 1u << (pi[e2] & 31);
            }
            VF_B(ix->lbits.ensure(bits.size() * 4));
            VF_B(cudaMemcpy(ix->lbits.p, bits.data(), bits.size() * 4, cudaMemcpyHostToDevice));
            VF_B(ix->lbit_slot.ensure(slot.size() * 2));
            VF_B(cudaMemcpy(ix->lbit_slot.p, slot.data(), slot.size() * 2, cudaMemcpyHostToDevice));
        }
    }
    if (!owner.empty()) {
        VF_B(ix->owner_dev.ensure(owner.size() * 4));
        VF_B(cudaMemcpy(ix->owner_dev.p, owner.data(), owner.size() * 4, cudaMemcpyHostToDevice));
    }
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
    D.lbits = n_bitmaps ? ix->lbits.as<uint32_t>() : nullptr;
    D.lbit_slot = n_bitmaps ? ix->lbit_slot.as<int16_t>() : nullptr;
    D.lbit_words = lbit_words;
    D.lsig = ix->lsig.as<unsigned long long>();
    D.owner = owner.empty() ? nullptr : ix->owner_dev.as<int32_t>();
    D.rank = rank;
    D.world = world;
    D.xn = tc_rows && !enc8 ? ix->xn.as<uint32_t>() : nullptr;
    D.xn_ls = tc_rows && !enc8 ? ix->xn_ls.as<uint32_t>() : nullptr;
    ix->enc8 = enc8;
    if (enc8) {                 // the u8 view: same directory / graphs / maps, u8 rows
        DevIndex &E = ix->dev8;
        E = D;
        E.dtype = VF_U8;
        E.row_bytes = row_bytes8;
        E.chunks = row_bytes8 / 16;
        E.X = ix->X8.as<uint8_t>();
        E.Xls = ix->Xls8.as<uint8_t>();
        E.xn = tc_rows ? ix->xn.as<uint32_t>() : nullptr;
        E.xn_ls = tc_rows ? ix->xn_ls.as<uint32_t>() : nullptr;
    }
    ix->scan_tc = tc_rows && scan_tc_encode(enc8 ? ix->dev8 : D, ls_rows_pad, ix->tm_ls, ix->tm_x);
    // query range check of the fast path (chk_hi < chk_lo: none)
    ix->chk_lo = enc8 ? 0.f : ix->scan_tc && d->dtype == VF_F32 ? -vmax : 1.f;
    ix->chk_hi = enc8 ? 255.f : ix->scan_tc && d->dtype == VF_F32 ? vmax : 0.f;
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
    I.bytes_predicate = (N + 1) * 8 + n_entries * 4 + (n_bitmaps ? n_bitmaps * lbit_words * 4 + (int64_t)L * 2 : 0) +
                        N * 8;   // + label signatures
    I.bytes_directory = (int64_t)L * sizeof(LabelDir) + (owner.empty() ? 0 : (int64_t)L * 4);
    I.bytes_norms = tc_rows ? (N + (int64_t)m_ls.size()) * 4 : 0;
    I.bytes_u8_store = enc8 ? (N + ls_rows_pad) * row_bytes8 : 0;
    I.bytes_total = I.bytes_vectors + I.bytes_graph + I.bytes_map_hs + I.bytes_ls_vectors + I.bytes_map_ls +
                    I.bytes_predicate + I.bytes_directory + I.bytes_norms + I.bytes_u8_store;
    I.world_size = world;
    I.rank = rank;
    I.owned_labels = n_hs + n_ls;
    *out = ix;
    return VF_OK;
#undef VF_B
}

static std::vector<int64_t> label_sizes(const vf_build_desc *d) {
    std::vector<int64_t> sz(d->n_labels);
    for (int l = 0; l < d->n_labels; l++) sz[l] = d->posting_offsets[l + 1] - d->posting_offsets[l];
    return sz;
}

extern "C" vf_status vf_build_index(const vf_build_desc *d, vf_index **out) {
    if (!out) return fail(VF_ERR_INVALID_ARG, "out is NULL");
    *out = nullptr;
    vf_status st = validate_desc(d);
    if (st != VF_OK) return st;
    const int world = d->world_size < 1 ? 1 : d->world_size;
    if (world > kMaxWorld) return fail(VF_ERR_INVALID_ARG, "world_size must be <= 16");
    if (world == 1) return build_one(d, 1, 0, {}, out);
    if (d->rank < 0 || d->rank >= world) return fail(VF_ERR_INVALID_ARG, "rank out of range");
    if (!d->nccl_unique_id) return fail(VF_ERR_INVALID_ARG, "world_size > 1 needs nccl_unique_id");
    std::vector<int64_t> sz = label_sizes(d);
    std::vector<int32_t> owner(std::max(d->n_labels, 1));
    shard_partition(d->n_labels, sz.data(), world, owner.data());
    owner.resize(d->n_labels);
    vf_index *ix = nullptr;
    st = build_one(d, world, d->rank, owner, &ix);
    if (st != VF_OK) return st;
    st = nccl_transport_create(d->nccl_unique_id, world, d->rank, &ix->transport);
    if (st != VF_OK) {
        delete ix;
        return st;
    }
    *out = ix;
    return VF_OK;
}

extern "C" vf_status vf_build_index_virtual_shards(const vf_build_desc *d, int32_t n_shards, vf_index **out) {
    if (!out) return fail(VF_ERR_INVALID_ARG, "out is NULL");
    *out = nullptr;
    vf_status st = validate_desc(d);
    if (st != VF_OK) return st;
    if (n_shards < 1 || n_shards > kMaxWorld) return fail(VF_ERR_INVALID_ARG, "n_shards must be in [1, 16]");
    std::vector<int64_t> sz = label_sizes(d);
    std::vector<int32_t> owner(std::max(d->n_labels, 1));
    shard_partition(d->n_labels, sz.data(), n_shards, owner.data());
    owner.resize(d->n_labels);
    vf_index *parent = new vf_index();
    parent->device = d->device;
    parent->world = n_shards;
    parent->owner = owner;
    for (int r = 0; r < n_shards; r++) {
        vf_index *sh = nullptr;
        st = build_one(d, n_shards, r, owner, &sh);
        if (st != VF_OK) {
            delete parent;
            return st;
        }
        parent->vshards.push_back(sh);
    }
    st = loopback_transport_create(&parent->transport);
    if (st != VF_OK) {
        delete parent;
        return st;
    }
    parent->info = parent->vshards[0]->info;
    parent->info.owned_labels = 0;
    parent->info.bytes_total = 0;
    for (vf_index *sh : parent->vshards) {
        parent->info.owned_labels += sh->info.owned_labels;
        parent->info.bytes_total += sh->info.bytes_total;
    }
    parent->dev = parent->vshards[0]->dev;
    *out = parent;
    return VF_OK;
}

extern "C" vf_status vf_partition_labels(int32_t n_labels, const int64_t *sizes, int32_t world, int32_t *owner) {
    if (n_labels < 0 || (n_labels > 0 && (!sizes || !owner))) return fail(VF_ERR_INVALID_ARG, "NULL argument");
    if (world < 1 || world > kMaxWorld) return fail(VF_ERR_INVALID_ARG, "world must be in [1, 16]");
    return shard_partition(n_labels, sizes, world, owner);
}

extern "C" vf_status vf_get_index_info(const vf_index *index, vf_index_info *info) {
    if (!index || !info) return fail(VF_ERR_INVALID_ARG, "NULL argument");
    *info = index->info;
    return VF_OK;
}

extern "C" vf_status vf_set_profiling(vf_index *index, int32_t enable) {
    if (!index) return fail(VF_ERR_INVALID_ARG, "NULL index");
    index->profiling = enable != 0;
    for (vf_index *s : index->vshards) s->profiling = enable != 0;
    // (re)enabling starts a new averaging window on every stream's scratch
    auto reset = [](vf_index *ix) {
        std::lock_guard<std::mutex> g(ix->mu);
        for (auto &kv : ix->scratch) kv.second->prof_first = kv.second->prof_n;
    };
    reset(index);
    for (vf_index *s : index->vshards) reset(s);
    return VF_OK;
}

// ------------------------------------------------------------------ search (Alg. 2)
namespace vf {

// Visited-set geometry of one beam search: a shared-memory table within ~7 KB per warp and an exact
// global overflow table large enough for every vertex the search can visit.
void beam_sizes(int itopk, int w, int R, int n_init, int max_iter, int *hash_slots, uint64_t *gslots,
                int warp_bytes) {
    // the visited table takes what the Top buffers leave of the warp's budget, in 32-slot steps
    // (any count: slots are found by multiply-high, kernels/graph_item.cuh), at least 1,024 slots,
    // at most 64 * itopk or 8,192
    const int64_t budget = (int64_t)warp_bytes - 16ll * itopk - 1024;
    int hs = (int)std::min<int64_t>(std::min<int64_t>(64ll * itopk, 8192), std::max<int64_t>(1024, budget / 4));
    hs = std::max(1024, hs & ~31);
    const int64_t v_bound = (int64_t)n_init + (int64_t)max_iter * w * R + 32;
    *hash_slots = hs;
    *gslots = pow2ceil((uint64_t)(2 * v_bound + 64));
}

static bool getenv_pack() {          // read per search (A/B tests toggle it)
    const char *e = getenv("VF_PACK");
    return e ? atoi(e) != 0 : true;
}

int graph_warp_kb_default(int itopk) { return itopk >= 128 ? 7 : 7; }

vf_status plan_search(vf_index *ix, Scratch *sc, int64_t n, int64_t n_slots, const vf_search_params *p,
                      cudaStream_t s, Plan *out) {
    const DevIndex &D = ix->dev;
    const int R = D.R, k = p->k;
    const int w = p->search_width < 1 ? 1 : p->search_width;
    // labels the scan may stream: LS lists, or every list in exact mode / with f3 AND routing
    // labels the scan may stream: LS lists; every list in exact mode / with T' > T; with f3 AND
    // routing an HS l* whose AND set is estimated below the threshold: est >= |C_l*|^2 / N (the
    // other labels are at least as large), so |C_l*| < sqrt(threshold * N) bounds those lists
    int scan_max = ix->max_ls_size;
    if (p->exact || p->scan_threshold > D.T) {
        scan_max = ix->max_label_size;
    } else if (p->and_scan_threshold > 0) {
        const double b = std::ceil(std::sqrt((double)p->and_scan_threshold * (double)D.n_points)) + 1.0;
        scan_max = std::max(scan_max, (int)std::min<double>(ix->max_label_size, b));
    }
    // row tiles: small in the normal path (load balance across SMs; a label split over several
    // tiles is finalised in-kernel), large in exact mode (<= 256 tiles per label)
    // (the tensor-core scan finalises a label split over tiles with a grid-wide fence and a merge,
    // which costs more than its streaming loses to imbalance: whole LS labels per tile there)
    int tile_rows = p->exact ? 4096 : (ix->scan_tc ? 2048 : 512);
    if (!p->exact) {
        static const int env_tile = [] { const char *e = getenv("VF_TILE_ROWS"); return e ? atoi(e) : 0; }();
        if (env_tile >= 64) tile_rows = env_tile & ~63;   // experiment knob (scripts/ab.py)
    }
    if ((scan_max + 255) / 256 > tile_rows) tile_rows = (((scan_max + 255) / 256) + 63) & ~63;  // x64 rows
    const int mtpl = std::max(1, (scan_max + tile_rows - 1) / tile_rows);
    Plan &pl = *out;
    pl = Plan();
    pl.n_slots = n_slots;
    pl.multi = mtpl > 1;
    // segments must fit every scan kernel that may run: the fast one (tensor-core scan, on the u8
    // view when enc8) and, when a query-range check is active, k_scan on the fp32 rows (a batch
    // with a query outside the exact range falls back to it on the device)
    const DevIndex &F = ix->enc8 ? ix->dev8 : D;
    const int tc_qg = ix->scan_tc ? scan_tc_qg(F.row_bytes, k) : 0;
    pl.tc = tc_qg > 0;
    pl.checked = ix->chk_hi >= ix->chk_lo;
    pl.qg = pl.tc ? tc_qg : scan_qg(F.row_bytes, k);
    if (pl.checked) pl.qg = std::min(pl.qg, scan_qg(D.row_bytes, k));
    const int64_t slots = std::max<int64_t>(n_slots, 1);
    pl.max_tiles = slots * mtpl;
    const int n_init = p->n_init > 0 ? p->n_init : R * w;
    const int max_iter = p->max_iterations > 0 ? p->max_iterations : 2 * ((p->itopk + w - 1) / w) + 16;
    int hs = 0;
    uint64_t gslots = 0;
    // per-warp shared memory of the batched graph kernel: the visited table takes what the Top
    // buffers leave; more bytes per warp = fewer visited ids spilling to the global table (long
    // searches) but fewer resident warps (VF_GRAPH_WARP_KB, read per search)
    const char *wk = getenv("VF_GRAPH_WARP_KB");
    const int warp_kb = wk ? std::max(4, atoi(wk)) : graph_warp_kb_default(p->itopk);
    beam_sizes(p->itopk, w, R, n_init, max_iter, &hs, &gslots, warp_kb * 1024);

    SearchArgs &a = pl.a;
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
    a.and_scan_thr = p->and_scan_threshold;
    a.scan_thr = std::max(D.T, p->scan_threshold);
    a.tile_rows = tile_rows;
    {
        // f3-only segments (every tile pre-filtered): VF_F3_TILE rows per tile (read per search)
        const char *e = getenv("VF_F3_TILE");
        const int f3t = e ? atoi(e) : kF3TileRows;
        a.tile_rows_f3 = std::max(tile_rows, f3t >= 64 ? (f3t & ~63) : tile_rows);
    }
    a.max_tiles_per_label = mtpl;
    a.max_tiles = (int32_t)std::min<int64_t>(pl.max_tiles, INT32_MAX);
    a.hash_slots = hs;
    a.gtab_slots = (int64_t)gslots;
    a.chk_lo = ix->chk_lo;
    a.chk_hi = ix->chk_hi;
    a.q8 = nullptr;
    a.q8_row_bytes = ix->enc8 ? ix->dev8.row_bytes : 0;
    a.gate = 0;
    // AND items are pre-filtered for the tensor-core scan (k_and_filter); the survivor
    // pool is sized per search, overflow is exact (the scan then verifies by itself)
    pl.filter = pl.tc && p->op == VF_AND;
    a.pool = nullptr;
    a.pool_bits = nullptr;
    a.pool_norm = nullptr;
    a.tc_xn = F.xn;
    a.tc_xn_ls = F.xn_ls;
    a.pool_cap = 0;
    a.filt_list = nullptr;
    a.n_slots = n_slots;
    a.max_nl = ix->world > 1 ? kRecLabels : kMaxQueryLabels;
    a.pack_list = nullptr;
    a.pack_max_nq = 0;
    a.pack_group = 0;
    a.packq_base = 0;
    {
        const char *e = getenv("VF_TC_PARTS");
        a.tc_parts = e ? atoi(e) : 1;
        const char *kn = getenv("VF_KNOBS");
        a.knobs = kn ? (int32_t)strtol(kn, nullptr, 0) : kDefaultKnobs;
    }
    pl.graph_ctas = graph_max_ctas(a);
    if (pl.graph_ctas <= 0) return fail(VF_ERR_INTERNAL, "no graph kernel for this row size");
    size_t nwarp = (size_t)pl.graph_ctas * kWarpsPerGraphCta;
    if (ix->enc8) {
        SearchArgs a8 = a;
        a8.ix = ix->dev8;
        pl.graph_ctas8 = graph_max_ctas(a8);
        if (pl.graph_ctas8 <= 0) return fail(VF_ERR_INTERNAL, "no graph kernel for the u8 row size");
        nwarp = std::max(nwarp, (size_t)pl.graph_ctas8 * kWarpsPerGraphCta);
    }

    bool fresh = false;
    VF_CUDA(sc->Qp.ensure((size_t)std::max<int64_t>(n, 1) * D.row_bytes));
    if (pl.filter || (pl.tc && getenv_pack())) {
        int64_t cap = 64ll << 20;                       // 256 MB of survivor ids + 512 MB of pass bits
        if (const char *e = getenv("VF_POOL_CAP")) cap = std::max<int64_t>(1, atoll(e));   // overflow tests
        VF_CUDA(sc->pool.ensure((size_t)cap * 4));
        VF_CUDA(sc->pool_bits.ensure((size_t)cap * 8));
        VF_CUDA(sc->pool_norm.ensure((size_t)cap * 4));
        a.pool = sc->pool.as<int32_t>();
        a.pool_bits = sc->pool_bits.as<unsigned long long>();
        a.pool_norm = F.xn ? sc->pool_norm.as<uint32_t>() : nullptr;
        a.pool_cap = (int32_t)cap;
        if (pl.filter) {
            VF_CUDA(sc->filt_list.ensure((size_t)std::max<int64_t>(pl.max_tiles, 1) * 4));
            a.filt_list = sc->filt_list.as<int32_t>();
        }
    }
    if (ix->enc8) {
        VF_CUDA(sc->Q8.ensure((size_t)std::max<int64_t>(n, 1) * ix->dev8.row_bytes));
        a.q8 = sc->Q8.as<uint8_t>();
    }
    VF_CUDA(sc->qoff.ensure((size_t)(n + 1) * 8));
    VF_CUDA(sc->qlab.ensure((size_t)slots * 4));
    VF_CUDA(sc->qinfo.ensure((size_t)std::max<int64_t>(n, 1) * sizeof(QueryInfo)));
    VF_CUDA(sc->items.ensure((size_t)slots * sizeof(Item)));
    VF_CUDA(sc->item_ctr.ensure((size_t)slots * 12));
    VF_CUDA(sc->graph_list.ensure((size_t)slots * kGraphClasses * 4));
    VF_CUDA(sc->scan_slots.ensure((size_t)slots * 4));
    // tile packing (k_pack; VF_PACK=0 off): small single-tile segments of the tensor-core scan
    pl.pack = pl.tc && getenv_pack() && pl.a.pool != nullptr;
    VF_CUDA(sc->scan_q.ensure((size_t)slots * (pl.pack ? 2 : 1) * sizeof(ScanQuery)));
    VF_CUDA(sc->segs.ensure((size_t)slots * sizeof(Segment)));
    VF_CUDA(sc->tiles.ensure((size_t)(pl.max_tiles + (pl.pack ? slots : 0)) * sizeof(Tile)));
    if (pl.pack) {
        VF_CUDA(sc->pack_list.ensure((size_t)slots * 4));
        a.pack_list = sc->pack_list.as<int32_t>();
        a.pack_max_nq = std::max(1, pl.qg / 8);                 // segments of <= qg/8 queries
        a.pack_group = std::min(16, pl.qg / a.pack_max_nq);     // <= qg queries per packed tile
        a.packq_base = slots;
    }
    VF_CUDA(sc->item_seg.ensure((size_t)slots * 4));
    VF_CUDA(sc->item_res.ensure((size_t)slots * k * 8));
    if (pl.multi) VF_CUDA(sc->partials.ensure((size_t)slots * a.max_tiles_per_label * k * 8));
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
    a.gtab_slots = (int64_t)sc->gtab_slots;   // the kernels index the tables with the allocated geometry
    a.n_warp_slots = (int32_t)sc->gtab_warps;
    if (!sc->ev_ok) {
        for (auto &set : sc->evs)
            for (auto &e : set) VF_CUDA(cudaEventCreate(&e));
        sc->ev_ok = true;
    }
    sc->ev = sc->evs[sc->prof_n % Scratch::kProfRing];
    a.Qp = sc->Qp.as<uint8_t>();
    a.q_off = sc->qoff.as<int64_t>();
    a.qlab = sc->qlab.as<int32_t>();
    a.qlab_in = nullptr;
    a.qinfo = sc->qinfo.as<QueryInfo>();
    a.items = sc->items.as<Item>();
    a.item_ctr = sc->item_ctr.as<int32_t>();
    a.ls_count = sc->ls_count.as<int32_t>();
    a.ls_segbase = sc->ls_segbase.as<int32_t>();
    a.ls_itembase = sc->ls_itembase.as<int32_t>();
    a.graph_list = sc->graph_list.as<int32_t>();
    a.graph_stride = slots;
    a.scan_slots = sc->scan_slots.as<int32_t>();
    a.scan_q = sc->scan_q.as<ScanQuery>();
    a.segs = sc->segs.as<Segment>();
    a.tiles = sc->tiles.as<Tile>();
    a.tile_cls = nullptr;
    if (pl.tc) {
        VF_CUDA(sc->tile_cls.ensure((size_t)kTileClasses * (size_t)std::max<int64_t>(a.max_tiles, 1) * 4));
        a.tile_cls = sc->tile_cls.as<int32_t>();
    }
    a.item_seg = sc->item_seg.as<int32_t>();
    a.item_res = sc->item_res.as<unsigned long long>();
    a.partials = pl.multi ? sc->partials.as<unsigned long long>() : nullptr;
    a.ctr = sc->ctr.as<Counters>();
    a.gtab = sc->gtab.as<unsigned long long>();
    return VF_OK;
}

static inline int D_dtype(const vf_index *ix) { return ix->dev.dtype; }

vf_status run_local(vf_index *ix, Scratch *sc, Plan &pl, cudaStream_t s, const uint8_t *recv, int64_t n_recv,
                    int rec_bytes, int *launches) {
    vf_status st = run_route(ix, sc, pl, s, recv, n_recv, rec_bytes, launches);
    if (st != VF_OK) return st;
    return run_compute(ix, sc, pl, s, launches);
}

// a1: routing (items, graph lists); the bucketing and pre-filter of the scan items run in
// run_compute, concurrently with the graph kernels
vf_status run_route(vf_index *ix, Scratch *sc, Plan &pl, cudaStream_t s, const uint8_t *recv, int64_t n_recv,
                    int rec_bytes, int *launches) {
    SearchArgs &a = pl.a;
    const bool prof = ix->profiling;
    VF_CUDA(cudaMemsetAsync(sc->ctr.p, 0, sizeof(Counters), s));
    if (prof) VF_CUDA(cudaEventRecord(sc->ev[1], s));
    int nl = 0;
    if (recv) {
        nl += launch_unpack_items(a, s, recv, n_recv, rec_bytes);
    } else {
        if (pl.clear_items && pl.n_slots > 0) VF_CUDA(cudaMemsetAsync(a.items, 0, (size_t)pl.n_slots * sizeof(Item), s));
        nl += launch_prepare(a, s);
    }
    if (prof) VF_CUDA(cudaEventRecord(sc->ev[2], s));
    VF_CUDA(cudaGetLastError());
    *launches += nl;
    return VF_OK;
}

// a2 / a3: the scan and graph kernels of the routed items (concurrently, on forked streams)
vf_status run_compute(vf_index *ix, Scratch *sc, Plan &pl, cudaStream_t s, int *launches) {
    SearchArgs &a = pl.a;
    const bool prof = ix->profiling;
    int nl = 0;
    const int tb = (int)std::min<int64_t>(pl.max_tiles, INT32_MAX);
    // scan and graph items are independent (Alg. 2 L418 / L428): the graph kernels run on a side
    // stream concurrently with the scan; graph CTAs take whatever each SM has left and pull items
    // dynamically. VF_OVERLAP=0 serialises them (A/B knobs: VF_TC_CTAS, VF_GRAPH_FIRST,
    // VF_GRAPH_PER_SM; scripts/ab_overlap.sh).
    // VF_OVERLAP (read per search): 1 always, 0 never, 2 (default) unless the f3 threshold makes the
    // AND pre-filter heavy (>= kOverlapMaxF3): the persistent graph CTAs fill the SMs first and the
    // pre-filter, which the scan waits for, would run in their leftovers (profiles/r02ss)
    const char *ov_e = getenv("VF_OVERLAP");
    const int ov_mode = ov_e ? atoi(ov_e) : 2;
    const int overlap_env = ov_mode == 2 ? (a.and_scan_thr < kOverlapMaxF3 ? 1 : 0) : ov_mode;
    static const int tc_ctas_env = [] { const char *e = getenv("VF_TC_CTAS"); return e ? atoi(e) : 2; }();
    const bool overlap = overlap_env != 0 && pl.tc;
    // Both become runnable at the fork; the scan goes on a high-priority stream so the block
    // scheduler always places the scan CTAs first (otherwise whichever kernel wins the race takes
    // the SMs and step times become bimodal).
    cudaStream_t gs = s, ss = s;
    if (overlap) {
        if (!sc->side) {
            int lo = 0, hi = 0;
            VF_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
            VF_CUDA(cudaStreamCreateWithFlags(&sc->side, cudaStreamNonBlocking));
            VF_CUDA(cudaStreamCreateWithPriority(&sc->side_hi, cudaStreamNonBlocking, hi));
            VF_CUDA(cudaEventCreateWithFlags(&sc->ev_fork, cudaEventDisableTiming));
            VF_CUDA(cudaEventCreateWithFlags(&sc->ev_join, cudaEventDisableTiming));
            VF_CUDA(cudaEventCreateWithFlags(&sc->ev_join2, cudaEventDisableTiming));
        }
        VF_CUDA(cudaEventRecord(sc->ev_fork, s));
        VF_CUDA(cudaStreamWaitEvent(sc->side_hi, sc->ev_fork, 0));
        VF_CUDA(cudaStreamWaitEvent(sc->side, sc->ev_fork, 0));
        gs = sc->side;
        ss = sc->side_hi;
    }
    // Fast kernels gated on "no query outside the exact range" (gate 1), the fp32 FFMA kernels on
    // the opposite (gate 2); without a range check only the fast set runs (gate 0).
    SearchArgs fast = a, slow = a;
    if (ix->enc8) {
        fast.ix = ix->dev8;
        fast.Qp = sc->Q8.as<uint8_t>();
        fast.q8 = nullptr;
    }
    fast.gate = pl.checked ? 1 : 0;
    slow.gate = 2;
    // read per search (A/B: scripts/ab_env.py)
    const char *gf_e = getenv("VF_GRAPH_FIRST"), *gps_e = getenv("VF_GRAPH_PER_SM");
    const int graph_first_env = gf_e ? atoi(gf_e) : 0;
    const int graph_per_sm_env = gps_e ? atoi(gps_e) : 0;
    auto launch_scans = [&]() -> int {
        int sl = pl.tc ? launch_scan_tc(fast, ss, tb, ix->tm_ls, ix->tm_x, overlap ? tc_ctas_env : 0)
                       : launch_scan(fast, ss, tb);
        if (sl >= 0 && pl.checked) {
            const int s2 = launch_scan(slow, ss, tb);
            sl = s2 < 0 ? s2 : sl + s2;
        }
        return sl;
    };
    auto launch_graphs = [&]() -> int {
        const int gb = (int)std::min<int64_t>(pl.n_slots, INT32_MAX);
        auto cap = [&](int ctas) { return overlap && graph_per_sm_env > 0 ? std::min(ctas, graph_per_sm_env * 148) : ctas; };
        int gl;
        if (ix->enc8) {
            gl = launch_graph(fast, gs, gb, cap(pl.graph_ctas8));
            const int g2 = gl < 0 ? 0 : launch_graph(slow, gs, gb, cap(pl.graph_ctas));
            gl = g2 < 0 ? g2 : gl + g2;
        } else {
            SearchArgs ga = a;
            ga.gate = 0;
            gl = launch_graph(ga, gs, gb, cap(pl.graph_ctas));
        }
        return gl;
    };
    // the scan items' bucketing, AND pre-filter and packing run on the scan stream: with overlap
    // they proceed while the graph kernels (launched first when VF_GRAPH_FIRST=1) search
    int gl = 0;
    if (overlap && graph_first_env) {
        gl = launch_graphs();
        if (gl < 0) return fail(VF_ERR_INTERNAL, "graph kernel dispatch failed");
    }
    nl += launch_bucket(a, ss, pl.n_slots, pl.qg);
    if (pl.filter) nl += launch_and_filter(a, ss);
    if (pl.pack) nl += launch_pack(a, ss);
    if (prof) VF_CUDA(cudaEventRecord(sc->ev[8], ss));
    // VF_GRAPH_AFTER=1 (read per search): the graph kernels start once the pre-filter is done, so
    // the pre-filter runs on the whole GPU and the graph search shares it with the scan instead
    const char *ga_e = getenv("VF_GRAPH_AFTER");
    if (overlap && !graph_first_env && ga_e && atoi(ga_e) == 1) {
        if (!sc->ev_filt) VF_CUDA(cudaEventCreateWithFlags(&sc->ev_filt, cudaEventDisableTiming));
        VF_CUDA(cudaEventRecord(sc->ev_filt, ss));
        VF_CUDA(cudaStreamWaitEvent(gs, sc->ev_filt, 0));
    }
    const int sl = launch_scans();
    if (sl < 0) return fail(VF_ERR_INTERNAL, "scan kernel dispatch failed");
    nl += sl;
    if (prof) VF_CUDA(cudaEventRecord(sc->ev[3], ss));
    if (!(overlap && graph_first_env)) {
        gl = launch_graphs();
        if (gl < 0) return fail(VF_ERR_INTERNAL, "graph kernel dispatch failed");
    }
    nl += gl;
    if (overlap) {
        if (prof) VF_CUDA(cudaEventRecord(sc->ev[7], gs));     // graph phase end (side stream)
        VF_CUDA(cudaEventRecord(sc->ev_join, gs));
        VF_CUDA(cudaEventRecord(sc->ev_join2, ss));
        VF_CUDA(cudaStreamWaitEvent(s, sc->ev_join, 0));
        VF_CUDA(cudaStreamWaitEvent(s, sc->ev_join2, 0));
    }
    sc->overlapped = overlap;
    if (prof) sc->evov[sc->prof_n % Scratch::kProfRing] = overlap;
    if (prof) VF_CUDA(cudaEventRecord(sc->ev[4], s));
    VF_CUDA(cudaGetLastError());
    *launches += nl;
    return VF_OK;
}

// Small batches take the per-query path (f1, small.cu) unless VF_SMALL_BATCH=0; VF_SMALL_BATCH=<n>
// sets the largest batch that takes it (default kSmallMaxBatch).
static bool use_small_path(vf_index *ix, const vf_search_params *p, int64_t n) {
    static const int limit = [] {
        const char *e = getenv("VF_SMALL_BATCH");
        return e ? atoi(e) : kSmallMaxBatch;
    }();
    if (n <= 0 || n > limit || ix->world > 1) return false;
    const DevIndex &F = ix->enc8 ? ix->dev8 : ix->dev;
    return small_supported(F, ix->dev, ix->enc8, p->k);
}

static vf_status check_params(vf_index *ix, const vf_search_params *p) {
    if (!p) return fail(VF_ERR_INVALID_ARG, "params is NULL");
    if (p->k < 1 || p->k > kMaxK) return fail(VF_ERR_INVALID_ARG, "k must be in [1, 256]");
    if (p->itopk < p->k || p->itopk > kMaxItopk) return fail(VF_ERR_INVALID_ARG, "itopk must be in [k, 1024]");
    const int w = p->search_width < 1 ? 1 : p->search_width;
    if (w * ix->dev.R > 64) return fail(VF_ERR_INVALID_ARG, "search_width * R must be <= 64");
    if (p->op < 0 || p->op > 2) return fail(VF_ERR_INVALID_ARG, "op must be VF_SINGLE, VF_OR or VF_AND");
    if (p->recall_mode < 0 || p->recall_mode > 1) return fail(VF_ERR_INVALID_ARG, "bad recall_mode");
    return VF_OK;
}

}  // namespace vf

extern "C" vf_status vf_search(vf_index *ix, const void *queries, int64_t n, const int64_t *qoff,
                               const int32_t *qlab, const vf_search_params *p, int32_t *out_ids,
                               float *out_dists, void *cuda_stream) {
    if (!ix) return fail(VF_ERR_INVALID_ARG, "index is NULL");
    vf_status st = check_params(ix, p);
    if (st != VF_OK) return st;
    if (n < 0) return fail(VF_ERR_INVALID_ARG, "n_queries < 0");
    if (n > 0 && (!queries || !qoff || !out_ids || !out_dists))
        return fail(VF_ERR_INVALID_ARG, "NULL queries / offsets / outputs");
    VF_CUDA(cudaSetDevice(ix->device));
    cudaStream_t s = (cudaStream_t)cuda_stream;
    const int64_t n_max_labels = ix->world > 1 ? kRecLabels : kMaxQueryLabels;

    const bool off_dev = is_device_ptr(qoff);
    const bool lab_dev = is_device_ptr(qlab);
    if (n > 0 && !off_dev) {
        if (qoff[0] != 0) return fail(VF_ERR_INVALID_ARG, "qlabel_offsets[0] must be 0");
        for (int64_t i = 0; i < n; i++) {
            const int64_t c = qoff[i + 1] - qoff[i];
            if (c < 0 || c > n_max_labels)
                return fail(VF_ERR_INVALID_ARG, "query " + std::to_string(i) + " has a bad label count (max " +
                                                    std::to_string(n_max_labels) + ")");
            if (p->op == VF_SINGLE && c > 1 && !lab_dev) {
                for (int64_t e = qoff[i] + 1; e < qoff[i + 1]; e++)
                    if (qlab[e] != qlab[qoff[i]])
                        return fail(VF_ERR_INVALID_ARG, "VF_SINGLE query " + std::to_string(i) + " has more than one label");
            }
        }
    }
    // -- label-sharded index: virtual shards on this device (loopback) or one rank of an NCCL group
    if (ix->world > 1) {
        std::vector<vf_index *> shards;
        std::vector<const void *> qs;
        std::vector<int64_t> nq;
        std::vector<const int64_t *> qo;
        std::vector<const int32_t *> ql;
        std::vector<int32_t *> oi;
        std::vector<float *> od;
        if (!ix->vshards.empty()) {
            // the caller's batch is split into contiguous chunks, one per virtual origin rank
            if (n > 0 && (off_dev || lab_dev || is_device_ptr(queries) || is_device_ptr(out_ids)))
                return fail(VF_ERR_INVALID_ARG, "virtual shards take host query / result buffers");
            const int W = (int)ix->vshards.size();
            const size_t qbytes = (size_t)ix->dev.dim * elem_size(ix->dev.dtype);
            for (int r = 0; r < W; r++) {
                const int64_t lo = n * r / W, hi = n * (r + 1) / W;
                shards.push_back(ix->vshards[r]);
                qs.push_back(static_cast<const uint8_t *>(queries) + lo * qbytes);
                nq.push_back(hi - lo);
                qo.push_back(qoff + lo);
                ql.push_back(qlab);
                oi.push_back(out_ids + lo * p->k);
                od.push_back(out_dists + lo * p->k);
            }
        } else {
            shards.push_back(ix);
            qs.push_back(queries);
            nq.push_back(n);
            qo.push_back(qoff);
            ql.push_back(qlab);
            oi.push_back(out_ids);
            od.push_back(out_dists);
        }
        return sharded_search(shards, qs, nq, qo, ql, p, oi, od, ix->transport, s);
    }
    if (n == 0) return VF_OK;

    Scratch *sc = get_scratch(ix, s, 0);
    const DevIndex &D = ix->dev;
    const int k = p->k;
    const bool q_dev = is_device_ptr(queries);
    const bool out_dev = is_device_ptr(out_ids);
    if (out_dev != is_device_ptr(out_dists))
        return fail(VF_ERR_INVALID_ARG, "out_ids and out_dists must both be host or both be device");
    int64_t n_slots = 0;
    if (!off_dev) {
        n_slots = qoff[n];
    } else if (p->n_query_labels > 0) {
        n_slots = p->n_query_labels;             // the caller's label-array length (no sync)
    } else {
        VF_CUDA(cudaMemcpyAsync(&n_slots, qoff + n, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
        VF_CUDA(cudaStreamSynchronize(s));
    }
    if (n_slots > 0 && !qlab) return fail(VF_ERR_INVALID_ARG, "qlabels is NULL");
    if (n_slots >= (1ll << 31)) return fail(VF_ERR_INVALID_ARG, "too many query labels");

    Plan pl;
    st = plan_search(ix, sc, n, n_slots, p, s, &pl);
    if (st != VF_OK) return st;
    pl.clear_items = off_dev;
    SearchArgs &a = pl.a;
    const int raw_bytes = D.dim * elem_size(D.dtype);
    if (!q_dev) VF_CUDA(sc->raw.ensure((size_t)n * raw_bytes));
    if (!out_dev) {
        VF_CUDA(sc->out_ids.ensure((size_t)n * k * 4));
        VF_CUDA(sc->out_dists.ensure((size_t)n * k * 4));
    }
    const bool prof = ix->profiling;
    if (prof) VF_CUDA(cudaEventRecord(sc->ev[0], s));
    // -- inputs to the device
    if (!q_dev) VF_CUDA(cudaMemcpyAsync(sc->raw.p, queries, (size_t)n * raw_bytes, cudaMemcpyHostToDevice, s));
    if (off_dev) a.q_off = qoff;
    else VF_CUDA(cudaMemcpyAsync(sc->qoff.p, qoff, (size_t)(n + 1) * 8, cudaMemcpyHostToDevice, s));
    // f1 per-query path (small.cu): small batches are answered by one launch, one CTA per query
    const bool small_path = use_small_path(ix, p, n);
    // host labels are copied in; device labels are read in place by the per-query path and copied
    // by k_prepare itself on the batched path (no separate device-to-device copy)
    a.qlab_in = nullptr;
    if (n_slots > 0 && !lab_dev)
        VF_CUDA(cudaMemcpyAsync(sc->qlab.p, qlab, (size_t)n_slots * 4, cudaMemcpyHostToDevice, s));
    else if (n_slots > 0 && !small_path)
        a.qlab_in = qlab;
    a.Qraw = q_dev ? reinterpret_cast<const uint8_t *>(queries) : sc->raw.as<uint8_t>();
    a.out_ids = out_dev ? out_ids : sc->out_ids.as<int32_t>();
    a.out_dists = out_dev ? out_dists : sc->out_dists.as<float>();

    int launches = 0;
    if (small_path) {
        SearchArgs f = a;
        if (ix->enc8) f.ix = ix->dev8;
        {   // the per-query path keeps the default 7 KB per warp (its CTAs also hold row stages)
            uint64_t gs_ = 0;
            beam_sizes(p->itopk, f.w, D.R, f.n_init, f.max_iter, &f.hash_slots, &gs_, 7168);
        }
        if (lab_dev) f.qlab = const_cast<int32_t *>(qlab);
        VF_CUDA(cudaMemsetAsync(sc->ctr.p, 0, sizeof(Counters), s));
        if (prof) {
            VF_CUDA(cudaEventRecord(sc->ev[1], s));
            VF_CUDA(cudaEventRecord(sc->ev[2], s));
            VF_CUDA(cudaEventRecord(sc->ev[8], s));
            VF_CUDA(cudaEventRecord(sc->ev[3], s));
        }
        // a small batch spreads each query over several CTAs (scan items split by rows, graph items
        // round robin over the CTAs' warps) so that one query can use several SMs
        const int nparts = (int)std::max<int64_t>(1, std::min<int64_t>(8, 148 / n));
        bool fresh = false;
        VF_CUDA(sc->small_part.ensure((size_t)n * nparts * kMaxQueryLabels * kSmallMaxK * 8));
        VF_CUDA(sc->small_cnt.ensure((size_t)std::max<int64_t>(n, kSmallMaxBatch) * 4 + 256, &fresh));
        if (fresh) VF_CUDA(cudaMemsetAsync(sc->small_cnt.p, 0, sc->small_cnt.n, s));
        const int l = launch_small(f, D, ix->enc8, raw_bytes, nparts, sc->small_part.as<unsigned long long>(),
                                   sc->small_cnt.as<int32_t>(), s);
        if (l < 0) return fail(VF_ERR_INTERNAL, "per-query kernel dispatch failed");
        launches += l;
        if (prof) VF_CUDA(cudaEventRecord(sc->ev[4], s));
    } else {
        st = run_local(ix, sc, pl, s, nullptr, 0, 0, &launches);
        if (st != VF_OK) return st;
        const bool need_merge = p->op == VF_OR || (p->op == VF_AND && p->recall_mode == VF_RECALL_PARALLEL);
        if (need_merge) launches += launch_merge(a, s);
    }
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
    if (prof) sc->prof_n++;
    sc->has_last = true;
    if (!out_dev) VF_CUDA(cudaStreamSynchronize(s));
    return VF_OK;
}

extern "C" vf_status vf_get_last_stats(vf_index *ix, void *cuda_stream, vf_search_stats *st) {
    if (!ix || !st) return fail(VF_ERR_INVALID_ARG, "NULL argument");
    if (!ix->vshards.empty()) ix = ix->vshards[0];
    VF_CUDA(cudaSetDevice(ix->device));
    cudaStream_t s = (cudaStream_t)cuda_stream;
    Scratch *sc = get_scratch(ix, s, 0);
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
    st->n_invalid_queries = c.n_invalid;
    st->prefilter_words = c.pool_used;
    st->kernel_launches = sc->last_launches;
    st->row_bytes = ix->enc8 && !c.exact_fallback ? ix->dev8.row_bytes : ix->dev.row_bytes;   // rows the kernels read
    auto span = [](unsigned long long t0_inv, unsigned long long t1) {
        const unsigned long long t0 = ~t0_inv;
        return (t0_inv && t1 > t0) ? (double)(t1 - t0) / 1e6 : 0.0;
    };
    st->ms_scan_active = span(c.scan_t0_inv, c.scan_t1);
    st->ms_graph_active = span(c.graph_t0_inv, c.graph_t1);
    // with scan / graph overlap the graph phase runs from the fork (ev[2]) to its own end (ev[7])
    // route = k_prepare; filter = bucket + AND pre-filter + packing; scan = the scan kernels
    auto phases = [](cudaEvent_t *e, bool ov, double *out) {
        float t;
        cudaEventElapsedTime(&t, e[1], e[2]); out[0] = t;
        cudaEventElapsedTime(&t, e[8], e[3]); out[1] = t;
        cudaEventElapsedTime(&t, e[2], e[8]); out[6] = t;
        cudaEventElapsedTime(&t, ov ? e[2] : e[3], ov ? e[7] : e[4]); out[2] = t;
        cudaEventElapsedTime(&t, e[4], e[5]); out[3] = t;
        float c0, c1;
        cudaEventElapsedTime(&c0, e[0], e[1]);
        cudaEventElapsedTime(&c1, e[5], e[6]);
        out[4] = c0 + c1;
        cudaEventElapsedTime(&t, e[0], e[6]); out[5] = t;
    };
    if (sc->profiled && sc->prof_n > 0) {
        double v[7];
        phases(sc->evs[(sc->prof_n - 1) % Scratch::kProfRing], sc->evov[(sc->prof_n - 1) % Scratch::kProfRing], v);
        st->ms_route = v[0]; st->ms_scan = v[1]; st->ms_graph = v[2];
        st->ms_merge = v[3]; st->ms_copy = v[4]; st->ms_total = v[5]; st->ms_filter = v[6];
        const int64_t lo = std::max(sc->prof_first, sc->prof_n - Scratch::kProfRing);
        double sum[7] = {0, 0, 0, 0, 0, 0, 0};
        for (int64_t i = lo; i < sc->prof_n; i++) {
            phases(sc->evs[i % Scratch::kProfRing], sc->evov[i % Scratch::kProfRing], v);
            for (int j = 0; j < 7; j++) sum[j] += v[j];
        }
        const int64_t m = sc->prof_n - lo;
        st->n_profiled = m;
        if (m > 0) {
            st->mean_ms_route = sum[0] / m; st->mean_ms_scan = sum[1] / m; st->mean_ms_graph = sum[2] / m;
            st->mean_ms_merge = sum[3] / m; st->mean_ms_copy = sum[4] / m; st->mean_ms_total = sum[5] / m;
            st->mean_ms_filter = sum[6] / m;
        }
    }
    return VF_OK;
}

extern "C" vf_status vf_get_last_items(vf_index *ix, void *cuda_stream, int64_t max_items, int32_t *rec,
                                       int64_t *n_items) {
    if (!ix || !n_items) return fail(VF_ERR_INVALID_ARG, "NULL argument");
    if (!ix->vshards.empty()) return fail(VF_ERR_INVALID_ARG, "per-item records are kept per shard");
    VF_CUDA(cudaSetDevice(ix->device));
    cudaStream_t s = (cudaStream_t)cuda_stream;
    Scratch *sc = get_scratch(ix, s, 0);
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
            const bool g = path == PATH_GRAPH && !(items[i].meta & META_REMOTE);
            r[3] = g ? ctr[i * 3 + 0] : 0;
            r[4] = g ? ctr[i * 3 + 1] : 0;
            r[5] = g ? ctr[i * 3 + 2] : 0;
        }
        m++;
    }
    *n_items = m;
    return VF_OK;
}
