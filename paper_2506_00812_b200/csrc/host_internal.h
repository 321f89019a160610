// Host-side internals shared by vf_api.cpp (index build, single-index search) and shard.cpp (label
// sharding, §8(e)). Not part of the C-ABI.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <mutex>
#include <string>
#include <unordered_map>
#include <vector>

#include "vf.h"
#include "vf_internal.h"

namespace vf {

vf_status fail(vf_status s, const std::string &m);

#define VF_CUDA(x)                                                                               \
    do {                                                                                         \
        cudaError_t e_ = (x);                                                                    \
        if (e_ != cudaSuccess) {                                                                 \
            vf_status st_ = e_ == cudaErrorMemoryAllocation ? VF_ERR_OUT_OF_MEMORY : VF_ERR_CUDA; \
            return ::vf::fail(st_, std::string(#x) + ": " + cudaGetErrorString(e_));            \
        }                                                                                        \
    } while (0)

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
    // grow to at least `bytes` (contents not preserved)
    cudaError_t ensure(size_t bytes, bool *fresh = nullptr) {
        if (fresh) *fresh = false;
        if (bytes <= n && p) return cudaSuccess;
        release();
        const size_t want = bytes < 256 ? 256 : bytes;
        cudaError_t e = cudaMalloc(&p, want);
        if (e != cudaSuccess) {
            p = nullptr;
            return e;
        }
        n = want;
        if (fresh) *fresh = true;
        return cudaSuccess;
    }
    template <class T> T *as() const { return reinterpret_cast<T *>(p); }
};

// Per-stream (and per role) scratch of a search.
struct Scratch {
    DevBuf raw, Qp, Q8, pool, pool_bits, pool_norm, filt_list, pack_list, qoff, qlab, qinfo, items, item_ctr, graph_list, scan_slots, scan_q, segs, tiles, item_seg,
        item_res, partials, ctr, out_ids, out_dists, ls_count, ls_segbase, ls_itembase, gtab;
    // label sharding: item records out / in, returned results, slots of the sent items
    DevBuf send, recv, res_ids, res_dists, back_ids, back_dists, sent_slots, dst_off;
    // per-query path (f1): per-CTA item lists of a query split over several CTAs, completion counters
    DevBuf small_part, small_cnt;
    DevBuf tile_cls;            // scan tiles by row-count class (claim order of the tensor-core scan)
    // scan / graph overlap: the graph kernels run on a side stream forked after routing
    cudaStream_t side = nullptr, side_hi = nullptr;   // graph kernels; scan kernels (high priority)
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr, ev_join2 = nullptr, ev_filt = nullptr;
    // label sharding: the exchange stream, its events and the pinned copy of the routed counters
    cudaStream_t xs = nullptr;
    cudaEvent_t ev_routed = nullptr, ev_cnt = nullptr, ev_xdone = nullptr;
    Counters *hctr = nullptr;
    size_t gtab_slots = 0, gtab_warps = 0;
    // profiled searches record their phase events into a ring: ev points at the current set, so
    // the mean over every search since profiling was enabled (<= kProfRing of them) is readable
    // without a host sync between searches
    static constexpr int kProfRing = 64;
    cudaEvent_t evs[kProfRing][9];
    cudaEvent_t *ev = evs[0];
    int64_t prof_n = 0, prof_first = 0;
    bool ev_ok = false;
    bool profiled = false;
    bool overlapped = false;        // last search ran scan and graph concurrently (phases overlap)
    bool evov[kProfRing] = {};      // per profiled search: graph phase = ev[2] -> ev[7] (side stream)
    SearchArgs last{};
    int64_t last_slots = 0;
    int last_launches = 0;
    bool has_last = false;
    ~Scratch() {
        if (ev_ok)
            for (auto &set : evs)
                for (auto &e : set) cudaEventDestroy(e);
        if (side) cudaStreamDestroy(side);
        if (side_hi) cudaStreamDestroy(side_hi);
        if (ev_fork) cudaEventDestroy(ev_fork);
        if (ev_join) cudaEventDestroy(ev_join);
        if (ev_join2) cudaEventDestroy(ev_join2);
        if (ev_filt) cudaEventDestroy(ev_filt);
        if (xs) cudaStreamDestroy(xs);
        if (ev_routed) cudaEventDestroy(ev_routed);
        if (ev_cnt) cudaEventDestroy(ev_cnt);
        if (ev_xdone) cudaEventDestroy(ev_xdone);
        if (hctr) cudaFreeHost(hctr);
    }
};

struct Transport;

struct vf_index_impl;
}  // namespace vf

struct vf_index {
    vf::DevIndex dev{};
    int device = 0;
    vf::DevBuf X, dir, G, M_hs, Xls, M_ls, pt_off, pt_lab, owner_dev, xn, xn_ls, X8, Xls8, lbits, lbit_slot, lsig;
    bool enc8 = false;                          // lossless u8 row store of integer-valued fp32 rows
    vf::DevIndex dev8{};                        // ... and the u8 view the fast kernels read
    alignas(64) unsigned char tm_ls[128];       // CUtensorMap of X_LS (tensor-core scan)
    alignas(64) unsigned char tm_x[128];        // CUtensorMap of X rows (HS gathers)
    bool scan_tc = false;                       // tensor-core scan available (for dev8 when enc8)
    float chk_lo = 1.f, chk_hi = 0.f;           // fast-path query range check (hi < lo: none)
    vf_index_info info{};
    int32_t max_ls_size = 0, max_label_size = 0;
    std::mutex mu;
    std::unordered_map<uint64_t, vf::Scratch *> scratch;   // (stream, role) -> scratch
    bool profiling = false;
    // label sharding (§8(e))
    int world = 1, rank = 0;
    std::vector<int32_t> owner;                 // [n_labels] owning rank (host copy)
    vf::Transport *transport = nullptr;         // NCCL (one rank per process) or loopback
    std::vector<vf_index *> vshards;            // virtual shards on one device (loopback transport)
    ~vf_index();
};

namespace vf {

Scratch *get_scratch(vf_index *ix, cudaStream_t s, int role);
bool is_device_ptr(const void *p);

// Plan of one search pass over a batch on one index (shard).
struct Plan {
    SearchArgs a{};
    int64_t n_slots = 0;
    int qg = 0;
    bool tc = false;          // tensor-core scan (scan_tc.cu)
    bool checked = false;     // fast path with a query-range check (fp32 fallback kernels launched too)
    bool filter = false;      // AND pre-filter of the scan tiles (k_and_filter)
    int graph_ctas8 = 0;      // graph grid on the u8 view (enc8)
    int64_t max_tiles = 0;
    int graph_ctas = 0;
    bool multi = false;
    bool pack = false;        // small scan segments packed into shared tiles (k_pack)
    bool clear_items = false; // device offsets: item slots start as PATH_NONE (a rejected query's
                              // slots are never read stale; k_prepare's device-side check)
};

// Size every scratch buffer for a batch of n queries / n_slots item slots and fill the SearchArgs
// (queries, labels and outputs are bound by the caller).
vf_status plan_search(vf_index *ix, Scratch *sc, int64_t n, int64_t n_slots, const vf_search_params *p,
                      cudaStream_t s, Plan *out);
// route (k_prepare) or unpack received items, then bucket, scan and graph for the local items
// (= run_route + run_compute).
vf_status run_local(vf_index *ix, Scratch *sc, Plan &pl, cudaStream_t s, const uint8_t *recv, int64_t n_recv,
                    int rec_bytes, int *launches);
vf_status run_route(vf_index *ix, Scratch *sc, Plan &pl, cudaStream_t s, const uint8_t *recv, int64_t n_recv,
                    int rec_bytes, int *launches);
vf_status run_compute(vf_index *ix, Scratch *sc, Plan &pl, cudaStream_t s, int *launches);

// Label sharding entry points (shard.cpp).
vf_status shard_partition(int32_t n_labels, const int64_t *sizes, int32_t world, int32_t *owner);
vf_status nccl_transport_create(const void *unique_id, int world, int rank, Transport **out);
vf_status loopback_transport_create(Transport **out);
void transport_destroy(Transport *t);
vf_status sharded_search(std::vector<vf_index *> &shards, std::vector<const void *> &queries,
                         std::vector<int64_t> &nq, std::vector<const int64_t *> &qoff,
                         std::vector<const int32_t *> &qlab, const vf_search_params *p,
                         std::vector<int32_t *> &out_ids, std::vector<float *> &out_dists, Transport *tr,
                         cudaStream_t s);

}  // namespace vf
