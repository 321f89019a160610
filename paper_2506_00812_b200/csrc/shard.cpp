// Label sharding (BASELINE.json configs[4]): labels are independent units, so an index
// is split across ranks by label -- greedy LPT over |C_l| -- with X and the predicate table
// replicated. A search has exactly one exchange step each way:
//   1. every rank routes its own queries (a1); items of labels it owns run locally (a2/a3);
//   2. items of other ranks' labels are packed as records (query row, label set, content hash)
//      and sent to their owners (grouped point-to-point, NCCL over NVLink in production);
//   3. owners run the received items as a batch of single-item queries (same kernels);
//   4. the per-item top-k lists go back to the origin, which merges per query (a5).
// Items are independent and the entry sampler keys on query content (reading #34), so any number of
// ranks returns results bit-identical to one rank. Two transports: NCCL (one rank per process,
// loaded with dlopen) and an in-process loopback over several shards on one device ("virtual
// shards"), which runs the same protocol on a single GPU for parity tests.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstring>
#include <numeric>

#include "host_internal.h"

namespace vf {

// ------------------------------------------------------------------ partition
vf_status shard_partition(int32_t L, const int64_t *sizes, int32_t world, int32_t *owner) {
    std::vector<int32_t> order(L);
    std::iota(order.begin(), order.end(), 0);
    std::stable_sort(order.begin(), order.end(), [&](int32_t a, int32_t b) { return sizes[a] > sizes[b]; });
    std::vector<int64_t> load(world, 0);
    for (int32_t l : order) {
        int best = 0;
        for (int r = 1; r < world; r++)
            if (load[r] < load[best]) best = r;
        owner[l] = best;
        load[best] += sizes[l];
    }
    return VF_OK;
}

// ------------------------------------------------------------------ transports
struct Transport {
    virtual ~Transport() {}
    virtual bool loopback() const = 0;
    virtual vf_status exchange_counts(const int64_t *send_cnt, int64_t *recv_cnt, int world, int rank,
                                      cudaStream_t s) = 0;
    virtual vf_status alltoallv(const uint8_t *send, const int64_t *soff, const int64_t *sbytes, uint8_t *recv,
                                const int64_t *roff, const int64_t *rbytes, int world, int rank, cudaStream_t s) = 0;
};

struct LoopbackTransport : Transport {
    bool loopback() const override { return true; }
    vf_status exchange_counts(const int64_t *, int64_t *, int, int, cudaStream_t) override {
        return fail(VF_ERR_INTERNAL, "loopback exchange is done across shards");
    }
    vf_status alltoallv(const uint8_t *, const int64_t *, const int64_t *, uint8_t *, const int64_t *,
                        const int64_t *, int, int, cudaStream_t) override {
        return fail(VF_ERR_INTERNAL, "loopback exchange is done across shards");
    }
};

struct NcclApi {
    void *h = nullptr;
    ncclResult_t (*commInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*send)(const void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*recv)(void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*groupStart)() = nullptr;
    ncclResult_t (*groupEnd)() = nullptr;
    const char *(*errstr)(ncclResult_t) = nullptr;
    bool load() {
        if (h) return true;
        for (const char *name : {"libnccl.so.2", "libnccl.so"}) {
            h = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
            if (h) break;
        }
        if (!h) return false;
        commInitRank = (decltype(commInitRank))dlsym(h, "ncclCommInitRank");
        commDestroy = (decltype(commDestroy))dlsym(h, "ncclCommDestroy");
        send = (decltype(send))dlsym(h, "ncclSend");
        recv = (decltype(recv))dlsym(h, "ncclRecv");
        groupStart = (decltype(groupStart))dlsym(h, "ncclGroupStart");
        groupEnd = (decltype(groupEnd))dlsym(h, "ncclGroupEnd");
        errstr = (decltype(errstr))dlsym(h, "ncclGetErrorString");
        return commInitRank && commDestroy && send && recv && groupStart && groupEnd && errstr;
    }
};
static NcclApi g_nccl;

#define VF_NCCL(x)                                                                     \
    do {                                                                               \
        ncclResult_t r_ = (x);                                                         \
        if (r_ != ncclSuccess) return fail(VF_ERR_NCCL, std::string(#x) + ": " + g_nccl.errstr(r_)); \
    } while (0)

struct NcclTransport : Transport {
    ncclComm_t comm = nullptr;
    DevBuf cnt;
    ~NcclTransport() override {
        if (comm) g_nccl.commDestroy(comm);
    }
    bool loopback() const override { return false; }
    vf_status exchange_counts(const int64_t *send_cnt, int64_t *recv_cnt, int world, int rank,
                              cudaStream_t s) override {
        VF_CUDA(cnt.ensure(2 * world * sizeof(int64_t)));
        int64_t *d = cnt.as<int64_t>();
        VF_CUDA(cudaMemcpyAsync(d, send_cnt, world * sizeof(int64_t), cudaMemcpyHostToDevice, s));
        VF_NCCL(g_nccl.groupStart());
        for (int p = 0; p < world; p++) {
            if (p == rank) continue;
            VF_NCCL(g_nccl.send(d + p, 1, ncclInt64, p, comm, s));
            VF_NCCL(g_nccl.recv(d + world + p, 1, ncclInt64, p, comm, s));
        }
        VF_NCCL(g_nccl.groupEnd());
        VF_CUDA(cudaMemcpyAsync(recv_cnt, d + world, world * sizeof(int64_t), cudaMemcpyDeviceToHost, s));
        VF_CUDA(cudaStreamSynchronize(s));
        recv_cnt[rank] = send_cnt[rank];
        return VF_OK;
    }
    vf_status alltoallv(const uint8_t *send, const int64_t *soff, const int64_t *sbytes, uint8_t *recv,
                        const int64_t *roff, const int64_t *rbytes, int world, int rank, cudaStream_t s) override {
        if (sbytes[rank] > 0)
            VF_CUDA(cudaMemcpyAsync(recv + roff[rank], send + soff[rank], sbytes[rank], cudaMemcpyDeviceToDevice, s));
        VF_NCCL(g_nccl.groupStart());
        for (int p = 0; p < world; p++) {
            if (p == rank) continue;
            if (sbytes[p] > 0) VF_NCCL(g_nccl.send(send + soff[p], sbytes[p], ncclUint8, p, comm, s));
            if (rbytes[p] > 0) VF_NCCL(g_nccl.recv(recv + roff[p], rbytes[p], ncclUint8, p, comm, s));
        }
        VF_NCCL(g_nccl.groupEnd());
        return VF_OK;
    }
};

vf_status nccl_transport_create(const void *unique_id, int world, int rank, Transport **out) {
    if (!g_nccl.load()) return fail(VF_ERR_NCCL, "cannot load libnccl.so.2");
    NcclTransport *t = new NcclTransport();
    ncclUniqueId id;
    std::memcpy(&id, unique_id, sizeof(id));
    ncclResult_t r = g_nccl.commInitRank(&t->comm, world, id, rank);
    if (r != ncclSuccess) {
        t->comm = nullptr;
        delete t;
        return fail(VF_ERR_NCCL, std::string("ncclCommInitRank: ") + g_nccl.errstr(r));
    }
    *out = t;
    return VF_OK;
}

vf_status loopback_transport_create(Transport **out) {
    *out = new LoopbackTransport();
    return VF_OK;
}

void transport_destroy(Transport *t) { delete t; }

// ------------------------------------------------------------------ the sharded search
struct ShardJob {
    vf_index *ix = nullptr;
    Scratch *own = nullptr, *exec = nullptr;
    Plan po, pe;                        // origin batch, received-items batch
    int64_t n = 0, n_slots = 0;
    bool out_dev = false;
    int32_t *out_ids = nullptr;
    float *out_dists = nullptr;
    std::vector<int64_t> send_cnt, recv_cnt, send_off, recv_off;
    int64_t n_send = 0, n_recv = 0;
};

// The exchange runs on a second stream of the origin scratch (xs) so that the local items' scan /
// graph kernels (on the caller's stream) overlap it: the only host waits are for the routed
// per-owner counts (they size the exchange) and the count exchange itself, both right after
// routing; the item records, the owners' searches and the results travel while the local
// kernels run, and the caller's stream joins the exchange stream only for the final merge.
static vf_status exchange_stream(Scratch *sc) {
    if (!sc->xs) {
        VF_CUDA(cudaStreamCreateWithFlags(&sc->xs, cudaStreamNonBlocking));
        VF_CUDA(cudaEventCreateWithFlags(&sc->ev_routed, cudaEventDisableTiming));
        VF_CUDA(cudaEventCreateWithFlags(&sc->ev_cnt, cudaEventDisableTiming));
        VF_CUDA(cudaEventCreateWithFlags(&sc->ev_xdone, cudaEventDisableTiming));
        VF_CUDA(cudaHostAlloc((void **)&sc->hctr, sizeof(Counters), cudaHostAllocDefault));
    }
    return VF_OK;
}

vf_status sharded_search(std::vector<vf_index *> &shards, std::vector<const void *> &queries,
                         std::vector<int64_t> &nq, std::vector<const int64_t *> &qoff,
                         std::vector<const int32_t *> &qlab, const vf_search_params *p,
                         std::vector<int32_t *> &out_ids, std::vector<float *> &out_dists, Transport *tr,
                         cudaStream_t s) {
    const int W = shards[0]->world;
    const int J = (int)shards.size();
    const int k = p->k;
    const DevIndex &D0 = shards[0]->dev;
    const int raw_bytes = D0.dim * (D0.dtype == VF_U8 ? 1 : 4);
    const int rec_bytes = (int)sizeof(ItemRecord) + D0.row_bytes;
    if (!tr) return fail(VF_ERR_INTERNAL, "sharded index without transport");
    std::vector<ShardJob> jobs(J);
    bool any_host_out = false;

    // ---- phase 1: every origin routes its queries; local items start on s, counts go to the host
    for (int j = 0; j < J; j++) {
        ShardJob &jb = jobs[j];
        vf_index *ix = shards[j];
        jb.ix = ix;
        jb.n = nq[j];
        jb.own = get_scratch(ix, s, 0);
        jb.exec = get_scratch(ix, s, 1);
        VF_CUDA(cudaSetDevice(ix->device));
        vf_status st = exchange_stream(jb.own);
        if (st != VF_OK) return st;
        const bool q_dev = is_device_ptr(queries[j]), off_dev = is_device_ptr(qoff[j]);
        const bool lab_dev = is_device_ptr(qlab[j]);
        jb.out_dev = is_device_ptr(out_ids[j]);
        any_host_out |= !jb.out_dev;
        jb.out_ids = out_ids[j];
        jb.out_dists = out_dists[j];
        int64_t lo = 0, hi = 0;
        if (jb.n > 0) {
            if (!off_dev) {
                lo = qoff[j][0];
                hi = qoff[j][jb.n];
            } else if (J == 1 && p->n_query_labels > 0) {
                hi = p->n_query_labels;        // device offsets of the caller's batch: qoff[0] == 0
            } else {
                VF_CUDA(cudaMemcpyAsync(&lo, qoff[j], 8, cudaMemcpyDeviceToHost, s));
                VF_CUDA(cudaMemcpyAsync(&hi, qoff[j] + jb.n, 8, cudaMemcpyDeviceToHost, s));
                VF_CUDA(cudaStreamSynchronize(s));
            }
        }
        jb.n_slots = hi - lo;
        Scratch *sc = jb.own;
        st = plan_search(ix, sc, jb.n, jb.n_slots, p, s, &jb.po);
        if (st != VF_OK) return st;
        SearchArgs &a = jb.po.a;
        VF_CUDA(sc->raw.ensure((size_t)std::max<int64_t>(jb.n, 1) * raw_bytes));
        VF_CUDA(sc->out_ids.ensure((size_t)std::max<int64_t>(jb.n, 1) * k * 4));
        VF_CUDA(sc->out_dists.ensure((size_t)std::max<int64_t>(jb.n, 1) * k * 4));
        if (jb.n > 0) {
            VF_CUDA(cudaMemcpyAsync(sc->raw.p, queries[j], (size_t)jb.n * raw_bytes,
                                    q_dev ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, s));
            if (off_dev && lo == 0) {
                VF_CUDA(cudaMemcpyAsync(sc->qoff.p, qoff[j], (jb.n + 1) * 8, cudaMemcpyDeviceToDevice, s));
            } else {
                // offsets rebased to this chunk's first label
                std::vector<int64_t> ho(jb.n + 1);
                if (off_dev) VF_CUDA(cudaMemcpy(ho.data(), qoff[j], (jb.n + 1) * 8, cudaMemcpyDeviceToHost));
                else std::memcpy(ho.data(), qoff[j], (jb.n + 1) * 8);
                for (auto &v : ho) v -= lo;
                VF_CUDA(cudaMemcpy(sc->qoff.p, ho.data(), (jb.n + 1) * 8, cudaMemcpyHostToDevice));
            }
            if (jb.n_slots > 0)
                VF_CUDA(cudaMemcpyAsync(sc->qlab.p, qlab[j] + lo, (size_t)jb.n_slots * 4,
                                        lab_dev ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, s));
        }
        a.Qraw = sc->raw.as<uint8_t>();
        a.out_ids = sc->out_ids.as<int32_t>();
        a.out_dists = sc->out_dists.as<float>();
        int launches = 0;
        if (ix->profiling) VF_CUDA(cudaEventRecord(sc->ev[0], s));
        st = run_route(ix, sc, jb.po, s, nullptr, 0, 0, &launches);
        if (st != VF_OK) return st;
        VF_CUDA(cudaEventRecord(sc->ev_routed, s));
        VF_CUDA(cudaStreamWaitEvent(sc->xs, sc->ev_routed, 0));
        VF_CUDA(cudaMemcpyAsync(sc->hctr, sc->ctr.p, sizeof(Counters), cudaMemcpyDeviceToHost, sc->xs));
        VF_CUDA(cudaEventRecord(sc->ev_cnt, sc->xs));
        st = run_compute(ix, sc, jb.po, s, &launches);       // local items, overlapping the exchange
        if (st != VF_OK) return st;
        sc->last_launches = launches;
    }
    for (auto &jb : jobs) {
        VF_CUDA(cudaEventSynchronize(jb.own->ev_cnt));
        jb.send_cnt.assign(W, 0);
        for (int r = 0; r < W; r++) jb.send_cnt[r] = jb.own->hctr->remote[r];
    }
    cudaStream_t xs = jobs[0].own->xs;       // one stream carries the exchange (per process)

    // ---- phase 2: exchange the per-destination counts
    for (int j = 0; j < J; j++) jobs[j].recv_cnt.assign(W, 0);
    if (tr->loopback()) {
        for (int src = 0; src < J; src++)
            for (int dst = 0; dst < J; dst++) jobs[dst].recv_cnt[src] = jobs[src].send_cnt[dst];
    } else {
        vf_status st = tr->exchange_counts(jobs[0].send_cnt.data(), jobs[0].recv_cnt.data(), W, shards[0]->rank, xs);
        if (st != VF_OK) return st;
    }
    for (auto &jb : jobs) {
        jb.send_off.assign(W + 1, 0);
        jb.recv_off.assign(W + 1, 0);
        for (int r = 0; r < W; r++) {
            jb.send_off[r + 1] = jb.send_off[r] + jb.send_cnt[r];
            jb.recv_off[r + 1] = jb.recv_off[r] + jb.recv_cnt[r];
        }
        jb.n_send = jb.send_off[W];
        jb.n_recv = jb.recv_off[W];
    }

    // ---- phase 3: pack the remote items and ship them to their owners (exchange stream)
    for (auto &jb : jobs) {
        Scratch *sc = jb.own;
        VF_CUDA(cudaSetDevice(jb.ix->device));
        if (jb.own->xs != xs) {           // loopback shards: every shard's exchange work on xs
            VF_CUDA(cudaEventRecord(jb.own->ev_routed, s));
            VF_CUDA(cudaStreamWaitEvent(xs, jb.own->ev_routed, 0));
        }
        VF_CUDA(sc->send.ensure((size_t)std::max<int64_t>(jb.n_send, 1) * rec_bytes));
        VF_CUDA(sc->sent_slots.ensure((size_t)std::max<int64_t>(jb.n_send, 1) * 4));
        VF_CUDA(sc->dst_off.ensure((size_t)(W + 1) * 8));
        VF_CUDA(cudaMemcpyAsync(sc->dst_off.p, jb.send_off.data(), (W + 1) * 8, cudaMemcpyHostToDevice, xs));
        launch_pack_remote(jb.po.a, xs, jb.n_slots, sc->send.as<uint8_t>(), sc->dst_off.as<int64_t>(),
                           sc->sent_slots.as<int32_t>(), rec_bytes);
        VF_CUDA(jb.exec->recv.ensure((size_t)std::max<int64_t>(jb.n_recv, 1) * rec_bytes));
    }
    auto exchange = [&](bool forward, int which) -> vf_status {
        // forward: origin send regions (per dst) -> owner recv regions (per src), item records;
        // backward: owner result regions (per src) -> origin back regions (per dst), ids or dists
        const int64_t unit = forward ? rec_bytes : (int64_t)k * 4;
        auto sbuf = [&](ShardJob &jb) -> uint8_t * {
            if (forward) return jb.own->send.as<uint8_t>();
            return which == 0 ? jb.exec->res_ids.as<uint8_t>() : jb.exec->res_dists.as<uint8_t>();
        };
        auto rbuf = [&](ShardJob &jb) -> uint8_t * {
            if (forward) return jb.exec->recv.as<uint8_t>();
            return which == 0 ? jb.own->back_ids.as<uint8_t>() : jb.own->back_dists.as<uint8_t>();
        };
        if (tr->loopback()) {
            for (int src = 0; src < J; src++)
                for (int dst = 0; dst < J; dst++) {
                    // forward: src's items for dst; backward: dst-owner's results for origin src
                    ShardJob &a_ = jobs[src], &b_ = jobs[dst];
                    const int64_t cnt = forward ? a_.send_cnt[dst] : b_.recv_cnt[src];
                    if (cnt == 0) continue;
                    const uint8_t *from = forward ? sbuf(a_) + a_.send_off[dst] * unit : sbuf(b_) + b_.recv_off[src] * unit;
                    uint8_t *to = forward ? rbuf(b_) + b_.recv_off[src] * unit : rbuf(a_) + a_.send_off[dst] * unit;
                    VF_CUDA(cudaMemcpyAsync(to, from, cnt * unit, cudaMemcpyDeviceToDevice, xs));
                }
            return VF_OK;
        }
        ShardJob &jb = jobs[0];
        std::vector<int64_t> soff(W), sb(W), roff(W), rb(W);
        for (int r = 0; r < W; r++) {
            if (forward) {
                soff[r] = jb.send_off[r] * unit; sb[r] = jb.send_cnt[r] * unit;
                roff[r] = jb.recv_off[r] * unit; rb[r] = jb.recv_cnt[r] * unit;
            } else {
                soff[r] = jb.recv_off[r] * unit; sb[r] = jb.recv_cnt[r] * unit;
                roff[r] = jb.send_off[r] * unit; rb[r] = jb.send_cnt[r] * unit;
            }
        }
        return tr->alltoallv(sbuf(jb), soff.data(), sb.data(), rbuf(jb), roff.data(), rb.data(), W,
                             jb.ix->rank, xs);
    };
    vf_status st = exchange(true, 0);
    if (st != VF_OK) return st;

    // ---- phase 4: owners run the received items (single-item queries, results written directly)
    for (auto &jb : jobs) {
        vf_index *ix = jb.ix;
        Scratch *sc = jb.exec;
        st = plan_search(ix, sc, jb.n_recv, jb.n_recv, p, xs, &jb.pe);
        if (st != VF_OK) return st;
        VF_CUDA(sc->qlab.ensure((size_t)std::max<int64_t>(jb.n_recv, 1) * kRecLabels * 4));
        VF_CUDA(sc->res_ids.ensure((size_t)std::max<int64_t>(jb.n_recv, 1) * k * 4));
        VF_CUDA(sc->res_dists.ensure((size_t)std::max<int64_t>(jb.n_recv, 1) * k * 4));
        SearchArgs &a = jb.pe.a;
        a.qlab = sc->qlab.as<int32_t>();
        a.out_ids = sc->res_ids.as<int32_t>();
        a.out_dists = sc->res_dists.as<float>();
        int launches = 0;
        st = run_local(ix, sc, jb.pe, xs, sc->recv.as<uint8_t>(), jb.n_recv, rec_bytes, &launches);
        if (st != VF_OK) return st;
        jb.own->last_launches += launches;
        VF_CUDA(jb.own->back_ids.ensure((size_t)std::max<int64_t>(jb.n_send, 1) * k * 4));
        VF_CUDA(jb.own->back_dists.ensure((size_t)std::max<int64_t>(jb.n_send, 1) * k * 4));
    }

    // ---- phase 5: results go back to the origins
    st = exchange(false, 0);
    if (st != VF_OK) return st;
    st = exchange(false, 1);
    if (st != VF_OK) return st;
    VF_CUDA(cudaEventRecord(jobs[0].own->ev_xdone, xs));
    VF_CUDA(cudaStreamWaitEvent(s, jobs[0].own->ev_xdone, 0));

    // ---- phase 6: origins merge local and returned lists per query (a5)
    for (auto &jb : jobs) {
        Scratch *sc = jb.own;
        SearchArgs &a = jb.po.a;
        int launches = launch_scatter_results(a, s, sc->back_ids.as<int32_t>(), sc->back_dists.as<float>(),
                                              sc->sent_slots.as<int32_t>(), jb.n_send);
        launches += launch_merge(a, s);
        if (jb.ix->profiling) VF_CUDA(cudaEventRecord(sc->ev[5], s));
        if (jb.n > 0) {
            const cudaMemcpyKind kind = jb.out_dev ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
            VF_CUDA(cudaMemcpyAsync(jb.out_ids, a.out_ids, (size_t)jb.n * k * 4, kind, s));
            VF_CUDA(cudaMemcpyAsync(jb.out_dists, a.out_dists, (size_t)jb.n * k * 4, kind, s));
        }
        if (jb.ix->profiling) VF_CUDA(cudaEventRecord(sc->ev[6], s));
        sc->last = a;
        sc->last_slots = jb.n_slots;
        sc->last_launches += launches;
        sc->profiled = jb.ix->profiling;
        if (sc->profiled) sc->prof_n++;
        sc->has_last = true;
    }
    VF_CUDA(cudaGetLastError());
    // host outputs or no stream: the results must be there on return (device outputs with a
    // stream: asynchronous like vf_search)
    if (any_host_out || s == nullptr) VF_CUDA(cudaStreamSynchronize(s));
    return VF_OK;
}

}  // namespace vf
