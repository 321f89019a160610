// f1 -- one CTA answers one query end to end: route (a1), every item (a2 scan / a3 beam search),
// predicate (a4) and merge (a5) inside a single launch. PAPER.md P:L474-L493 ("Persistent
// Kernel-based Search for Small Batch Queries"): small batches pay the batched pipeline's chain of
// launches (route, bucket, scan, graph, merge) for very little work, so VecFlow maps each query to
// one thread block. The same per-query body serves
//   k_small  -- one launch per small vf_search batch (grid = one CTA per query), and
//   k_serve  -- the persistent kernel: resident CTAs claim jobs from a ring in host-mapped memory
//               (atomic job counter, host-published head), answer them and publish the results
//               with a sequence number; no launch and no host synchronisation per query.
// Results are identical to the batched path: the same routing function, the same beam search
// (beam_item), exact integer / fp32 distances under the same (dist, id) total order.
#include "graph_item.cuh"
#include "small.h"

#ifndef VF_SERVE_SYSLD
#define VF_SERVE_SYSLD 0
#endif

namespace vf {

// ---------------------------------------------------------------- shared-memory layout
static SmallLayout small_layout(int itopk, int hash_slots, int row_native, int row_fast, int k) {
    // X_LS stages: as many ~24 KB stages as fit next to the rest (2..kSmallStages), so one CTA keeps
    // enough bytes in flight to stream a list
    SmallLayout L;
    const GraphLayout G = graph_layout(itopk, hash_slots);
    L.itopk = G.itopk; L.hash_slots = G.hash_slots;
    L.off_topA = G.off_topA; L.off_topB = G.off_topB; L.off_cbuf = G.off_cbuf; L.off_fgid = G.off_fgid;
    L.off_floc = G.off_floc; L.off_par = G.off_par; L.off_hash = G.off_hash; L.warp_bytes = G.warp_bytes;
    (void)k;
    size_t o = 0;
    L.off_warps = o; o += G.warp_bytes * kSmallWarps;
    o = (o + 127) & ~(size_t)127;
    L.off_qs = o; o += (size_t)row_native;
    L.off_qf = o; o += (size_t)row_fast;
    L.off_lab = o; o += (size_t)kMaxQueryLabels * 4;
    L.off_items = o; o += (size_t)kMaxQueryLabels * 8;
    L.off_res = o; o += (size_t)kMaxQueryLabels * kSmallMaxK * 8;
    L.off_mrg = o; o += (size_t)kSmallWarps * 32 * 8;
    o = (o + 127) & ~(size_t)127;
    // TMA stages for contiguous X_LS rows: whole rows, ~24 KB each
    const int rb = row_fast > row_native ? row_fast : row_native;
    int rows = kSmallStageBytes / rb;
    if (rows < 1) rows = 1;
    L.stage_rows = rows;
    L.stage_bytes = rows * rb;
    const size_t budget = 220 * 1024;
    int ns = kSmallStages;
    while (ns > 2 && o + (size_t)L.stage_bytes * ns + 16 * ns + 256 > budget) ns--;
    L.n_stages = ns;
    L.off_stage = o; o += (size_t)L.stage_bytes * ns;
    L.off_bar = o; o += 16 * ns;
    L.off_misc = o; o += 64;
    L.bytes = (o + 127) & ~(size_t)127;
    return L;
}

struct SmallSmem {
    uint8_t *warps;
    uint8_t *qs, *qf;
    int32_t *lab;
    int32_t *items;      // [t] label, [64 + t] path | pred
    ull *res;            // [item][kSmallMaxK]
    ull *mrg;            // [warp][32]
    uint8_t *stage;
    uint64_t *bar;
    int32_t *misc;       // [0] nl, [1] nch, [2] fast view ok, [3] pred, [4] qh
};

__device__ __forceinline__ GraphLayout graph_of(const SmallLayout &L) {
    GraphLayout G;
    G.itopk = L.itopk; G.hash_slots = L.hash_slots;
    G.off_topA = L.off_topA; G.off_topB = L.off_topB; G.off_cbuf = L.off_cbuf; G.off_fgid = L.off_fgid;
    G.off_floc = L.off_floc; G.off_par = L.off_par; G.off_hash = L.off_hash; G.warp_bytes = L.warp_bytes;
    return G;
}

__device__ __forceinline__ SmallSmem small_smem(uint8_t *smem, const SmallLayout &L) {
    SmallSmem s;
    s.warps = smem + L.off_warps;
    s.qs = smem + L.off_qs;
    s.qf = smem + L.off_qf;
    s.lab = reinterpret_cast<int32_t *>(smem + L.off_lab);
    s.items = reinterpret_cast<int32_t *>(smem + L.off_items);
    s.res = reinterpret_cast<ull *>(smem + L.off_res);
    s.mrg = reinterpret_cast<ull *>(smem + L.off_mrg);
    s.stage = smem + L.off_stage;
    s.bar = reinterpret_cast<uint64_t *>(smem + L.off_bar);
    s.misc = reinterpret_cast<int32_t *>(smem + L.off_misc);
    return s;
}

// Merge the 4 warps' sorted k-lists in s.mrg into one sorted list (warp 0 calls; k <= 32).
__device__ __forceinline__ ull merge_warp_lists(const ull *mrg, int k, int lane) {
    ull Li = lane < k ? mrg[lane] : KEY_INF;
    for (int w = 1; w < kSmallWarps; w++) Li = warp_merge_topk(Li, lane < k ? mrg[w * 32 + lane] : KEY_INF, k, lane);
    return Li;
}

// ---------------------------------------------------------------- a2 scan of one item by the CTA
// Exact squared-L2 top-k over the label's posting list, AND predicate applied
// before the distance. LS lists are contiguous in X_LS and arrive by 1-D TMA bulk copies
// (double-buffered); lists scanned on an HS label (f2 / f3 / exact) are gathered through M_HS.
template <int DT, int TEAM, int CPL>
__device__ void small_scan_item(const SearchArgs &a, const DevIndex &v, const SmallLayout &L, const SmallSmem &s,
                                const uint8_t *qrow, int32_t label, bool has_pred, int np, ull *out,
                                uint32_t &bar_phase, int part, int nparts) {
    typedef Acc<DT> A;
    constexpr int RP = 32 / TEAM;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int team = lane / TEAM, tl = lane % TEAM;
    const int k = a.k, chunks = v.chunks, rb = v.row_bytes;
    const LabelDir d = v.dir[label];
    const bool hs = d.size >= v.T;
    // this CTA's slice of the list (a small batch splits each scan item over nparts CTAs)
    const int32_t rlo = (int32_t)((int64_t)d.size * part / nparts);
    const int32_t S = (int32_t)((int64_t)d.size * (part + 1) / nparts) - rlo;
    uint4 qreg[CPL];
    const uint4 *q4 = reinterpret_cast<const uint4 *>(qrow);
#pragma unroll
    for (int j = 0; j < CPL; j++) {
        const int c = tl + j * TEAM;
        qreg[j] = c < chunks ? q4[c] : make_uint4(0, 0, 0, 0);
    }
    ull Li = KEY_INF;
    auto offer = [&](int32_t gid, const uint4 *row, bool ok) {
        // one row per team: distance, then the warp's register top-k
        typename A::T acc = 0;
        if (ok) {
#pragma unroll
            for (int j = 0; j < CPL; j++) {
                const int c = tl + j * TEAM;
                if (c < chunks) A::add(acc, qreg[j], row[c]);
            }
        }
#pragma unroll
        for (int o = TEAM / 2; o > 0; o >>= 1) acc += __shfl_xor_sync(FULL, acc, o);
        const ull key = (ok && tl == 0) ? make_key(A::to_float(acc), (uint32_t)gid) : KEY_INF;
        Li = warp_merge_topk(Li, key, k, lane);
    };
    const int32_t *P = s.lab;
    if (!hs) {
        // contiguous rows: TMA bulk stages of L.stage_rows rows
        const uint8_t *src = v.Xls + (d.base + rlo) * (int64_t)rb;
        const int SR = L.stage_rows, NS = L.n_stages;
        const int nst = (S + SR - 1) / SR;
        if (threadIdx.x == 0) {
            for (int st = 0; st < NS && st < nst; st++) {
                const int r0 = st * SR, nr = min(SR, S - r0);
                mbar_arrive_expect_tx(s.bar + 2 * st, (uint32_t)(nr * rb));
                tma_load_1d(s.stage + (size_t)st * L.stage_bytes, src + (int64_t)r0 * rb, (uint32_t)(nr * rb),
                            s.bar + 2 * st);
            }
        }
        for (int st = 0; st < nst; st++) {
            const int buf = st % NS;
            mbar_wait(s.bar + 2 * buf, (bar_phase >> buf) & 1u);
            const int r0 = st * SR, nr = min(SR, S - r0);
            const uint8_t *stg = s.stage + (size_t)buf * L.stage_bytes;
            // keys carry the row's position in the list: local order = global-id order (C_l is
            // ascending), so the (dist, id) tie-break is unchanged; the k winners are
            // mapped through M_LS at the end. AND items need the global id first (predicate).
            for (int rr = wid * RP; rr < nr; rr += kSmallWarps * RP) {
                const int r = rr + team;
                const bool live = r < nr;
                bool ok = live;
                if (ok && has_pred) ok = verify_pred(v, __ldg(v.M_ls + d.base + rlo + r0 + r), P, np, label);
                offer(rlo + r0 + r, reinterpret_cast<const uint4 *>(stg + (size_t)(live ? r : 0) * rb), ok);
            }
            __syncthreads();                                   // stage consumed by every warp
            bar_phase ^= 1u << buf;                            // every thread tracks the parity
            if (threadIdx.x == 0 && st + NS < nst) {
                const int r1 = (st + NS) * SR, n1 = min(SR, S - r1);
                mbar_arrive_expect_tx(s.bar + 2 * buf, (uint32_t)(n1 * rb));
                tma_load_1d(s.stage + (size_t)buf * L.stage_bytes, src + (int64_t)r1 * rb, (uint32_t)(n1 * rb),
                            s.bar + 2 * buf);
            }
        }
    } else {
        // HS list scanned (f2 / f3 / exact): rows gathered through M_HS, predicate first
        for (int rr = wid * RP; rr < S; rr += kSmallWarps * RP) {
            const int r = rr + team;
            const bool live = r < S;
            int32_t gid = live ? __ldg(v.M_hs + d.base + rlo + r) : 0;
            bool ok = live;
            if (ok && has_pred) ok = verify_pred(v, gid, P, np, label);
            offer(gid, reinterpret_cast<const uint4 *>(v.X + (int64_t)(ok ? gid : 0) * rb), ok);
        }
    }
    if (lane < 32) s.mrg[wid * 32 + lane] = Li;
    __syncthreads();
    if (wid == 0) {
        ull m = merge_warp_lists(s.mrg, k, lane);
        if (!hs && m != KEY_INF)                                   // local position -> global id
            m = (m & 0xFFFFFFFF00000000ull) | (uint32_t)__ldg(v.M_ls + d.base + (int32_t)(uint32_t)m);
        if (lane < k) out[lane] = m;
    }
    if (threadIdx.x == 0 && S > 0) atomicAdd(&a.ctr->scan_rows, (ull)S);
    __syncthreads();
}

// ---------------------------------------------------------------- the per-query body
// The items are routed (s.items), the query rows are in shared memory. Scan items first (all
// warps), then graph items (one warp each, round robin), then the merge (warp 0).
template <int DT, int TEAM, int CPL>
__device__ void small_items(const SearchArgs &a, const DevIndex &v, const SmallLayout &L, const SmallSmem &s,
                            const uint8_t *qrow, ull *gtab_base, uint32_t *epochs, int warp_slot0,
                            int32_t item_slot0, int32_t qid, uint32_t &bar_phase, int part, int nparts) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int nl = s.misc[0], nch = s.misc[1];
    const bool has_pred = s.misc[3] != 0;
    const uint32_t qh = (uint32_t)s.misc[4];
    for (int i = threadIdx.x; i < nch * kSmallMaxK; i += blockDim.x) s.res[i] = KEY_INF;
    __syncthreads();
    for (int t = 0; t < nch; t++)
        if ((s.items[64 + t] & 3) == PATH_SCAN)
            small_scan_item<DT, TEAM, CPL>(a, v, L, s, qrow, s.items[t], has_pred, nl, s.res + t * kSmallMaxK,
                                           bar_phase, part, nparts);
    int g = 0;
    for (int t = 0; t < nch; t++) {
        if ((s.items[64 + t] & 3) != PATH_GRAPH) continue;
        const int gw = g++ % (kSmallWarps * nparts);      // graph items round robin over the warps
        if (gw != part * kSmallWarps + wid) continue;       // of every CTA of the query
        const int32_t label = s.items[t];
        const LabelDir d = v.dir[label];
        BeamItem bi;
        bi.label = label;
        bi.S = d.size;
        bi.base = d.base;
        bi.has_pred = has_pred;
        bi.P = s.lab;
        bi.np = nl;
        bi.qh = qh;
        bi.qrow = qrow;
        const int ws = warp_slot0 + wid;
        ull *gtab = gtab_base + (size_t)ws * a.gtab_slots;
        uint32_t ep = epochs[ws] + 1;
        if (lane == 0) epochs[ws] = ep;
        __syncwarp();
        const BeamOut bo = beam_item<DT, TEAM, CPL>(a, v, graph_of(L), s.warps + (size_t)wid * L.warp_bytes, gtab,
                                                    (uint64_t)a.gtab_slots - 1, ep, bi, lane);
        for (int i = lane; i < a.k; i += 32) {
            ull key = KEY_INF;
            if (i < bo.ntop) {
                const ull kk = bo.top[i];
                const int32_t j = (int32_t)((uint32_t)kk >> 1);
                key = (kk & 0xFFFFFFFF00000000ull) | (uint32_t)__ldg(v.M_hs + d.base + j);
            }
            s.res[t * kSmallMaxK + i] = key;
        }
        if (lane == 0) {
            if (item_slot0 >= 0) {
                a.item_ctr[(size_t)(item_slot0 + t) * 3 + 0] = bo.nvis;
                a.item_ctr[(size_t)(item_slot0 + t) * 3 + 1] = bo.E;
                a.item_ctr[(size_t)(item_slot0 + t) * 3 + 2] = bo.iters;
            }
            atomicAdd(&a.ctr->graph_V, (ull)bo.nvis);
            atomicAdd(&a.ctr->graph_E, (ull)bo.E);
            atomicAdd(&a.ctr->graph_iters, (ull)bo.iters);
            atomicMax(&a.ctr->graph_V_max, (ull)bo.nvis);
        }
        __syncwarp();
    }
    (void)qid;
    __syncthreads();
}

// Merge (a5): union of the items' lists, dedup by global id (equal ids carry equal keys), best k
// by (dist, id) (Alg. 2). Warp 0; returns lane i's i-th key.
__device__ __forceinline__ ull small_merge(const SmallSmem &s, int k, int lane) {
    const int nch = s.misc[1];
    if (nch == 0) return KEY_INF;
    ull Li = lane < k ? s.res[lane] : KEY_INF;
    for (int t = 1; t < nch; t++) {
        ull key = lane < k ? s.res[t * kSmallMaxK + lane] : KEY_INF;
        bool dup = false;
        for (int j = 0; j < k; j++) dup |= key == __shfl_sync(FULL, Li, j);
        if (dup) key = KEY_INF;
        Li = warp_merge_topk(Li, key, k, lane);
    }
    return Li;
}

// Route + prepare one query into shared memory (whole CTA). raw: the caller's row (dim elements of
// the index's element type); lab / nraw: its labels. Writes the padded native row (s.qs), the
// fast-view u8 row (s.qf, when the index has one and the query is in its exact range), the content
// hash, the routed items. Returns nothing; everything lands in s.misc / s.items.
__device__ void small_prepare(const SearchArgs &a, const DevIndex &native, const SmallSmem &s, const uint8_t *raw,
                              int raw_bytes, const int32_t *lab, int nraw, bool have_fast) {
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int nwords = (raw_bytes + 3) >> 2, dwords = native.row_bytes >> 2;
    for (int i = tid; i < nraw; i += blockDim.x) s.lab[i] = lab[i];
    if (wid == 0) {
        uint32_t hacc = 0;
        for (int w = lane; w < dwords; w += 32) {
            uint32_t word = 0;
            if (w < nwords) {
                if ((raw_bytes & 3) == 0) {
                    word = reinterpret_cast<const uint32_t *>(raw)[w];
                } else {
                    for (int t = 0; t < 4; t++) {
                        const int p = w * 4 + t;
                        const uint32_t b = p < raw_bytes ? (uint32_t)raw[p] : 0u;
                        word |= b << (8 * t);
                    }
                }
                hacc += fmix32(word + (uint32_t)w * 0x9E3779B9u);
            }
            reinterpret_cast<uint32_t *>(s.qs)[w] = word;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) hacc += __shfl_xor_sync(FULL, hacc, o);
        if (lane == 0) s.misc[4] = (int32_t)fmix32(hacc);
    }
    __syncthreads();
    if (wid == 0) {
        bool bad = false;
        if (have_fast) {
            const float *row = reinterpret_cast<const float *>(s.qs);
            for (int i = lane; i < native.dim; i += 32) {
                const float x = row[i];
                bad |= !(x == rintf(x) && x >= a.chk_lo && x <= a.chk_hi);
            }
            for (int i = lane; i < a.q8_row_bytes; i += 32) {
                const float x = i < native.dim ? row[i] : 0.f;
                s.qf[i] = (uint8_t)(x >= 0.f && x <= 255.f ? (int)x : 0);
            }
        }
        bad = __any_sync(FULL, bad);
        if (lane == 0) {
            s.misc[2] = have_fast && !bad;
            int32_t chosen[kMaxQueryLabels];
            uint32_t cpath[kMaxQueryLabels];
            int nl = 0, nch = 0;
            uint32_t pred = 0;
            route_labels(a, s.lab, nraw, &nl, chosen, cpath, &nch, &pred);
            s.misc[0] = nl;
            s.misc[1] = nch;
            s.misc[3] = pred ? 1 : 0;
            for (int t = 0; t < nch; t++) {
                s.items[t] = chosen[t];
                s.items[64 + t] = (int32_t)cpath[t];
            }
        }
    }
    __syncthreads();
}

// Record the items (vf_get_last_items) and write the k results of query q.
__device__ __forceinline__ void small_finish(const SearchArgs &a, const SmallSmem &s, ull key, int32_t qid,
                                             int32_t item_slot0, int nraw, int32_t *out_ids, float *out_d) {
    const int lane = threadIdx.x & 31;
    const int nch = s.misc[1];
    if (lane < a.k) {
        out_ids[lane] = key == KEY_INF ? -1 : (int32_t)key_id(key);
        out_d[lane] = key == KEY_INF ? __uint_as_float(0x7f800000u) : key_dist(key);
    }
    if (item_slot0 >= 0) {
        for (int t = lane; t < nraw; t += 32) {
            Item it;
            it.qid = qid;
            it.rank = 0;
            it.label = t < nch ? s.items[t] : -1;
            it.meta = t < nch ? ((uint32_t)s.items[64 + t] | (s.misc[3] ? META_PRED : 0u) | (nch == 1 ? META_DIRECT : 0u))
                              : PATH_NONE;
            a.items[item_slot0 + t] = it;
        }
    }
    if (lane == 0) {
        int ng = 0, ns = 0;
        for (int t = 0; t < nch; t++) {
            ng += (s.items[64 + t] & 3) == PATH_GRAPH;
            ns += (s.items[64 + t] & 3) == PATH_SCAN;
        }
        if (ng) atomicAdd(&a.ctr->n_graph, ng);
        if (ns) atomicAdd(&a.ctr->n_scan_items, ns);
    }
}

// One whole query by the CTA: prepare, items on the fast or native view, merge, output.
// Returns true in the CTA that wrote the query's results (with nparts > 1: the last to finish).
// partials: [nparts][pstride][kSmallMaxK] keys (pstride >= the query's item count).
template <int DTF, int TF, int CF, int TS, int CS>
__device__ bool small_query(const SearchArgs &a, const DevIndex &native, const SmallLayout &L, uint8_t *smem,
                            const uint8_t *raw, int raw_bytes, const int32_t *lab, int nraw, int32_t qid,
                            int32_t item_slot0, int32_t *out_ids, float *out_d, int warp_slot0, uint32_t *epochs,
                            uint32_t &bar_phase, int part = 0, int nparts = 1, ull *partials = nullptr,
                            int32_t *done_ctr = nullptr, int pstride = kMaxQueryLabels) {
    const SmallSmem s = small_smem(smem, L);
    const bool have_fast = TS > 0;   // a u8 row store in front of a fp32 index
    small_prepare(a, native, s, raw, raw_bytes, lab, nraw, have_fast);
    if (!have_fast || s.misc[2]) {
        small_items<DTF, TF, CF>(a, a.ix, L, s, have_fast ? s.qf : s.qs, a.gtab, epochs, warp_slot0, item_slot0,
                                 qid, bar_phase, part, nparts);
    } else {
        // every index array of the fp32 view is read through `native`; `a` only supplies parameters
        small_items<1, (TS > 0 ? TS : 1), (CS > 0 ? CS : 1)>(a, native, L, s, s.qs, a.gtab, epochs, warp_slot0,
                                                             item_slot0, qid, bar_phase, part, nparts);
    }
    if (nparts > 1) {
        // publish this CTA's per-item lists; the last CTA of the query merges all of them
        const int nch = s.misc[1];
        ull *mine = partials + (size_t)part * pstride * kSmallMaxK;
        for (int i = threadIdx.x; i < nch * kSmallMaxK; i += blockDim.x) mine[i] = s.res[i];
        __threadfence();
        __syncthreads();
        if (threadIdx.x == 0) s.misc[12] = atomicAdd(done_ctr, 1) == nparts - 1;
        __syncthreads();
        if (!s.misc[12]) return false;                // not the last: this CTA is done
        __threadfence();
        if ((threadIdx.x >> 5) == 0) {
            const int lane = threadIdx.x & 31;
            for (int t = 0; t < nch; t++) {
                ull Li = KEY_INF;
                for (int c = 0; c < nparts; c++) {
                    const ull key = lane < a.k ? __ldcg(partials + ((size_t)c * pstride + t) * kSmallMaxK + lane)
                                               : KEY_INF;
                    Li = warp_merge_topk(Li, key, a.k, lane);   // slices hold distinct rows
                }
                s.res[t * kSmallMaxK + lane] = Li;
            }
            if (lane == 0) *done_ctr = 0;                 // ready for the next search
        }
        __syncthreads();
    }
    if ((threadIdx.x >> 5) == 0) {
        const ull key = small_merge(s, a.k, threadIdx.x & 31);
        small_finish(a, s, key, qid, item_slot0, nraw, out_ids, out_d);
    }
    __syncthreads();
    return true;
}

__device__ __forceinline__ void small_init_bars(const SmallSmem &s, int n_stages) {
    if (threadIdx.x == 0) {
        for (int i = 0; i < n_stages; i++) mbar_init(s.bar + 2 * i, 1);
        fence_mbar_init();
    }
    __syncthreads();
}

// ---------------------------------------------------------------- k_small: one CTA per query
template <int DTF, int TF, int CF, int TS, int CS>
__global__ void __launch_bounds__(32 * kSmallWarps) k_small(SearchArgs a, DevIndex native, SmallLayout L,
                                                            int raw_bytes, uint32_t *epochs, int nparts,
                                                            ull *partials, int32_t *done_ctr) {
    extern __shared__ __align__(128) uint8_t smem[];
    const int64_t q = blockIdx.x / nparts;
    const int part = (int)(blockIdx.x % nparts);
    if (q >= a.n_q) return;
    const SmallSmem s = small_smem(smem, L);
    small_init_bars(s, L.n_stages);
    uint32_t bar_phase = 0;
    int64_t lo = a.q_off[q];
    const int64_t hi = a.q_off[q + 1];
    // device-side check of the caller's offsets (empty row + n_invalid; see SearchArgs)
    const bool bad = lo < 0 || hi < lo || hi > a.n_slots || hi - lo > a.max_nl;
    if (bad && part == 0 && threadIdx.x == 0) atomicAdd(&a.ctr->n_invalid, 1);
    if (bad) lo = 0;
    const int nraw = bad ? 0 : (int)(hi - lo);
    small_query<DTF, TF, CF, TS, CS>(a, native, L, smem, a.Qraw + q * (int64_t)raw_bytes, raw_bytes, a.qlab + lo,
                                     nraw, (int32_t)q, bad ? -1 : (int32_t)lo, a.out_ids + q * a.k, a.out_dists + q * a.k,
                                     (int)blockIdx.x * kSmallWarps, epochs, bar_phase, part, nparts,
                                     partials + (size_t)q * nparts * kMaxQueryLabels * kSmallMaxK, done_ctr + q);
}

// ---------------------------------------------------------------- k_serve: the persistent kernel
// Job j lives in slot j % cap of the host-mapped ring. The host writes the slot's query row and
// labels, then publishes head = j + 1 (release). The last CTA is the dispatcher: it alone polls the
// host-mapped head / stop words over PCIe and mirrors them into device memory. Every other CTA
// claims j from the device job counter, waits on the device mirror for head > j (or stop), answers
// the query, writes ids / dists into the slot and publishes done[slot] = j + 1 after a system-scope
// fence.
template <int DTF, int TF, int CF, int TS, int CS>
__global__ void __launch_bounds__(32 * kSmallWarps) k_serve(SearchArgs a, DevIndex native, SmallLayout L,
                                                            int raw_bytes, uint32_t *epochs, ServeRing ring) {
    extern __shared__ __align__(128) uint8_t smem[];
    if (blockIdx.x == 0) {
        // dispatcher: the only CTA that reads the host ring. New jobs are copied in bulk (all 128
        // threads, 16-byte loads, a job's slot per 40 threads) into the device-memory ring, then
        // published through the device head; workers never touch PCIe for their inputs.
        long long *sh = reinterpret_cast<long long *>(smem);
        long long copied = 0;
        unsigned long long last_job = 0;
        if (threadIdx.x == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(last_job));
        const int qv = ring.raw_stride / 16;             // 16-byte words of a query slot
        const int per_job = qv + kServeLabels / 4 + 1;   // + labels (4 x 16 B) + the count
        for (;;) {
            if (threadIdx.x == 0) {
                long long h;
                int32_t st;
                for (;;) {
                    st = *(volatile const int32_t *)ring.stop;
                    __threadfence_system();
                    h = *(volatile const long long *)ring.head;
                    if (h != copied || st) break;
                    if (ring.idle_ns) {
                        // idle exit: no job published for idle_ns (e.g. a profiler serialises the
                        // launch, so the host can never submit); answered like a stop
                        unsigned long long now;
                        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
                        if (now - last_job > ring.idle_ns) { st = 1; break; }
                    }
                    __nanosleep(64);
                }
                if (h != copied) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(last_job));
                sh[0] = h;
                sh[1] = st;
            }
            __syncthreads();
            const long long h = sh[0];
            const bool st = sh[1] != 0;
            const long long n_new = h - copied;
            // 4 PCIe reads in flight per thread before their stores (latency-bound otherwise)
            constexpr int U = 4;
            const long long total = n_new * per_job;
            for (long long e0 = threadIdx.x; e0 < total; e0 += (long long)U * blockDim.x) {
                uint4 v[U];
                uint4 *dst[U];
#pragma unroll
                for (int u = 0; u < U; u++) {
                    const long long e = e0 + (long long)u * blockDim.x;
                    dst[u] = nullptr;
                    if (e >= total) continue;
                    const long long j = copied + e / per_job;
                    const int w = (int)(e % per_job);
                    const int64_t slot = j % ring.cap;
                    if (w < qv) {
                        v[u] = __ldcv(reinterpret_cast<const uint4 *>(ring.queries + slot * ring.raw_stride) + w);
                        dst[u] = reinterpret_cast<uint4 *>(ring.dq + slot * ring.raw_stride) + w;
                    } else if (w < per_job - 1) {
                        const int l = w - qv;
                        v[u] = __ldcv(reinterpret_cast<const uint4 *>(ring.labels + slot * kServeLabels) + l);
                        dst[u] = reinterpret_cast<uint4 *>(ring.dlab + slot * kServeLabels) + l;
                    } else {
                        v[u].x = (uint32_t)__ldcv(ring.nlab + slot);
                        ring.dnlab[slot] = (int32_t)v[u].x;
                    }
                }
#pragma unroll
                for (int u = 0; u < U; u++)
                    if (dst[u]) *dst[u] = v[u];
            }
            __threadfence();
            __syncthreads();
            if (threadIdx.x == 0) {
                copied = h;
                *(volatile long long *)ring.dev_head = h;
                if (st) *(volatile int32_t *)ring.dev_stop = 1;
                __threadfence();
            }
            if (threadIdx.x != 0) copied = h;
            if (st) break;
            __syncthreads();
        }
        return;
    }
    const SmallSmem s = small_smem(smem, L);
    small_init_bars(s, L.n_stages);
    uint32_t bar_phase = 0;
    long long *s_job = reinterpret_cast<long long *>(s.misc + 8);   // no static smem: the dynamic
    auto now = [] { unsigned long long t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t; };
    for (;;) {                                                      // size may use all 227 KB
        unsigned long long t0 = 0, t1 = 0, t2 = 0;
        if (threadIdx.x == 0) {
            t0 = now();
            // claim c = (job j, part c % nparts): a job is answered by nparts CTAs together
            const long long c = (long long)atomicAdd(ring.next, 1ull);
            long long j = c / ring.nparts;
            s.misc[13] = (int32_t)(c % ring.nparts);
            // wait until job j is published (device mirror of the host head), or stop
            for (;;) {
                const long long h = *(volatile long long *)ring.dev_head;
                if (h > j) break;
                if (*(volatile int32_t *)ring.dev_stop) {
                    __threadfence();
                    if (*(volatile long long *)ring.dev_head > j) break;
                    j = -1;
                    break;
                }
                __nanosleep(32);
            }
            *s_job = j;
        }
        __syncthreads();
        const long long j = *s_job;
        const int part = s.misc[13];
        if (j < 0) break;
        if (threadIdx.x == 0) t1 = now();
        const int slot = (int)(j % ring.cap);
        // the job's query and labels into shared memory
        uint8_t *rawbuf = s.stage;
        int32_t *labbuf = reinterpret_cast<int32_t *>(s.stage + ring.raw_stride);
        const uint4 *src = reinterpret_cast<const uint4 *>(ring.queries + (int64_t)slot * ring.raw_stride);
#if VF_SERVE_SYSLD == 2
        // system-scope relaxed loads: coherent with the host's stores, vectorised
        for (int i = threadIdx.x; i < ring.raw_stride / 16; i += blockDim.x) {
            uint4 v;
            asm volatile("ld.relaxed.sys.global.v4.u32 {%0,%1,%2,%3}, [%4];"
                         : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(src + i));
            reinterpret_cast<uint4 *>(rawbuf)[i] = v;
        }
        for (int i = threadIdx.x; i < kServeLabels; i += blockDim.x) {
            int32_t v;
            asm volatile("ld.relaxed.sys.global.s32 %0, [%1];" : "=r"(v) : "l"(ring.labels + (int64_t)slot * kServeLabels + i));
            labbuf[i] = v;
        }
        int32_t nl_raw;
        asm volatile("ld.relaxed.sys.global.s32 %0, [%1];" : "=r"(nl_raw) : "l"(ring.nlab + slot));
        const int nraw = min(nl_raw, kServeLabels);
#else
        // the dispatcher copied the slot into device memory: read it from L2 (ld.cg; an earlier job
        // in this slot may still sit in this SM's L1)
        const uint4 *dsrc = reinterpret_cast<const uint4 *>(ring.dq + (int64_t)slot * ring.raw_stride);
        for (int i = threadIdx.x; i < ring.raw_stride / 16; i += blockDim.x)
            reinterpret_cast<uint4 *>(rawbuf)[i] = __ldcg(dsrc + i);
        for (int i = threadIdx.x; i < kServeLabels; i += blockDim.x)
            labbuf[i] = __ldcg(ring.dlab + (int64_t)slot * kServeLabels + i);
        const int nraw = min(__ldcg(ring.dnlab + slot), kServeLabels);
        (void)src;
#endif
        __syncthreads();
        if (threadIdx.x == 0) t2 = now();
        const bool wrote = small_query<DTF, TF, CF, TS, CS>(
            a, native, L, smem, rawbuf, raw_bytes, labbuf, nraw, -1, -1, ring.out_ids + (int64_t)slot * a.k,
            ring.out_dists + (int64_t)slot * a.k, (int)(blockIdx.x - 1) * kSmallWarps, epochs, bar_phase, part,
            ring.nparts, ring.partials + (size_t)slot * ring.nparts * kServeLabels * kSmallMaxK,
            ring.part_done + slot, kServeLabels);
        // only warp 0 wrote results into the slot: its lanes make them visible to the host, then the
        // done word publishes the job
        if (wrote && threadIdx.x < 32) {
            __threadfence_system();
            __syncwarp();
            if (threadIdx.x == 0) *(volatile long long *)(ring.done + slot) = j + 1;
        }
        if (threadIdx.x == 0 && ring.stats) {       // [0] wait for the job, [1] slot copy, [2] search, [3] parts
            const unsigned long long t3 = now();
            atomicAdd(ring.stats + 0, t1 - t0);
            atomicAdd(ring.stats + 1, t2 - t1);
            atomicAdd(ring.stats + 2, t3 - t2);
            atomicAdd(ring.stats + 3, 1ull);
        }
        __syncthreads();
    }
}

// ---------------------------------------------------------------- dispatch
typedef void (*small_fn)(SearchArgs, DevIndex, SmallLayout, int, uint32_t *, int, ull *, int32_t *);
typedef void (*serve_fn)(SearchArgs, DevIndex, SmallLayout, int, uint32_t *, ServeRing);

struct SmallPick { small_fn f; serve_fn g; };

// Instantiations: the fast view's (dtype, team, chunks/lane) and, for a u8 row store in front of a
// fp32 index, the fp32 view's (team, chunks/lane); others are served by the batched path.
static SmallPick small_pick(int dt, int team, int cpl, int team_s, int cpl_s) {
#define VF_SP(D_, T_, C_, TS_, CS_)                                                                     \
    if (dt == D_ && team == T_ && cpl <= C_ && team_s == TS_ && cpl_s <= CS_)                           \
        return SmallPick{k_small<D_, T_, C_, TS_, CS_>, k_serve<D_, T_, C_, TS_, CS_>};
    VF_SP(0, 1, 2, 0, 0) VF_SP(0, 2, 4, 0, 0) VF_SP(0, 4, 4, 0, 0) VF_SP(0, 8, 4, 0, 0)
    VF_SP(1, 2, 4, 0, 0) VF_SP(1, 8, 4, 0, 0) VF_SP(1, 16, 4, 0, 0)
    VF_SP(0, 1, 2, 2, 4) VF_SP(0, 2, 4, 8, 4) VF_SP(0, 4, 4, 16, 4)
#undef VF_SP
    return SmallPick{nullptr, nullptr};
}

static SmallPick small_kernel(const DevIndex &fast, const DevIndex &native, bool two_views) {
    int t, c, ts = 0, cs = 0;
    team_for(fast.chunks, &t, &c);
    if (two_views) team_for(native.chunks, &ts, &cs);
    return small_pick(fast.dtype, t, c, ts, cs);
}

bool small_supported(const DevIndex &fast, const DevIndex &native, bool two_views, int k) {
    return k <= kSmallMaxK && small_kernel(fast, native, two_views).f != nullptr;
}

int small_smem_bytes(const SearchArgs &a, const DevIndex &native, bool two_views) {
    const SmallLayout L = small_layout(a.itopk, a.hash_slots, native.row_bytes, two_views ? a.ix.row_bytes : 16, a.k);
    return (int)L.bytes;
}

static void set_smem_attr(const void *f) {
    static thread_local const void *done[32];
    static thread_local int nd = 0;
    for (int i = 0; i < nd; i++) if (done[i] == f) return;
    cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    if (nd < 32) done[nd++] = f;
}

int launch_small(const SearchArgs &a, const DevIndex &native, bool two_views, int raw_bytes, int nparts,
                 unsigned long long *partials, int32_t *done_ctr, cudaStream_t s) {
    const SmallPick p = small_kernel(a.ix, native, two_views);
    if (!p.f || a.n_q <= 0) return a.n_q <= 0 ? 0 : -1;
    const SmallLayout L = small_layout(a.itopk, a.hash_slots, native.row_bytes, two_views ? a.ix.row_bytes : 16, a.k);
    set_smem_attr((const void *)p.f);
    uint32_t *epochs = reinterpret_cast<uint32_t *>(a.gtab + (size_t)a.n_warp_slots * a.gtab_slots);
    p.f<<<(unsigned)(a.n_q * nparts), 32 * kSmallWarps, L.bytes, s>>>(a, native, L, raw_bytes, epochs, nparts,
                                                                      partials, done_ctr);
    return 1;
}

int launch_serve(const SearchArgs &a, const DevIndex &native, bool two_views, int raw_bytes, int n_ctas,
                 const ServeRing &ring, cudaStream_t s) {
    const SmallPick p = small_kernel(a.ix, native, two_views);
    if (!p.g) return -1;
    const SmallLayout L = small_layout(a.itopk, a.hash_slots, native.row_bytes, two_views ? a.ix.row_bytes : 16, a.k);
    set_smem_attr((const void *)p.g);
    uint32_t *epochs = reinterpret_cast<uint32_t *>(a.gtab + (size_t)a.n_warp_slots * a.gtab_slots);
    p.g<<<n_ctas + 1, 32 * kSmallWarps, L.bytes, s>>>(a, native, L, raw_bytes, epochs, ring);   // + dispatcher
    return 1;
}

int serve_max_ctas(const SearchArgs &a, const DevIndex &native, bool two_views) {
    const SmallPick p = small_kernel(a.ix, native, two_views);
    if (!p.g) return 0;
    const SmallLayout L = small_layout(a.itopk, a.hash_slots, native.row_bytes, two_views ? a.ix.row_bytes : 16, a.k);
    cudaError_t e = cudaFuncSetAttribute((const void *)p.g, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L.bytes);
    if (e != cudaSuccess) return -(int)e;
    int per_sm = 0, dev = 0, nsm = 148;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, p.g, 32 * kSmallWarps, L.bytes);
    if (e != cudaSuccess) return -(int)e;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    return per_sm * nsm;
}

}  // namespace vf
