// a2 -- IVF-BFS for low-specificity labels (Alg. 2), redesigned
// for sm_100a as a label-grouped scan: all queries routed to one LS label in this batch (a
// "segment", up to QG of them) share ONE pass over the label's rows, so every touched posting
// list is read from HBM once per batch. HBM-bound at every workload (arithmetic
// intensity ~ 2 x queries-per-label ops/byte), so the design goal is bytes in flight, not FLOPs.
//
// Persistent CTAs (one per SM), warp-specialised, 288 threads:
//   warp 0 (producer): claims row tiles (<= tile_rows rows of one segment) with an atomic
//     counter. Per tile it first prefetches the segment's query rows and item metadata into one of
//     two query buffers (mbarrier pair qfull/qempty), then streams the tile's rows into a ring of
//     shared-memory stages: one 1-D TMA bulk copy (cp.async.bulk + mbarrier complete_tx) of the
//     contiguous X_LS rows per stage; in exact mode an HS label's rows are gathered from X through
//     M_HS with one bulk copy per row.
//   warps 1-8 (consumers): "teams" of TS lanes split each row's 16-byte chunks (lane tl owns chunks
//     tl, tl+TS, ...), so each lane keeps its query chunks in registers; NV rows per team are
//     accumulated at once and a butterfly reduces the NV x TS partial sums in (NV-1)+log2(TS/NV)
//     shuffles, leaving one exact distance per "owner" lane (u8: vabsdiff4+dp4a int32; f32: FFMA,
//     exact for integer-valued data), written to a shared distance tile; AND items mark rows that
//     fail the predicate (equivalent to the paper's pre-filter, reading #21). After one named
//     barrier per stage the warp owning each query merges the tile into that query's single
//     register-resident top-k list (ballot against the k-th, insert by shuffle). A segment split
//     over several tiles is finalised by the CTA that completes its last tile (partial lists in
//     global memory, last-block-done counter).
#include "common.cuh"

namespace vf {

constexpr int kScanConsumers = 8;
constexpr int kScanThreads = 32 * (1 + kScanConsumers);
enum : int { ST_FIRST = 1, ST_LAST = 2, ST_END = 4 };

struct ScanLayout {
    int nst, rps, qg, k, row_bytes, ts, cpl;
    size_t off_full, off_empty, off_qfull, off_qempty, off_meta, off_tinfo, off_stage, off_qbuf,
        off_qmeta, off_lists, off_lcnt, off_scratch, off_flag, off_dist, off_gid, total;
};
constexpr uint32_t DIST_EXCL = 0xFFFFFFFFu;   // distance slot of an invalid / filtered row

struct QMeta {          // per query of the current segment
    int64_t p_off;      // offset of the query's sorted labels (predicate)
    int32_t slot, qid;
    uint32_t meta;
    int32_t nl;
    int32_t pad[2];
};

struct TInfo {          // per tile, written by the producer with the query prefetch
    int64_t base;       // first row of the label in X_LS (or M_HS in exact mode)
    int32_t tile, seg, label, nq, tile_in_seg, n_tiles, hs, pad;
};

static void scan_team(int chunks, int *ts, int *cpl) {
    for (int t = 32; t >= 2; t >>= 1)
        if (chunks % t == 0 && chunks / t <= 4) { *ts = t; *cpl = chunks / t; return; }
    *ts = 32;
    *cpl = (chunks + 31) / 32;
}

// Shared-memory plan: a ring of row stages, two query buffers, a double-buffered distance tile
// D[2][qg][rps] (+ the stage rows' global ids) and one top-k list per query of the segment.
static ScanLayout scan_layout(int row_bytes, int k) {
    ScanLayout L;
    L.row_bytes = row_bytes;
    L.k = k;
    scan_team(row_bytes / 16, &L.ts, &L.cpl);
    const int nv = L.ts < 8 ? L.ts : 8;
    const int br = nv * (32 / L.ts);                    // rows per warp batch
    int rb = 1;
    while (rb < 4 && kScanConsumers * br * rb * 2 <= 256 &&
           (size_t)kScanConsumers * br * (rb * 2) * row_bytes <= 32 * 1024)
        rb *= 2;
    L.rps = kScanConsumers * br * rb;
    int qg = kScanQG;
    while (qg > 1 && ((size_t)qg * row_bytes > 16 * 1024 || (size_t)qg * k * 8 > 16 * 1024 ||
                      (size_t)qg * L.rps > 8192))
        qg >>= 1;
    L.qg = qg;
    const size_t stage = (size_t)L.rps * row_bytes;
    size_t fixed = 2 * (size_t)qg * row_bytes + 2 * (size_t)qg * sizeof(QMeta) + (size_t)qg * k * 8 +
                   (size_t)kScanConsumers * (32 + 2 * k) * 8 + (size_t)qg * 4 + 2 * (size_t)qg * L.rps * 4 +
                   2 * (size_t)L.rps * 4 + 1024;
    L.nst = (int)((200 * 1024 - fixed) / stage);
    if (L.nst < 2) L.nst = 2;
    if (L.nst > 8) L.nst = 8;
    size_t o = 0;
    L.off_full = o; o += 8 * L.nst;
    L.off_empty = o; o += 8 * L.nst;
    L.off_qfull = o; o += 16;
    L.off_qempty = o; o += 16;
    L.off_meta = o; o += 16 * L.nst;
    L.off_tinfo = o; o += 2 * sizeof(TInfo);
    L.off_flag = o; o += 16;
    o = (o + 127) & ~(size_t)127;
    L.off_stage = o; o += stage * L.nst;
    L.off_qbuf = o; o += 2 * (size_t)qg * row_bytes;
    L.off_qmeta = o; o += 2 * (size_t)qg * sizeof(QMeta);
    L.off_lists = o; o += (size_t)qg * k * 8;
    L.off_scratch = o; o += (size_t)kScanConsumers * (32 + 2 * k) * 8;
    L.off_dist = o; o += 2 * (size_t)qg * L.rps * 4;
    L.off_gid = o; o += 2 * (size_t)L.rps * 4;
    L.off_lcnt = o; o += (size_t)qg * 4;
    L.total = o;
    return L;
}

int scan_qg(int row_bytes, int k) { return scan_layout(row_bytes, k).qg; }

// warp-level top-k update of one query's per-warp list with 32 candidate keys (one per lane)
__device__ __forceinline__ void warp_topk_update(ull *L, int *cnt_p, ull key, int k, ull *cbuf, ull *tmp,
                                                 int lane) {
    const int cnt = *cnt_p;
    const ull thr = cnt < k ? KEY_INF : L[k - 1];
    const bool take = key < thr;
    const unsigned m = __ballot_sync(FULL, take);
    if (m == 0) return;
    const ull s = warp_sort32(take ? key : KEY_INF, lane);
    cbuf[lane] = s;
    __syncwarp();
    const int nn = warp_merge(L, cnt, cbuf, __popc(m), tmp, k, lane);
    for (int i = lane; i < nn; i += 32) L[i] = tmp[i];
    __syncwarp();
    if (lane == 0) *cnt_p = nn;
    __syncwarp();
}

// Write one item's final list to its destination (direct output row or the item's result slot).
__device__ __forceinline__ void write_final(const SearchArgs &a, const QMeta &q, const ull *L, int n, int k,
                                            int lane) {
    for (int t = lane; t < k; t += 32) {
        const ull key = t < n ? L[t] : KEY_INF;
        if (q.meta & META_DIRECT) {
            a.out_ids[(int64_t)q.qid * k + t] = key == KEY_INF ? -1 : (int32_t)key_id(key);
            a.out_dists[(int64_t)q.qid * k + t] = key == KEY_INF ? __uint_as_float(0x7f800000u) : key_dist(key);
        } else {
            a.item_res[(size_t)q.slot * k + t] = key;
        }
    }
}

// Distances of NQB queries against the NV rows of this lane's team; after the butterfly the owner
// lane of each row holds that row's distance for every query (see file header).
template <int DT, int TS, int CPLMAX, int NQB>
__device__ __forceinline__ void batch_dist(const uint8_t *__restrict__ rows, int row_bytes, int cpl, int tl,
                                           const uint4 (&q)[4][CPLMAX], typename Acc<DT>::T (&out)[4], int lane) {
    typedef Acc<DT> A;
    constexpr int NV = TS < 8 ? TS : 8;
    typename A::T acc[NQB][NV];
#pragma unroll
    for (int g = 0; g < NQB; g++)
#pragma unroll
        for (int i = 0; i < NV; i++) acc[g][i] = 0;
#pragma unroll
    for (int i = 0; i < NV; i++) {
        const uint4 *r = reinterpret_cast<const uint4 *>(rows + (size_t)i * row_bytes);
#pragma unroll
        for (int j = 0; j < CPLMAX; j++) {
            if (j < cpl) {
                const uint4 x = r[tl + j * TS];
#pragma unroll
                for (int g = 0; g < NQB; g++) A::add(acc[g][i], q[g][j], x);
            }
        }
    }
    // butterfly: halve the NV values per lane log2(NV) times, then full-reduce the rest of the team
#pragma unroll
    for (int g = 0; g < NQB; g++) {
#pragma unroll
        for (int s = 0; (1 << s) < NV; s++) {
            const int o = TS >> (s + 1);
            const int half = NV >> (s + 1);
            const bool up = (lane & o) != 0;
#pragma unroll
            for (int i = 0; i < half; i++) {
                const typename A::T send = up ? acc[g][i] : acc[g][i + half];
                const typename A::T keep = up ? acc[g][i + half] : acc[g][i];
                acc[g][i] = keep + __shfl_xor_sync(FULL, send, o);
            }
        }
#pragma unroll
        for (int o = TS / (2 * NV); o >= 1; o >>= 1) acc[g][0] += __shfl_xor_sync(FULL, acc[g][0], o);
        out[g] = acc[g][0];
    }
}

template <int DT, int TS, int CPLMAX>
__global__ void __launch_bounds__(kScanThreads, 1) k_scan(SearchArgs a, ScanLayout SL) {
    constexpr int NV = TS < 8 ? TS : 8;
    constexpr int BR = NV * (32 / TS);               // rows per warp batch
    typedef Acc<DT> A;
    extern __shared__ __align__(128) uint8_t smem[];
    uint64_t *full = reinterpret_cast<uint64_t *>(smem + SL.off_full);
    uint64_t *empty = reinterpret_cast<uint64_t *>(smem + SL.off_empty);
    uint64_t *qfull = reinterpret_cast<uint64_t *>(smem + SL.off_qfull);
    uint64_t *qempty = reinterpret_cast<uint64_t *>(smem + SL.off_qempty);
    int4 *meta = reinterpret_cast<int4 *>(smem + SL.off_meta);
    TInfo *tinfo = reinterpret_cast<TInfo *>(smem + SL.off_tinfo);
    int *flag = reinterpret_cast<int *>(smem + SL.off_flag);
    uint8_t *stages = smem + SL.off_stage;
    uint8_t *qbuf = smem + SL.off_qbuf;
    QMeta *qmeta = reinterpret_cast<QMeta *>(smem + SL.off_qmeta);
    ull *lists = reinterpret_cast<ull *>(smem + SL.off_lists);
    ull *scratch = reinterpret_cast<ull *>(smem + SL.off_scratch);
    int *lcnt = reinterpret_cast<int *>(smem + SL.off_lcnt);
    uint32_t *dtile = reinterpret_cast<uint32_t *>(smem + SL.off_dist);   // [2][qg][rps] distance bits
    int32_t *gtile = reinterpret_cast<int32_t *>(smem + SL.off_gid);      // [2][rps] global ids

    const DevIndex &ix = a.ix;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nst = SL.nst, rps = SL.rps, k = SL.k, qg = SL.qg, row_bytes = ix.row_bytes;
    if (gate_skip(a)) return;     // the tensor-core / u8 kernels took this batch

    if (threadIdx.x == 0) {
        for (int i = 0; i < nst; i++) {
            mbar_init(full + i, 1);
            mbar_init(empty + i, kScanConsumers);
        }
        for (int i = 0; i < 2; i++) {
            mbar_init(qfull + i, 1);
            mbar_init(qempty + i, kScanConsumers);
        }
        fence_mbar_init();
    }
    __syncthreads();

    if (warp == 0) {
        // ------------------------------------------------------------ producer
        uint32_t n = 0, tc = 0;
        const int ntiles = a.ctr->n_tiles;
        for (;;) {
            int t = 0;
            if (lane == 0) t = atomicAdd(&a.ctr->scan_next, 1);
            t = __shfl_sync(FULL, t, 0);
            if (t >= ntiles) {
                if (lane == 0) {
                    const int slot = n % nst;
                    mbar_wait(empty + slot, ((n / nst) & 1) ^ 1);
                    meta[slot] = make_int4(-1, 0, 0, ST_END);
                    mbar_arrive(full + slot);
                }
                break;
            }
            const Tile tl = a.tiles[t];
            const Segment sg = a.segs[tl.seg];
            const LabelDir d = ix.dir[sg.label];
            const bool hs = d.size >= ix.T;
            // -- query prefetch for this tile (double buffer by tile parity)
            const int tp = tc & 1;
            if (lane == 0) mbar_wait(qempty + tp, ((tc >> 1) & 1) ^ 1);
            __syncwarp();
            const int nq = sg.n_items;
            QMeta *qm = qmeta + (size_t)tp * qg;
            for (int g = lane; g < nq; g += 32) {
                const int s = a.scan_slots[sg.item_base + g];
                const Item it = a.items[s];
                QMeta m;
                m.p_off = a.q_off[it.qid];
                m.slot = s;
                m.qid = it.qid;
                m.meta = it.meta;
                m.nl = a.qinfo[it.qid].nl;
                m.pad[0] = m.pad[1] = 0;
                qm[g] = m;
            }
            if (lane == 0) {
                TInfo ti;
                ti.base = d.base;
                ti.tile = t; ti.seg = tl.seg; ti.label = sg.label; ti.nq = nq;
                ti.tile_in_seg = tl.tile_in_seg; ti.n_tiles = sg.n_tiles; ti.hs = hs; ti.pad = 0;
                tinfo[tp] = ti;
            }
            __syncwarp();
            __threadfence_block();
            if (lane == 0) mbar_arrive_expect_tx(qfull + tp, (uint32_t)nq * row_bytes);
            __syncwarp();
            for (int g = lane; g < nq; g += 32)
                tma_load_1d(qbuf + ((size_t)tp * qg + g) * row_bytes, a.Qp + (int64_t)qm[g].qid * row_bytes,
                            (uint32_t)row_bytes, qfull + tp);
            tc++;
            // -- row stages
            for (int r0 = tl.row_begin; r0 < tl.row_end; r0 += rps) {
                const int nr = min(rps, tl.row_end - r0);
                const int slot = n % nst;
                uint8_t *dst = stages + (size_t)slot * rps * row_bytes;
                const uint32_t bytes = (uint32_t)nr * row_bytes;
                if (lane == 0) {
                    mbar_wait(empty + slot, ((n / nst) & 1) ^ 1);
                    const int flags = (r0 == tl.row_begin ? ST_FIRST : 0) | (r0 + nr >= tl.row_end ? ST_LAST : 0);
                    meta[slot] = make_int4(t, r0, nr, flags);
                    mbar_arrive_expect_tx(full + slot, bytes);
                    if (!hs) tma_load_1d(dst, ix.Xls + (d.base + r0) * (int64_t)row_bytes, bytes, full + slot);
                }
                __syncwarp();
                if (hs) {
                    for (int r = lane; r < nr; r += 32) {
                        const int32_t gid = __ldg(ix.M_hs + d.base + r0 + r);
                        tma_load_1d(dst + (size_t)r * row_bytes, ix.X + (int64_t)gid * row_bytes,
                                    (uint32_t)row_bytes, full + slot);
                    }
                }
                n++;
            }
        }
        return;
    }

    // ---------------------------------------------------------------- consumers
    // Per stage: (1) every warp computes the exact distances of its rows for all queries of the
    // segment into the distance tile D[buf]; (2) one named barrier; (3) the warp owning query g
    // (g = cw mod 8) streams D[buf][g] into that query's single top-k list. One list per query
    // means ~k(1 + ln(rows/k)) insertions per tile instead of one re-filling list per warp.
    const int cw = warp - 1;
    const int ct = threadIdx.x - 32;
    const int tm = lane / TS, tl = lane % TS;
    const int r_own = tl / (TS / NV);                 // row of the team this lane owns after reduction
    const bool owner = (tl % (TS / NV)) == 0;
    const int cpl = SL.cpl;
    ull *cbuf = scratch + (size_t)cw * (32 + 2 * k);
    ull *tmp = cbuf + 32;
    ull *fin2 = tmp + k;
    unsigned long long my_rows = 0, my_qrows = 0;
    uint32_t n = 0, tc = 0;
    TInfo ti;
    ti.nq = 0;
    const QMeta *qm = qmeta;
    const uint8_t *qb = qbuf;
    const int32_t *gmap = ix.M_ls;
    int tp = 0;
    for (;;) {
        const int slot = n % nst;
        mbar_wait(full + slot, (n / nst) & 1);
        const int4 m = meta[slot];
        if (m.w & ST_END) break;
        if (m.w & ST_FIRST) {
            tp = tc & 1;
            mbar_wait(qfull + tp, (tc >> 1) & 1);
            ti = tinfo[tp];
            qm = qmeta + (size_t)tp * qg;
            qb = qbuf + (size_t)tp * qg * row_bytes;
            gmap = ti.hs ? ix.M_hs : ix.M_ls;
            for (int g = cw; g < ti.nq; g += kScanConsumers) {          // my queries' lists
                for (int e = lane; e < k; e += 32) lists[(size_t)g * k + e] = KEY_INF;
                if (lane == 0) lcnt[g] = 0;
            }
            __syncwarp();
        }
        const int nq = ti.nq, nr = m.z;
        const int buf = n & 1;
        uint32_t *D = dtile + (size_t)buf * qg * rps;
        int32_t *Gd = gtile + (size_t)buf * rps;
        const uint8_t *stage = stages + (size_t)slot * rps * row_bytes;
        // (1) distances
        for (int b0 = cw * BR; b0 < nr; b0 += kScanConsumers * BR) {
            const int trow0 = b0 + tm * NV;
            const int orow = trow0 + r_own;
            const bool ovalid = owner && orow < nr;
            const int32_t gid = ovalid ? __ldg(gmap + ti.base + m.y + orow) : -1;
            if (owner && orow < rps) Gd[orow] = gid;
            for (int g0 = 0; g0 < nq; g0 += 4) {
                const int nb = min(4, nq - g0);
                uint4 q[4][CPLMAX];
#pragma unroll
                for (int g = 0; g < 4; g++)
#pragma unroll
                    for (int j = 0; j < CPLMAX; j++)
                        q[g][j] = (g < nb && j < cpl)
                                      ? reinterpret_cast<const uint4 *>(qb + (size_t)(g0 + g) * row_bytes)[tl + j * TS]
                                      : make_uint4(0, 0, 0, 0);
                typename A::T dist[4];
                const uint8_t *rows = stage + (size_t)trow0 * row_bytes;
                if (nb == 1) batch_dist<DT, TS, CPLMAX, 1>(rows, row_bytes, cpl, tl, q, dist, lane);
                else if (nb == 2) batch_dist<DT, TS, CPLMAX, 2>(rows, row_bytes, cpl, tl, q, dist, lane);
                else batch_dist<DT, TS, CPLMAX, 4>(rows, row_bytes, cpl, tl, q, dist, lane);
                if (owner && orow < rps) {
                    for (int g = 0; g < nb; g++) {
                        uint32_t bits = DIST_EXCL;
                        if (ovalid) {
                            bits = __float_as_uint(A::to_float(dist[g]));
                            const QMeta &qq = qm[g0 + g];
                            if ((qq.meta & META_PRED) && !verify_pred(ix, gid, a.qlab + qq.p_off, qq.nl, ti.label))
                                bits = DIST_EXCL;
                        }
                        D[(size_t)(g0 + g) * rps + orow] = bits;
                    }
                }
            }
        }
        if (ct == 0) { my_rows += nr; my_qrows += (unsigned long long)nr * nq; }
        __syncwarp();
        if (lane == 0) mbar_arrive(empty + slot);
        // (2) the distance tile is complete
        named_bar_sync(1, 32 * kScanConsumers);
        // (3) selection: my queries' lists absorb this stage's keys
        for (int g = cw; g < nq; g += kScanConsumers) {
            ull *L = lists + (size_t)g * k;
            const uint32_t *Dg = D + (size_t)g * rps;
            if (k <= 32) {
                ull Li = lane < k ? L[lane] : KEY_INF;
                for (int r0 = 0; r0 < nr; r0 += 32) {
                    const int r = r0 + lane;
                    const uint32_t bits = r < nr ? Dg[r] : DIST_EXCL;
                    const ull key = bits == DIST_EXCL ? KEY_INF : (((ull)bits << 32) | (uint32_t)Gd[r]);
                    Li = warp_insert_topk(Li, key, k, lane);
                }
                if (lane < k) L[lane] = Li;
            } else {
                for (int r0 = 0; r0 < nr; r0 += 32) {
                    const int r = r0 + lane;
                    const uint32_t bits = r < nr ? Dg[r] : DIST_EXCL;
                    const ull key = bits == DIST_EXCL ? KEY_INF : (((ull)bits << 32) | (uint32_t)Gd[r]);
                    warp_topk_update(L, lcnt + g, key, k, cbuf, tmp, lane);
                }
            }
            __syncwarp();
        }
        if (m.w & ST_LAST) {
            const bool multi = ti.n_tiles > 1;
            for (int g = cw; g < nq; g += kScanConsumers) {
                const ull *L = lists + (size_t)g * k;
                const int na = k <= 32 ? __popc(__ballot_sync(FULL, lane < k && L[lane < k ? lane : 0] != KEY_INF))
                                       : lcnt[g];
                if (multi) {
                    for (int t = lane; t < k; t += 32)
                        a.partials[((size_t)qm[g].slot * a.max_tiles_per_label + ti.tile_in_seg) * k + t] =
                            t < na ? L[t] : KEY_INF;
                } else {
                    write_final(a, qm[g], L, na, k, lane);
                }
                __syncwarp();
            }
            if (multi) {
                // last-block-done: the CTA completing the segment's last tile merges the partials
                __threadfence();
                named_bar_sync(1, 32 * kScanConsumers);
                if (ct == 0) flag[0] = atomicAdd(&a.segs[ti.seg].done, 1) == ti.n_tiles - 1;
                named_bar_sync(1, 32 * kScanConsumers);
                if (flag[0]) {
                    __threadfence();
                    for (int g = cw; g < nq; g += kScanConsumers) {
                        ull *A0 = tmp, *B0 = fin2;
                        int na = 0;
                        for (int t2 = 0; t2 < ti.n_tiles; t2++) {
                            const volatile ull *P =
                                a.partials + ((size_t)qm[g].slot * a.max_tiles_per_label + t2) * k;
                            ull *C = cbuf;                    // stage the partial list 32 keys at a time
                            for (int c0 = 0; c0 < k; c0 += 32) {
                                const int cn = min(32, k - c0);
                                ull v = lane < cn ? P[c0 + lane] : KEY_INF;
                                C[lane] = v;
                                __syncwarp();
                                int nc = __popc(__ballot_sync(FULL, v != KEY_INF));
                                na = warp_merge(A0, na, C, nc, B0, k, lane);
                                ull *t3 = A0; A0 = B0; B0 = t3;
                                __syncwarp();
                            }
                        }
                        write_final(a, qm[g], A0, na, k, lane);
                        __syncwarp();
                    }
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(qempty + tp);   // this warp is done with the tile's queries
            tc++;
        }
        n++;
    }
    if (ct == 0 && my_rows) {
        atomicAdd(&a.ctr->scan_rows, my_rows);
        atomicAdd(&a.ctr->scan_qrows, my_qrows);
    }
}

// ------------------------------------------------------------------ dispatch
typedef void (*scan_fn)(SearchArgs, ScanLayout);

template <int DT>
static scan_fn scan_pick(int ts, int cpl) {
#define VF_S(T_, C_) if (ts == T_ && cpl <= C_) return k_scan<DT, T_, C_>;
    VF_S(32, 1) VF_S(32, 2) VF_S(32, 4) VF_S(32, 8) VF_S(16, 1) VF_S(16, 2) VF_S(16, 4)
    VF_S(8, 1) VF_S(8, 2) VF_S(8, 4) VF_S(4, 1) VF_S(4, 2) VF_S(4, 4) VF_S(2, 1) VF_S(2, 2) VF_S(2, 4)
#undef VF_S
    return nullptr;
}

int launch_scan(const SearchArgs &a, cudaStream_t s, int max_tiles_bound) {
    if (max_tiles_bound <= 0) return 0;
    const ScanLayout SL = scan_layout(a.ix.row_bytes, a.k);
    scan_fn f = a.ix.dtype == 0 ? scan_pick<0>(SL.ts, SL.cpl) : scan_pick<1>(SL.ts, SL.cpl);
    if (!f) return -1;
    // per-(kernel, device) setup cached: attribute calls cost microseconds per small batch
    struct Key { scan_fn f; int dev, smem, nsm; };
    static thread_local Key cache[16];
    static thread_local int ncache = 0;
    int dev = 0, nsm = -1;
    cudaGetDevice(&dev);
    for (int i = 0; i < ncache && i < 16; i++)
        if (cache[i].f == f && cache[i].dev == dev && cache[i].smem == (int)SL.total) nsm = cache[i].nsm;
    if (nsm < 0) {
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
        cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);   // ceiling, per function
        cache[ncache % 16] = Key{f, dev, (int)SL.total, nsm};
        ncache++;
    }
    int grid = nsm;
    if (grid > max_tiles_bound) grid = max_tiles_bound;
    f<<<grid, kScanThreads, SL.total, s>>>(a, SL);
    return 1;
}

}  // namespace vf
