// a2 -- IVF-BFS for low-specificity labels (Alg. 2), redesigned
// for sm_100a as a label-grouped scan: all queries routed to one LS label in this batch (a
// "segment", up to QG of them) share ONE pass over the label's rows, so every touched posting
// list is read from HBM once per batch.
//
// Persistent CTAs, warp-specialised:
//   warp 0 (producer, one elected lane): claims row tiles with an atomic counter and streams each
//     tile's rows -- contiguous in the label-grouped X_LS store -- into a ring of shared-memory
//     stages with 1-D TMA bulk copies (cp.async.bulk, completion counted in bytes on an mbarrier).
//   warps 1-4 (consumers): one row per thread per stage; exact squared L2 against every query of
//     the segment held in shared memory (u8: vabsdiff4+dp4a int32; f32: FFMA), then a warp top-k
//     update (ballot against the k-th key, bitonic sort + rank merge only when a key qualifies).
//     AND items mask rows that fail the predicate (equivalent to the paper's pre-filter, reading
//     #21). At a tile's last stage the four warp lists are merged and written.
// The row-to-thread mapping reads the 16-byte chunks of a row in a lane-rotated order, so the 8
// lanes of a quarter-warp hit 8 different bank groups (conflict-free for 512-byte rows).
#include "common.cuh"

namespace vf {

constexpr int kScanConsumers = 4;
constexpr int kScanThreads = 32 * (1 + kScanConsumers);
enum : int { ST_FIRST = 1, ST_LAST = 2, ST_END = 4 };

struct ScanLayout {
    int nst, rps, qg, k, row_bytes;
    size_t off_full, off_empty, off_meta, off_stage, off_q, off_lists, off_lcnt, off_scratch,
        off_qmeta, total;
};

static ScanLayout scan_layout(int row_bytes, int k, int qg) {
    ScanLayout L;
    L.row_bytes = row_bytes;
    L.k = k;
    L.qg = qg;
    L.rps = 32 * kScanConsumers;
    while (L.rps > 32 && (size_t)L.rps * row_bytes * 2 > 112 * 1024) L.rps -= 32;
    const size_t stage = (size_t)L.rps * row_bytes;
    L.nst = (int)((120 * 1024) / stage);
    if (L.nst < 2) L.nst = 2;
    if (L.nst > 8) L.nst = 8;
    size_t o = 0;
    L.off_full = o; o += 8 * L.nst;
    L.off_empty = o; o += 8 * L.nst;
    L.off_meta = o; o += 16 * L.nst;
    o = (o + 127) & ~(size_t)127;
    L.off_stage = o; o += stage * L.nst;
    L.off_q = o; o += (size_t)qg * row_bytes;
    L.off_lists = o; o += (size_t)kScanConsumers * qg * k * 8;
    L.off_scratch = o; o += (size_t)kScanConsumers * (32 + 2 * k) * 8;
    L.off_lcnt = o; o += (size_t)kScanConsumers * qg * 4;
    L.off_qmeta = o; o += (size_t)qg * 32;
    L.total = o;
    return L;
}

int scan_qg(int row_bytes, int k) {
    int qg = kScanQG;
    while (qg > 1 && ((size_t)qg * row_bytes > 32 * 1024 ||
                      (size_t)kScanConsumers * qg * k * 8 > 40 * 1024))
        qg >>= 1;
    return qg;
}

struct QMeta {          // per query of the current segment
    int64_t p_off;      // offset of the query's sorted labels (predicate)
    int32_t slot, qid;
    uint32_t meta;
    int32_t nl;
    int32_t pad[2];
};

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

template <int DT>
__global__ void __launch_bounds__(kScanThreads, 1) k_scan(SearchArgs a, ScanLayout SL) {
    extern __shared__ __align__(128) uint8_t smem[];
    uint64_t *full = reinterpret_cast<uint64_t *>(smem + SL.off_full);
    uint64_t *empty = reinterpret_cast<uint64_t *>(smem + SL.off_empty);
    int4 *meta = reinterpret_cast<int4 *>(smem + SL.off_meta);
    uint8_t *stages = smem + SL.off_stage;
    const uint4 *qsm = reinterpret_cast<const uint4 *>(smem + SL.off_q);
    ull *lists = reinterpret_cast<ull *>(smem + SL.off_lists);
    ull *scratch = reinterpret_cast<ull *>(smem + SL.off_scratch);
    int *lcnt = reinterpret_cast<int *>(smem + SL.off_lcnt);
    QMeta *qm = reinterpret_cast<QMeta *>(smem + SL.off_qmeta);

    const DevIndex &ix = a.ix;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nst = SL.nst, rps = SL.rps, k = SL.k, row_bytes = ix.row_bytes;

    if (threadIdx.x == 0) {
        for (int i = 0; i < nst; i++) {
            mbar_init(full + i, 1);
            mbar_init(empty + i, kScanConsumers);
        }
        fence_mbar_init();
    }
    __syncthreads();

    if (warp == 0) {
        // ------------------------------------------------------------ producer (warp 0)
        // LS labels: one bulk copy of the tile's contiguous X_LS rows per stage. In exact mode an
        // HS label is scanned too; its rows are gathered from X through M_HS, one bulk copy per row
        // issued by all 32 lanes (no duplicated vectors).
        uint32_t n = 0;
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
    typedef Acc<DT> A;
    const int cw = warp - 1;                 // consumer warp 0..3
    const int ct = threadIdx.x - 32;         // consumer thread 0..127
    const int chunks = ix.chunks;
    ull *cbuf = scratch + (size_t)cw * (32 + 2 * k);
    ull *tmp = cbuf + 32;
    ull *fin2 = tmp + k;
    int nq = 0, label = 0, tile_in_seg = 0;
    int64_t lbase = 0;
    const int32_t *gmap = ix.M_ls;   // local row -> global id (M_LS, or M_HS in exact mode)
    unsigned long long my_rows = 0, my_qrows = 0;
    uint32_t n = 0;
    for (;;) {
        const int slot = n % nst;
        mbar_wait(full + slot, (n / nst) & 1);
        const int4 m = meta[slot];
        if (m.w & ST_END) break;
        if (m.w & ST_FIRST) {
            named_bar_sync(1, 32 * kScanConsumers);
            const Tile tl = a.tiles[m.x];
            const Segment sg = a.segs[tl.seg];
            nq = sg.n_items;
            label = sg.label;
            tile_in_seg = tl.tile_in_seg;
            lbase = ix.dir[label].base;
            gmap = ix.dir[label].size >= ix.T ? ix.M_hs : ix.M_ls;
            if (ct < nq) {
                const int s = a.scan_slots[sg.item_base + ct];
                const Item it = a.items[s];
                QMeta q;
                q.slot = s; q.qid = it.qid; q.meta = it.meta;
                q.p_off = a.q_off[it.qid];
                q.nl = a.qinfo[it.qid].nl;
                qm[ct] = q;
            }
            for (int i = ct; i < nq * kScanConsumers; i += 32 * kScanConsumers) lcnt[i] = 0;
            named_bar_sync(1, 32 * kScanConsumers);
            uint4 *qdst = reinterpret_cast<uint4 *>(smem + SL.off_q);
            for (int e = ct; e < nq * chunks; e += 32 * kScanConsumers) {
                const int g = e / chunks, c = e - g * chunks;
                qdst[e] = __ldg(reinterpret_cast<const uint4 *>(a.Qp + (int64_t)qm[g].qid * row_bytes) + c);
            }
            named_bar_sync(1, 32 * kScanConsumers);
        }
        // -- compute: thread ct owns row ct of the stage
        const int nr = m.z;
        const bool valid = ct < nr;
        const uint4 *rowp = reinterpret_cast<const uint4 *>(stages + (size_t)slot * rps * row_bytes +
                                                            (size_t)ct * row_bytes);
        const int32_t gid = valid ? __ldg(gmap + lbase + m.y + ct) : -1;
        const int rot = ct % chunks;
        for (int g0 = 0; g0 < nq; g0 += 8) {
            typename A::T acc[8];
#pragma unroll
            for (int g = 0; g < 8; g++) acc[g] = 0;
            if (valid) {
                int cc = rot;
                for (int c = 0; c < chunks; c++) {
                    const uint4 xv = rowp[cc];
#pragma unroll
                    for (int g = 0; g < 8; g++)
                        if (g0 + g < nq) A::add(acc[g], qsm[(g0 + g) * chunks + cc], xv);
                    cc = cc + 1 == chunks ? 0 : cc + 1;
                }
            }
#pragma unroll
            for (int g = 0; g < 8; g++) {
                if (g0 + g >= nq) break;
                ull key = KEY_INF;
                if (valid) {
                    key = make_key(A::to_float(acc[g]), (uint32_t)gid);
                    const QMeta &q = qm[g0 + g];
                    if ((q.meta & META_PRED) && !verify_pred(ix, gid, a.qlab + q.p_off, q.nl, label))
                        key = KEY_INF;
                }
                const int li = cw * nq + g0 + g;
                warp_topk_update(lists + (size_t)li * k, lcnt + li, key, k, cbuf, tmp, lane);
            }
        }
        if (ct == 0) { my_rows += nr; my_qrows += (unsigned long long)nr * nq; }
        __syncwarp();
        if (lane == 0) mbar_arrive(empty + slot);
        if (m.w & ST_LAST) {
            // -- merge the four warp lists of every query and write the tile's results
            named_bar_sync(1, 32 * kScanConsumers);
            for (int g = cw; g < nq; g += kScanConsumers) {
                ull *A0 = tmp, *B0 = fin2;
                int na = lcnt[0 * nq + g];
                for (int i = lane; i < na; i += 32) A0[i] = lists[(size_t)(0 * nq + g) * k + i];
                __syncwarp();
                for (int w2 = 1; w2 < kScanConsumers; w2++) {
                    const int li = w2 * nq + g;
                    na = warp_merge(A0, na, lists + (size_t)li * k, lcnt[li], B0, k, lane);
                    ull *t2 = A0; A0 = B0; B0 = t2;
                }
                const QMeta &q = qm[g];
                for (int t = lane; t < k; t += 32) {
                    const ull key = t < na ? A0[t] : KEY_INF;
                    if (q.meta & META_MULTI) {
                        a.partials[((size_t)q.slot * a.max_tiles_per_label + tile_in_seg) * k + t] = key;
                    } else if (q.meta & META_DIRECT) {
                        a.out_ids[(int64_t)q.qid * k + t] = key == KEY_INF ? -1 : (int32_t)key_id(key);
                        a.out_dists[(int64_t)q.qid * k + t] =
                            key == KEY_INF ? __uint_as_float(0x7f800000u) : key_dist(key);
                    } else {
                        a.item_res[(size_t)q.slot * k + t] = key;
                    }
                }
                __syncwarp();
            }
            named_bar_sync(1, 32 * kScanConsumers);
        }
        n++;
    }
    if (ct == 0 && my_rows) {
        atomicAdd(&a.ctr->scan_rows, my_rows);
        atomicAdd(&a.ctr->scan_qrows, my_qrows);
    }
}

int launch_scan(const SearchArgs &a, cudaStream_t s, int max_tiles_bound) {
    if (max_tiles_bound <= 0) return 0;
    const int qg = scan_qg(a.ix.row_bytes, a.k);
    const ScanLayout SL = scan_layout(a.ix.row_bytes, a.k, qg);
    int dev = 0, nsm = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    int grid = nsm;
    if (grid > max_tiles_bound) grid = max_tiles_bound;
    if (a.ix.dtype == 0) {
        cudaFuncSetAttribute(k_scan<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SL.total);
        k_scan<0><<<grid, kScanThreads, SL.total, s>>>(a, SL);
    } else {
        cudaFuncSetAttribute(k_scan<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SL.total);
        k_scan<1><<<grid, kScanThreads, SL.total, s>>>(a, SL);
    }
    return 1;
}

}  // namespace vf
