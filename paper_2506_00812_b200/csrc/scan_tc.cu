// a2 on the 5th-generation tensor cores -- the label-grouped exact scan (Alg. 2;
// P:L466-L469) as a tcgen05 contraction: kind::i8 for u8 vectors and
// kind::tf32 for fp32 vectors whose values are integers small enough that every product and
// partial sum is exact in fp32 (C5; checked per index at build and per batch for the queries --
// a batch with any other query runs k_scan instead).
//
// Same work decomposition as k_scan (scan.cu): persistent CTAs claim row tiles of one segment
// (an LS label with up to QG of this batch's queries). What changes is where the distances come
// from. For u8, ||x - q||^2 = ||x||^2 + ||q||^2 - 2 q.x with every term an exact int32 (D*255^2 <
// 2^24), so the query-group x row-tile dot products are one tcgen05.mma.kind::i8 per 32-byte K
// step (M = 128 rows, N = the segment's queries padded to 16), accumulated exactly in TMEM.
//
// 352 threads, warp-specialised (an epilogue and a selection group pipelined through mbarriers):
//   warp 10 tile scheduler: claims tiles and resolves their metadata into a double-buffered tile
//           slot ahead of the producer (no global round trip between consecutive tiles' stages).
//   warp 0  producer: claims tiles, prefetches the segment's query rows + metadata (double buffer
//           by tile parity), and per 128-row stage issues 2-D TMA tensor loads of the rows in the
//           128/64/32-byte-swizzled K-major layout the MMA reads (LS: one box per K chunk of the
//           label-contiguous X_LS; HS rows in exact / f3 mode: TMA tile::gather4 of 4 rows per chunk from
//           X through M_HS), plus the rows' global ids and precomputed norms.
//   warp 1  MMA: owns the TMEM allocation (2 accumulator buffers); per tile it converts the query
//           rows into the swizzled B operand, per stage one elected lane issues the K-step MMAs
//           and commits them to the accumulator's mbarrier.
//   warps 2-5 epilogue: a warp reads its TMEM lane quarter (32 rows) for every query column,
//           forms exact distances, drops every (row, query) pair whose key is not below the
//           query's current k-th key (a stale threshold only lets more through) or that fails the
//           AND predicate, and publishes survivors as per-query 128-bit masks (double-buffered).
//   warps 6-9 selection: the warp owning a query inserts only its surviving rows into the
//           query's register-resident top-k list while the epilogue works on the next stage.
//           Multi-tile segments are finished as in k_scan.
#include <cuda.h>
#include <cstdio>
#include <cstdlib>
#include "common.cuh"
#include "tc_common.cuh"

namespace vf {

namespace {

constexpr int kTcThreads = 352;
constexpr int kTcEpiW = 4;            // epilogue warps (one per TMEM lane quarter)
constexpr int kTcSelW = 4;            // selection warps
constexpr int kTcRows = 128;          // rows per stage = MMA M
enum : int { TS_FIRST = 1, TS_LAST = 2, TS_END = 4 };

struct TcQMeta {
    int64_t p_off;
    int32_t slot, qid;
    uint32_t meta;
    int32_t nl;
    int32_t pad[2];
};

struct TcTInfo {
    int64_t base;
    int32_t tile, seg, label, nq, tile_in_seg, n_tiles, hs, row_begin, row_end, n_pieces, bits_off;
    int32_t piece_off[kMaxPieces], piece_cnt[kMaxPieces];
};

}  // namespace

struct TcLayout {
    int nst, qg, k, row_bytes, cw, nch, kpad, nmax, tmem_cols, ctas;
    size_t off_bar, off_misc, off_meta, off_tinfo, off_rows, off_sid, off_snorm, off_sbits, off_qbuf, off_bsm, off_qmeta,
        off_qn, off_thr, off_lists, off_lcnt, off_scratch, off_dist, off_gid, off_mask, off_sinfo, total;
};

constexpr int kTcCtasPerSm = 2;       // up to two independent pipelines per SM (latency-bound chains)

// K chunk (swizzle width) of the row tiles: the largest of 128 / 64 / 32 B dividing the row, or with
// VF_TC_CW=128 always 128 B (rows padded to a multiple of 128 in shared memory: the TMA fills the
// bytes past the row with zeros without reading them, so a 192-B row costs 2 tile::gather4 requests
// per 4 rows instead of 3; the zero columns add nothing to the dot products). Read once per process:
// the tensor maps (index build) and the layout (each search) must agree.
static int tc_chunk_bytes(int row_bytes) {
    static const int force = [] { const char *e = getenv("VF_TC_CW"); return e ? atoi(e) : 0; }();
    if (force == 128 && row_bytes > 64) return 128;
    return row_bytes % 128 == 0 ? 128 : row_bytes % 64 == 0 ? 64 : 32;
}

static TcLayout tc_layout_for(int row_bytes, int k, int ctas) {
    TcLayout L{};
    L.ctas = ctas;
    L.row_bytes = row_bytes;
    L.k = k;
    L.cw = tc_chunk_bytes(row_bytes);
    L.kpad = (row_bytes + L.cw - 1) / L.cw * L.cw;
    L.nch = L.kpad / L.cw;
    const size_t stage = (size_t)kTcRows * L.kpad;
    auto stages_for = [&](int qg) {
        const size_t nmax = (size_t)(qg + 15) / 16 * 16;
        const size_t fixed = 2048 + 2 * (size_t)qg * row_bytes + 2 * (size_t)L.nch * nmax * L.cw + 2 * (size_t)qg * 32 +
                             2 * (size_t)qg * 4 + 2 * (size_t)qg * 8 + 2 * (size_t)qg * k * 8 + 2 * (size_t)qg * 4 +
                             (size_t)kTcSelW * (32 + 2 * k) * 8 + 2 * (size_t)qg * kTcRows * 4 + 2 * kTcRows * 4 +
                             2 * (size_t)qg * 16 + 4096;
        const size_t budget = (227 * 1024) / ctas - 2048;
        return fixed >= budget ? 0 : (int)((budget - fixed) / (stage + 2 * kTcRows * 4 + kTcRows * 8));
    };
    // queries per segment: as many as keep >= 3 row stages in flight per CTA (>= 2 for wide rows)
    int qg = kScanQG;
    while (qg > 16 && ((size_t)qg * k * 8 > 8 * 1024 || (size_t)qg * row_bytes > 8 * 1024 || stages_for(qg) < 3))
        qg >>= 1;
    L.qg = qg;
    L.nmax = (qg + 15) / 16 * 16;
    int cols = 32;
    while (cols < 2 * L.nmax) cols <<= 1;
    L.tmem_cols = cols;
    int nst = stages_for(qg);
    if (nst > 6) nst = 6;
    L.nst = nst;
    size_t o = 0;
    auto take = [&](size_t bytes, size_t align) {
        o = (o + align - 1) / align * align;
        const size_t r = o;
        o += bytes;
        return r;
    };
    L.off_bar = take(8 * (2 * (size_t)nst + 16), 8);
    L.off_misc = take(16, 16);
    L.off_sinfo = take(2 * 16, 16);
    L.off_meta = take(16 * (size_t)nst, 16);
    L.off_tinfo = take(2 * sizeof(TcTInfo), 16);
    L.off_rows = take(stage * nst, 1024);
    L.off_bsm = take(2 * (size_t)L.nch * L.nmax * L.cw, 1024);
    L.off_sid = take((size_t)nst * kTcRows * 4, 16);
    L.off_snorm = take((size_t)nst * kTcRows * 4, 16);
    L.off_sbits = take((size_t)nst * kTcRows * 8, 16);
    L.off_qbuf = take(2 * (size_t)qg * row_bytes, 16);
    L.off_qmeta = take(2 * (size_t)qg * sizeof(TcQMeta), 16);
    L.off_qn = take(2 * (size_t)qg * 4, 16);
    L.off_thr = take(2 * (size_t)qg * 8, 16);           // per tile parity
    L.off_lists = take(2 * (size_t)qg * k * 8, 16);
    L.off_lcnt = take(2 * (size_t)qg * 4, 16);
    L.off_scratch = take((size_t)kTcSelW * (32 + 2 * k) * 8, 16);
    L.off_dist = take(2 * (size_t)qg * kTcRows * 4, 16);
    L.off_gid = take(2 * (size_t)kTcRows * 4, 16);
    L.off_mask = take(2 * (size_t)qg * 16, 16);
    L.total = o + 1024;     // slack for aligning the dynamic window to 1024 bytes
    if (L.total > (size_t)(227 * 1024) / ctas) L.nst = 0;
    return L;
}

// two CTAs per SM when the row size leaves >= 2 stages each, else one (nst < 2: k_scan instead)
static TcLayout tc_layout(int row_bytes, int k) {
    // VF_TC_LAYOUT_CTAS=1 / 2 forces the layout's CTAs per SM (read once; A/B of pipeline depth:
    // one CTA holds more stages in flight, two run two independent chains)
    static const int force = [] { const char *e = getenv("VF_TC_LAYOUT_CTAS"); return e ? atoi(e) : 0; }();
    if (force == 1 || force == 2) {
        const TcLayout F = tc_layout_for(row_bytes, k, force);
        if (F.nst >= 2) return F;
    }
    const TcLayout L2 = tc_layout_for(row_bytes, k, 2);
    return L2.nst >= 2 ? L2 : tc_layout_for(row_bytes, k, 1);
}

int scan_tc_qg(int row_bytes, int k) {
    const TcLayout L = tc_layout(row_bytes, k);
    return L.nst >= 2 ? L.qg : 0;     // 0: this (row size, k) does not fit the tensor-core scan
}

// Diagnostics build (-DVF_TC_PROF): per-role cycle breakdown of CTAs 0-1, printed at exit.
#ifdef VF_TC_PROF
#define TP_DECL unsigned long long tp_acc[8] = {0, 0, 0, 0, 0, 0, 0, 0}, tp_t0 = clock64();
#define TP_MARK(i) { const unsigned long long t1_ = clock64(); tp_acc[i] += t1_ - tp_t0; tp_t0 = t1_; }
#define TP_DUMP(name) if (lane == 0 && blockIdx.x < 2) \
    printf("TCPROF blk %d warp %d %s: %llu %llu %llu %llu %llu %llu %llu %llu\n", blockIdx.x, warp, name, tp_acc[0], \
           tp_acc[1], tp_acc[2], tp_acc[3], tp_acc[4], tp_acc[5], tp_acc[6], tp_acc[7]);
#else
#define TP_DECL
#define TP_MARK(i)
#define TP_DUMP(name)
#endif

// position of the j-th (0-based) set bit of w (j < popc(w)): binary search on popcounts
__device__ __forceinline__ int nth_bit(uint32_t w, int j) {
    int pos = 0;
#pragma unroll
    for (int sh = 16; sh > 0; sh >>= 1) {
        const int c = __popc(w & ((1u << sh) - 1));
        if (j >= c) { j -= c; w >>= sh; pos += sh; }
    }
    return pos;
}

// The survivors of one 128-row stage for one query, compacted: candidate c (c < popc(mask & wsel))
// of the stage's four 32-row words lands in lane c (lanes past the count get KEY_INF). Words not
// selected by `wsel` (bit w4) belong to another warp. Returns the number of candidates.
__device__ __forceinline__ int stage_candidates(const uint32_t *Mk4, unsigned wsel, const uint32_t *Dg,
                                                const int32_t *Gd, int base, int lane, ull &key) {
    const uint4 mw = *reinterpret_cast<const uint4 *>(Mk4);
    const uint32_t w0 = (wsel & 1) ? mw.x : 0u, w1 = (wsel & 2) ? mw.y : 0u;
    const uint32_t w2 = (wsel & 4) ? mw.z : 0u, w3 = (wsel & 8) ? mw.w : 0u;
    const int c0 = __popc(w0), c1 = c0 + __popc(w1), c2 = c1 + __popc(w2), c3 = c2 + __popc(w3);
    const int c = base + lane;
    key = KEY_INF;
    if (c < c3) {
        int r;
        if (c < c0) r = nth_bit(w0, c);
        else if (c < c1) r = 32 + nth_bit(w1, c - c0);
        else if (c < c2) r = 64 + nth_bit(w2, c - c1);
        else r = 96 + nth_bit(w3, c - c2);
        key = ((ull)Dg[r] << 32) | (uint32_t)Gd[r];
    }
    return c3;
}

// Out-of-line copies of the large warp helpers: eleven warps in five roles share one instruction
// cache, and inlining these (bitonic networks, binary searches) at every call site tripled the
// kernel's code size (ncu: no_instructions stalls).
__device__ __noinline__ ull merge_topk_ol(ull Li, ull key, int k, int lane) {
    return warp_merge_topk(Li, key, k, lane);
}
__device__ __noinline__ bool verify_pred_ol(const DevIndex &ix, int32_t gid, const int32_t *P, int np,
                                            int32_t excl) {
    return verify_pred(ix, gid, P, np, excl);
}

__device__ __forceinline__ void write_final_tc(const SearchArgs &a, const TcQMeta &q, const ull *L, int n, int k,
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

__device__ __noinline__ void topk_update_tc(ull *L, int *cnt_p, ull key, int k, ull *cbuf, ull *tmp, int lane) {
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
__global__ void __launch_bounds__(kTcThreads, kTcCtasPerSm)
    k_scan_tc(SearchArgs a, TcLayout SL, const __grid_constant__ CUtensorMap tm_ls,
              const __grid_constant__ CUtensorMap tm_x) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
    const int nst = SL.nst, qg = SL.qg, k = SL.k, row_bytes = SL.row_bytes, cw = SL.cw, nch = SL.nch;
    const int kpad = SL.kpad, nmax = SL.nmax;
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem + SL.off_bar);
    uint64_t *full = bars, *empty = bars + nst;
    uint64_t *qfull = bars + 2 * nst, *qempty = qfull + 2, *accfull = qfull + 4, *accempty = qfull + 6;
    uint64_t *tready = qfull + 8, *dready = qfull + 10, *dfree = qfull + 12, *tfree = qfull + 14;
    int4 *sinfo = reinterpret_cast<int4 *>(smem + SL.off_sinfo);
    uint32_t *misc = reinterpret_cast<uint32_t *>(smem + SL.off_misc);   // [0] TMEM base, [1] flag
    int4 *meta = reinterpret_cast<int4 *>(smem + SL.off_meta);
    TcTInfo *tinfo = reinterpret_cast<TcTInfo *>(smem + SL.off_tinfo);
    uint8_t *rows = smem + SL.off_rows;
    uint8_t *bsm = smem + SL.off_bsm;
    int32_t *sid = reinterpret_cast<int32_t *>(smem + SL.off_sid);
    uint32_t *snorm = reinterpret_cast<uint32_t *>(smem + SL.off_snorm);
    unsigned long long *sbits = reinterpret_cast<unsigned long long *>(smem + SL.off_sbits);
    uint8_t *qbuf = smem + SL.off_qbuf;
    TcQMeta *qmeta = reinterpret_cast<TcQMeta *>(smem + SL.off_qmeta);
    uint32_t *qn = reinterpret_cast<uint32_t *>(smem + SL.off_qn);
    ull *thr = reinterpret_cast<ull *>(smem + SL.off_thr);
    ull *lists = reinterpret_cast<ull *>(smem + SL.off_lists);
    int *lcnt = reinterpret_cast<int *>(smem + SL.off_lcnt);
    ull *scratch = reinterpret_cast<ull *>(smem + SL.off_scratch);
    uint32_t *dtile = reinterpret_cast<uint32_t *>(smem + SL.off_dist);
    int32_t *gtile = reinterpret_cast<int32_t *>(smem + SL.off_gid);
    uint32_t *mask = reinterpret_cast<uint32_t *>(smem + SL.off_mask);

    const DevIndex &ix = a.ix;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const size_t stage_bytes = (size_t)kTcRows * kpad;
    if (gate_skip(a)) return;     // a batch outside the exact range runs k_scan instead
    if (threadIdx.x == 0) atomicMax(&a.ctr->scan_t0_inv, ~gtimer());
#ifdef VF_TC_PROF
    const unsigned long long cta_t0 = gtimer();
#endif

    if (threadIdx.x == 0) {
        for (int i = 0; i < nst; i++) {
            mbar_init(full + i, 1);
            mbar_init(empty + i, kTcEpiW);
        }
        for (int i = 0; i < 2; i++) {
            mbar_init(qfull + i, 1);
            mbar_init(qempty + i, kTcSelW);
            mbar_init(accfull + i, 1);
            mbar_init(accempty + i, kTcEpiW);
            mbar_init(tready + i, 1);
            mbar_init(dready + i, kTcEpiW);
            mbar_init(dfree + i, kTcSelW);
            mbar_init(tfree + i, kTcSelW);
        }
        fence_mbar_init();
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(misc)),
                     "r"(SL.tmem_cols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    for (int i = threadIdx.x; i < 2 * qg * k; i += kTcThreads) lists[i] = KEY_INF;
    for (int i = threadIdx.x; i < 2 * qg; i += kTcThreads) { thr[i] = KEY_INF; lcnt[i] = 0; }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tbase = misc[0];

    if (warp == 10) {
        // ------------------------------------------------------------ tile scheduler
        // Claims tiles and resolves their metadata (Tile record, per-query ScanQuery records) into
        // the tile slot of its parity ahead of the producer, so no dependent global round trip sits
        // between one tile's last row stage and the next tile's first.
        uint32_t tc = 0;
        const bool by_cls = a.tile_cls != nullptr;          // longest tiles first (row-count classes)
        int cum[kTileClasses + 1];
        cum[0] = 0;
        for (int c = 0; c < kTileClasses; c++) cum[c + 1] = cum[c] + (by_cls ? a.ctr->n_tile_cls[c] : 0);
        // with the claim lists every claimable tile is listed there (packed segments are not,
        // their packed tile is)
        const int ntiles = by_cls ? cum[kTileClasses] : a.ctr->n_tiles;
        TP_DECL
        for (;;) {
            const int tp = tc & 1;
            TP_MARK(3)
            if (lane == 0) mbar_wait(qempty + tp, ((tc >> 1) & 1) ^ 1);
            __syncwarp();
            TP_MARK(0)
            int t = 0;
            if (lane == 0) t = atomicAdd(&a.ctr->scan_next, 1);
            t = __shfl_sync(FULL, t, 0);
            if (t < ntiles && by_cls) {
                int c = 0;
                while (c + 1 < kTileClasses && t >= cum[c + 1]) c++;
                t = a.tile_cls[(int64_t)c * a.max_tiles + (t - cum[c])];
            } else if (t >= ntiles) t = INT32_MAX;
            if (t == INT32_MAX) {
                if (lane == 0) {
                    tinfo[tp].tile = -1;
                    mbar_arrive(tready + tp);
                }
                break;
            }
            const Tile tl = a.tiles[t];
            TP_MARK(1)
            const int nq = tl.nq;
            TcQMeta *qm = qmeta + (size_t)tp * qg;
            for (int g = lane; g < nq; g += 32) {
                const ScanQuery sq = a.scan_q[tl.item_base + g];
                TcQMeta m;
                m.p_off = sq.p_off;
                m.slot = sq.slot;
                m.qid = sq.qid;
                m.meta = sq.meta;
                m.nl = sq.nl;
                m.pad[0] = m.pad[1] = 0;
                qm[g] = m;
            }
            if (lane == 0) {
                TcTInfo ti;
                ti.base = tl.base;
                ti.tile = t; ti.seg = tl.seg; ti.label = tl.label; ti.nq = nq;
                ti.tile_in_seg = tl.tile_in_seg; ti.n_tiles = tl.n_tiles; ti.hs = tl.hs != 0;
                ti.row_begin = tl.row_begin; ti.row_end = tl.row_end; ti.n_pieces = tl.n_pieces;
                ti.bits_off = tl.bits_off;
                for (int i = 0; i < kMaxPieces; i++) { ti.piece_off[i] = tl.piece_off[i]; ti.piece_cnt[i] = tl.piece_cnt[i]; }
                tinfo[tp] = ti;
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(tready + tp);
            TP_MARK(2)
            tc++;
        }
        TP_DUMP("sched(qempty,claim+tile,scanq,other)")
    } else if (warp == 0) {
        // ------------------------------------------------------------ producer
        uint32_t n = 0, tc = 0;
        TP_DECL
        for (;;) {
            const int tp = tc & 1;
            TP_MARK(3)
            if (lane == 0) mbar_wait(tready + tp, (tc >> 1) & 1);
            __syncwarp();
            TP_MARK(0)
            const TcTInfo tl = tinfo[tp];
            if (tl.tile < 0) {
                if (lane == 0) {
                    const int slot = n % nst;
                    mbar_wait(empty + slot, ((n / nst) & 1) ^ 1);
                    meta[slot] = make_int4(-1, 0, 0, TS_END);
                    mbar_arrive(full + slot);
                }
                break;
            }
            const int t = tl.tile;
            const bool hs = tl.hs != 0;
            const int nq = tl.nq;
            const TcQMeta *qm = qmeta + (size_t)tp * qg;
            if (lane == 0) mbar_arrive_expect_tx(qfull + tp, (uint32_t)nq * row_bytes);
            __syncwarp();
            for (int g = lane; g < nq; g += 32)
                tma_load_1d(qbuf + ((size_t)tp * qg + g) * row_bytes, a.Qp + (int64_t)qm[g].qid * row_bytes,
                            (uint32_t)row_bytes, qfull + tp);
            tc++;
            // rows of the tile: its range of the label, or only the AND pre-filter's survivors
            const bool filt = tl.n_pieces >= 0;
            const bool rbits = !filt && tl.bits_off >= 0;     // per-row pass bits of a mixed tile
            int total = tl.row_end - tl.row_begin;
            if (filt) {
                total = 0;
                for (int i = 0; i < tl.n_pieces; i++) total += tl.piece_cnt[i];
            }
            const int nstage = max(1, (total + kTcRows - 1) / kTcRows);
#ifdef VF_TC_PROF
            if (lane == 0 && nstage > 40)
                printf("TCBIG blk %d tile %d stages %d rows %d..%d pieces %d bits %d hs %d nq %d label %d ntiles %d\n",
                       blockIdx.x, t, nstage, tl.row_begin, tl.row_end, tl.n_pieces, tl.bits_off, tl.hs, nq, tl.label,
                       tl.n_tiles);
#endif
            for (int si = 0; si < nstage; si++) {
                const int v0 = si * kTcRows;
                const int r0 = tl.row_begin + v0;
                const int nr = max(0, min(kTcRows, total - v0));
                const int slot = n % nst;
                uint8_t *dst = rows + (size_t)slot * stage_bytes;
                int32_t *dsid = sid + (size_t)slot * kTcRows;
                uint32_t *dnorm = snorm + (size_t)slot * kTcRows;
                unsigned long long *dbits = sbits + (size_t)slot * kTcRows;
                const int flags = (si == 0 ? TS_FIRST : 0) | (si == nstage - 1 ? TS_LAST : 0);
                TP_MARK(3)
                if (!hs && !filt) {
                    if (lane == 0) {
                        mbar_wait(empty + slot, ((n / nst) & 1) ^ 1);
                        TP_MARK(1)
                        meta[slot] = make_int4(t, r0, nr, flags);
                        const uint32_t idb = (uint32_t)((nr * 4 + 15) & ~15);
                        const uint32_t bb = rbits ? (uint32_t)((nr * 8 + 15) & ~15) : 0u;
                        mbar_arrive_expect_tx(full + slot, (uint32_t)stage_bytes + 2 * idb + bb);
                        const int64_t row0 = tl.base + r0;
                        for (int c = 0; c < nch; c++)
                            tma_load_2d(dst + (size_t)c * kTcRows * cw, &tm_ls, c * cw, (int)row0, full + slot);
                        tma_load_1d(dsid, ix.M_ls + row0, idb, full + slot);
                        tma_load_1d(dnorm, ix.xn_ls + row0, idb, full + slot);
                        if (rbits) tma_load_1d(dbits, a.pool_bits + tl.bits_off + v0, bb, full + slot);
                    }
                    __syncwarp();
                } else if (filt && a.pool_norm) {
                    // compacted tile: its pieces start at 4-row boundaries, 16-B aligned (k_and_filter),
                    // so per piece overlapping this stage ids / norms / pass bits move by bulk copies
                    // and the lanes read the ids (coalesced int4, the only wait) for tile::gather4
                    const int ng = (nr + 3) >> 2;
                    const uint32_t b4n = (uint32_t)((nr * 4 + 15) & ~15), b8n = (uint32_t)((nr * 8 + 15) & ~15);
                    if (lane == 0) {
                        mbar_wait(empty + slot, ((n / nst) & 1) ^ 1);
                        meta[slot] = make_int4(t, r0, nr, flags);
                        mbar_arrive_expect_tx(full + slot, (uint32_t)(ng * 4 * kpad) + 2 * b4n + b8n);
                        int ps = 0;                                       // first row of piece p
                        for (int p = 0; p < tl.n_pieces && nr > 0; p++) {
                            const int pc = tl.piece_cnt[p];
                            const int lo = max(ps, v0), hi = min(ps + pc, v0 + nr);
                            if (lo < hi) {
                                const int64_t po = tl.piece_off[p] + (lo - ps);
                                const int d = lo - v0, len = hi - lo;
                                tma_load_1d(dsid + d, a.pool + po, (uint32_t)((len * 4 + 15) & ~15), full + slot);
                                tma_load_1d(dnorm + d, a.pool_norm + po, (uint32_t)((len * 4 + 15) & ~15), full + slot);
                                tma_load_1d(dbits + d, a.pool_bits + po, (uint32_t)((len * 8 + 15) & ~15), full + slot);
                            }
                            ps += pc;
                        }
                    }
                    __syncwarp();
                    for (int q4 = lane; q4 < ng; q4 += 32) {
                        const int rr = q4 * 4, v = v0 + rr;
                        int p = 0, ps = 0;
                        while (p + 1 < tl.n_pieces && v >= ps + tl.piece_cnt[p]) { ps += tl.piece_cnt[p]; p++; }
                        const int64_t po = tl.piece_off[p] + (v - ps);
                        const int cnt = min(4, ps + tl.piece_cnt[p] - v);   // rows of this group in the piece
                        int32_t g4[4];
                        if (cnt == 4) {
                            const int4 v4 = __ldg(reinterpret_cast<const int4 *>(a.pool + po));
                            g4[0] = v4.x; g4[1] = v4.y; g4[2] = v4.z; g4[3] = v4.w;
                        } else {
#pragma unroll
                            for (int j = 0; j < 4; j++) g4[j] = __ldg(a.pool + po + min(j, cnt - 1));
                        }
                        for (int c = 0; c < nch; c++)
                            tma_gather4(dst + (size_t)c * kTcRows * cw + (size_t)q4 * 4 * cw, &tm_x, c * cw, g4,
                                        full + slot);
                    }
                    __syncwarp();
                } else {
                    // HS label (exact mode / f3): gather rows of X through M_HS, 4 rows per TMA
                    // tile::gather4 per K chunk (a short group repeats its last row; ignored)
                    const int ng = (nr + 3) >> 2;
                    if (lane == 0) {
                        mbar_wait(empty + slot, ((n / nst) & 1) ^ 1);
                        meta[slot] = make_int4(t, r0, nr, flags);
                        mbar_expect_tx(full + slot, (uint32_t)(ng * 4 * kpad));
                    }
                    __syncwarp();
                    for (int q4 = lane; q4 < ng; q4 += 32) {
                        int32_t g4[4];
                        unsigned long long b4[4] = {0, 0, 0, 0};
#pragma unroll
                        for (int j = 0; j < 4; j++) {
                            const int r = min(q4 * 4 + j, nr - 1);
                            if (filt) {
                                int v = v0 + r, p = 0;
                                while (v >= tl.piece_cnt[p]) { v -= tl.piece_cnt[p]; p++; }
                                g4[j] = __ldg(a.pool + tl.piece_off[p] + v);
                                b4[j] = __ldg(a.pool_bits + tl.piece_off[p] + v);
                            } else {
                                g4[j] = __ldg(ix.M_hs + tl.base + r0 + r);
                                if (rbits) b4[j] = __ldg(a.pool_bits + tl.bits_off + v0 + r);
                            }
                        }
                        for (int c = 0; c < nch; c++)
                            tma_gather4(dst + (size_t)c * kTcRows * cw + (size_t)q4 * 4 * cw, &tm_x, c * cw, g4,
                                        full + slot);
#pragma unroll
                        for (int j = 0; j < 4; j++) {
                            if (q4 * 4 + j < nr) {
                                dsid[q4 * 4 + j] = g4[j];
                                dnorm[q4 * 4 + j] = __ldg(ix.xn + g4[j]);
                                dbits[q4 * 4 + j] = b4[j];
                            }
                        }
                    }
                    __syncwarp();
                    if (lane == 0) mbar_arrive(full + slot);
                }
                TP_MARK(2)
                n++;
            }
        }
        TP_DUMP("producer(tready,empty,issue,other)")
    } else if (warp == 1) {
        // ------------------------------------------------------------ MMA issuer
        uint32_t n = 0, tc = 0;
        int tp = 0, npad = 16;
        TP_DECL
        for (;;) {
            const int slot = n % nst;
            TP_MARK(4)
            mbar_wait(full + slot, (n / nst) & 1);
            TP_MARK(0)
            const int4 m = meta[slot];
            if (m.w & TS_END) break;
            const int buf = n & 1;
            mbar_wait(accempty + buf, ((n >> 1) & 1) ^ 1);
            TP_MARK(1)
            if (m.w & TS_FIRST) {
                tp = tc & 1;
                mbar_wait(qfull + tp, (tc >> 1) & 1);
                const int nq = tinfo[tp].nq;
                npad = max(16, (nq + 15) & ~15);
                // queries -> swizzled K-major B operand (zero K padding past row_bytes)
                const uint8_t *qsrc = qbuf + (size_t)tp * qg * row_bytes;
                uint8_t *bdst = bsm + (size_t)tp * nch * nmax * cw;
                const int upr = kpad / 16, rb16 = row_bytes / 16, upc = cw / 16;
                for (int e = lane; e < nq * upr; e += 32) {
                    const int g = e / upr, u = e - g * upr;
                    const uint4 v = u < rb16 ? reinterpret_cast<const uint4 *>(qsrc + (size_t)g * row_bytes)[u]
                                             : make_uint4(0, 0, 0, 0);
                    const int c = u / upc;
                    *reinterpret_cast<uint4 *>(bdst + (size_t)c * nmax * cw + swz(g, u - c * upc, cw)) = v;
                }
                fence_async_smem();
                __syncwarp();
                tc++;
                TP_MARK(2)
            }
            tc_fence_after();
            if (lane == 0) {
                const uint32_t a0 = smem_u32(rows + (size_t)slot * stage_bytes);
                const uint32_t b0 = smem_u32(bsm + (size_t)tp * nch * nmax * cw);
                const uint32_t id = idesc_of<DT>(npad);
                const uint32_t td = tbase + (uint32_t)(buf * nmax);
                uint32_t acc = 0;
                for (int c = 0; c < nch; c++)
                    for (int s = 0; s < cw / 32; s++) {
                        mma_issue<DT>(td, smem_desc(a0 + c * kTcRows * cw + s * 32, cw),
                               smem_desc(b0 + c * nmax * cw + s * 32, cw), id, acc);
                        acc = 1;
                    }
                mma_commit(accfull + buf);
            }
            __syncwarp();
            TP_MARK(3)
            n++;
        }
        TP_DUMP("mma(full,accempty,first,issue,other)")
    } else if (warp < 2 + kTcEpiW) {
        // ------------------------------------------------------------ epilogue (4 warps)
        // Warp w owns TMEM lane quarter w & 3 (rows 32q .. 32q+31 of the stage) for every query
        // column; it hands each stage to the selection warps through dready / dfree and never waits
        // for their top-k work (the D buffers are double-buffered).
        const int e = warp - 2;                       // 0..3
        const int quarter = warp & 3;
        const int row = quarter * 32 + lane;
        unsigned long long my_rows = 0, my_qrows = 0;
        uint32_t n = 0, tc = 0;
        TcTInfo ti;
        ti.nq = 0;
        const TcQMeta *qm = qmeta;
        const uint32_t *qnp = qn;
        const ull *thrp = thr;
        int tp = 0;
        uint32_t first_n = 0;
        TP_DECL
        for (;;) {
            const int slot = n % nst;
            const int buf = n & 1;
            TP_MARK(7)
            mbar_wait(full + slot, (n / nst) & 1);
            TP_MARK(0)
            const int4 m = meta[slot];
            if (m.w & TS_END) {
                mbar_wait(dfree + buf, ((n >> 1) & 1) ^ 1);
                if (e == 0 && lane == 0) sinfo[buf] = make_int4(0, TS_END, tp, 0);
                __syncwarp();
                if (lane == 0) mbar_arrive(dready + buf);
                break;
            }
            if (m.w & TS_FIRST) {
                tp = tc & 1;
                first_n = n;
                mbar_wait(qfull + tp, (tc >> 1) & 1);
                ti = tinfo[tp];
                qm = qmeta + (size_t)tp * qg;
                // this parity's thresholds were reset by the selection warps after the tile two back
                mbar_wait(tfree + tp, ((tc >> 1) & 1) ^ 1);
                uint32_t *qnw = qn + (size_t)tp * qg;
                const uint8_t *qsrc = qbuf + (size_t)tp * qg * row_bytes;
                for (int g = e; g < ti.nq; g += kTcEpiW) {
                    uint32_t s = 0;
                    const uint32_t *w = reinterpret_cast<const uint32_t *>(qsrc + (size_t)g * row_bytes);
                    for (int i = lane; i < row_bytes / 4; i += 32) s = sq_word<DT>(w[i], s);
#pragma unroll
                    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(FULL, s, o);
                    if (lane == 0) qnw[g] = s;
                }
                qnp = qnw;
                thrp = thr + (size_t)tp * qg;
                named_bar_sync(2, 32 * kTcEpiW);       // every query norm of the tile is in place
                tc++;
                TP_MARK(1)
            }
            const int nq = ti.nq, nr = m.z;
            uint32_t *D = dtile + (size_t)buf * qg * kTcRows;
            int32_t *Gd = gtile + (size_t)buf * kTcRows;
            uint32_t *Mk = mask + (size_t)buf * qg * 4;
            mbar_wait(dfree + buf, ((n >> 1) & 1) ^ 1);    // the selection is done with stage n-2
            if (n == first_n + 1)                          // ... and, for the tile's second stage, with
                mbar_wait(dfree + (buf ^ 1), ((n - 1) >> 1) & 1);   // its first: thresholds are real
            TP_MARK(6)
            mbar_wait(accfull + buf, (n >> 1) & 1);
            TP_MARK(2)
            tc_fence_after();
            const bool valid = row < nr;
            const int32_t gid = sid[(size_t)slot * kTcRows + row];
            const int32_t xn = (int32_t)snorm[(size_t)slot * kTcRows + row];
            // AND predicate: pass bits from the pre-filter (k_and_filter) when it ran on this tile
            const bool use_bits = ti.n_pieces >= 0 || ti.bits_off >= 0;
            const unsigned long long pbits = use_bits && valid ? sbits[(size_t)slot * kTcRows + row] : 0ull;
            Gd[row] = valid ? gid : -1;
            for (int c0 = 0; c0 < nq; c0 += 8) {
                uint32_t v[8];
                tmem_ld8(tbase + ((uint32_t)(quarter * 32) << 16) + (uint32_t)(buf * nmax + c0), v);
                tmem_wait_ld();
#pragma unroll
                for (int j = 0; j < 8; j++) {
                    const int g = c0 + j;
                    if (g < nq) {
                        const int32_t dot = DT == 0 ? (int32_t)v[j] : __float2int_rn(__uint_as_float(v[j]));
                        const int32_t d = xn + (int32_t)qnp[g] - 2 * dot;
                        const uint32_t bits = __float_as_uint((float)d);
                        const ull key = ((ull)bits << 32) | (uint32_t)gid;
                        bool pass = valid && key < thrp[g];
                        if (pass) {
                            // pass bits (pre-filter / packed tile: the row's own segment's queries
                            // and their AND predicates), else the scan verifies the predicate itself
                            if (use_bits) pass = ((pbits >> g) & 1ull) != 0;
                            else if (qm[g].meta & META_PRED)
                                pass = verify_pred_ol(ix, gid, a.qlab + qm[g].p_off, qm[g].nl, ti.label);
                        }
                        if (pass) D[(size_t)g * kTcRows + row] = bits;
                        const unsigned b = __ballot_sync(FULL, pass);
                        if (lane == 0) Mk[g * 4 + quarter] = b;
                    }
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) {
                mbar_arrive(accempty + buf);
                mbar_arrive(empty + slot);
                if (e == 0) sinfo[buf] = make_int4(nr, m.w, tp, 0);
                mbar_arrive(dready + buf);
            }
            if (threadIdx.x == 64) { my_rows += nr; my_qrows += (unsigned long long)nr * nq; }
            TP_MARK(3)
            n++;
        }
        if (warp == 2) { TP_DUMP("epi(full,first,accfull,compute,-,-,dfree,other)") }
        if (threadIdx.x == 64 && my_rows) {
            atomicAdd(&a.ctr->scan_rows, my_rows);
            atomicAdd(&a.ctr->scan_qrows, my_qrows);
        }
    } else {
        // ------------------------------------------------------------ selection (4 warps)
        // The warp owning query g (g = sw mod 4) merges each stage's survivors into the query's
        // register-resident top-k and tightens its threshold; a tile with 1-2 queries splits each
        // query's 32-row words over 2-4 warps (private lists, atomicMin thresholds, merged at the
        // tile's last stage). After a tile this parity's lists / thresholds are reset for the tile
        // two ahead (tfree) and its query slot released (qempty).
        const int sw = warp - 2 - kTcEpiW;            // 0..3
        ull *cbuf = scratch + (size_t)sw * (32 + 2 * k);
        ull *tmp = cbuf + 32;
        ull *fin2 = tmp + k;
        uint32_t n = 0;
        int tp = 0, parts = 1, nq = 0;
        TcTInfo ti;
        ti.nq = 0;
        const TcQMeta *qm = qmeta;
        ull *L0 = lists, *thr0 = thr;
        int *lc0 = lcnt;
        TP_DECL
        for (;;) {
            const int buf = n & 1;
            TP_MARK(7)
            mbar_wait(dready + buf, (n >> 1) & 1);
            TP_MARK(0)
            const int4 si = sinfo[buf];               // (rows, flags, tile parity)
            if (si.y & TS_END) break;
            if (si.y & TS_FIRST) {
                tp = si.z;
                ti = tinfo[tp];
                nq = ti.nq;
                qm = qmeta + (size_t)tp * qg;
                parts = (k <= 32 && nq <= 2 && a.tc_parts) ? (nq == 1 ? 4 : 2) : 1;
                L0 = lists + (size_t)tp * qg * k;
                thr0 = thr + (size_t)tp * qg;
                lc0 = lcnt + (size_t)tp * qg;
                // the lists this warp will use in this tile start empty
                if (parts > 1) {
                    if (sw < nq * parts && lane < k) L0[(size_t)sw * k + lane] = KEY_INF;
                } else {
                    for (int g = sw; g < nq; g += kTcSelW) {
                        for (int t = lane; t < k; t += 32) L0[(size_t)g * k + t] = KEY_INF;
                        if (lane == 0) lc0[g] = 0;
                    }
                }
                __syncwarp();
            }
            const uint32_t *D = dtile + (size_t)buf * qg * kTcRows;
            const int32_t *Gd = gtile + (size_t)buf * kTcRows;
            const uint32_t *Mk = mask + (size_t)buf * qg * 4;
            if (parts > 1) {
                if (sw < nq * parts) {
                    const int g = sw / parts, part = sw % parts;
                    ull *L = L0 + (size_t)sw * k;
                    const uint32_t *Dg = D + (size_t)g * kTcRows;
                    ull Li = lane < k ? L[lane] : KEY_INF;
                    unsigned wsel = 0;
                    for (int w4 = 0; w4 < 4; w4++)
                        if ((int)((n * 4 + w4) % parts) == part) wsel |= 1u << w4;
                    for (int base = 0;; base += 32) {
                        ull key;
                        const int nc = stage_candidates(Mk + g * 4, wsel, Dg, Gd, base, lane, key);
                        if (base >= nc) break;
                        Li = merge_topk_ol(Li, key, k, lane);
                    }
                    if (lane < k) L[lane] = Li;
                    const ull kth = __shfl_sync(FULL, Li, k - 1);
                    if (lane == 0 && kth != KEY_INF) atomicMin(thr0 + g, kth);   // any part's k-th bounds
                }
            } else {
                for (int g = sw; g < nq; g += kTcSelW) {
                    ull *L = L0 + (size_t)g * k;
                    const uint32_t *Dg = D + (size_t)g * kTcRows;
                    if (k <= 32) {
                        ull Li = lane < k ? L[lane] : KEY_INF;
                        for (int base = 0;; base += 32) {
                            ull key;
                            const int nc = stage_candidates(Mk + g * 4, 0xFu, Dg, Gd, base, lane, key);
                            if (base >= nc) break;
                            Li = merge_topk_ol(Li, key, k, lane);
                        }
                        if (lane < k) L[lane] = Li;
                        const ull kth = __shfl_sync(FULL, Li, k - 1);
                        if (lane == 0) thr0[g] = kth;
                    } else {
                        for (int w4 = 0; w4 < 4; w4++) {
                            const uint32_t word = Mk[g * 4 + w4];
                            if (!word) continue;
                            const int r = w4 * 32 + lane;
                            const ull key = (word >> lane) & 1 ? (((ull)Dg[r] << 32) | (uint32_t)Gd[r]) : KEY_INF;
                            topk_update_tc(L, lc0 + g, key, k, cbuf, tmp, lane);
                        }
                        if (lane == 0) thr0[g] = lc0[g] >= k ? L[k - 1] : KEY_INF;
                    }
                    __syncwarp();
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(dfree + buf);
            TP_MARK(1)
            if (si.y & TS_LAST) {
                const bool multi = ti.n_tiles > 1;
                if (parts > 1) {
                    // every part's list is final: the warp of part 0 merges its query's parts
                    named_bar_sync(3, 32 * kTcSelW);
                    if (sw < nq * parts && sw % parts == 0) {
                        ull Li = L0[(size_t)sw * k + (lane < k ? lane : 0)];
                        if (lane >= k) Li = KEY_INF;
                        for (int q = 1; q < parts; q++) {
                            const ull o = lane < k ? L0[(size_t)(sw + q) * k + lane] : KEY_INF;
                            Li = merge_topk_ol(Li, o, k, lane);
                        }
                        if (lane < k) L0[(size_t)sw * k + lane] = Li;
                    }
                    named_bar_sync(3, 32 * kTcSelW);   // no list is reset before every merge is done
                }
                for (int g = (parts > 1 ? (sw % parts == 0 ? sw / parts : nq) : sw); g < nq;
                     g += (parts > 1 ? nq : kTcSelW)) {
                    const ull *L = L0 + (size_t)(parts > 1 ? sw : g) * k;
                    const int na = k <= 32 ? __popc(__ballot_sync(FULL, lane < k && L[lane < k ? lane : 0] != KEY_INF))
                                           : lc0[g];
                    if (multi) {
                        for (int t = lane; t < k; t += 32)
                            a.partials[((size_t)qm[g].slot * a.max_tiles_per_label + ti.tile_in_seg) * k + t] =
                                t < na ? L[t] : KEY_INF;
                    } else {
                        write_final_tc(a, qm[g], L, na, k, lane);
                    }
                    __syncwarp();
                }
                if (multi) {
                    // last-block-done: the CTA completing the segment's last tile merges the partials
                    __threadfence();
                    named_bar_sync(3, 32 * kTcSelW);
                    if (sw == 0 && lane == 0) misc[2] = atomicAdd(&a.segs[ti.seg].done, 1) == ti.n_tiles - 1;
                    named_bar_sync(3, 32 * kTcSelW);
                    if (misc[2]) {
                        __threadfence();
                        for (int g = sw; g < nq; g += kTcSelW) {
                            ull *A0 = tmp, *B0 = fin2;
                            int na = 0;
                            for (int t2 = 0; t2 < ti.n_tiles; t2++) {
                                const volatile ull *P =
                                    a.partials + ((size_t)qm[g].slot * a.max_tiles_per_label + t2) * k;
                                for (int c0 = 0; c0 < k; c0 += 32) {
                                    const int cn = min(32, k - c0);
                                    const ull v = lane < cn ? P[c0 + lane] : KEY_INF;
                                    cbuf[lane] = v;
                                    __syncwarp();
                                    const int nc = __popc(__ballot_sync(FULL, v != KEY_INF));
                                    na = warp_merge(A0, na, cbuf, nc, B0, k, lane);
                                    ull *t3 = A0; A0 = B0; B0 = t3;
                                    __syncwarp();
                                }
                            }
                            write_final_tc(a, qm[g], A0, na, k, lane);
                            __syncwarp();
                        }
                    }
                    named_bar_sync(3, 32 * kTcSelW);   // misc[2] is read before the next tile writes it
                }
                // reset the thresholds of this parity for the tile two ahead (lists are reset by
                // their warps when that tile starts)
                if (lane == 0)
                    for (int g = sw; g < nq; g += kTcSelW) thr0[g] = KEY_INF;
                __syncwarp();
                if (lane == 0) {
                    mbar_arrive(qempty + tp);
                    mbar_arrive(tfree + tp);
                }
                TP_MARK(6)
            }
            n++;
        }
        if (warp == 6) { TP_DUMP("sel(dready,select,-,-,-,-,last,other)") }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tbase), "r"(SL.tmem_cols));
    }
    if (threadIdx.x == 0) atomicMax(&a.ctr->scan_t1, gtimer());
#ifdef VF_TC_PROF
    if (threadIdx.x == 0) printf("TCCTA %d start %llu end %llu\n", blockIdx.x, cta_t0, gtimer());
#endif
}

// ---------------------------------------------------------------- row norms (build time)
// out[r] = ||X[ids ? ids[r] : r]||^2 as an exact int32 (ids < 0 -> 0).
template <int DT>
__global__ void k_row_norms(const uint8_t *__restrict__ X, int row_bytes, const int32_t *__restrict__ ids,
                            int64_t n, uint32_t *__restrict__ out) {
    const int lane = threadIdx.x & 31;
    const int64_t w0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t r = w0; r < n; r += nw) {
        const int64_t src = ids ? (int64_t)ids[r] : r;
        uint32_t s = 0;
        if (src >= 0) {
            const uint32_t *w = reinterpret_cast<const uint32_t *>(X + src * row_bytes);
            for (int i = lane; i < row_bytes / 4; i += 32) s = sq_word<DT>(w[i], s);
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(FULL, s, o);
        if (lane == 0) out[r] = s;
    }
}

void launch_row_norms(int dtype, const uint8_t *X, int row_bytes, const int32_t *ids, int64_t n, uint32_t *out,
                      cudaStream_t s) {
    if (n <= 0) return;
    if (dtype == 0) k_row_norms<0><<<148 * 8, 256, 0, s>>>(X, row_bytes, ids, n, out);
    else k_row_norms<1><<<148 * 8, 256, 0, s>>>(X, row_bytes, ids, n, out);
}

// fp32 rows: flag any value that is not an integer in [lo, hi]
__global__ void k_check_int_range(const float *__restrict__ X, int64_t n, int row_floats, int dim, float lo, float hi,
                                  int32_t *__restrict__ bad) {
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n * row_floats;
         e += (int64_t)gridDim.x * blockDim.x) {
        const float v = X[e];
        if ((int)(e % row_floats) < dim && !(v == rintf(v) && v >= lo && v <= hi)) atomicOr(bad, 1);
    }
}

// largest integer magnitude for which every tf32 product and partial sum is exact in fp32
float tf32_exact_vmax(int dim) {
    float v = 2047.f;
    while (v > 0 && (double)dim * v * v >= 16777216.0) v -= 1.f;
    return v;
}

bool rows_int_in_range(const uint8_t *X, int64_t n, int row_bytes, int dim, float lo, float hi, cudaStream_t s) {
    int32_t *bad = nullptr, h = 1;
    if (cudaMalloc(&bad, 4) != cudaSuccess) return false;
    cudaMemsetAsync(bad, 0, 4, s);
    if (n > 0)
        k_check_int_range<<<148 * 8, 256, 0, s>>>(reinterpret_cast<const float *>(X), n, row_bytes / 4, dim, lo, hi,
                                                  bad);
    cudaMemcpyAsync(&h, bad, 4, cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    cudaFree(bad);
    return h == 0;
}

// fp32 rows holding integers in [0, 255] -> their exact u8 copy (zero padded to row_bytes8)
__global__ void k_f32_to_u8(const float *__restrict__ X, int row_floats, int64_t n, int dim, uint8_t *__restrict__ X8,
                            int row_bytes8) {
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n * row_bytes8;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = e / row_bytes8;
        const int c = (int)(e - r * row_bytes8);
        X8[e] = c < dim ? (uint8_t)(int)X[r * row_floats + c] : 0;
    }
}

void launch_f32_to_u8(const uint8_t *X, int row_bytes, int64_t n, int dim, uint8_t *X8, int row_bytes8,
                      cudaStream_t s) {
    if (n <= 0) return;
    k_f32_to_u8<<<148 * 8, 256, 0, s>>>(reinterpret_cast<const float *>(X), row_bytes / 4, n, dim, X8, row_bytes8);
}

// ---------------------------------------------------------------- tensor maps + launch
typedef CUresult (*encode_tiled_fn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                    const cuuint64_t *, const cuuint32_t *, const cuuint32_t *,
                                    CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                                    CUtensorMapFloatOOBfill);

static encode_tiled_fn get_encoder() {
    static encode_tiled_fn fn = nullptr;
    if (!fn) {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<encode_tiled_fn>(p);
    }
    return fn;
}

// 2-D byte tensor [n_rows][row_bytes] with a box of `box_rows` rows x cw bytes, swizzled to cw.
// promote: L2 fill size for the map's loads -- 256 B for contiguous row tiles (X_LS), none for
// row gathers (X via tile::gather4: a 192-B row promoted to 256-B blocks would fetch up to 512 B)
static bool encode_rows(CUtensorMap *m, const void *base, int row_bytes, int64_t n_rows, int cw, int box_rows,
                        bool promote) {
    encode_tiled_fn enc = get_encoder();
    if (!enc || n_rows <= 0) return false;
    cuuint64_t dims[2] = {(cuuint64_t)row_bytes, (cuuint64_t)n_rows};
    cuuint64_t strides[1] = {(cuuint64_t)row_bytes};
    cuuint32_t box[2] = {(cuuint32_t)cw, (cuuint32_t)box_rows};
    cuuint32_t es[2] = {1, 1};
    const CUtensorMapSwizzle sw = cw == 128 ? CU_TENSOR_MAP_SWIZZLE_128B
                                  : cw == 64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_32B;
    return enc(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void *>(base), dims, strides, box, es,
               CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
               promote ? CU_TENSOR_MAP_L2_PROMOTION_L2_256B : CU_TENSOR_MAP_L2_PROMOTION_NONE,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// A row-tile map for other tensor-core kernels (graph builder): box of box_rows rows x cw bytes.
bool encode_row_map(void *map, const void *base, int row_bytes, int64_t n_rows, int cw, int box_rows) {
    return encode_rows(reinterpret_cast<CUtensorMap *>(map), base, row_bytes, n_rows, cw, box_rows, true);
}

// Encode the two maps the tensor-core scan reads (X_LS tiles, X rows); false if unsupported.
bool scan_tc_encode(const DevIndex &ix, int64_t ls_rows_pad, void *tm_ls, void *tm_x) {
    const int cw = tc_chunk_bytes(ix.row_bytes);
    static const bool gpromote = [] { const char *e = getenv("VF_GATHER_PROMOTE"); return e && atoi(e) == 1; }();
    bool ok = encode_rows(reinterpret_cast<CUtensorMap *>(tm_x), ix.X, ix.row_bytes, ix.n_points, cw, 1, gpromote);
    ok = ok && encode_rows(reinterpret_cast<CUtensorMap *>(tm_ls), ix.Xls, ix.row_bytes,
                           ls_rows_pad > 0 ? ls_rows_pad : 1, cw, kTcRows, true);
    return ok;
}

int launch_scan_tc(const SearchArgs &a, cudaStream_t s, int max_tiles_bound, const void *tm_ls, const void *tm_x,
                   int ctas_per_sm) {
    if (max_tiles_bound <= 0) return 0;
    const TcLayout SL = tc_layout(a.ix.row_bytes, a.k);
    if (SL.nst < 2) return -1;
    auto f = a.ix.dtype == 0 ? k_scan_tc<0> : k_scan_tc<1>;
    static thread_local int cached_dev[2] = {-1, -1}, cached_nsm = 0;
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev != cached_dev[a.ix.dtype]) {
        cudaDeviceGetAttribute(&cached_nsm, cudaDevAttrMultiProcessorCount, dev);
        cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
        cached_dev[a.ix.dtype] = dev;
    }
    int grid = cached_nsm * (ctas_per_sm > 0 && ctas_per_sm < SL.ctas ? ctas_per_sm : SL.ctas);
    if (grid > max_tiles_bound) grid = max_tiles_bound;
    f<<<grid, kTcThreads, SL.total, s>>>(a, SL, *reinterpret_cast<const CUtensorMap *>(tm_ls),
                                         *reinterpret_cast<const CUtensorMap *>(tm_x));
    return 1;
}

}  // namespace vf
