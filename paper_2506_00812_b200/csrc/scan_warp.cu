// a2 for small query groups -- the exact label-grouped scan (Alg. 2; P:L466-L469,
// P:L559) with one warp per row tile, for tiles of <= kWarpScanQ queries and <= kWarpScanRows rows.
//
// Most scan segments are small: YFCC-shaped batches average ~1.4 queries and a few hundred rows
// per segment, SIFT-like ~3 queries. There a staged tensor-core pipeline (scan_tc.cu) spends its
// time in per-stage synchronisation rather than on bytes, so these tiles go to a massively parallel
// design instead: every warp owns one tile, keeps its queries in shared memory, streams the rows
// with coalesced 16-byte loads (LR lanes per row, CPL chunks per lane, U steps in flight), forms
// exact distances (u8: vabsdiff4 + dp4a, int32; integer-valued fp32: FFMA, exact) and keeps one
// register-resident top-k list per query (ballot against the k-th key, shuffle insertion). AND
// items verify the predicate only for rows that beat the k-th key. A segment split over several
// tiles is finished by the warp completing its last tile (partials + last-block-done), as in k_scan.
// Used only when the tensor-core scan is enabled (integer data, exact on both kernels).
#include "common.cuh"

namespace vf {

namespace {
constexpr int kWsWarps = 8;          // warps per CTA
constexpr int kWsU = 2;              // row steps in flight per warp
}

template <int DT, int LR, int CPL>
__global__ void __launch_bounds__(32 * kWsWarps) k_scan_warp(SearchArgs a) {
    typedef Acc<DT> A;
    constexpr int RPS = 32 / LR;                    // rows per step
    extern __shared__ __align__(16) uint8_t smem[];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int grp = lane / LR, gl = lane % LR;
    const DevIndex &ix = a.ix;
    const int row_bytes = ix.row_bytes, k = a.k;
    uint8_t *qs = smem + (size_t)wid * kWarpScanQ * row_bytes;                       // query rows
    ull *scr = reinterpret_cast<ull *>(smem + (size_t)kWsWarps * kWarpScanQ * row_bytes) +
               (size_t)wid * (32 + 2 * k);                                           // merge scratch
    __shared__ int s_last[kWsWarps];
    if (gate_skip(a)) return;
    const int nwt = a.ctr->n_wtiles;
    unsigned long long my_rows = 0, my_qrows = 0;
    for (;;) {
        int t = 0;
        if (lane == 0) t = atomicAdd(&a.ctr->wscan_next, 1);
        t = __shfl_sync(FULL, t, 0);
        if (t >= nwt) break;
        const Tile tl = a.tiles[a.wtiles[t]];
        const int nq = tl.nq;
        // -- the tile's queries: records + padded rows into this warp's shared slot
        ScanQuery sq[kWarpScanQ];
#pragma unroll
        for (int g = 0; g < kWarpScanQ; g++)
            if (g < nq) sq[g] = a.scan_q[tl.item_base + g];
        for (int g = 0; g < nq; g++) {
            const uint4 *src = reinterpret_cast<const uint4 *>(a.Qp + (int64_t)sq[g].qid * row_bytes);
            for (int c = lane; c < row_bytes / 16; c += 32)
                reinterpret_cast<uint4 *>(qs + (size_t)g * row_bytes)[c] = src[c];
        }
        __syncwarp();
        // -- rows: the label's range of X_LS, its HS list through M_HS (exact / f3), or only the
        //    AND pre-filter's survivors
        const bool hs = tl.hs != 0;
        const bool filt = hs && tl.n_pieces >= 0;
        int total = tl.row_end - tl.row_begin;
        if (filt) {
            total = 0;
            for (int i = 0; i < tl.n_pieces; i++) total += tl.piece_cnt[i];
        }
        ull Li[kWarpScanQ], kth[kWarpScanQ];
#pragma unroll
        for (int g = 0; g < kWarpScanQ; g++) { Li[g] = KEY_INF; kth[g] = KEY_INF; }
        for (int v0 = 0; v0 < total; v0 += RPS * kWsU) {
            int32_t gid[kWsU];
            uint4 x[kWsU][CPL];
#pragma unroll
            for (int u = 0; u < kWsU; u++) {
                const int v = v0 + u * RPS + grp;
                gid[u] = -1;
                const uint8_t *rp = nullptr;
                if (v < total) {
                    if (filt) {
                        int vv = v, p = 0;
                        while (vv >= tl.piece_cnt[p]) { vv -= tl.piece_cnt[p]; p++; }
                        gid[u] = __ldg(a.pool + tl.piece_off[p] + vv);
                        rp = ix.X + (int64_t)gid[u] * row_bytes;
                    } else if (hs) {
                        gid[u] = __ldg(ix.M_hs + tl.base + tl.row_begin + v);
                        rp = ix.X + (int64_t)gid[u] * row_bytes;
                    } else {
                        gid[u] = __ldg(ix.M_ls + tl.base + tl.row_begin + v);
                        rp = ix.Xls + (tl.base + tl.row_begin + v) * (int64_t)row_bytes;
                    }
                }
#pragma unroll
                for (int j = 0; j < CPL; j++)
                    x[u][j] = rp ? __ldg(reinterpret_cast<const uint4 *>(rp) + gl + j * LR) : make_uint4(0, 0, 0, 0);
            }
#pragma unroll
            for (int u = 0; u < kWsU; u++) {
                const bool valid = gid[u] >= 0;
#pragma unroll
                for (int g = 0; g < kWarpScanQ; g++) {
                    if (g >= nq) break;
                    typename A::T acc = 0;
                    const uint4 *qv = reinterpret_cast<const uint4 *>(qs + (size_t)g * row_bytes);
#pragma unroll
                    for (int j = 0; j < CPL; j++) A::add(acc, qv[gl + j * LR], x[u][j]);
#pragma unroll
                    for (int o = LR / 2; o > 0; o >>= 1) acc += __shfl_xor_sync(FULL, acc, o);
                    const ull key = ((ull)__float_as_uint(A::to_float(acc)) << 32) | (uint32_t)gid[u];
                    bool pass = valid && gl == 0 && key < kth[g];
                    if (pass && (sq[g].meta & META_PRED))
                        pass = verify_pred(ix, gid[u], a.qlab + sq[g].p_off, sq[g].nl, tl.label);
                    unsigned m = __ballot_sync(FULL, pass);
                    while (m) {
                        const int src = __ffs(m) - 1;
                        m &= m - 1;
                        const ull kk = __shfl_sync(FULL, key, src);
                        if (kk < kth[g]) {
                            const int pos = __popc(__ballot_sync(FULL, lane < k && Li[g] < kk));
                            const ull up = __shfl_up_sync(FULL, Li[g], 1);
                            if (lane > pos) Li[g] = up;
                            else if (lane == pos) Li[g] = kk;
                            kth[g] = __shfl_sync(FULL, Li[g], k - 1);
                        }
                    }
                }
            }
        }
        if (lane == 0) { my_rows += total; my_qrows += (unsigned long long)total * nq; }
        // -- results: direct rows / item lists, or partials of a split segment
        const bool multi = tl.n_tiles > 1;
#pragma unroll
        for (int g = 0; g < kWarpScanQ; g++) {
            if (g >= nq) break;
            const ull key = lane < k ? Li[g] : KEY_INF;
            if (multi) {
                if (lane < k)
                    a.partials[((size_t)sq[g].slot * a.max_tiles_per_label + tl.tile_in_seg) * k + lane] = key;
            } else if (sq[g].meta & META_DIRECT) {
                if (lane < k) {
                    a.out_ids[(int64_t)sq[g].qid * k + lane] = key == KEY_INF ? -1 : (int32_t)key_id(key);
                    a.out_dists[(int64_t)sq[g].qid * k + lane] =
                        key == KEY_INF ? __uint_as_float(0x7f800000u) : key_dist(key);
                }
            } else if (lane < k) {
                a.item_res[(size_t)sq[g].slot * k + lane] = key;
            }
        }
        if (multi) {
            __threadfence();
            __syncwarp();
            if (lane == 0) s_last[wid] = atomicAdd(&a.segs[tl.seg].pad[0], 1) == tl.n_tiles - 1;
            __syncwarp();
            if (s_last[wid]) {
                __threadfence();
                ull *cbuf = scr, *A0 = scr + 32, *B0 = A0 + k;
#pragma unroll
                for (int g = 0; g < kWarpScanQ; g++) {
                    if (g >= nq) break;
                    int na = 0;
                    ull *P0 = A0, *P1 = B0;
                    for (int t2 = 0; t2 < tl.n_tiles; t2++) {
                        const volatile ull *P = a.partials + ((size_t)sq[g].slot * a.max_tiles_per_label + t2) * k;
                        const ull v = lane < k ? P[lane] : KEY_INF;
                        cbuf[lane] = v;
                        __syncwarp();
                        const int nc = __popc(__ballot_sync(FULL, v != KEY_INF));
                        na = warp_merge(P0, na, cbuf, nc, P1, k, lane);
                        ull *t3 = P0; P0 = P1; P1 = t3;
                        __syncwarp();
                    }
                    const ull key = lane < na ? P0[lane] : KEY_INF;
                    if (lane < k) {
                        if (sq[g].meta & META_DIRECT) {
                            a.out_ids[(int64_t)sq[g].qid * k + lane] = key == KEY_INF ? -1 : (int32_t)key_id(key);
                            a.out_dists[(int64_t)sq[g].qid * k + lane] =
                                key == KEY_INF ? __uint_as_float(0x7f800000u) : key_dist(key);
                        } else {
                            a.item_res[(size_t)sq[g].slot * k + lane] = key;
                        }
                    }
                    __syncwarp();
                }
            }
        }
        __syncwarp();
    }
    if (lane == 0 && my_rows) {
        atomicAdd(&a.ctr->scan_rows, my_rows);
        atomicAdd(&a.ctr->scan_qrows, my_qrows);
    }
}

typedef void (*wscan_fn)(SearchArgs);

template <int DT>
static wscan_fn wscan_pick(int chunks) {
    // lanes per row LR (power of two) and 16-byte chunks per lane CPL = chunks / LR <= 4
#define VF_W(LR_, CPL_) if (chunks == LR_ * CPL_) return k_scan_warp<DT, LR_, CPL_>;
    VF_W(1, 1) VF_W(1, 2) VF_W(1, 3) VF_W(1, 4) VF_W(2, 3) VF_W(2, 4) VF_W(4, 3) VF_W(4, 4)
    VF_W(8, 3) VF_W(8, 4) VF_W(16, 3) VF_W(16, 4) VF_W(32, 3) VF_W(32, 4)
#undef VF_W
    return nullptr;
}

bool warp_scan_supported(int dtype, int row_bytes, int k) {
    if (k > 32) return false;
    return (dtype == 0 ? wscan_pick<0>(row_bytes / 16) : wscan_pick<1>(row_bytes / 16)) != nullptr;
}

int launch_scan_warp(const SearchArgs &a, cudaStream_t s, int max_tiles_bound) {
    if (max_tiles_bound <= 0) return 0;
    wscan_fn f = a.ix.dtype == 0 ? wscan_pick<0>(a.ix.row_bytes / 16) : wscan_pick<1>(a.ix.row_bytes / 16);
    if (!f) return -1;
    const size_t smem = (size_t)kWsWarps * kWarpScanQ * a.ix.row_bytes + (size_t)kWsWarps * (32 + 2 * a.k) * 8;
    // per-(kernel, device) setup once: attribute calls cost microseconds of host time per search,
    // during which the GPU idles between the search's kernels
    struct Key { wscan_fn f; int dev; };
    static thread_local Key done[16];
    static thread_local int ndone = 0, cached_nsm = 148;
    int dev = 0;
    cudaGetDevice(&dev);
    bool seen = false;
    for (int i = 0; i < ndone && i < 16; i++) seen |= done[i].f == f && done[i].dev == dev;
    if (!seen) {
        cudaDeviceGetAttribute(&cached_nsm, cudaDevAttrMultiProcessorCount, dev);
        cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);   // + static s_last
        done[ndone % 16] = Key{f, dev};
        ndone++;
    }
    int grid = cached_nsm * 4;
    const int need = (max_tiles_bound + kWsWarps - 1) / kWsWarps;
    if (grid > need) grid = need;
    f<<<grid, 32 * kWsWarps, smem, s>>>(a);
    return 1;
}

}  // namespace vf
