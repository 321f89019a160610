// a1 -- route and bucket (Alg. 2 "ClassifyQueries"; routing equation; AND/OR
// policies P:L523). One warp per query pads the query row, hashes its content for
// the entry sampler, sorts/deduplicates its labels and emits its work items into the query's
// label slots. Two small grid-stride kernels then turn the per-label bucket counts into scan
// segments (<= QG queries of one LS label) and row tiles, and scatter the scan items.
#include "common.cuh"

namespace vf {

// ---------------------------------------------------------------- prepare: pad + hash + route
constexpr int kPrepWarps = 32;   // queries per block (block-aggregated atomics)

// Integer-valued fp32 fast paths (tf32 scan, u8 row store): flag the batch if this padded query row
// holds a value outside [chk_lo, chk_hi] or not an integer, and write its u8 copy (warp-wide call).
__device__ __forceinline__ void check_query_row(const SearchArgs &a, const float *row, int64_t q, int lane) {
    bool bad = false;
    for (int i = lane; i < a.ix.dim; i += 32) {
        const float v = row[i];
        bad |= !(v == rintf(v) && v >= a.chk_lo && v <= a.chk_hi);
    }
    if (a.q8) {
        uint8_t *d8 = a.q8 + q * (int64_t)a.q8_row_bytes;
        for (int i = lane; i < a.q8_row_bytes; i += 32) {
            const float v = i < a.ix.dim ? row[i] : 0.f;
            d8[i] = (uint8_t)(v >= 0.f && v <= 255.f ? (int)v : 0);
        }
    }
    if (__any_sync(FULL, bad) && lane == 0) atomicOr(&a.ctr->exact_fallback, 1);
}

__global__ void __launch_bounds__(32 * kPrepWarps) k_prepare(SearchArgs a, const uint8_t *__restrict__ raw,
                                                             int raw_bytes) {
    __shared__ int s_ngraph[kGraphClasses][kPrepWarps];
    __shared__ int s_gbase[kGraphClasses];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int64_t q = (int64_t)blockIdx.x * kPrepWarps + wid;
    const bool live = q < a.n_q;
    const DevIndex &ix = a.ix;
    int32_t chosen[kMaxQueryLabels];
    uint32_t cpath[kMaxQueryLabels];
    int nch = 0, nraw = 0;
    int ngc[kGraphClasses] = {0, 0, 0, 0};
    int64_t lo = 0;
    uint32_t pred = 0;

    if (live) {
        // -- padded copy of the query row + content hash (reading c.3)
        const uint8_t *src = raw + q * (int64_t)raw_bytes;
        uint8_t *dst = const_cast<uint8_t *>(a.Qp) + q * (int64_t)ix.row_bytes;
        const int nwords = (raw_bytes + 3) >> 2;
        const int dwords = ix.row_bytes >> 2;
        uint32_t hacc = 0;
        for (int w = lane; w < dwords; w += 32) {
            uint32_t word = 0;
            if (w < nwords) {
                if ((raw_bytes & 3) == 0) {
                    word = __ldg(reinterpret_cast<const uint32_t *>(src) + w);
                } else {
                    for (int t = 0; t < 4; t++) {
                        int p = w * 4 + t;
                        uint32_t b = p < raw_bytes ? (uint32_t)__ldg(src + p) : 0u;
                        word |= b << (8 * t);
                    }
                }
                hacc += fmix32(word + (uint32_t)w * 0x9E3779B9u);
            }
            reinterpret_cast<uint32_t *>(dst)[w] = word;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) hacc += __shfl_xor_sync(FULL, hacc, o);
        const uint32_t qh = fmix32(hacc);
        if (a.chk_hi >= a.chk_lo) {
            __syncwarp();
            check_query_row(a, reinterpret_cast<const float *>(dst), q, lane);
        }

        lo = a.q_off[q];
        const int64_t hi = a.q_off[q + 1];
        const bool bad = lo < 0 || hi < lo || hi > a.n_slots || hi - lo > a.max_nl;
        if (bad) {
            // never index outside the label array; a query whose own range is in bounds but too
            // long marks its slots empty (no stale item is ever read from them)
            if (lane == 0) atomicAdd(&a.ctr->n_invalid, 1);
            if (lo >= 0 && hi >= lo && hi <= a.n_slots)
                for (int64_t t = lo + lane; t < hi; t += 32) {
                    Item it;
                    it.qid = (int32_t)q; it.rank = 0; it.label = -1; it.meta = PATH_NONE;
                    a.items[t] = it;
                }
            lo = 0;
        }
        nraw = bad ? 0 : (int)(hi - lo);
        int32_t *L = a.qlab + lo;   // the search's private copy of the labels, sorted in place
        if (a.qlab_in)              // fused copy of the caller's device labels (no separate memcpy)
            for (int t = lane; t < nraw; t += 32) L[t] = a.qlab_in[lo + t];
        __syncwarp();
        if (lane == 0) {
            int nl = 0;
            route_labels(a, L, nraw, &nl, chosen, cpath, &nch, &pred);
            for (int t = 0; t < nch; t++)
                if (cpath[t] == PATH_GRAPH) ngc[graph_class(ix.dir[chosen[t]].size)]++;
            QueryInfo qi;
            qi.nl = nl; qi.n_items = nch; qi.qh = qh; qi.pad = 0;
            a.qinfo[q] = qi;
        }
    }
    if (lane == 0)
        for (int c = 0; c < kGraphClasses; c++) s_ngraph[c][wid] = ngc[c];
    __syncthreads();
    if (threadIdx.x < kGraphClasses) {          // one thread per size class: block prefix + one atomic
        const int c = threadIdx.x;
        int tot = 0;
        for (int i = 0; i < kPrepWarps; i++) { const int g = s_ngraph[c][i]; s_ngraph[c][i] = tot; tot += g; }
        s_gbase[c] = tot ? atomicAdd(&a.ctr->n_graph_cls[c], tot) : 0;
        if (tot) atomicAdd(&a.ctr->n_graph, tot);
    }
    __syncthreads();
    if (live && lane == 0) {
        int gpos[kGraphClasses];
        for (int c = 0; c < kGraphClasses; c++) gpos[c] = s_gbase[c] + s_ngraph[c][wid];
        for (int t = 0; t < nraw; t++) {
            Item it;
            it.qid = (int32_t)q;
            it.rank = 0;
            if (t < nch) {
                const int32_t l = chosen[t];
                it.label = l;
                const bool remote = (cpath[t] & META_REMOTE) != 0;
                it.meta = cpath[t] | pred | (nch == 1 && !remote ? META_DIRECT : 0u);
                if (remote) atomicAdd(&a.ctr->remote[ix.owner[l]], 1);
                else if (cpath[t] == PATH_SCAN) it.rank = atomicAdd(a.ls_count + ix.dir[l].bslot, 1);
                else {
                    const int c = graph_class(ix.dir[l].size);
                    a.graph_list[c * a.graph_stride + gpos[c]++] = (int32_t)(lo + t);
                }
            } else {
                it.label = -1;
                it.meta = PATH_NONE;
            }
            a.items[lo + t] = it;
        }
    }
    if (live && __shfl_sync(FULL, nch, 0) == 0) {    // empty result row: pad (reading #23)
        for (int t = lane; t < a.k; t += 32) {
            a.out_ids[q * a.k + t] = -1;
            a.out_dists[q * a.k + t] = __uint_as_float(0x7f800000u);
        }
    }
}

// ---------------------------------------------------------------- bucket: segments + tiles
// For the first item (rank 0) of each scanned label: allocate ceil(count / QG) segments and, per
// segment, ceil(|C_l| / tile_rows) row tiles.
__global__ void k_segments(SearchArgs a, int64_t n_slots, int qg) {
    for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < n_slots;
         s += (int64_t)gridDim.x * blockDim.x) {
        const Item it = a.items[s];
        if ((it.meta & (3u | META_REMOTE)) != PATH_SCAN || it.rank != 0) continue;
        const LabelDir d = a.ix.dir[it.label];
        const int count = a.ls_count[d.bslot];
        const int nseg = (count + qg - 1) / qg;
        const int tr = (!a.exact && d.size >= a.scan_thr) ? a.tile_rows_f3 : a.tile_rows;
        const int ntile = (d.size + tr - 1) / tr;
        const int total = nseg * ntile;
        const int seg0 = atomicAdd(&a.ctr->n_segs, nseg);
        const int ib = atomicAdd(&a.ctr->n_scan_items, count);
        int tb = atomicAdd(&a.ctr->n_tiles, total);
        a.ls_segbase[d.bslot] = seg0;
        a.ls_itembase[d.bslot] = ib;
        for (int g = 0; g < nseg; g++) {
            Segment sg;
            sg.label = it.label;
            sg.item_base = ib + g * qg;
            sg.n_items = min(qg, count - g * qg);
            sg.tile_base = tb;
            sg.n_tiles = ntile;
            sg.listed = 0;
            sg.done = 0;
            sg.pad = 0;
            a.segs[seg0 + g] = sg;
            for (int t = 0; t < ntile; t++) {
                Tile tl;
                tl.base = d.base;
                tl.seg = seg0 + g;
                tl.row_begin = t * tr;
                tl.row_end = min(d.size, (t + 1) * tr);
                tl.tile_in_seg = t;
                tl.label = it.label;
                tl.nq = sg.n_items;
                tl.item_base = sg.item_base;
                tl.n_tiles = ntile;
                tl.hs = d.size >= a.ix.T;
                tl.bits_off = -1;
                tl.n_pieces = -1;
                a.tiles[tb + t] = tl;
                if (a.pack_list && ntile == 1 && !tl.hs && sg.n_items <= a.pack_max_nq) {
                    a.pack_list[atomicAdd(&a.ctr->n_pack, 1)] = tb + t;     // packed by k_pack
                } else if (a.tile_cls) {
                    const int c = tile_class(tl.row_end - tl.row_begin);
                    a.tile_cls[(int64_t)c * a.max_tiles + atomicAdd(&a.ctr->n_tile_cls[c], 1)] = tb + t;
                }
            }
            tb += ntile;
        }
    }
}

__global__ void k_scatter(SearchArgs a, int64_t n_slots, int qg) {
    for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < n_slots;
         s += (int64_t)gridDim.x * blockDim.x) {
        Item it = a.items[s];
        if ((it.meta & (3u | META_REMOTE)) != PATH_SCAN) continue;
        const LabelDir d = a.ix.dir[it.label];
        const int seg = a.ls_segbase[d.bslot] + it.rank / qg;
        a.scan_slots[a.ls_itembase[d.bslot] + it.rank] = (int32_t)s;
        a.item_seg[s] = seg;
        const int ntile = a.segs[seg].n_tiles;     // written by k_segments
        if ((it.meta & META_PRED) && a.filt_list && atomicExch(&a.segs[seg].listed, 1) == 0) {
            // the segment's first predicate item lists its tiles for the AND pre-filter
            const int tb = a.segs[seg].tile_base;
            const int f0 = atomicAdd(&a.ctr->n_filt_tiles, ntile);
            for (int t = 0; t < ntile; t++) a.filt_list[f0 + t] = tb + t;
        }
        if (ntile > 1) {
            it.meta |= META_MULTI;       // finalised in the scan kernel (last tile done)
            a.items[s] = it;
        }
        ScanQuery sq;
        sq.p_off = a.q_off[it.qid];
        sq.slot = (int32_t)s;
        sq.qid = it.qid;
        sq.meta = it.meta;
        sq.nl = a.qinfo[it.qid].nl;
        sq.pad[0] = sq.pad[1] = 0;
        a.scan_q[a.ls_itembase[d.bslot] + it.rank] = sq;
        if (it.rank == 0) a.ls_count[d.bslot] = 0;   // bucket counters stay zero between searches
    }
}

// ---------------------------------------------------------------- AND pre-filter (scan tiles)
// "Before distance computation ... points that do not contain all required labels are filtered
// out": the predicate of every AND scan item is evaluated here, for every row of its tile,
// by the whole GPU (many independent rows per SM hide the dependent id -> labels chains), and the
// scan no longer checks it row by row inside its epilogue.
//   * tile whose queries ALL carry a predicate: rows passing some query are compacted into the
//     survivor pool with their per-query pass bits; the scan gathers only those rows;
//   * tile mixing predicate and plain queries: every row is kept, its pass bits go to pool_bits;
//   * pool exhausted / piece list full: the tile keeps -1 and the scan verifies by itself (exact).
// Membership: the segment's other labels (<= 64 distinct) become bit positions; a label with a
// membership bitmap costs one bit read per row (one sector), a label of this rank without one a
// binary search of the row's id in the label's ascending posting list (M_LS / M_HS: small lists,
// their upper levels stay in L1), and only a label owned by another rank (sharded index) one pass
// over the row's sorted label list; query g passes iff its labels' mask is a subset of the row's.
constexpr int kFiltThreads = 256;
constexpr int kFiltBuf = 2048;
constexpr int kFiltUnion = 64;
#ifndef VF_FILT_ROWS
#define VF_FILT_ROWS 4
#endif
constexpr int kFiltRows = VF_FILT_ROWS;   // rows per thread per round

template <int MINB>
__global__ void __launch_bounds__(kFiltThreads, MINB) k_and_filter(SearchArgs a) {
    __shared__ int32_t buf[kFiltBuf];
    __shared__ unsigned long long bbuf[kFiltBuf];
    __shared__ int64_t q_off[kScanQG];
    __shared__ int32_t q_nl[kScanQG];
    __shared__ int32_t p_off[kMaxPieces], p_cnt[kMaxPieces];
    __shared__ int s_tile, s_npred, s_n, s_np, s_bad, s_flush_off, s_nu, s_bits_off, s_ns;
    __shared__ int32_t s_u[kFiltUnion];           // union of the tile's other query labels, sorted
    __shared__ unsigned long long s_qm[kScanQG];  // per query: its labels' bits in s_u (0: no predicate)
    __shared__ unsigned long long s_plain;        // queries without a predicate (always pass)
    __shared__ unsigned long long s_one[kFiltUnion];   // queries whose mask is exactly bit j
    __shared__ unsigned long long s_multi;        // predicate queries with >= 2 mask bits (checked one by one)
    __shared__ int16_t s_slot[kFiltUnion];        // membership bitmap of each s_u label (-1: none)
    __shared__ const int32_t *s_pl[kFiltUnion];   // ... else its posting list on this rank (ascending ids)
    __shared__ int32_t s_pn[kFiltUnion];          // ... and its length (0: not on this rank -> label list)
    __shared__ unsigned long long s_sig[kFiltUnion];   // signature bits of each s_u label
    __shared__ uint8_t s_first[kFiltThreads];     // staged pair i holds the first copy of its label
    // only tiles holding a predicate query are listed (k_scatter), so none is visited for nothing
    const int ntiles = a.ctr->n_filt_tiles;
    for (;;) {
        if (threadIdx.x == 0) {
            const int i = atomicAdd(&a.ctr->filter_next, 1);
            s_tile = i < ntiles ? a.filt_list[i] : -1;
            s_npred = 0; s_n = 0; s_np = 0; s_bad = 0; s_plain = 0; s_bits_off = -1; s_ns = 0; s_multi = 0;
        }
        if (threadIdx.x < kFiltUnion) s_one[threadIdx.x] = 0;
        __syncthreads();
        const int t = s_tile;
        if (t < 0) break;
        const Tile tl = a.tiles[t];
        const int nq = tl.nq;
        if (threadIdx.x < nq) {
            const ScanQuery sq = a.scan_q[tl.item_base + threadIdx.x];
            q_off[threadIdx.x] = sq.p_off;
            q_nl[threadIdx.x] = (sq.meta & META_PRED) ? sq.nl : 0;
            if (sq.meta & META_PRED) atomicAdd(&s_npred, 1);
            else atomicOr(&s_plain, 1ull << threadIdx.x);
            s_qm[threadIdx.x] = 0;
        }
        __syncthreads();
        const int npred = s_npred;
        const bool compact = npred == nq;
        const int nrows = tl.row_end - tl.row_begin;
        // the tile's other labels -> bit positions (<= 64 distinct, else per-query verification),
        // in parallel: every (query, label) pair is staged (label in buf, query in bbuf), the
        // distinct labels ranked, and each label's membership structure looked up by its own thread
        if (threadIdx.x < nq) {
            const int g = threadIdx.x;
            for (int i = 0; i < q_nl[g]; i++) {
                const int32_t l = a.qlab[q_off[g] + i];
                if (l == tl.label) continue;
                const int p = atomicAdd(&s_ns, 1);
                if (p < kFiltThreads) { buf[p] = l; bbuf[p] = (unsigned long long)g; }
            }
        }
        __syncthreads();
        const int ns = s_ns;
        bool first = false;
        int32_t myl = 0;
        if (ns <= kFiltThreads && threadIdx.x < ns) {
            myl = buf[threadIdx.x];
            first = true;
            for (int j = 0; j < threadIdx.x; j++)
                if (buf[j] == myl) { first = false; break; }
            s_first[threadIdx.x] = first;
        }
        // number of distinct labels, and each distinct label's rank among them
        const int nd = ns <= kFiltThreads ? __syncthreads_count(first) : kFiltUnion + 1;
        if (first && nd <= kFiltUnion) {
            int r = 0;
            for (int j = 0; j < ns; j++) r += s_first[j] && buf[j] < myl;
            s_u[r] = myl;
        }
        if (threadIdx.x == 0) {
            s_nu = nd <= kFiltUnion ? nd : kFiltUnion + 1;
            if (!compact) {
                const int need = (nrows + 3) & ~3;        // 16-B aligned bulk copies of the words
                const int off = atomicAdd(&a.ctr->pool_used, need);
                s_bits_off = (int64_t)off + need > a.pool_cap ? -1 : off;
            }
        }
        __syncthreads();
        const int nu = s_nu;
        int lab_ok = 1, lab_nobm = 0;
        if (nu <= kFiltUnion && threadIdx.x < nu) {
            const int j = threadIdx.x;
            const int32_t l = s_u[j];
            const bool known = l >= 0 && l < a.ix.n_labels;
            const int sl = (known && a.ix.lbit_slot) ? a.ix.lbit_slot[l] : -1;
            s_slot[j] = (int16_t)sl;
            s_sig[j] = label_sig_bits(l);
            int pn = 0;
            const int32_t *pl = nullptr;
            if (sl < 0 && known) {
                const LabelDir dl = a.ix.dir[l];
                pn = dl.size;
                pl = (dl.size >= a.ix.T ? a.ix.M_hs : a.ix.M_ls) + dl.base;
            }
            s_pn[j] = pn;
            s_pl[j] = pl;
            lab_ok = !(sl < 0 && pn == 0);           // not on this rank: the label list decides
            lab_nobm = sl < 0;
        }
        if (nu <= kFiltUnion && threadIdx.x < ns) {   // each staged pair sets its query's mask bit
            int lo = 0, hi = nu - 1;
            const int32_t l = buf[threadIdx.x];
            while (lo < hi) { const int mid = (lo + hi) >> 1; if (s_u[mid] < l) lo = mid + 1; else hi = mid; }
            atomicOr(&s_qm[(int)bbuf[threadIdx.x]], 1ull << lo);
        }
        const bool allbits = nu <= kFiltUnion && __syncthreads_and(lab_ok);
        // a bitmap label costs one sector per row, as does the signature (a random 8-B read): with
        // every label on a bitmap the signature only adds a sector (VF_KNOBS bit 0)
        const bool anynobm = __syncthreads_or(lab_nobm);
        const bool needsig = !(a.knobs & KNOB_FILT_SIG_AUTO) || anynobm;
        const int bits_off = s_bits_off;
        if (!compact && bits_off < 0) {          // pool exhausted: the scan verifies this tile
            __syncthreads();
            continue;
        }
        // pass bits of a row = plain | OR of s_one[j] over its set label bits | multi-bit queries
        // whose whole mask is set
        if (nu <= kFiltUnion && threadIdx.x < nq && q_nl[threadIdx.x]) {
            const unsigned long long qm = s_qm[threadIdx.x];
            if (qm == 0) atomicOr(&s_plain, 1ull << threadIdx.x);        // its labels are all the tile's
            else if ((qm & (qm - 1)) == 0) atomicOr(&s_one[__ffsll((long long)qm) - 1], 1ull << threadIdx.x);
            else atomicOr(&s_multi, 1ull << threadIdx.x);
        }
        __syncthreads();
        const unsigned long long plain = s_plain;
        const unsigned long long multi = s_multi;
        const int32_t *rowid = tl.hs ? a.ix.M_hs + tl.base : a.ix.M_ls + tl.base;
        // survivors in buf -> one pool piece (ids, pass bits, norms); pieces are 16-B aligned
        // survivors in buf -> one pool piece (ids, pass bits, norms). Every piece but a tile's last
        // holds a multiple of 4 rows (up to 3 survivors wait in buf for the next piece) and every
        // allocation is rounded to 4 rows, so each piece starts 16-B aligned in pool, pool_norm and
        // pool_bits AND at a 4-row boundary of the tile: the scan moves any piece with bulk copies.
        auto flush = [&](bool final_piece) {
            const int n = final_piece ? s_n : (s_n & ~3);
            if (threadIdx.x == 0 && n > 0) {
                if (s_np == kMaxPieces) {
                    s_bad = 1;
                } else {
                    const int off = atomicAdd(&a.ctr->pool_used, (n + 3) & ~3);
                    if ((int64_t)off + n > a.pool_cap) {
                        s_bad = 1;
                    } else {
                        p_off[s_np] = off;
                        p_cnt[s_np] = n;
                        s_np++;
                        s_flush_off = off;
                    }
                }
            }
            __syncthreads();
            if (!s_bad && n > 0)
                for (int i = threadIdx.x; i < n; i += kFiltThreads) {
                    a.pool[s_flush_off + i] = buf[i];
                    a.pool_bits[s_flush_off + i] = bbuf[i];
                    if (a.pool_norm) a.pool_norm[s_flush_off + i] = __ldg(a.tc_xn + buf[i]);
                }
            __syncthreads();
            if (threadIdx.x < s_n - n) {          // the <= 3 survivors left over move to the front
                buf[threadIdx.x] = buf[n + threadIdx.x];
                bbuf[threadIdx.x] = bbuf[n + threadIdx.x];
            }
            __syncthreads();
            if (threadIdx.x == 0) s_n -= n;
            __syncthreads();
        };
        for (int r0 = tl.row_begin; r0 < tl.row_end; r0 += kFiltThreads * kFiltRows) {
            // kFiltRows rows per thread, their dependent chains (id -> label offsets -> labels)
            // interleaved so several memory latencies overlap
            int32_t gid[kFiltRows];
            unsigned long long pb[kFiltRows];
#pragma unroll
            for (int u = 0; u < kFiltRows; u++) {
                const int r = r0 + u * kFiltThreads + threadIdx.x;
                gid[u] = r < tl.row_end ? __ldg(rowid + r) : -1;
                pb[u] = 0;
            }
            if (nu > 64) {
#pragma unroll
                for (int u = 0; u < kFiltRows; u++) {
                    if (gid[u] < 0) continue;
                    unsigned long long b = plain;
                    for (int g = 0; g < nq; g++)
                        if (q_nl[g] && verify_pred(a.ix, gid[u], a.qlab + q_off[g], q_nl[g], tl.label)) b |= 1ull << g;
                    pb[u] = b;
                }
            } else {
                unsigned long long lb[kFiltRows];
                if (allbits) {
                    // membership bitmaps (one bit read per (row, label), independent loads) and
                    // binary searches in the short posting lists of labels without one
                    unsigned long long sg[kFiltRows];
#pragma unroll
                    for (int u = 0; u < kFiltRows; u++)
                        sg[u] = gid[u] >= 0 && a.ix.lsig && needsig ? ld_keep(a.ix.lsig + gid[u]) : ~0ull;
#pragma unroll
                    for (int u = 0; u < kFiltRows; u++) {
                        lb[u] = 0;
                        if (gid[u] < 0) continue;
                        for (int j = 0; j < nu; j++) {
                            bool in;
                            if (!sig_may_have(sg[u], s_sig[j])) {
                                in = false;                 // the signature rules the label out
                            } else if (s_slot[j] >= 0) {
                                in = has_label_bit(a.ix, s_slot[j], gid[u]);
                            } else {
                                const int32_t *pl = s_pl[j];
                                int lo = 0, hi = s_pn[j];
                                while (lo < hi) {
                                    const int mid = (lo + hi) >> 1;
                                    if (__ldg(pl + mid) < gid[u]) lo = mid + 1; else hi = mid;
                                }
                                in = lo < s_pn[j] && __ldg(pl + lo) == gid[u];
                            }
                            if (in) lb[u] |= 1ull << j;
                        }
                    }
                } else {
                    int64_t lo[kFiltRows], hi[kFiltRows];
#pragma unroll
                    for (int u = 0; u < kFiltRows; u++) {
                        lo[u] = gid[u] >= 0 ? __ldg(a.ix.pt_off + gid[u]) : 0;
                        hi[u] = gid[u] >= 0 ? __ldg(a.ix.pt_off + gid[u] + 1) : 0;
                    }
                    const int32_t umax = nu > 0 ? s_u[nu - 1] : -1;
#pragma unroll
                    for (int u = 0; u < kFiltRows; u++) {
                        lb[u] = 0;
                        if (gid[u] < 0) continue;
                        // the point's sorted labels, 8 independent loads per round
                        for (int64_t e0 = lo[u]; e0 < hi[u]; e0 += 8) {
                            int32_t l8[8];
#pragma unroll
                            for (int t8 = 0; t8 < 8; t8++) l8[t8] = e0 + t8 < hi[u] ? __ldg(a.ix.pt_lab + e0 + t8) : INT32_MAX;
                            bool stop = false;
#pragma unroll
                            for (int t8 = 0; t8 < 8; t8++) {
                                const int32_t l = l8[t8];
                                if (l > umax) { stop = true; break; }
                                int b0 = 0, b1 = nu - 1;
                                while (b0 < b1) { const int mid = (b0 + b1) >> 1; if (s_u[mid] < l) b0 = mid + 1; else b1 = mid; }
                                if (s_u[b0] == l) lb[u] |= 1ull << b0;
                            }
                            if (stop) break;
                        }
                    }
                }
#pragma unroll
                for (int u = 0; u < kFiltRows; u++) {
                    if (gid[u] < 0) continue;
                    unsigned long long b = plain;
                    for (unsigned long long m = lb[u]; m; m &= m - 1) b |= s_one[__ffsll((long long)m) - 1];
                    for (unsigned long long m = multi; m; m &= m - 1) {
                        const int g = __ffsll((long long)m) - 1;
                        if ((lb[u] & s_qm[g]) == s_qm[g]) b |= 1ull << g;
                    }
                    pb[u] = b;
                }
            }
            if (!compact) {
#pragma unroll
                for (int u = 0; u < kFiltRows; u++) {
                    const int r = r0 + u * kFiltThreads + threadIdx.x;
                    if (r < tl.row_end) a.pool_bits[bits_off + (r - tl.row_begin)] = pb[u];
                }
                continue;
            }
#pragma unroll
            for (int u = 0; u < kFiltRows; u++)
                if (gid[u] >= 0 && pb[u]) {
                    const int i = atomicAdd(&s_n, 1);
                    buf[i] = gid[u];
                    bbuf[i] = pb[u];
                }
            __syncthreads();
            const bool last = r0 + kFiltThreads * kFiltRows >= tl.row_end;
            // a tile of <= kFiltBuf rows flushes once: its survivors form ONE contiguous piece,
            // which the scan's producer moves with bulk copies (ids, norms, pass bits)
            const bool one_piece = nrows <= kFiltBuf;
            if (last && s_n > 0) flush(true);
            else if (!one_piece && s_n > kFiltBuf - kFiltThreads * kFiltRows) flush(false);
            if (s_bad) break;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            Tile *T = a.tiles + t;
            if (!compact) {
                T->bits_off = bits_off;
            } else if (s_bad) {
                T->n_pieces = -1;
            } else {
                for (int i = 0; i < s_np; i++) { T->piece_off[i] = p_off[i]; T->piece_cnt[i] = p_cnt[i]; }
                T->n_pieces = s_np;
            }
        }
        __syncthreads();
    }
}

// ---------------------------------------------------------------- tile packing
// The YFCC-shaped batch holds ~36K scan segments of ~1.4 queries and a few hundred rows: one tile
// each, the tensor-core scan's per-tile chain (claim, query load, B operand, thresholds, results)
// dominated its time. pack_group such segments become ONE tile: its queries are the segments'
// queries side by side (<= 64), its rows the segments' rows (after the AND pre-filter), each row
// carrying the pass bits of exactly its own segment's queries -- every other (row, query) pair of
// the packed tile is masked in the scan's epilogue, so each query still sees exactly its label's
// rows (reading #50). One CTA per group.
constexpr int kPackThreads = 256;
constexpr int kPackMaxGroup = 16;
constexpr int kPackRows = 1024;      // a segment with more rows (after the pre-filter) stays alone;
                                     // a packed tile closes once it holds this many rows

// rows of a (pre-filtered) tile
__device__ __forceinline__ int tile_rows_now(const Tile &T) {
    if (T.n_pieces < 0) return T.row_end - T.row_begin;
    int r = 0;
    for (int p = 0; p < T.n_pieces; p++) r += T.piece_cnt[p];
    return r;
}

__device__ __forceinline__ void list_tile(const SearchArgs &a, int t, int rows) {
    const int c = tile_class(rows);
    a.tile_cls[(int64_t)c * a.max_tiles + atomicAdd(&a.ctr->n_tile_cls[c], 1)] = t;
}

__global__ void __launch_bounds__(kPackThreads) k_pack(SearchArgs a) {
    __shared__ Tile st[kPackMaxGroup];
    __shared__ int s_idx[kPackMaxGroup], s_rows[kPackMaxGroup];
    __shared__ int s_q0[kPackMaxGroup + 1], s_r0[kPackMaxGroup + 1];
    __shared__ int s_pack[kPackMaxGroup];        // packed tile (0..) of each sub, -1 alone
    __shared__ int s_off[kPackMaxGroup], s_cnt[kPackMaxGroup], s_pq[kPackMaxGroup], s_nq[kPackMaxGroup];
    __shared__ int s_npk;
    const int n_pack = a.ctr->n_pack;
    const int G = a.pack_group;
    const int n_groups = (n_pack + G - 1) / G;
    for (int gidx = blockIdx.x; gidx < n_groups; gidx += gridDim.x) {
        const int i0 = gidx * G, ng = min(G, n_pack - i0);
        if (threadIdx.x < ng) {
            s_idx[threadIdx.x] = a.pack_list[i0 + threadIdx.x];
            st[threadIdx.x] = a.tiles[s_idx[threadIdx.x]];
            s_rows[threadIdx.x] = tile_rows_now(st[threadIdx.x]);
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            // consecutive subs of <= kPackRows rows fill packed tiles up to kPackRows rows and the
            // scan's query capacity; bigger subs stay tiles of their own
            int npk = 0, q = 0, r = 0;
            for (int s = 0; s < ng; s++) {
                if (s_rows[s] > kPackRows) { s_pack[s] = -1; continue; }
                if (npk == 0 || q + st[s].nq > a.pack_max_nq * G || r >= kPackRows) {
                    if (npk > 0) { s_nq[npk - 1] = q; s_cnt[npk - 1] = r; }
                    npk++; q = 0; r = 0;
                }
                s_pack[s] = npk - 1;
                s_q0[s] = q;
                s_r0[s] = r;
                q += st[s].nq;
                r += s_rows[s];
            }
            if (npk > 0) { s_nq[npk - 1] = q; s_cnt[npk - 1] = r; }
            for (int p2 = 0; p2 < npk; p2++) {
                const int off = atomicAdd(&a.ctr->pool_used, (s_cnt[p2] + 3) & ~3);
                const bool ok = s_nq[p2] <= 64 && (int64_t)off + s_cnt[p2] <= a.pool_cap;
                s_off[p2] = ok ? off : -1;
                s_pq[p2] = ok ? atomicAdd(&a.ctr->packq_used, s_nq[p2]) : 0;
                s_cnt[p2] = 0;                                  // rows written so far
            }
            for (int s = 0; s < ng; s++)                        // alone, or no room: its own tile
                if (s_pack[s] < 0 || s_off[s_pack[s]] < 0) {
                    list_tile(a, s_idx[s], s_rows[s]);
                    s_pack[s] = -1;
                }
            s_npk = npk;
        }
        __syncthreads();
        for (int s = 0; s < ng; s++) {
            const int pk = s_pack[s];
            if (pk < 0) continue;
            const Tile &T = st[s];
            const int q0 = s_q0[s];
            for (int g = threadIdx.x; g < T.nq; g += kPackThreads)        // query records side by side
                a.scan_q[a.packq_base + s_pq[pk] + q0 + g] = a.scan_q[T.item_base + g];
            const unsigned long long mine = (T.nq >= 64 ? ~0ull : ((1ull << T.nq) - 1)) << q0;
            const int nrows = s_rows[s];
            for (int i0r = 0; i0r < nrows; i0r += kPackThreads) {
                const int i = i0r + threadIdx.x;
                int32_t gid = -1;
                uint32_t nrm = 0;
                unsigned long long bits = 0;
                if (i < nrows) {
                    if (T.n_pieces >= 0) {
                        int v = i, p = 0;
                        while (v >= T.piece_cnt[p]) { v -= T.piece_cnt[p]; p++; }
                        const int64_t e = T.piece_off[p] + v;
                        gid = __ldg(a.pool + e);
                        nrm = __ldg(a.pool_norm + e);
                        bits = __ldg(a.pool_bits + e) << q0;
                    } else {
                        const int64_t r = T.base + T.row_begin + i;
                        gid = __ldg(a.ix.M_ls + r);
                        nrm = __ldg(a.tc_xn_ls + r);
                        bits = T.bits_off >= 0 ? (__ldg(a.pool_bits + T.bits_off + i) << q0) : mine;
                    }
                }
                const bool keep = bits != 0;
                const unsigned m = __ballot_sync(FULL, keep);
                int base = 0;
                if ((threadIdx.x & 31) == 0 && m) base = atomicAdd(&s_cnt[pk], __popc(m));
                base = __shfl_sync(FULL, base, 0);
                if (keep) {
                    const int o = s_off[pk] + base + __popc(m & ((1u << (threadIdx.x & 31)) - 1));
                    a.pool[o] = gid;
                    a.pool_norm[o] = nrm;
                    a.pool_bits[o] = bits;
                }
            }
        }
        __syncthreads();
        if (threadIdx.x < s_npk && s_off[threadIdx.x] >= 0) {
            const int pk = threadIdx.x;
            const int pi = atomicAdd(&a.ctr->n_packed, 1);
            Tile P;
            P.base = 0;
            P.seg = -1;
            P.row_begin = 0;
            P.row_end = s_cnt[pk];
            P.tile_in_seg = 0;
            P.label = -1;
            P.nq = s_nq[pk];
            P.item_base = (int32_t)(a.packq_base + s_pq[pk]);
            P.n_tiles = 1;
            P.hs = 0;
            P.bits_off = -1;
            P.n_pieces = 1;
            P.piece_off[0] = s_off[pk];
            P.piece_cnt[0] = s_cnt[pk];
            for (int i = 1; i < kMaxPieces; i++) { P.piece_off[i] = 0; P.piece_cnt[i] = 0; }
            P.pad2[0] = P.pad2[1] = P.pad2[2] = 0;
            const int t = a.max_tiles + pi;
            a.tiles[t] = P;
            list_tile(a, t, s_cnt[pk]);
        }
        __syncthreads();
    }
}

int launch_pack(const SearchArgs &a, cudaStream_t s) {
    if (!a.pack_list) return 0;
    k_pack<<<148 * 4, kPackThreads, 0, s>>>(a);
    return 1;
}

int launch_and_filter(const SearchArgs &a, cudaStream_t s) {
    if (!a.pool || a.pool_cap <= 0 || !a.filt_list) return 0;
    // VF_KNOBS bit 4: 6 resident CTAs per SM (<= 40 registers) instead of 4 (64 registers)
    if (a.knobs & KNOB_FILT_OCC6) k_and_filter<6><<<148 * 6, kFiltThreads, 0, s>>>(a);
    else k_and_filter<4><<<148 * 4, kFiltThreads, 0, s>>>(a);
    return 1;
}

int launch_prepare(const SearchArgs &a, cudaStream_t s) {
    if (a.n_q == 0) return 0;
    const int64_t blocks = (a.n_q + kPrepWarps - 1) / kPrepWarps;
    const int raw_bytes = a.ix.dim * (a.ix.dtype == 0 ? 1 : 4);
    k_prepare<<<(unsigned)blocks, kPrepWarps * 32, 0, s>>>(a, a.Qraw, raw_bytes);
    return 1;
}

int launch_bucket(const SearchArgs &a, cudaStream_t s, int64_t n_slots, int qg) {
    if (n_slots == 0) return 0;
    int64_t blocks = (n_slots + 255) / 256;
    if (blocks > 148 * 16) blocks = 148 * 16;
    k_segments<<<(unsigned)blocks, 256, 0, s>>>(a, n_slots, qg);
    k_scatter<<<(unsigned)blocks, 256, 0, s>>>(a, n_slots, qg);
    return 2;
}

// ---------------------------------------------------------------- build-time helpers
__global__ void k_gather_rows(const uint8_t *__restrict__ X, int row_bytes, const int32_t *__restrict__ ids,
                              int64_t n, uint8_t *__restrict__ out) {
    const int words = row_bytes >> 4;
    const int64_t total = n * words;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = e / words;
        const int c = (int)(e - r * words);
        const int32_t id = ids[r];                    // -1: alignment padding row -> zeros
        reinterpret_cast<uint4 *>(out + r * row_bytes)[c] =
            id < 0 ? make_uint4(0, 0, 0, 0) : __ldg(reinterpret_cast<const uint4 *>(X + (int64_t)id * row_bytes) + c);
    }
}

__global__ void k_pad_rows(const uint8_t *__restrict__ src, int src_bytes, int64_t n, int row_bytes,
                           uint8_t *__restrict__ dst) {
    const int64_t total = n * row_bytes;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = e / row_bytes;
        const int c = (int)(e - r * row_bytes);
        dst[e] = c < src_bytes ? src[r * src_bytes + c] : 0;
    }
}

void launch_gather_rows(const uint8_t *X, int row_bytes, const int32_t *ids, int64_t n, uint8_t *out,
                        cudaStream_t s) {
    if (n == 0) return;
    k_gather_rows<<<148 * 8, 256, 0, s>>>(X, row_bytes, ids, n, out);
}

void launch_pad_rows(const uint8_t *src, int src_bytes, int64_t n, int row_bytes, uint8_t *dst,
                     cudaStream_t s) {
    if (n == 0) return;
    k_pad_rows<<<148 * 8, 256, 0, s>>>(src, src_bytes, n, row_bytes, dst);
}

// ---------------------------------------------------------------- label sharding (§8(e))
// Origin rank: pack every remote item into the send buffer region of its owner.
__global__ void k_pack_remote(SearchArgs a, int64_t n_slots, uint8_t *__restrict__ send,
                              const int64_t *__restrict__ dst_off, int32_t *__restrict__ sent_slots, int rec_bytes) {
    const int lane = threadIdx.x & 31;
    const int64_t s = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;   // warp per slot
    if (s >= n_slots) return;
    const Item it = a.items[s];
    if (!(it.meta & META_REMOTE)) return;
    const int dst = a.ix.owner[it.label];
    int pos = 0;
    if (lane == 0) pos = atomicAdd(&a.ctr->remote_pos[dst], 1);
    pos = __shfl_sync(FULL, pos, 0);
    const int64_t idx = dst_off[dst] + pos;
    uint8_t *rec = send + idx * (int64_t)rec_bytes;
    ItemRecord *h = reinterpret_cast<ItemRecord *>(rec);
    const QueryInfo qi = a.qinfo[it.qid];
    const int32_t *L = a.qlab + a.q_off[it.qid];
    if (lane == 0) {
        h->origin_slot = (int32_t)s;
        h->label = it.label;
        h->nl = qi.nl;
        h->pred = it.meta & META_PRED;
        h->qh = qi.qh;
        h->pad[0] = (int32_t)(it.meta & 3u);     // the origin's routing decision (path)
        h->pad[1] = h->pad[2] = 0;
        sent_slots[idx] = (int32_t)s;
    }
    if (lane < kRecLabels) h->labels[lane] = lane < qi.nl ? L[lane] : -1;
    const uint4 *src = reinterpret_cast<const uint4 *>(a.Qp + (int64_t)it.qid * a.ix.row_bytes);
    uint4 *dst_row = reinterpret_cast<uint4 *>(rec + sizeof(ItemRecord));
    for (int c = lane; c < a.ix.chunks; c += 32) dst_row[c] = src[c];
}

// Owner rank: received records become a batch of single-item queries (query i = record i, item
// slot i, labels at qlab[i * kRecLabels]) whose results are written directly to out_ids/out_dists.
__global__ void k_unpack_items(SearchArgs a, const uint8_t *__restrict__ recv, int64_t n, int rec_bytes) {
    const int lane = threadIdx.x & 31;
    const int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (i >= n) return;
    const uint8_t *rec = recv + i * (int64_t)rec_bytes;
    const ItemRecord *h = reinterpret_cast<const ItemRecord *>(rec);
    const uint4 *src = reinterpret_cast<const uint4 *>(rec + sizeof(ItemRecord));
    uint4 *dst = reinterpret_cast<uint4 *>(const_cast<uint8_t *>(a.Qp) + i * (int64_t)a.ix.row_bytes);
    for (int c = lane; c < a.ix.chunks; c += 32) dst[c] = src[c];
    __syncwarp();
    if (a.chk_hi >= a.chk_lo) check_query_row(a, reinterpret_cast<const float *>(dst), i, lane);
    if (lane < kRecLabels) a.qlab[i * kRecLabels + lane] = h->labels[lane];
    if (lane == 0) {
        int64_t *qoff = const_cast<int64_t *>(a.q_off);
        qoff[i] = i * kRecLabels;
        if (i == n - 1) qoff[n] = n * kRecLabels;
        const int32_t l = h->label;
        const LabelDir d = a.ix.dir[l];
        QueryInfo qi;
        qi.nl = h->nl; qi.n_items = 1; qi.qh = h->qh; qi.pad = 0;
        a.qinfo[i] = qi;
        const uint32_t path = (uint32_t)h->pad[0];   // as routed by the origin (a1)
        Item it;
        it.qid = (int32_t)i;
        it.label = l;
        it.rank = 0;
        it.meta = path | h->pred | META_DIRECT;
        if (path == PATH_SCAN) it.rank = atomicAdd(a.ls_count + d.bslot, 1);
        else {
            const int c = graph_class(d.size);
            a.graph_list[c * a.graph_stride + atomicAdd(&a.ctr->n_graph_cls[c], 1)] = (int32_t)i;
            atomicAdd(&a.ctr->n_graph, 1);
        }
        a.items[i] = it;
    }
}

// Origin rank: results returned by the owners (in send order) become the remote items' keys.
__global__ void k_scatter_results(SearchArgs a, const int32_t *__restrict__ ids, const float *__restrict__ dists,
                                  const int32_t *__restrict__ sent_slots, int64_t n) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= n * a.k) return;
    const int64_t j = e / a.k;
    const int t = (int)(e - j * a.k);
    const int32_t id = ids[e];
    a.item_res[(size_t)sent_slots[j] * a.k + t] = id < 0 ? KEY_INF : make_key(dists[e], (uint32_t)id);
}

int launch_pack_remote(const SearchArgs &a, cudaStream_t s, int64_t n_slots, uint8_t *send, const int64_t *dst_off,
                       int32_t *sent_slots, int rec_bytes) {
    if (n_slots == 0) return 0;
    k_pack_remote<<<(unsigned)((n_slots * 32 + 255) / 256), 256, 0, s>>>(a, n_slots, send, dst_off, sent_slots, rec_bytes);
    return 1;
}

int launch_unpack_items(const SearchArgs &a, cudaStream_t s, const uint8_t *recv, int64_t n, int rec_bytes) {
    if (n == 0) return 0;
    k_unpack_items<<<(unsigned)((n * 32 + 255) / 256), 256, 0, s>>>(a, recv, n, rec_bytes);
    return 1;
}

int launch_scatter_results(const SearchArgs &a, cudaStream_t s, const int32_t *ids, const float *dists,
                           const int32_t *sent_slots, int64_t n) {
    if (n == 0) return 0;
    k_scatter_results<<<(unsigned)((n * a.k + 255) / 256), 256, 0, s>>>(a, ids, dists, sent_slots, n);
    return 1;
}

}  // namespace vf
