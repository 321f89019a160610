// a3 -- IVF-Graph beam search for high-specificity labels (Alg. 2; P:L442-L444;
// AND inline filtering P:L549-L550), following the deterministic reading of DESIGN.md §2 c.2.
//
// One warp per (query, label) item, persistent warps pulling items from an atomic counter.
// Per warp in shared memory: the top-M list (itopk keys, double-buffered), 32 candidate keys,
// and an open-addressing visited set of local ids; when the visited set would pass half its
// capacity new ids spill into a per-warp global-memory table (64-bit entries tagged with an item
// epoch, so it is never cleared) -- the visited set is exact, never "forgettable", which is what
// makes the result schedule-independent (reading #12).
// Per iteration: the first w unexpanded entries of Top become parents (Alg. 2); their G_l
// rows are read -- each edge carries (local id, global id), i.e. the M_HS mapping of P:L444 is
// folded into the row so a child costs no dependent M_HS gather; children are de-duplicated within
// the batch (match.any), checked/inserted in the visited set, filtered by the AND predicate, and their vector rows gathered with 16-byte loads by "teams" of
// lanes (TEAM lanes per row, up to 8 rows' loads in flight per lane); team-reduced exact distances
// become keys (dist, local id << 1 | expanded) that are bitonic-sorted across the warp and merged
// into Top by rank.
#include "common.cuh"

namespace vf {

struct GraphLayout {
    int itopk, hash_slots;
    size_t off_topA, off_topB, off_cbuf, off_fgid, off_floc, off_par, off_hash, warp_bytes;
};

static GraphLayout graph_layout(int itopk, int hash_slots) {
    GraphLayout L;
    L.itopk = itopk;
    L.hash_slots = hash_slots;
    size_t o = 0;
    L.off_topA = o; o += (size_t)itopk * 8;
    L.off_topB = o; o += (size_t)itopk * 8;
    L.off_cbuf = o; o += 32 * 8;
    L.off_fgid = o; o += 32 * 4;
    L.off_floc = o; o += 32 * 4;
    L.off_par = o; o += 64 * 4;
    L.off_hash = o; o += (size_t)hash_slots * 4;
    L.warp_bytes = (o + 15) & ~(size_t)15;
    return L;
}

__device__ __forceinline__ uint32_t vis_hash(int32_t c) { return (uint32_t)c * 0x9E3779B1u; }

__device__ __forceinline__ bool smem_find(const int32_t *tab, uint32_t mask, int32_t c) {
    uint32_t h = vis_hash(c) & mask;
    for (;;) {
        const int32_t v = tab[h];
        if (v == c) return true;
        if (v < 0) return false;
        h = (h + 1) & mask;
    }
}
__device__ __forceinline__ void smem_insert(int32_t *tab, uint32_t mask, int32_t c) {
    uint32_t h = vis_hash(c) & mask;
    for (;;) {
        const int32_t old = atomicCAS(tab + h, -1, c);
        if (old == -1 || old == c) return;
        h = (h + 1) & mask;
    }
}
__device__ __forceinline__ bool gtab_find(const ull *tab, uint64_t mask, uint32_t epoch, int32_t c) {
    uint64_t h = vis_hash(c) & mask;
    for (;;) {
        const ull v = *(volatile const ull *)(tab + h);
        if ((uint32_t)(v >> 32) != epoch) return false;
        if ((int32_t)(uint32_t)v == c) return true;
        h = (h + 1) & mask;
    }
}
__device__ __forceinline__ void gtab_insert(ull *tab, uint64_t mask, uint32_t epoch, int32_t c) {
    uint64_t h = vis_hash(c) & mask;
    const ull want = ((ull)epoch << 32) | (uint32_t)c;
    for (;;) {
        const ull v = *(volatile ull *)(tab + h);
        if ((uint32_t)(v >> 32) != epoch) {
            if (atomicCAS(tab + h, v, want) == v) return;
            continue;
        }
        if ((int32_t)(uint32_t)v == c) return;
        h = (h + 1) & mask;
    }
}

template <int DT, int TEAM, int MAXCPL>
__global__ void __launch_bounds__(32 * kWarpsPerGraphCta, 8) k_graph(SearchArgs a, GraphLayout GL,
                                                                  uint32_t *gtab_epoch) {
    extern __shared__ __align__(16) uint8_t smem[];
    typedef Acc<DT> A;
    constexpr int RP = 32 / TEAM;                       // rows per pass
    constexpr int GROUP = MAXCPL >= 8 ? 1 : (MAXCPL >= 4 ? 2 : 8 / MAXCPL);  // passes in flight together
    if (gate_skip(a)) return;     // u8 row store: the other view's kernel takes this batch
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int team = lane / TEAM, tl = lane % TEAM;
    uint8_t *wb = smem + (size_t)wid * GL.warp_bytes;
    ull *topA = reinterpret_cast<ull *>(wb + GL.off_topA);
    ull *topB = reinterpret_cast<ull *>(wb + GL.off_topB);
    ull *cbuf = reinterpret_cast<ull *>(wb + GL.off_cbuf);
    int32_t *fgid = reinterpret_cast<int32_t *>(wb + GL.off_fgid);
    int32_t *floc = reinterpret_cast<int32_t *>(wb + GL.off_floc);
    int32_t *spar = reinterpret_cast<int32_t *>(wb + GL.off_par);
    int32_t *htab = reinterpret_cast<int32_t *>(wb + GL.off_hash);

    const DevIndex &ix = a.ix;
    const int M = GL.itopk, H = GL.hash_slots, R = ix.R, k = a.k;
    const int chunks = ix.chunks, row_bytes = ix.row_bytes;
    const uint32_t hmask = (uint32_t)H - 1;
    const int r_shift = (R & (R - 1)) == 0 ? __ffs(R) - 1 : -1;
    const int warp_slot = blockIdx.x * kWarpsPerGraphCta + wid;
    ull *gtab = a.gtab + (size_t)warp_slot * a.gtab_slots;
    const uint64_t gmask = (uint64_t)a.gtab_slots - 1;
    uint32_t epoch = gtab_epoch[warp_slot];
    const int n_graph = a.ctr->n_graph;
    const unsigned lt_mask = (1u << lane) - 1u;

    for (;;) {
        int gi = 0;
        if (lane == 0) gi = atomicAdd(&a.ctr->graph_next, 1);
        gi = __shfl_sync(FULL, gi, 0);
        if (gi >= n_graph) break;
        const int32_t slot = a.graph_list[gi];
        const Item it = a.items[slot];
        const LabelDir d = ix.dir[it.label];
        const int32_t S = d.size;
        const int64_t base = d.base;
        const QueryInfo qi = a.qinfo[it.qid];
        const bool has_pred = (it.meta & META_PRED) != 0;
        const int32_t *P = a.qlab + a.q_off[it.qid];
        const int np = qi.nl;

        uint4 qreg[MAXCPL];
        const uint4 *qrow = reinterpret_cast<const uint4 *>(a.Qp + (int64_t)it.qid * row_bytes);
#pragma unroll
        for (int j = 0; j < MAXCPL; j++) {
            const int c = tl + j * TEAM;
            qreg[j] = c < chunks ? __ldg(qrow + c) : make_uint4(0, 0, 0, 0);
        }
        for (int i = lane; i < H; i += 32) htab[i] = -1;
        epoch++;
        bool g_used = false;
        int n_smem = 0, nvis = 0, ntop = 0, E = 0, iters = 0;
        ull *cur = topA, *oth = topB;
        __syncwarp();

        // Process one batch of candidate local ids (one per lane, -1 = none): visited-set
        // check/insert, M_HS mapping, predicate, distances, merge into Top.
        auto process = [&](int32_t c, int32_t gid) {
            bool v = c >= 0;
            const unsigned same = __match_any_sync(FULL, v ? c : -1 - lane);
            if (v && (__ffs(same) - 1) != lane) v = false;          // duplicate within the batch
            bool found = false;
            if (v) {
                found = smem_find(htab, hmask, c);
                if (!found && g_used) found = gtab_find(gtab, gmask, epoch, c);
            }
            const bool isnew = v && !found;
            const unsigned nm = __ballot_sync(FULL, isnew);
            const int nnew = __popc(nm);
            const bool use_smem = 2 * (n_smem + nnew) <= H;
            __syncwarp();
            if (isnew) {
                if (use_smem) smem_insert(htab, hmask, c);
                else gtab_insert(gtab, gmask, epoch, c);
            }
            if (nnew) { if (use_smem) n_smem += nnew; else g_used = true; }
            nvis += nnew;
            if (isnew && gid < 0) gid = __ldg(ix.M_hs + base + c);   // entry samples only
            bool pass = isnew;
            if (pass && has_pred) pass = verify_pred(ix, gid, P, np, it.label);
            const unsigned pm = __ballot_sync(FULL, pass);
            const int nc = __popc(pm);
            if (nc == 0) return;
            if (pass) {
                const int ci = __popc(pm & lt_mask);
                fgid[ci] = gid;
                floc[ci] = c;
            }
            __syncwarp();
            if (nc > RP * GROUP) {
                // more rows than one load group: put every row's 128-byte lines in flight to L2 now,
                // so the later groups do not each pay a full DRAM round trip
                const int lines = (row_bytes + 127) >> 7;
                for (int e = lane; e < nc * lines; e += 32) {
                    const int r = e / lines, l = e - r * lines;
                    asm volatile("prefetch.global.L2 [%0];" ::"l"(ix.X + (int64_t)fgid[r] * row_bytes + l * 128));
                }
            }
            for (int p0 = 0; p0 < nc; p0 += RP * GROUP) {
                uint4 xv[GROUP][MAXCPL];
#pragma unroll
                for (int g = 0; g < GROUP; g++) {
                    const int r = p0 + g * RP + team;
                    const uint4 *row = reinterpret_cast<const uint4 *>(
                        ix.X + (int64_t)(r < nc ? fgid[r] : 0) * row_bytes);
#pragma unroll
                    for (int j = 0; j < MAXCPL; j++) {
                        const int cc = tl + j * TEAM;
                        xv[g][j] = (r < nc && cc < chunks) ? __ldg(row + cc) : make_uint4(0, 0, 0, 0);
                    }
                }
#pragma unroll
                for (int g = 0; g < GROUP; g++) {
                    typename A::T acc = 0;
#pragma unroll
                    for (int j = 0; j < MAXCPL; j++) A::add(acc, qreg[j], xv[g][j]);
#pragma unroll
                    for (int o = TEAM / 2; o > 0; o >>= 1) acc += __shfl_xor_sync(FULL, acc, o);
                    const int r = p0 + g * RP + team;
                    if (tl == 0 && r < nc)
                        cbuf[r] = make_key(A::to_float(acc), (uint32_t)floc[r] << 1);
                }
            }
            __syncwarp();
            ull ck = lane < nc ? cbuf[lane] : KEY_INF;
            // a full Top keeps its best M keys: a child not below the M-th can never enter it, so
            // it is dropped before the sort / merge (it is already counted as visited)
            if (ntop == M && ck >= cur[M - 1]) ck = KEY_INF;
            const unsigned sm = __ballot_sync(FULL, ck != KEY_INF);
            const int ns = __popc(sm);
            if (ns == 0) return;
            if (M <= 32) {
                // Top fits one key per lane: merge in registers (no shared-memory rank search)
                ull Li = lane < ntop ? cur[lane] : KEY_INF;
                if (ns <= 4) {
                    // few survivors (the common case once Top is full): insert one at a time
                    // (ballot for the position, shift up) instead of a 32-key sort; the register
                    // list stays sorted, and lanes >= M are never written back
                    unsigned rem = sm;
                    while (rem) {
                        const ull kk = __shfl_sync(FULL, ck, __ffs(rem) - 1);
                        rem &= rem - 1;
                        const int pos = __popc(__ballot_sync(FULL, Li < kk));
                        const ull up = __shfl_up_sync(FULL, Li, 1);
                        if (lane > pos) Li = up;
                        else if (lane == pos) Li = kk;
                    }
                } else {
                    // the 32 smallest of two sorted lists: min against the reversed candidates is a
                    // bitonic sequence, sorted by five compare-exchange steps
                    const ull srt = warp_sort32(ck, lane);
                    const ull r = __shfl_sync(FULL, srt, 31 - lane);
                    Li = Li < r ? Li : r;
#pragma unroll
                    for (int j = 16; j > 0; j >>= 1) {
                        const ull o = __shfl_xor_sync(FULL, Li, j);
                        Li = ((lane & j) == 0) ? (Li < o ? Li : o) : (Li < o ? o : Li);
                    }
                }
                if (lane < M) cur[lane] = Li;
                ntop = min(M, ntop + ns);
                __syncwarp();
                return;
            }
            if (ns == 1) {
                ck = __shfl_sync(FULL, ck, __ffs(sm) - 1);
                if (lane == 0) cbuf[0] = ck;
            } else {
                ck = warp_sort32(ck, lane);
                cbuf[lane] = ck;
            }
            __syncwarp();
            ntop = warp_merge(cur, ntop, cbuf, ns, oth, M, lane);
            ull *t2 = cur; cur = oth; oth = t2;
        };

        // ---- INIT: entries = all of [0, S) if S <= n_init, else the hashed samples (reading c.3)
        const int n_entry = S <= a.n_init ? S : a.n_init;
        const uint32_t hbase = fmix32(a.seed ^ qi.qh ^ fmix32((uint32_t)it.label * 0x9E3779B9u));
        for (int e0 = 0; e0 < n_entry; e0 += 32) {
            const int i = e0 + lane;
            int32_t c = -1;
            if (i < n_entry)
                c = S <= a.n_init ? i : (int32_t)(fmix32(hbase + (uint32_t)i * 0x9E3779B9u) % (uint32_t)S);
            process(c, -1);
        }
        // ---- LOOP (Alg. 2)
        for (int iter = 0; iter < a.max_iter; iter++) {
            int npar = 0;
            for (int b = 0; b < ntop && npar < a.w; b += 32) {
                const int i = b + lane;
                const bool unexp = i < ntop && !(cur[i] & 1ull);
                unsigned m = __ballot_sync(FULL, unexp);
                while (m && npar < a.w) {
                    const int l = __ffs(m) - 1;
                    m &= m - 1;
                    if (lane == l) {
                        spar[npar] = (int32_t)((uint32_t)cur[i] >> 1);
                        cur[i] |= 1ull;                             // mark expanded
                    }
                    npar++;
                }
            }
            __syncwarp();
            if (npar == 0) break;                                    // reading #10
            E += npar;
            iters++;
            const int nch = npar * R;
            for (int cb = 0; cb < nch; cb += 32) {
                const int l = cb + lane;
                int32_t c = -1, cg = -1;
                if (l < nch) {
                    // R is a power of two in practice (16): shift instead of a division
                    const int pi = r_shift >= 0 ? (l >> r_shift) : l / R;
                    const int p = spar[pi];
                    const int2 e = __ldg(ix.G + (base + p) * (int64_t)R + (l - pi * R));
                    c = e.x;
                    cg = e.y;
                    if (c < 0 || c >= S) c = -1;                     // reading #15
                }
                process(c, cg);
            }
        }
        // ---- OUTPUT: first min(k, |Top|) entries mapped to global ids (Alg. 2)
        const bool direct = (it.meta & META_DIRECT) != 0;
        for (int t = lane; t < k; t += 32) {
            ull key = KEY_INF;
            if (t < ntop) {
                const ull kk = cur[t];
                const int32_t j = (int32_t)((uint32_t)kk >> 1);
                key = (kk & 0xFFFFFFFF00000000ull) | (uint32_t)__ldg(ix.M_hs + base + j);
            }
            if (direct) {
                a.out_ids[(int64_t)it.qid * k + t] = key == KEY_INF ? -1 : (int32_t)key_id(key);
                a.out_dists[(int64_t)it.qid * k + t] =
                    key == KEY_INF ? __uint_as_float(0x7f800000u) : key_dist(key);
            } else {
                a.item_res[(size_t)slot * k + t] = key;
            }
        }
        if (lane == 0) {
            a.item_ctr[(size_t)slot * 3 + 0] = nvis;
            a.item_ctr[(size_t)slot * 3 + 1] = E;
            a.item_ctr[(size_t)slot * 3 + 2] = iters;
            atomicAdd(&a.ctr->graph_V, (ull)nvis);
            atomicAdd(&a.ctr->graph_E, (ull)E);
            atomicAdd(&a.ctr->graph_iters, (ull)iters);
            atomicMax(&a.ctr->graph_V_max, (ull)nvis);
        }
        __syncwarp();
    }
    if (lane == 0) gtab_epoch[warp_slot] = epoch;
}

// ------------------------------------------------------------------ dispatch
typedef void (*graph_fn)(SearchArgs, GraphLayout, uint32_t *);

template <int DT>
static graph_fn pick(int team, int cpl) {
#define VF_CASE(T_, C_) if (team == T_ && cpl <= C_) return k_graph<DT, T_, C_>;
    VF_CASE(1, 2) VF_CASE(1, 4) VF_CASE(2, 4) VF_CASE(4, 4) VF_CASE(8, 4) VF_CASE(16, 4)
    VF_CASE(32, 4) VF_CASE(32, 8)
#undef VF_CASE
    return nullptr;
}

// TEAM lanes per row with ~4 16-byte chunks per lane: fewer shuffles per distance than a full
// warp per row and several rows' loads in flight per lane.
static void team_for(int chunks, int *team, int *cpl) {
    const int want = (chunks + 3) / 4;
    int t = 1;
    while (t < want && t < 32) t <<= 1;
    *team = t;
    *cpl = (chunks + t - 1) / t;
}

static graph_fn graph_kernel(const SearchArgs &a) {
    int team, cpl;
    team_for(a.ix.chunks, &team, &cpl);
    return a.ix.dtype == 0 ? pick<0>(team, cpl) : pick<1>(team, cpl);
}

int graph_smem_bytes(const SearchArgs &a) {
    return (int)(graph_layout(a.itopk, a.hash_slots).warp_bytes * kWarpsPerGraphCta);
}

int graph_max_ctas(const SearchArgs &a) {
    graph_fn f = graph_kernel(a);
    if (!f) return 0;
    const int smem = graph_smem_bytes(a);
    // occupancy queries cost microseconds: cache per (kernel, device, smem) -- small-batch latency
    struct Key { graph_fn f; int dev, smem, ctas; };
    static thread_local Key cache[16];
    static thread_local int ncache = 0;
    int dev = 0;
    cudaGetDevice(&dev);
    for (int i = 0; i < ncache; i++)
        if (cache[i].f == f && cache[i].dev == dev && cache[i].smem == smem) return cache[i].ctas;
    // the attribute is per function: set the ceiling once, never a smaller value a later call needs
    cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    int per_sm = 0, nsm = 148;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, f, 32 * kWarpsPerGraphCta, smem);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    const int ctas = per_sm * nsm;
    cache[ncache % 16] = Key{f, dev, smem, ctas};
    ncache++;
    return ctas;
}

int launch_graph(const SearchArgs &a, cudaStream_t s, int graph_items_bound, int grid_ctas) {
    if (graph_items_bound <= 0) return 0;
    graph_fn f = graph_kernel(a);
    if (!f) return -1;
    const int smem = graph_smem_bytes(a);
    int grid = grid_ctas;
    const int need = (graph_items_bound + kWarpsPerGraphCta - 1) / kWarpsPerGraphCta;
    if (grid > need) grid = need;
    if (grid < 1) grid = 1;
    // the epoch array follows the global visited tables
    uint32_t *epochs = reinterpret_cast<uint32_t *>(a.gtab + (size_t)a.n_warp_slots * a.gtab_slots);
    f<<<grid, 32 * kWarpsPerGraphCta, smem, s>>>(a, graph_layout(a.itopk, a.hash_slots), epochs);
    return 1;
}

}  // namespace vf
