// a3 -- IVF-Graph beam search for high-specificity labels (Alg. 2; P:L442-L444;
// AND inline filtering P:L549-L550), following the deterministic reading of DESIGN.md §2 c.2.
//
// One warp per (query, label) item, persistent warps pulling items from an atomic counter; the
// search of one item is beam_item() (graph_item.cuh).
#include "graph_item.cuh"

#ifndef VF_GRAPH_MINB
#define VF_GRAPH_MINB 7      // CTAs per SM the register budget is sized for (7: 72 registers; r02aa A/B)
#endif

namespace vf {

template <int DT, int TEAM, int MAXCPL>
__global__ void __launch_bounds__(32 * kWarpsPerGraphCta, VF_GRAPH_MINB) k_graph(SearchArgs a, GraphLayout GL,
                                                                  uint32_t *gtab_epoch) {
    extern __shared__ __align__(16) uint8_t smem[];
    if (gate_skip(a)) return;     // u8 row store: the other view's kernel takes this batch
    if (threadIdx.x == 0) atomicMax(&a.ctr->graph_t0_inv, ~gtimer());
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    uint8_t *wb = smem + (size_t)wid * GL.warp_bytes;
    const DevIndex &ix = a.ix;
    const int k = a.k;
    const int warp_slot = blockIdx.x * kWarpsPerGraphCta + wid;
    ull *gtab = a.gtab + (size_t)warp_slot * a.gtab_slots;
    const uint64_t gmask = (uint64_t)a.gtab_slots - 1;
    uint32_t epoch = gtab_epoch[warp_slot];
    const int n_graph = a.ctr->n_graph;
    int cum[kGraphClasses + 1];                 // claim order: size classes, largest labels first
    cum[0] = 0;
    for (int c = 0; c < kGraphClasses; c++) cum[c + 1] = cum[c] + a.ctr->n_graph_cls[c];

    for (;;) {
        int gi = 0;
        if (lane == 0) gi = atomicAdd(&a.ctr->graph_next, 1);
        gi = __shfl_sync(FULL, gi, 0);
        if (gi >= n_graph) break;
        int c = 0;
        while (c + 1 < kGraphClasses && gi >= cum[c + 1]) c++;
        const int32_t slot = a.graph_list[c * a.graph_stride + (gi - cum[c])];
        const Item it = a.items[slot];
        const LabelDir d = ix.dir[it.label];
        const QueryInfo qi = a.qinfo[it.qid];
        BeamItem bi;
        bi.label = it.label;
        bi.S = d.size;
        bi.base = d.base;
        bi.has_pred = (it.meta & META_PRED) != 0;
        bi.P = a.qlab + a.q_off[it.qid];
        bi.np = qi.nl;
        bi.qh = qi.qh;
        bi.qrow = a.Qp + (int64_t)it.qid * ix.row_bytes;
        epoch++;
        const BeamOut bo = beam_item<DT, TEAM, MAXCPL>(a, ix, GL, wb, gtab, gmask, epoch, bi, lane);
        const int64_t base = d.base;
        const int ntop = bo.ntop, nvis = bo.nvis, E = bo.E, iters = bo.iters;
        const ull *cur = bo.top;
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
    if (lane == 0) {
        gtab_epoch[warp_slot] = epoch;
        atomicMax(&a.ctr->graph_t1, gtimer());
    }
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
