// a5 -- "Merge results and map to global IDs" (Alg. 2; OR P:L523; parallel AND P:L555).
// Per query: the union of its items' top-k lists, de-duplicated by global id (reading #20), best k by (dist, gid), padded.
// Queries whose single item already wrote its row directly are skipped. The lists are short
// (k entries, a handful of items), so one lane per query runs a k-way merge over the list heads.
#include "common.cuh"

namespace vf {

// merge sorted list `L` (k keys, KEY_INF padded) into the running result res[0..*n) (sorted,
// unique gids), keeping the best k; an id already present is skipped (same point reached by two
// items of a query, reading #20).
__device__ __forceinline__ void merge_into(ull *res, int *n, ull *tmp, const ull *L, int k) {
    int i = 0, j = 0, o = 0;
    const int na = *n;
    while (o < k) {
        const ull x = i < na ? res[i] : KEY_INF;
        ull y = j < k ? L[j] : KEY_INF;
        if (x == KEY_INF && y == KEY_INF) break;
        ull v;
        if (x <= y) { v = x; i++; if (x == y) j++; }
        else { v = y; j++; }
        bool dup = false;
        for (int t = 0; t < o && !dup; t++) dup = key_id(tmp[t]) == key_id(v);
        if (!dup) tmp[o++] = v;
    }
    for (int t = 0; t < o; t++) res[t] = tmp[t];
    *n = o;
}

__global__ void __launch_bounds__(128) k_merge(SearchArgs a) {
    const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= a.n_q) return;
    const QueryInfo qi = a.qinfo[q];
    if (qi.n_items == 0) return;
    const int64_t lo = a.q_off[q], hi = a.q_off[q + 1];
    const int k = a.k;
    bool all_direct = true;
    for (int64_t s = lo; s < hi; s++) {
        const Item it = a.items[s];
        if ((it.meta & 3u) != PATH_NONE && !(it.meta & META_DIRECT)) all_direct = false;
    }
    if (all_direct) return;   // the single item wrote the output row itself
    ull res[kMaxK], tmp[kMaxK];
    int n = 0;
    for (int64_t s = lo; s < hi; s++) {
        const Item it = a.items[s];
        if ((it.meta & 3u) == PATH_NONE) continue;
        merge_into(res, &n, tmp, a.item_res + (size_t)s * k, k);
    }
    for (int t = 0; t < k; t++) {
        a.out_ids[q * k + t] = t < n ? (int32_t)key_id(res[t]) : -1;
        a.out_dists[q * k + t] = t < n ? key_dist(res[t]) : __uint_as_float(0x7f800000u);
    }
}

int launch_merge(const SearchArgs &a, cudaStream_t s) {
    if (a.n_q == 0) return 0;
    const int64_t blocks = (a.n_q + 127) / 128;
    k_merge<<<(unsigned)blocks, 128, 0, s>>>(a);
    return 1;
}

int launch_finish_keys(const SearchArgs &, cudaStream_t) { return 0; }

}  // namespace vf
