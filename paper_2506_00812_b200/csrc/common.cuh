// Device helpers shared by the kernels: result keys, exact distances, the predicate, warp sort /
// merge, TMA-bulk + mbarrier wrappers.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include "vf_internal.h"

namespace vf {

typedef unsigned long long ull;
constexpr ull KEY_INF = ~0ull;
constexpr unsigned FULL = 0xffffffffu;

// A result key orders by (distance, id) (reading #6): the distance is a non-negative float whose
// IEEE bits order like unsigned integers, placed above the 32-bit id.
__device__ __forceinline__ ull make_key(float d, uint32_t id) {
    return ((ull)__float_as_uint(d) << 32) | (ull)id;
}
__device__ __forceinline__ float key_dist(ull k) { return __uint_as_float((uint32_t)(k >> 32)); }
__device__ __forceinline__ uint32_t key_id(ull k) { return (uint32_t)k; }

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

__device__ __forceinline__ uint32_t fmix32(uint32_t h) {
    h ^= h >> 16; h *= 0x85EBCA6Bu; h ^= h >> 13; h *= 0xC2B2AE35u; h ^= h >> 16;
    return h;
}

// ---------------------------------------------------------------- exact squared-L2 distances
// One 16-byte chunk of a query against one 16-byte chunk of a data row.
// u8: |q-x| per byte (vabsdiffu4) then dot of the differences with themselves (dp4a): exact int32.
// f32: (q-x)^2 accumulated with FFMA in fp32 (exact for integer-valued data < 2^24).
template <int DT> struct Acc;
template <> struct Acc<0> {
    typedef uint32_t T;
    __device__ __forceinline__ static void add(T &acc, const uint4 &q, const uint4 &x) {
        uint32_t d;
        d = __vabsdiffu4(q.x, x.x); acc = __dp4a(d, d, acc);
        d = __vabsdiffu4(q.y, x.y); acc = __dp4a(d, d, acc);
        d = __vabsdiffu4(q.z, x.z); acc = __dp4a(d, d, acc);
        d = __vabsdiffu4(q.w, x.w); acc = __dp4a(d, d, acc);
    }
    __device__ __forceinline__ static float to_float(T a) { return (float)a; }
};
template <> struct Acc<1> {
    typedef float T;
    __device__ __forceinline__ static void add(T &acc, const uint4 &q, const uint4 &x) {
        float t;
        t = __uint_as_float(q.x) - __uint_as_float(x.x); acc = fmaf(t, t, acc);
        t = __uint_as_float(q.y) - __uint_as_float(x.y); acc = fmaf(t, t, acc);
        t = __uint_as_float(q.z) - __uint_as_float(x.z); acc = fmaf(t, t, acc);
        t = __uint_as_float(q.w) - __uint_as_float(x.w); acc = fmaf(t, t, acc);
    }
    __device__ __forceinline__ static float to_float(T a) { return a; }
};

// ---------------------------------------------------------------- predicate
// verify(gid) <=> every label of the sorted query label list P[0..np) except `excl` is in the
// point's sorted label segment. Boundary-narrowing order of P:L537: smallest, largest, then the
// middle labels only inside the bracket found by the first two searches.
__device__ __forceinline__ int64_t bsearch_lab(const int32_t *__restrict__ lab, int64_t lo, int64_t hi,
                                               int32_t key) {
    while (lo < hi) {
        int64_t mid = (lo + hi) >> 1;
        int32_t v = __ldg(lab + mid);
        if (v == key) return mid;
        if (v < key) lo = mid + 1; else hi = mid;
    }
    return -1;
}

__device__ __forceinline__ bool has_label_bit(const DevIndex &ix, int slot, int32_t gid) {
    return (__ldg(ix.lbits + (int64_t)slot * ix.lbit_words + (gid >> 5)) >> (gid & 31)) & 1u;
}

// Out of line (its registers stay out of the callers' hot loops; only AND items call it), with the
// index arrays passed as scalars so no parameter struct is spilled to the stack.
static __device__ __noinline__ bool verify_pred_x(const int64_t *__restrict__ pt_off, const int32_t *__restrict__ pt_lab,
                                           const uint32_t *__restrict__ lbits, const int16_t *__restrict__ lslot,
                                           int64_t lwords, int32_t n_labels, int32_t gid, const int32_t *P, int np,
                                           int32_t excl) {
    // fast path: every label to check has a membership bitmap -> one bit per label, no search
    if (lslot) {
        bool all = true, ok = true;
        for (int t = 0; t < np && all; t++) {
            const int32_t l = P[t];
            if (l == excl) continue;
            const int sl = (l >= 0 && l < n_labels) ? lslot[l] : -1;
            if (sl < 0) all = false;
            else ok = ok && ((__ldg(lbits + (int64_t)sl * lwords + (gid >> 5)) >> (gid & 31)) & 1u);
        }
        if (all) return ok;
    }
    int i0 = 0, i1 = np - 1;
    if (i0 <= i1 && P[i0] == excl) i0++;
    if (i0 <= i1 && P[i1] == excl) i1--;
    if (i0 > i1) return true;
    const int64_t lo = __ldg(pt_off + gid), hi = __ldg(pt_off + gid + 1);
    const int64_t a = bsearch_lab(pt_lab, lo, hi, P[i0]);
    if (a < 0) return false;
    if (i0 == i1) return true;
    const int64_t b = bsearch_lab(pt_lab, a + 1, hi, P[i1]);
    if (b < 0) return false;
    for (int t = i0 + 1; t < i1; t++) {
        if (P[t] == excl) continue;
        if (bsearch_lab(pt_lab, a + 1, b, P[t]) < 0) return false;
    }
    return true;
}

// 8-byte load that asks L2 to keep the line (the signatures are re-read by every AND item)
__device__ __forceinline__ unsigned long long ld_keep(const unsigned long long *p) {
    unsigned long long v;
    asm volatile(
        "{\n.reg .b64 pol;\ncreatepolicy.fractional.L2::evict_last.b64 pol, 1.0;\n"
        "ld.global.nc.L2::cache_hint.u64 %0, [%1], pol;\n}\n"
        : "=l"(v) : "l"(p));
    return v;
}

// the labels' signature bits all set in the point's signature (else: certainly not a member)
__device__ __forceinline__ bool sig_may_have(unsigned long long sig, unsigned long long need) {
    return (sig & need) == need;
}

__device__ __forceinline__ bool verify_pred(const DevIndex &ix, int32_t gid, const int32_t *P, int np,
                                            int32_t excl) {
    if (ix.lsig) {
        unsigned long long need = 0;
        for (int t = 0; t < np; t++)
            if (P[t] != excl) need |= label_sig_bits(P[t]);
        if (!sig_may_have(ld_keep(ix.lsig + gid), need)) return false;
    }
    return verify_pred_x(ix.pt_off, ix.pt_lab, ix.lbits, ix.lbit_slot, ix.lbit_words, ix.n_labels, gid, P, np, excl);
}

// ---------------------------------------------------------------- routing of one query (a1)
// ClassifyQueries (Alg. 2) for one query, by ONE thread: sorts and deduplicates its labels in
// place (reading #22), then emits its items -- SINGLE / OR: one per non-empty label (
// reading #19); AND greedy: l* = argmin(|C_l|, l) with the other labels as predicate;
// AND parallel: every label -- each routed by the routing equation against the
// search's threshold max(T, scan_threshold) (f2), exact mode, or the f3 selectivity estimate.
__device__ __forceinline__ void route_labels(const SearchArgs &a, int32_t *L, int nraw, int *nl_out,
                                             int32_t *chosen, uint32_t *cpath, int *nch_out, uint32_t *pred_out) {
    const DevIndex &ix = a.ix;
    for (int i = 1; i < nraw; i++) {
        int32_t v = L[i];
        int j = i - 1;
        while (j >= 0 && L[j] > v) { L[j + 1] = L[j]; j--; }
        L[j + 1] = v;
    }
    int nl = 0, nch = 0;
    uint32_t pred = 0;
    for (int i = 0; i < nraw; i++)
        if (nl == 0 || L[i] != L[nl - 1]) L[nl++] = L[i];
    auto lsize = [&](int32_t l) -> int32_t {
        return (l >= 0 && l < ix.n_labels) ? ix.dir[l].size : 0;   // reading #19
    };
    if (a.op == 0 || a.op == 1) {             // SINGLE / OR: one item per non-empty label
        if (!(a.op == 0 && nl > 1))
            for (int t = 0; t < nl; t++) if (lsize(L[t]) > 0) chosen[nch++] = L[t];
    } else {                                  // AND
        bool any_empty = nl == 0;
        for (int t = 0; t < nl; t++) any_empty |= lsize(L[t]) == 0;
        if (!any_empty) {
            pred = nl > 1 ? META_PRED : 0;
            if (a.recall_mode == 0) {         // greedy: l* = argmin(|C_l|, l)
                int best = 0;
                for (int t = 1; t < nl; t++) if (lsize(L[t]) < lsize(L[best])) best = t;
                chosen[nch++] = L[best];
            } else {                          // parallel: every label
                for (int t = 0; t < nl; t++) chosen[nch++] = L[t];
            }
        }
    }
    // selectivity-aware AND routing (f3, beyond the paper; include/vf.h): expected AND-set
    // size of the greedy item under label independence, fp64, labels in ascending order
    bool and_scan = false;
    if (a.and_scan_thr > 0 && a.op == 2 && a.recall_mode == 0 && nch == 1 && nl > 1) {
        double est = (double)lsize(chosen[0]);
        for (int t = 0; t < nl; t++)
            if (L[t] != chosen[0]) est = __ddiv_rn(__dmul_rn(est, (double)lsize(L[t])), (double)ix.n_points);
        and_scan = est < (double)a.and_scan_thr;
    }
    for (int t = 0; t < nch; t++) {           // routing equation
        const int32_t s = lsize(chosen[t]);
        cpath[t] = (a.exact || s < a.scan_thr || and_scan) ? PATH_SCAN : PATH_GRAPH;
        // label sharding: an item whose label lives on another rank is shipped there
        if (ix.owner && ix.owner[chosen[t]] != ix.rank) cpath[t] |= META_REMOTE;
    }
    *nl_out = nl;
    *nch_out = nch;
    *pred_out = pred;
}

// ---------------------------------------------------------------- warp sort / merge of keys
// Bitonic sort of 32 keys, one per lane, ascending across lanes.
__device__ __forceinline__ ull warp_sort32(ull key, int lane) {
#pragma unroll
    for (int k = 2; k <= 32; k <<= 1) {
#pragma unroll
        for (int j = k >> 1; j > 0; j >>= 1) {
            ull other = __shfl_xor_sync(FULL, key, j);
            bool keep_min = ((lane & j) == 0) == ((lane & k) == 0);
            ull mn = key < other ? key : other;
            ull mx = key < other ? other : key;
            key = keep_min ? mn : mx;
        }
    }
    return key;
}

// Merge two sorted lists of DISTINCT keys, A[0..na) and C[0..nc) (both in shared memory), into
// B[0..min(cap, na+nc)) by rank: an element's output position is its index plus the number of
// elements of the other list smaller than it. Whole warp; returns the new length.
__device__ __forceinline__ int warp_merge(const ull *A, int na, const ull *C, int nc, ull *B, int cap,
                                          int lane) {
    for (int i = lane; i < na; i += 32) {
        ull a = A[i];
        int lo = 0, hi = nc;
        while (lo < hi) { int mid = (lo + hi) >> 1; if (C[mid] < a) lo = mid + 1; else hi = mid; }
        int pos = i + lo;
        if (pos < cap) B[pos] = a;
    }
    for (int j = lane; j < nc; j += 32) {
        ull c = C[j];
        int lo = 0, hi = na;
        while (lo < hi) { int mid = (lo + hi) >> 1; if (A[mid] < c) lo = mid + 1; else hi = mid; }
        int pos = j + lo;
        if (pos < cap) B[pos] = c;
    }
    __syncwarp();
    int n = na + nc;
    return n < cap ? n : cap;
}

// Register-resident top-k (k <= 32): lane i holds the i-th best key of a sorted, KEY_INF-padded
// list. Every lane offers one key; the keys beating the current k-th are inserted one at a time
// (ballot for the position, shuffle-up to shift) -- a handful of instructions per insertion, no
// shared-memory sort. Keys must be distinct (they carry the point id).
__device__ __forceinline__ ull warp_insert_topk(ull Li, ull key, int k, int lane) {
    unsigned m = __ballot_sync(FULL, key < __shfl_sync(FULL, Li, k - 1));
    while (m) {
        const int src = __ffs(m) - 1;
        m &= m - 1;
        const ull kk = __shfl_sync(FULL, key, src);
        if (kk < __shfl_sync(FULL, Li, k - 1)) {
            const int pos = __popc(__ballot_sync(FULL, lane < k && Li < kk));
            const ull up = __shfl_up_sync(FULL, Li, 1);
            if (lane > pos) Li = up;
            else if (lane == pos) Li = kk;
        }
    }
    return Li;
}

// Same contract as warp_insert_topk, for batches where many of the 32 offered keys may qualify:
// sort them (bitonic), then keep the 32 smallest of the two sorted lists -- min against the
// reversed candidates is a bitonic sequence -- and clean it up in 5 compare-exchange steps.
__device__ __forceinline__ ull warp_merge_topk(ull Li, ull key, int k, int lane) {
    const ull kth = __shfl_sync(FULL, Li, k - 1);
    const unsigned m = __ballot_sync(FULL, key < kth);
    if (m == 0) return Li;
    if (__popc(m) <= 4) return warp_insert_topk(Li, key, k, lane);
    const ull s = warp_sort32(key < kth ? key : KEY_INF, lane);
    const ull r = __shfl_sync(FULL, s, 31 - lane);
    ull c = Li < r ? Li : r;
#pragma unroll
    for (int j = 16; j > 0; j >>= 1) {
        const ull o = __shfl_xor_sync(FULL, c, j);
        const bool lo = (lane & j) == 0;
        c = lo ? (c < o ? c : o) : (c < o ? o : c);
    }
    return lane < k ? c : KEY_INF;
}

// ---------------------------------------------------------------- TMA bulk copy + mbarrier
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    uint32_t addr = smem_u32(bar);
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(addr), "r"(parity) : "memory");
}
// 1-D bulk copy global -> shared (TMA engine), completion counted on `bar` in bytes.
__device__ __forceinline__ void tma_load_1d(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
        ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void named_bar_sync(int id, int nthreads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

}  // namespace vf
