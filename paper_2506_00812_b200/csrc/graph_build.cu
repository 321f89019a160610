// f4 -- GPU construction of the per-label graphs G_l (VecFlow builds
// each high-specificity label's graph with CAGRA, "NN-descent" + "rank-based reordering"; Alg. 1
// L393 BuildGraph(C_l)). DESIGN.md §6 / reading #45-#48.
//
//  1. kNN lists: the K nearest other members of every point of an HS label, by (distance, row).
//     A tensor-core self-join (k_join): one CTA per 128-query block, candidate tiles of 256 rows
//     streamed by TMA through a smem ring, tcgen05.mma kind::i8 (u8 rows) into a double-buffered
//     128 x 256 TMEM accumulator, and an epilogue where each thread owns one query and keeps its
//     running top-K in registers (keys ||c||^2 - 2 q.c, exact int32; the per-query constant ||q||^2
//     does not change the order). Labels up to `exact_max` points are joined against all their
//     members (exact kNN); larger labels are clustered (k-means with the same join as the
//     assignment step) and each cell's points are joined against the members of its `probes`
//     nearest cells (IVF probing: approximate kNN).
//  2. CAGRA-style rank pruning (k_prune): edge x -> y (rank j in x's list) counts the "detours"
//     x -> z -> y with z at rank i < j in x's list and y at rank < j in z's list; the R neighbours
//     with the fewest detours (ties by rank) are kept.
//  3. Reverse edges (k_rev_*): y <- x for every kept x -> y (priority = its position); each point
//     keeps the R/2 best by (position, x).
//  4. Rows (k_rows): the first R/2 kept forward edges, then the reverse edges, then the remaining
//     forward edges, duplicates skipped, padded with -1.
// All arithmetic on ids is deterministic (atomic orders are re-sorted), so a build is
// reproducible bit for bit.
#include <algorithm>
#include <chrono>
#include <cstring>
#include <string>
#include <vector>

#include "host_internal.h"
#include "tc_common.cuh"

namespace vf {

constexpr int kJoinN = 256;            // candidate rows per stage (MMA N)
constexpr int kJoinM = 128;            // queries per job (MMA M = TMEM lanes)
constexpr int kJoinEpiW = 8;           // epilogue warps: 4 TMEM lane quarters x 2 column halves
constexpr int kJoinThreads = 32 * (2 + kJoinEpiW);
constexpr uint32_t kKeyBias = 1u << 25;   // ||c||^2 - 2 q.c >= -2 * 192 * 255^2 > -2^25

struct JoinJob {
    int64_t q_row;     // first query row (in the query source)
    int32_t nq;        // queries (<= 128)
    int32_t r_off;     // first candidate range
    int32_t nr;        // candidate ranges
    int32_t pad;
};
struct JoinRange {
    int64_t row;       // first candidate row (in the candidate source)
    int32_t n;
    int32_t pad;
};

struct JoinArgs {
    const JoinJob *jobs;
    int32_t n_jobs;
    int32_t *next;               // job counter (zeroed by the host)
    const JoinRange *ranges;
    const uint32_t *cn;          // candidate norms, by candidate row
    ull *out;                    // [query row - out_base][2][K] keys (bias-shifted key << 32 | cand row)
    int64_t out_base;
    int32_t exclude_self;        // query and candidate sources are the same rows: skip row == row
    int32_t nch, cw, kpad, nst;
};

struct JoinLayout {
    size_t off_bar, off_meta, off_a, off_st, st_bytes, off_lists, total;
};

// per epilogue thread, a running top-K list in shared memory ([K][256] keys: entry i of thread t at
// i * 256 + t); insertion shifts only the tail it displaces (new keys land near the end)
constexpr int kJoinListK = 32;

__host__ __device__ static JoinLayout join_layout(int kpad, int nst) {
    JoinLayout L{};
    size_t o = 0;
    L.off_bar = 0;
    o = 8 * (2 * (size_t)nst + 8);
    o = (o + 15) / 16 * 16;
    L.off_meta = o;
    o += 32 * (size_t)nst;
    o = (o + 1023) / 1024 * 1024;
    L.off_a = o;
    o += 2 * (size_t)kJoinM * kpad;
    L.st_bytes = ((size_t)kJoinN * kpad + kJoinN * 4 + 1023) / 1024 * 1024;
    o = (o + 1023) / 1024 * 1024;
    L.off_st = o;
    o += L.st_bytes * nst;
    L.off_lists = o;
    o += (size_t)kJoinListK * 32 * kJoinEpiW * 8;
    L.total = o + 1024;
    return L;
}

enum : int { JF_FIRST = 1, JF_LAST = 2, JF_END = 4 };

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&v)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
        "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
          "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
          "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
        : "r"(taddr));
}

// insert `key` (< Ls[K-1]) into the ascending shared-memory list Ls[i * S] (i < K); returns the
// new K-th key
template <int K>
__device__ __noinline__ ull list_insert_s(ull *Ls, ull key) {
    constexpr int S = 32 * kJoinEpiW;
    int i = K - 1;
    while (i > 0) {
        const ull prev = Ls[(i - 1) * S];
        if (!(key < prev)) break;
        Ls[i * S] = prev;
        i--;
    }
    Ls[i * S] = key;
    return Ls[(K - 1) * S];
}

// Stage meta (32 B): q_row, nq, flags | abuf << 8 | (job parity) << 9, candidate row0, ncols
struct JMeta {
    int64_t q_row;
    int32_t nq, flags, row0, ncols, pad0, pad1;
};

template <int K>
__global__ void __launch_bounds__(kJoinThreads, 1)
    k_join(JoinArgs A, const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_c) {
    static_assert(K <= kJoinListK, "list capacity");
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
    const int nst = A.nst, nch = A.nch, cw = A.cw, kpad = A.kpad;
    const JoinLayout SL = join_layout(kpad, nst);
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem + SL.off_bar);
    uint64_t *full = bars, *empty = bars + nst;
    uint64_t *afull = bars + 2 * nst, *aempty = afull + 2, *accfull = afull + 4, *accempty = afull + 6;
    JMeta *meta = reinterpret_cast<JMeta *>(smem + SL.off_meta);
    uint8_t *abuf_s = smem + SL.off_a;
    uint8_t *st = smem + SL.off_st;
    __shared__ uint32_t s_tmem;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    if (threadIdx.x == 0) {
        for (int i = 0; i < nst; i++) { mbar_init(full + i, 1); mbar_init(empty + i, kJoinEpiW); }
        for (int i = 0; i < 2; i++) {
            mbar_init(afull + i, 1);
            mbar_init(aempty + i, 1);
            mbar_init(accfull + i, 1);
            mbar_init(accempty + i, kJoinEpiW);
        }
        fence_mbar_init();
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&s_tmem)),
                     "r"(2 * kJoinN));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tbase = s_tmem;
    const size_t a_bytes = (size_t)kJoinM * kpad;

    if (warp == 0) {
        // ------------------------------------------------------------ producer
        uint32_t n = 0, jc = 0;
        for (;;) {
            int j = 0;
            if (lane == 0) j = atomicAdd(A.next, 1);
            j = __shfl_sync(FULL, j, 0);
            const bool end = j >= A.n_jobs;
            const JoinJob jb = end ? JoinJob{} : A.jobs[j];
            const int ab = jc & 1;
            if (!end && lane == 0) {
                // the query block (A operand), once per job
                mbar_wait(aempty + ab, ((jc >> 1) & 1) ^ 1);
                mbar_arrive_expect_tx(afull + ab, (uint32_t)(nch * kJoinM * cw));
                for (int c = 0; c < nch; c++)
                    tma_load_2d(abuf_s + (size_t)ab * a_bytes + (size_t)c * kJoinM * cw, &tm_q, c * cw, (int)jb.q_row,
                                afull + ab);
            }
            // candidate stages: every range of the job in tiles of <= 256 rows
            int total = 0;
            if (!end)
                for (int r = 0; r < jb.nr; r++) total += (A.ranges[jb.r_off + r].n + kJoinN - 1) / kJoinN;
            int si = 0;
            for (int r = 0; end ? si == 0 : r < jb.nr; r++) {
                const JoinRange rg = end ? JoinRange{0, 0, 0} : A.ranges[jb.r_off + r];
                const int ntile = end ? 1 : (rg.n + kJoinN - 1) / kJoinN;
                for (int t = 0; t < ntile; t++, si++) {
                    const int slot = n % nst;
                    uint8_t *sp = st + (size_t)slot * SL.st_bytes;
                    uint32_t *scn = reinterpret_cast<uint32_t *>(sp + (size_t)kJoinN * kpad);
                    if (lane == 0) mbar_wait(empty + slot, ((n / nst) & 1) ^ 1);
                    __syncwarp();
                    const int64_t row0 = rg.row + (int64_t)t * kJoinN;
                    const int ncols = end ? 0 : min(kJoinN, rg.n - t * kJoinN);
                    // candidate norms by the lanes (any alignment), then the TMA tiles
                    for (int c = lane; c < ncols; c += 32) scn[c] = __ldg(A.cn + row0 + c);
                    __syncwarp();
                    if (lane == 0) {
                        JMeta m;
                        m.q_row = jb.q_row;
                        m.nq = jb.nq;
                        m.flags = end ? JF_END
                                      : ((si == 0 ? JF_FIRST : 0) | (si == total - 1 ? JF_LAST : 0) | (ab << 8) |
                                         ((int)((jc >> 1) & 1) << 9));
                        m.row0 = (int32_t)row0;
                        m.ncols = ncols;
                        meta[slot] = m;
                        if (end) {
                            mbar_arrive(full + slot);
                        } else {
                            mbar_arrive_expect_tx(full + slot, (uint32_t)(nch * kJoinN * cw));
                            for (int c = 0; c < nch; c++) {
                                uint8_t *dst = sp + (size_t)c * kJoinN * cw;
                                tma_load_2d(dst, &tm_c, c * cw, (int)row0, full + slot);
                                tma_load_2d(dst + (size_t)kJoinM * cw, &tm_c, c * cw, (int)row0 + kJoinM, full + slot);
                            }
                        }
                    }
                    __syncwarp();
                    n++;
                }
            }
            if (end) break;
            jc++;
        }
    } else if (warp == 1) {
        // ------------------------------------------------------------ MMA issuer
        uint32_t n = 0;
        for (;;) {
            const int slot = n % nst, buf = n & 1;
            mbar_wait(full + slot, (n / nst) & 1);
            const JMeta m = meta[slot];
            if (m.flags & JF_END) break;
            const int ab = (m.flags >> 8) & 1;
            if (m.flags & JF_FIRST) mbar_wait(afull + ab, (m.flags >> 9) & 1);
            mbar_wait(accempty + buf, ((n >> 1) & 1) ^ 1);
            tc_fence_after();
            if (lane == 0) {
                const uint32_t a0 = smem_u32(abuf_s + (size_t)ab * a_bytes);
                const uint32_t b0 = smem_u32(st + (size_t)slot * SL.st_bytes);
                const uint32_t id = idesc_of<0>(kJoinN);
                const uint32_t td = tbase + (uint32_t)(buf * kJoinN);
                uint32_t acc = 0;
                for (int c = 0; c < nch; c++)
                    for (int s = 0; s < cw / 32; s++) {
                        mma_issue<0>(td, smem_desc(a0 + c * kJoinM * cw + s * 32, cw),
                                     smem_desc(b0 + c * kJoinN * cw + s * 32, cw), id, acc);
                        acc = 1;
                    }
                if (m.flags & JF_LAST) mma_commit(aempty + ab);
                mma_commit(accfull + buf);
            }
            __syncwarp();
            n++;
        }
    } else {
        // ------------------------------------------------------------ epilogue (8 warps)
        const int quarter = warp & 3, half = (warp - 2) >> 2;
        const int r = quarter * 32 + lane;                 // query of this thread (TMEM lane)
        ull *Ls = reinterpret_cast<ull *>(smem + SL.off_lists) + (threadIdx.x - 64);
        constexpr int LS = 32 * kJoinEpiW;
        for (int i = 0; i < K; i++) Ls[i * LS] = KEY_INF;
        ull kth = KEY_INF;
        uint32_t n = 0;
        for (;;) {
            const int slot = n % nst, buf = n & 1;
            mbar_wait(full + slot, (n / nst) & 1);
            const JMeta m = meta[slot];
            if (m.flags & JF_END) break;
            mbar_wait(accfull + buf, (n >> 1) & 1);
            tc_fence_after();
            const uint32_t *scn = reinterpret_cast<const uint32_t *>(st + (size_t)slot * SL.st_bytes + (size_t)kJoinN * kpad);
            const bool valid = r < m.nq;
            const int64_t qrow = m.q_row + r;
            uint32_t thr = (uint32_t)(kth >> 32);
            const int c_lo = half * (kJoinN / 2);
#pragma unroll 1
            for (int c0 = c_lo; c0 < c_lo + kJoinN / 2; c0 += 32) {
                if (c0 >= m.ncols) break;                 // warp-uniform
                uint32_t v[32];
                tmem_ld32(tbase + ((uint32_t)(quarter * 32) << 16) + (uint32_t)(buf * kJoinN + c0), v);
                tmem_wait_ld();
                if (!valid) continue;
#pragma unroll
                for (int j4 = 0; j4 < 32; j4 += 4) {
                    const uint4 cn4 = *reinterpret_cast<const uint4 *>(scn + c0 + j4);
                    const uint32_t cnv[4] = {cn4.x, cn4.y, cn4.z, cn4.w};
#pragma unroll
                    for (int jj = 0; jj < 4; jj++) {
                        const int col = c0 + j4 + jj;
                        const uint32_t key32 = (uint32_t)((int32_t)cnv[jj] - 2 * (int32_t)v[j4 + jj]) + kKeyBias;
                        if (key32 <= thr && col < m.ncols) {
                            const int64_t crow = (int64_t)m.row0 + col;
                            if (!(A.exclude_self && crow == qrow)) {
                                const ull key = ((ull)key32 << 32) | (uint32_t)crow;
                                if (key < kth) {
                                    kth = list_insert_s<K>(Ls, key);
                                    thr = (uint32_t)(kth >> 32);
                                }
                            }
                        }
                    }
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) {
                mbar_arrive(accempty + buf);
                mbar_arrive(empty + slot);
            }
            if (m.flags & JF_LAST) {
                if (valid) {
                    ull *o = A.out + ((qrow - A.out_base) * 2 + half) * K;
                    for (int i = 0; i < K; i++) o[i] = Ls[i * LS];
                }
                for (int i = 0; i < K; i++) Ls[i * LS] = KEY_INF;
                kth = KEY_INF;
            }
            n++;
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tbase), "r"(2 * kJoinN));
    }
}

// Merge the two column halves of every query: the K smallest keys, mapped through `rowmap`
// (candidate row -> output id; nullptr: row - map_base) into out_ids[q][K] (-1 padded).
template <int K>
__global__ void k_join_merge(const ull *__restrict__ part, int64_t n, const int32_t *__restrict__ rowmap,
                             int64_t map_base, int32_t *__restrict__ out_ids) {
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x) {
        const ull *a = part + q * 2 * K, *b = a + K;
        int i = 0, j = 0;
        for (int t = 0; t < K; t++) {
            const ull x = a[i], y = b[j];
            const ull m = x < y ? x : y;
            if (x < y) i++; else j++;
            int32_t id = -1;
            if (m != KEY_INF) {
                const int64_t row = (int64_t)(uint32_t)m;
                id = rowmap ? rowmap[row] : (int32_t)(row - map_base);
            }
            out_ids[q * K + t] = id;
        }
    }
}

// ---------------------------------------------------------------- rows, norms, k-means helpers
// out[r] = X[ids[r]] (u8 rows of row_bytes), norms[r] = ||out[r]||^2 (exact int32)
__global__ void k_gather_u8(const uint8_t *__restrict__ X, int row_bytes, const int32_t *__restrict__ ids,
                            int64_t n, uint8_t *__restrict__ out, uint32_t *__restrict__ norms) {
    const int lane = threadIdx.x & 31;
    const int64_t w0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int words = row_bytes >> 2;
    for (int64_t r = w0; r < n; r += nw) {
        const uint32_t *src = reinterpret_cast<const uint32_t *>(X + (int64_t)ids[r] * row_bytes);
        uint32_t *dst = reinterpret_cast<uint32_t *>(out + r * row_bytes);
        uint32_t s = 0;
        for (int i = lane; i < words; i += 32) {
            const uint32_t v = __ldg(src + i);
            dst[i] = v;
            s = __dp4a(v, v, s);
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(FULL, s, o);
        if (lane == 0) norms[r] = s;
    }
}

// k-means update: per-cell coordinate sums (u32: <= 8.45M * 255 < 2^32) and counts
__global__ void k_cell_sums(const uint8_t *__restrict__ X, int row_bytes, int dim, int64_t n,
                            const int32_t *__restrict__ cell, uint32_t *__restrict__ sums, uint32_t *__restrict__ cnt) {
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n * dim; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = e / dim;
        const int d = (int)(e - r * dim);
        const int c = cell[r];
        atomicAdd(sums + (int64_t)c * dim + d, (uint32_t)X[r * row_bytes + d]);
        if (d == 0) atomicAdd(cnt + c, 1u);
    }
}

// centroid = rounded mean (u8 row), unchanged when the cell is empty; its norm
__global__ void k_cell_means(const uint32_t *__restrict__ sums, const uint32_t *__restrict__ cnt, int dim, int row_bytes,
                             int64_t B, uint8_t *__restrict__ C, uint32_t *__restrict__ cn) {
    const int lane = threadIdx.x & 31;
    const int64_t w0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t b = w0; b < B; b += nw) {
        const uint32_t c = cnt[b];
        uint32_t s = 0;
        for (int d = lane; d < row_bytes; d += 32) {
            uint32_t v = C[b * row_bytes + d];
            if (c > 0 && d < dim) v = (uint32_t)((sums[b * dim + d] + c / 2) / c);
            if (d >= dim) v = 0;
            C[b * row_bytes + d] = (uint8_t)v;
            s += v * v;
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(FULL, s, o);
        if (lane == 0) cn[b] = s;
    }
}

// ---------------------------------------------------------------- pruning, reverse edges, rows
// CAGRA rank-based pruning, one warp per point x of a label: lane j holds y_j = knn[x][j]; for every
// i < K, z = y_i's list is loaded (lane t holds knn[z][t]); y_j gains a detour when it appears in
// z's list at a rank < j (and i < j). The R entries with the fewest detours (then rank) are kept.
__global__ void k_prune(const int32_t *__restrict__ knn, int K, int64_t n, const int64_t *__restrict__ node_base,
                        int R, int32_t *__restrict__ pruned) {
    const int lane = threadIdx.x & 31;
    const int64_t w0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t x = w0; x < n; x += nw) {
        const int64_t base = node_base[x];               // first row of x's label
        const int32_t y = lane < K ? knn[x * K + lane] : -1;
        int det = 0;
        for (int i = 0; i + 1 < K; i++) {
            const int32_t z = __shfl_sync(FULL, y, i);
            if (z < 0) break;                            // lists are -1 padded at the end
            const int32_t zt = lane < K ? knn[(base + z) * K + lane] : -2;
            for (int t = 0; t < K; t++) {
                const int32_t v = __shfl_sync(FULL, zt, t);
                if (lane > i && t < lane && v == y && y >= 0) det++;
            }
        }
        // sort lanes by (valid, detours, rank)
        const uint32_t key = y < 0 ? 0xFFFFFFFFu : ((uint32_t)det << 8) | (uint32_t)lane;
        const ull s = warp_sort32(((ull)key << 32) | (uint32_t)y, lane);
        if (lane < R) pruned[x * R + lane] = (uint32_t)(s >> 32) == 0xFFFFFFFFu ? -1 : (int32_t)(uint32_t)s;
    }
}

// reverse-edge candidates: count, then fill (key = position << 32 | source local id)
__global__ void k_rev_count(const int32_t *__restrict__ pruned, int R, int64_t n, const int64_t *__restrict__ node_base,
                            uint32_t *__restrict__ cnt) {
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n * R; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t x = e / R;
        const int32_t y = pruned[e];
        if (y >= 0) atomicAdd(cnt + node_base[x] + y, 1u);
    }
}
__global__ void k_rev_fill(const int32_t *__restrict__ pruned, int R, int64_t n, const int64_t *__restrict__ node_base,
                           const int64_t *__restrict__ off, uint32_t *__restrict__ fill, ull *__restrict__ keys) {
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n * R; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t x = e / R;
        const int p = (int)(e - x * R);
        const int32_t y = pruned[e];
        if (y < 0) continue;
        const int64_t yy = node_base[x] + y;
        const uint32_t pos = atomicAdd(fill + yy, 1u);
        keys[off[yy] + pos] = ((ull)p << 32) | (uint32_t)(x - node_base[x]);
    }
}

// final rows, one warp per point: forward[:h] + the h best reverse keys + forward[h:], no duplicates
constexpr int kRowsThreads = 256;
__global__ void __launch_bounds__(kRowsThreads) k_rows(const int32_t *__restrict__ pruned, int R, int64_t n,
                                                       const int64_t *__restrict__ off, const ull *__restrict__ keys,
                                                       int32_t *__restrict__ rows) {
    __shared__ int32_t sb[kRowsThreads / 32][96];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int64_t w0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int h = R / 2;
    int32_t *b = sb[wid];
    for (int64_t x = w0; x < n; x += nw) {
        // the h smallest reverse keys (deterministic: sorted, whatever the atomic fill order)
        ull best = KEY_INF;           // lane t < h: the t-th smallest so far
        const int64_t lo = off[x], hi = off[x + 1];
        for (int64_t e0 = lo; e0 < hi; e0 += 32) {
            const ull v = e0 + lane < hi ? keys[e0 + lane] : KEY_INF;
            const ull s = warp_sort32(v, lane);
            // the 32 smallest of best (ascending in lanes < h) and s (ascending): min against the
            // reversed s is bitonic, five compare-exchange steps sort it
            const ull r = __shfl_sync(FULL, s, 31 - lane);
            ull m = lane < h ? best : KEY_INF;
            m = m < r ? m : r;
#pragma unroll
            for (int j = 16; j > 0; j >>= 1) {
                const ull o = __shfl_xor_sync(FULL, m, j);
                m = ((lane & j) == 0) ? (m < o ? m : o) : (m < o ? o : m);
            }
            best = m;
        }
        if (lane < R) b[lane] = pruned[x * R + lane];
        if (lane < h) b[64 + lane] = best != KEY_INF ? (int32_t)(uint32_t)best : -1;
        __syncwarp();
        if (lane == 0) {
            int32_t *out = b + 32;
            int no = 0;
            auto push = [&](int32_t v) {
                if (v < 0 || no >= R) return;
                for (int t = 0; t < no; t++) if (out[t] == v) return;
                out[no++] = v;
            };
            for (int t = 0; t < h; t++) push(b[t]);
            for (int t = 0; t < h; t++) push(b[64 + t]);
            for (int t = h; t < R; t++) push(b[t]);
            for (int t = no; t < R; t++) out[t] = -1;
        }
        __syncwarp();
        if (lane < R) rows[x * R + lane] = b[32 + lane];
        __syncwarp();
    }
}

}  // namespace vf

// ================================================================ host: vf_build_graphs
namespace vf {

// Merge kernel with id maps (see k_join_merge): query q's output row is qmap[q] (or q); candidate
// row c maps to rowmap[c] (or c - qbase[q] / c - base_const).
template <int K>
__global__ void k_join_merge_map(const ull *__restrict__ part, int64_t n, const int32_t *__restrict__ rowmap,
                                 const int64_t *__restrict__ qbase, int64_t base_const, const int32_t *__restrict__ qmap,
                                 int32_t *__restrict__ out_ids) {
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x) {
        const ull *a = part + q * 2 * K, *b = a + K;
        const int64_t orow = qmap ? qmap[q] : q;
        const int64_t base = qbase ? qbase[q] : base_const;
        int i = 0, j = 0;
        for (int t = 0; t < K; t++) {
            const ull x = i < K ? a[i] : KEY_INF, y = j < K ? b[j] : KEY_INF;
            const bool ta = x < y;
            const ull m = ta ? x : y;
            if (ta) i++; else j++;
            int32_t id = -1;
            if (m != KEY_INF) {
                const int64_t row = (int64_t)(uint32_t)m;
                id = rowmap ? rowmap[row] : (int32_t)(row - base);
            }
            out_ids[orow * K + t] = id;
        }
    }
}

}  // namespace vf

using namespace vf;

namespace {

struct JoinGeom {
    int rb, cw, kpad, nch, nst;
    size_t smem;
};

JoinGeom join_geom(int rb) {
    JoinGeom g{};
    g.rb = rb;
    g.cw = rb % 128 == 0 ? 128 : rb % 64 == 0 ? 64 : 32;
    g.kpad = (rb + g.cw - 1) / g.cw * g.cw;
    g.nch = g.kpad / g.cw;
    int nst = 8;
    while (nst > 1 && join_layout(g.kpad, nst).total > 227 * 1024 - 256) nst--;   // + static smem
    g.nst = nst;
    g.smem = join_layout(g.kpad, nst).total;
    return g;
}

struct Joiner {
    JoinGeom g;
    DevBuf jobs, ranges, ctr;
    int nsm = 148;
    int64_t pairs = 0;
    cudaStream_t s = nullptr;

    template <int K>
    vf_status run(const std::vector<JoinJob> &jv, const std::vector<JoinRange> &rv, const void *tm_q,
                  const void *tm_c, const uint32_t *cn, ull *part, int64_t out_base, int exclude_self) {
        if (jv.empty()) return VF_OK;
        VF_CUDA(jobs.ensure(jv.size() * sizeof(JoinJob)));
        VF_CUDA(ranges.ensure(std::max<size_t>(rv.size(), 1) * sizeof(JoinRange)));
        VF_CUDA(ctr.ensure(64));
        VF_CUDA(cudaMemcpyAsync(jobs.p, jv.data(), jv.size() * sizeof(JoinJob), cudaMemcpyHostToDevice, s));
        if (!rv.empty()) VF_CUDA(cudaMemcpyAsync(ranges.p, rv.data(), rv.size() * sizeof(JoinRange), cudaMemcpyHostToDevice, s));
        VF_CUDA(cudaMemsetAsync(ctr.p, 0, 64, s));
        for (const JoinJob &j : jv)
            for (int r = 0; r < j.nr; r++) pairs += (int64_t)j.nq * rv[(size_t)j.r_off + r].n;
        JoinArgs A{};
        A.jobs = jobs.as<JoinJob>();
        A.n_jobs = (int32_t)jv.size();
        A.next = ctr.as<int32_t>();
        A.ranges = ranges.as<JoinRange>();
        A.cn = cn;
        A.out = part;
        A.out_base = out_base;
        A.exclude_self = exclude_self;
        A.nch = g.nch;
        A.cw = g.cw;
        A.kpad = g.kpad;
        A.nst = g.nst;
        VF_CUDA(cudaFuncSetAttribute(k_join<K>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)g.smem));
        const int grid = (int)std::min<size_t>(jv.size(), (size_t)nsm);
        k_join<K><<<grid, kJoinThreads, g.smem, s>>>(A, *reinterpret_cast<const CUtensorMap *>(tm_q),
                                                     *reinterpret_cast<const CUtensorMap *>(tm_c));
        VF_CUDA(cudaGetLastError());
        return VF_OK;
    }
};

double ms_since(std::chrono::steady_clock::time_point t0) {
    return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
}

}  // namespace

extern "C" vf_status vf_build_graphs(const vf_graph_desc *d, int64_t *goff, int32_t *gids, vf_graph_report *rep) {
    auto T0 = std::chrono::steady_clock::now();
    if (!d || !goff || !d->vectors || !d->posting_offsets || (d->n_labels > 0 && !d->posting_ids))
        return fail(VF_ERR_INVALID_ARG, "NULL argument");
    if (d->n_points < 1 || d->n_points >= (1ll << 31) || d->dim < 1 || d->dim > 256 || d->n_labels < 0)
        return fail(VF_ERR_INVALID_ARG, "bad n_points / dim (1..256) / n_labels");
    const int R = d->degree_R;
    if (R < 2 || R > 32 || (R & 1)) return fail(VF_ERR_INVALID_ARG, "degree_R must be even, in [2, 32]");
    if (d->threshold_T < 1) return fail(VF_ERR_INVALID_ARG, "threshold_T must be >= 1");
    int K = d->knn_k > 0 ? d->knn_k : std::min(32, 2 * R);
    if (K < R || K > 32) return fail(VF_ERR_INVALID_ARG, "knn_k must be in [degree_R, 32]");
    K = K <= 16 ? 16 : 32;                                 // kNN list lengths the join is built for
    const int64_t exact_max = d->exact_max == 0 ? 200000 : (d->exact_max < 0 ? INT64_MAX : d->exact_max);
    const int cell = d->ivf_cell > 0 ? d->ivf_cell : 2048;
    const int P = d->ivf_probes > 0 ? std::min(16, d->ivf_probes) : 16;
    const int iters = d->kmeans_iters > 0 ? d->kmeans_iters : 4;
    const int64_t N = d->n_points;
    const int L = d->n_labels;
    const int64_t *po = d->posting_offsets;
    const int32_t *pi = d->posting_ids;
    vf_graph_report rp{};
    rp.knn_k = 0;

    // ---- labels with graphs, their rows (label order), node -> label base
    std::vector<int32_t> glab;
    goff[0] = 0;
    for (int l = 0; l < L; l++) {
        const int64_t S = po[l + 1] - po[l];
        if (S < 0) return fail(VF_ERR_INVALID_ARG, "posting_offsets must be non-decreasing");
        goff[l + 1] = goff[l] + (S >= d->threshold_T ? S : 0);
        if (S >= d->threshold_T && S > 0) glab.push_back(l);
    }
    const int64_t RT = goff[L];
    rp.n_graph_labels = (int64_t)glab.size();
    rp.rows = RT;
    if (RT == 0) {
        rp.ms_total = ms_since(T0);
        if (rep) *rep = rp;
        return VF_OK;
    }
    if (!gids) return fail(VF_ERR_INVALID_ARG, "graph_local_ids is NULL");
    if (RT >= (1ll << 31)) return fail(VF_ERR_INVALID_ARG, "too many graph rows");
    for (int32_t l : glab)
        for (int64_t e = po[l]; e < po[l + 1]; e++)
            if (pi[e] < 0 || pi[e] >= N || (e > po[l] && pi[e] <= pi[e - 1]))
                return fail(VF_ERR_INVALID_ARG, "posting lists must be strictly ascending ids in [0, n_points)");

    // ---- u8 rows (zero padded to a multiple of 32 bytes)
    const int dim = d->dim;
    const int rb = (dim + 31) / 32 * 32;
    std::vector<uint8_t> X8((size_t)N * rb, 0);
    if (d->dtype == VF_U8) {
        const uint8_t *src = static_cast<const uint8_t *>(d->vectors);
        for (int64_t i = 0; i < N; i++) std::memcpy(&X8[(size_t)i * rb], src + (size_t)i * dim, dim);
    } else if (d->dtype == VF_F32) {
        const float *src = static_cast<const float *>(d->vectors);
        for (int64_t i = 0; i < N; i++)
            for (int c = 0; c < dim; c++) {
                const float v = src[(size_t)i * dim + c];
                if (!(v >= 0.f && v <= 255.f && v == (float)(int)v))
                    return fail(VF_ERR_INVALID_ARG, "the graph builder needs u8 vectors or fp32 integers in [0, 255]");
                X8[(size_t)i * rb + c] = (uint8_t)(int)v;
            }
    } else {
        return fail(VF_ERR_INVALID_ARG, "bad dtype");
    }
    VF_CUDA(cudaSetDevice(d->device));
    cudaStream_t s;
    VF_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    struct StreamGuard { cudaStream_t s; ~StreamGuard() { cudaStreamDestroy(s); } } sg{s};
    int nsm = 148;
    VF_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, d->device));

    auto t0 = std::chrono::steady_clock::now();
    DevBuf dX, dIds, XG, XGn, nbase;
    VF_CUDA(dX.ensure(X8.size()));
    VF_CUDA(cudaMemcpyAsync(dX.p, X8.data(), X8.size(), cudaMemcpyHostToDevice, s));
    {
        std::vector<int32_t> ids((size_t)RT);
        std::vector<int64_t> nb((size_t)RT);
        for (int32_t l : glab)
            for (int64_t e = po[l]; e < po[l + 1]; e++) {
                ids[(size_t)(goff[l] + e - po[l])] = pi[e];
                nb[(size_t)(goff[l] + e - po[l])] = goff[l];
            }
        VF_CUDA(dIds.ensure((size_t)RT * 4));
        VF_CUDA(nbase.ensure((size_t)RT * 8));
        VF_CUDA(cudaMemcpyAsync(dIds.p, ids.data(), (size_t)RT * 4, cudaMemcpyHostToDevice, s));
        VF_CUDA(cudaMemcpyAsync(nbase.p, nb.data(), (size_t)RT * 8, cudaMemcpyHostToDevice, s));
        VF_CUDA(XG.ensure((size_t)RT * rb));
        VF_CUDA(XGn.ensure((size_t)RT * 4));
        k_gather_u8<<<nsm * 8, 256, 0, s>>>(dX.as<uint8_t>(), rb, dIds.as<int32_t>(), RT, XG.as<uint8_t>(), XGn.as<uint32_t>());
        VF_CUDA(cudaStreamSynchronize(s));
    }
    dIds.release();
    rp.ms_upload = ms_since(t0);

    Joiner J;
    J.g = join_geom(rb);
    J.nsm = nsm;
    J.s = s;
    alignas(64) unsigned char tm_xg[128];
    if (!encode_row_map(tm_xg, XG.p, rb, RT, J.g.cw, kJoinM)) return fail(VF_ERR_CUDA, "tensor map (graph rows)");
    DevBuf knn, part;
    VF_CUDA(knn.ensure((size_t)RT * K * 4));
    const int64_t kChunkRows = 1 << 22;
    VF_CUDA(part.ensure((size_t)std::min<int64_t>(RT, kChunkRows + exact_max) * 2 * K * 8 + 256));
    auto merge = [&](int64_t n, const int32_t *rowmap, const int64_t *qbase, int64_t base_const, const int32_t *qmap,
                     int32_t *out) -> vf_status {
        if (n <= 0) return VF_OK;
        if (K == 16) k_join_merge_map<16><<<nsm * 8, 256, 0, s>>>(part.as<ull>(), n, rowmap, qbase, base_const, qmap, out);
        else k_join_merge_map<32><<<nsm * 8, 256, 0, s>>>(part.as<ull>(), n, rowmap, qbase, base_const, qmap, out);
        VF_CUDA(cudaGetLastError());
        return VF_OK;
    };
    auto join_k = [&](const std::vector<JoinJob> &jv, const std::vector<JoinRange> &rv, const void *tq, const void *tc,
                      const uint32_t *cn, int64_t out_base, int excl) -> vf_status {
        return K == 16 ? J.run<16>(jv, rv, tq, tc, cn, part.as<ull>(), out_base, excl)
                       : J.run<32>(jv, rv, tq, tc, cn, part.as<ull>(), out_base, excl);
    };

    // ---- 1a. exact kNN: labels of <= exact_max points, in chunks of consecutive labels
    t0 = std::chrono::steady_clock::now();
    {
        size_t gi = 0;
        while (gi < glab.size()) {
            std::vector<int32_t> chunk;
            int64_t rows = 0;
            while (gi < glab.size()) {
                const int32_t l = glab[gi];
                const int64_t S = po[l + 1] - po[l];
                if (S > exact_max) {                  // an IVF label ends the chunk (rows stay contiguous)
                    gi++;
                    if (chunk.empty()) continue;
                    break;
                }
                if (!chunk.empty() && rows + S > kChunkRows) break;
                chunk.push_back(l);
                rows += S;
                gi++;
            }
            if (chunk.empty()) continue;
            // chunk rows [r0, r1) of XG: consecutive exact labels (label order)
            const int64_t r0 = goff[chunk.front()], r1 = goff[chunk.back() + 1];
            std::vector<int32_t> bysize(chunk);
            std::stable_sort(bysize.begin(), bysize.end(),
                             [&](int32_t a, int32_t b) { return po[a + 1] - po[a] > po[b + 1] - po[b]; });
            std::vector<JoinJob> jv;
            std::vector<JoinRange> rv;
            for (int32_t l : bysize) {
                const int64_t S = po[l + 1] - po[l];
                rv.push_back(JoinRange{goff[l], (int32_t)S, 0});
                for (int64_t q = 0; q < S; q += kJoinM)
                    jv.push_back(JoinJob{goff[l] + q, (int32_t)std::min<int64_t>(kJoinM, S - q), (int32_t)rv.size() - 1, 1, 0});
            }
            if ((size_t)(r1 - r0) * 2 * K * 8 > part.n) VF_CUDA(part.ensure((size_t)(r1 - r0) * 2 * K * 8));
            vf_status st = join_k(jv, rv, tm_xg, tm_xg, XGn.as<uint32_t>(), r0, 1);
            if (st != VF_OK) return st;
            // every row of [r0, r1): the two column halves -> K local ids
            st = merge(r1 - r0, nullptr, nbase.as<int64_t>() + r0, 0, nullptr, knn.as<int32_t>() + r0 * K);
            if (st != VF_OK) return st;
            rp.n_exact_labels += (int64_t)chunk.size();
        }
        VF_CUDA(cudaStreamSynchronize(s));
    }
    rp.ms_knn_exact = ms_since(t0);

    // ---- 1b. IVF-probed kNN for the larger labels
    for (int32_t l : glab) {
        const int64_t S = po[l + 1] - po[l];
        if (S <= exact_max) continue;
        rp.n_ivf_labels++;
        auto tk = std::chrono::steady_clock::now();
        const int64_t lb = goff[l];
        const int64_t B = std::max<int64_t>(2, (S + cell / 2) / cell);
        DevBuf C, Cn, sums, cnt, assign, tmpi;
        VF_CUDA(C.ensure((size_t)B * rb));
        VF_CUDA(Cn.ensure((size_t)B * 4));
        VF_CUDA(sums.ensure((size_t)B * dim * 4));
        VF_CUDA(cnt.ensure((size_t)B * 4));
        VF_CUDA(assign.ensure((size_t)S * 4));
        {
            std::vector<int32_t> init((size_t)B);
            for (int64_t i = 0; i < B; i++) init[(size_t)i] = (int32_t)(i * S / B);
            VF_CUDA(tmpi.ensure((size_t)B * 4));
            VF_CUDA(cudaMemcpyAsync(tmpi.p, init.data(), (size_t)B * 4, cudaMemcpyHostToDevice, s));
            k_gather_u8<<<nsm * 4, 256, 0, s>>>(XG.as<uint8_t>() + (size_t)lb * rb, rb, tmpi.as<int32_t>(), B,
                                                 C.as<uint8_t>(), Cn.as<uint32_t>());
        }
        alignas(64) unsigned char tm_c[128];
        if (!encode_row_map(tm_c, C.p, rb, B, J.g.cw, kJoinM)) return fail(VF_ERR_CUDA, "tensor map (centroids)");
        std::vector<JoinJob> jq;
        std::vector<JoinRange> rq{JoinRange{0, (int32_t)B, 0}};
        for (int64_t q = 0; q < S; q += kJoinM)
            jq.push_back(JoinJob{lb + q, (int32_t)std::min<int64_t>(kJoinM, S - q), 0, 1, 0});
        if ((size_t)S * 2 * 16 * 8 > part.n) VF_CUDA(part.ensure((size_t)S * 2 * 16 * 8));
        for (int it = 0; it <= iters; it++) {
            // assignment: the nearest centroid of every point (a K = 1 join)
            vf_status st = J.run<1>(jq, rq, tm_xg, tm_c, Cn.as<uint32_t>(), part.as<ull>(), lb, 0);
            if (st != VF_OK) return st;
            k_join_merge_map<1><<<nsm * 8, 256, 0, s>>>(part.as<ull>(), S, nullptr, nullptr, 0, nullptr, assign.as<int32_t>());
            if (it == iters) break;
            VF_CUDA(cudaMemsetAsync(sums.p, 0, (size_t)B * dim * 4, s));
            VF_CUDA(cudaMemsetAsync(cnt.p, 0, (size_t)B * 4, s));
            k_cell_sums<<<nsm * 8, 256, 0, s>>>(XG.as<uint8_t>() + (size_t)lb * rb, rb, dim, S, assign.as<int32_t>(),
                                                 sums.as<uint32_t>(), cnt.as<uint32_t>());
            k_cell_means<<<nsm * 4, 256, 0, s>>>(sums.as<uint32_t>(), cnt.as<uint32_t>(), dim, rb, B, C.as<uint8_t>(),
                                                  Cn.as<uint32_t>());
        }
        // points in cell order (counting sort on the host), cell ranges
        std::vector<int32_t> a((size_t)S), perm((size_t)S);
        VF_CUDA(cudaMemcpyAsync(a.data(), assign.p, (size_t)S * 4, cudaMemcpyDeviceToHost, s));
        VF_CUDA(cudaStreamSynchronize(s));
        std::vector<int64_t> coff((size_t)B + 1, 0);
        for (int64_t i = 0; i < S; i++) coff[(size_t)a[(size_t)i] + 1]++;
        for (int64_t b = 0; b < B; b++) coff[(size_t)b + 1] += coff[(size_t)b];
        {
            std::vector<int64_t> fillp(coff.begin(), coff.end() - 1);
            for (int64_t i = 0; i < S; i++) perm[(size_t)fillp[(size_t)a[(size_t)i]]++] = (int32_t)i;
        }
        DevBuf dperm, XC, XCn;
        VF_CUDA(dperm.ensure((size_t)S * 4));
        VF_CUDA(cudaMemcpyAsync(dperm.p, perm.data(), (size_t)S * 4, cudaMemcpyHostToDevice, s));
        VF_CUDA(XC.ensure((size_t)S * rb));
        VF_CUDA(XCn.ensure((size_t)S * 4));
        k_gather_u8<<<nsm * 8, 256, 0, s>>>(XG.as<uint8_t>() + (size_t)lb * rb, rb, dperm.as<int32_t>(), S, XC.as<uint8_t>(),
                                            XCn.as<uint32_t>());
        // probe lists: each cell's 16 nearest centroids (itself first)
        std::vector<JoinJob> jc;
        for (int64_t q = 0; q < B; q += kJoinM) jc.push_back(JoinJob{q, (int32_t)std::min<int64_t>(kJoinM, B - q), 0, 1, 0});
        vf_status st = J.run<16>(jc, rq, tm_c, tm_c, Cn.as<uint32_t>(), part.as<ull>(), 0, 0);
        if (st != VF_OK) return st;
        DevBuf dprobe;
        VF_CUDA(dprobe.ensure((size_t)B * 16 * 4));
        k_join_merge_map<16><<<nsm * 4, 256, 0, s>>>(part.as<ull>(), B, nullptr, nullptr, 0, nullptr, dprobe.as<int32_t>());
        std::vector<int32_t> probe((size_t)B * 16);
        VF_CUDA(cudaMemcpyAsync(probe.data(), dprobe.p, probe.size() * 4, cudaMemcpyDeviceToHost, s));
        VF_CUDA(cudaStreamSynchronize(s));
        rp.ms_kmeans += ms_since(tk);
        tk = std::chrono::steady_clock::now();
        alignas(64) unsigned char tm_xc[128];
        if (!encode_row_map(tm_xc, XC.p, rb, S, J.g.cw, kJoinM)) return fail(VF_ERR_CUDA, "tensor map (cells)");
        std::vector<JoinJob> jv;
        std::vector<JoinRange> rv;
        for (int64_t b = 0; b < B; b++) {
            if (coff[(size_t)b + 1] == coff[(size_t)b]) continue;
            // itself first, then its nearest other cells (P in all)
            std::vector<int32_t> pr{(int32_t)b};
            for (int t = 0; t < 16 && (int)pr.size() < P; t++) {
                const int32_t c = probe[(size_t)b * 16 + t];
                if (c >= 0 && c != b) pr.push_back(c);
            }
            const int32_t r_off = (int32_t)rv.size();
            for (int32_t c : pr)
                if (coff[(size_t)c + 1] > coff[(size_t)c])
                    rv.push_back(JoinRange{coff[(size_t)c], (int32_t)(coff[(size_t)c + 1] - coff[(size_t)c]), 0});
            const int32_t nr = (int32_t)rv.size() - r_off;
            for (int64_t q = coff[(size_t)b]; q < coff[(size_t)b + 1]; q += kJoinM)
                jv.push_back(JoinJob{q, (int32_t)std::min<int64_t>(kJoinM, coff[(size_t)b + 1] - q), r_off, nr, 0});
        }
        if ((size_t)S * 2 * K * 8 > part.n) VF_CUDA(part.ensure((size_t)S * 2 * K * 8));
        st = join_k(jv, rv, tm_xc, tm_xc, XCn.as<uint32_t>(), 0, 1);
        if (st != VF_OK) return st;
        // cell-order rows -> local ids, written at the query's local row
        st = merge(S, dperm.as<int32_t>(), nullptr, 0, dperm.as<int32_t>(), knn.as<int32_t>() + lb * K);
        if (st != VF_OK) return st;
        VF_CUDA(cudaStreamSynchronize(s));
        rp.ms_knn_ivf += ms_since(tk);
    }
    rp.join_pairs = J.pairs;
    rp.knn_k = K;
    if (d->knn_lists) {
        VF_CUDA(cudaMemcpyAsync(d->knn_lists, knn.p, (size_t)RT * K * 4, cudaMemcpyDeviceToHost, s));
        VF_CUDA(cudaStreamSynchronize(s));
    }
    part.release();
    XG.release();
    XGn.release();
    dX.release();

    // ---- 2. pruning, 3. reverse edges, 4. rows
    t0 = std::chrono::steady_clock::now();
    DevBuf pruned;
    VF_CUDA(pruned.ensure((size_t)RT * R * 4));
    k_prune<<<nsm * 16, 256, 0, s>>>(knn.as<int32_t>(), K, RT, nbase.as<int64_t>(), R, pruned.as<int32_t>());
    VF_CUDA(cudaGetLastError());
    VF_CUDA(cudaStreamSynchronize(s));
    knn.release();
    rp.ms_prune = ms_since(t0);
    t0 = std::chrono::steady_clock::now();
    DevBuf cntb, off, fillb, keys, rows;
    VF_CUDA(cntb.ensure((size_t)RT * 4));
    VF_CUDA(cudaMemsetAsync(cntb.p, 0, (size_t)RT * 4, s));
    k_rev_count<<<nsm * 16, 256, 0, s>>>(pruned.as<int32_t>(), R, RT, nbase.as<int64_t>(), cntb.as<uint32_t>());
    std::vector<uint32_t> hc((size_t)RT);
    VF_CUDA(cudaMemcpyAsync(hc.data(), cntb.p, (size_t)RT * 4, cudaMemcpyDeviceToHost, s));
    VF_CUDA(cudaStreamSynchronize(s));
    std::vector<int64_t> ho((size_t)RT + 1, 0);
    for (int64_t i = 0; i < RT; i++) ho[(size_t)i + 1] = ho[(size_t)i] + hc[(size_t)i];
    VF_CUDA(off.ensure(((size_t)RT + 1) * 8));
    VF_CUDA(cudaMemcpyAsync(off.p, ho.data(), ((size_t)RT + 1) * 8, cudaMemcpyHostToDevice, s));
    VF_CUDA(fillb.ensure((size_t)RT * 4));
    VF_CUDA(cudaMemsetAsync(fillb.p, 0, (size_t)RT * 4, s));
    VF_CUDA(keys.ensure((size_t)std::max<int64_t>(ho[(size_t)RT], 1) * 8));
    k_rev_fill<<<nsm * 16, 256, 0, s>>>(pruned.as<int32_t>(), R, RT, nbase.as<int64_t>(), off.as<int64_t>(),
                                        fillb.as<uint32_t>(), keys.as<ull>());
    VF_CUDA(rows.ensure((size_t)RT * R * 4));
    k_rows<<<nsm * 16, kRowsThreads, 0, s>>>(pruned.as<int32_t>(), R, RT, off.as<int64_t>(), keys.as<ull>(),
                                             rows.as<int32_t>());
    VF_CUDA(cudaGetLastError());
    VF_CUDA(cudaStreamSynchronize(s));
    rp.ms_rows = ms_since(t0);
    t0 = std::chrono::steady_clock::now();
    VF_CUDA(cudaMemcpyAsync(gids, rows.p, (size_t)RT * R * 4, cudaMemcpyDeviceToHost, s));
    VF_CUDA(cudaStreamSynchronize(s));
    rp.ms_download = ms_since(t0);
    rp.ms_total = ms_since(T0);
    if (rep) *rep = rp;
    return VF_OK;
}
