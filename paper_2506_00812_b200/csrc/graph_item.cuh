// a3 -- the beam search of ONE (query, label) item by one warp (Alg. 2; P:L442-L444;
// AND inline filtering P:L549-L550), following the deterministic reading of DESIGN.md §2 c.2.
// Shared by the batched graph kernel (graph.cu: persistent warps over the batch's graph items) and
// the per-query CTA path (small.cu: small batches and the persistent serving kernel).
//
// Per warp in shared memory: the top-M list (itopk keys, double-buffered), 32 candidate keys,
// and an open-addressing visited set of local ids; when the visited set would pass half its
// capacity new ids spill into a per-warp global-memory table (64-bit entries tagged with an item
// epoch, so it is never cleared) -- the visited set is exact, never "forgettable", which is what
// makes the result schedule-independent (reading #12).
// Per iteration: the first w unexpanded entries of Top become parents (Alg. 2); their G_l
// rows are read -- each edge carries (local id, global id), i.e. the M_HS mapping of P:L444 is
// folded into the row so a child costs no dependent M_HS gather; children are de-duplicated within
// the batch (match.any), checked/inserted in the visited set, filtered by the AND predicate, and
// their vector rows gathered with 16-byte loads by "teams" of lanes (TEAM lanes per row, up to 8
// rows' loads in flight per lane); team-reduced exact distances become keys
// (dist, local id << 1 | expanded) merged into Top (single insertions for a few survivors, else a
// warp bitonic sort + merge).
#pragma once
#include "common.cuh"

#ifndef VF_PREFETCH_ADJ
#define VF_PREFETCH_ADJ 1
#endif

namespace vf {

struct GraphLayout {
    int itopk, hash_slots;
    size_t off_topA, off_topB, off_cbuf, off_fgid, off_floc, off_par, off_hash, warp_bytes;
};

static inline GraphLayout graph_layout(int itopk, int hash_slots) {
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

// the shared table has any number H of slots: a slot is the high word of hash * H, probing wraps
__device__ __forceinline__ uint32_t vis_slot(int32_t c, uint32_t H) { return __umulhi(vis_hash(c), H); }
__device__ __forceinline__ uint32_t vis_next(uint32_t h, uint32_t H) { return h + 1 == H ? 0u : h + 1; }
__device__ __forceinline__ bool smem_find(const int32_t *tab, uint32_t H, int32_t c) {
    uint32_t h = vis_slot(c, H);
    for (;;) {
        const int32_t v = tab[h];
        if (v == c) return true;
        if (v < 0) return false;
        h = vis_next(h, H);
    }
}
__device__ __forceinline__ void smem_insert(int32_t *tab, uint32_t H, int32_t c) {
    uint32_t h = vis_slot(c, H);
    for (;;) {
        const int32_t old = atomicCAS(tab + h, -1, c);
        if (old == -1 || old == c) return;
        h = vis_next(h, H);
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

// TEAM lanes per row with ~4 16-byte chunks per lane: fewer shuffles per distance than a full
// warp per row and several rows' loads in flight per lane.
static inline void team_for(int chunks, int *team, int *cpl) {
    const int want = (chunks + 3) / 4;
    int t = 1;
    while (t < want && t < 32) t <<= 1;
    *team = t;
    *cpl = (chunks + t - 1) / t;
}

// One item: the label's graph G_l (S points at rows [base, base+S) of G_HS / M_HS), the query's
// padded row (global or shared memory), its content hash and, for AND items, its sorted labels.
struct BeamItem {
    int32_t label, S;
    int64_t base;
    bool has_pred;
    const int32_t *P;
    int np;
    uint32_t qh;
    const uint8_t *qrow;
};
struct BeamOut {
    const ull *top;   // shared memory: ntop keys (dist, local id << 1 | expanded), ascending
    int ntop, nvis, E, iters;
};

// The whole warp calls it; `wb` = this warp's GL.warp_bytes of shared memory, `gtab` its global
// overflow table (gmask + 1 slots) and `epoch` a value never used before with that table.
template <int DT, int TEAM, int MAXCPL>
__device__ __forceinline__ BeamOut beam_item(const SearchArgs &a, const DevIndex &ix, const GraphLayout &GL,
                                             uint8_t *wb, ull *gtab, uint64_t gmask, uint32_t epoch,
                                             const BeamItem &bi, int lane) {
    typedef Acc<DT> A;
    constexpr int RP = 32 / TEAM;                       // rows per pass
    constexpr int GROUP = MAXCPL >= 8 ? 1 : (MAXCPL >= 4 ? 2 : 8 / MAXCPL);  // passes in flight together
    const int team = lane / TEAM, tl = lane % TEAM;
    ull *topA = reinterpret_cast<ull *>(wb + GL.off_topA);
    ull *topB = reinterpret_cast<ull *>(wb + GL.off_topB);
    ull *cbuf = reinterpret_cast<ull *>(wb + GL.off_cbuf);
    int32_t *fgid = reinterpret_cast<int32_t *>(wb + GL.off_fgid);
    int32_t *floc = reinterpret_cast<int32_t *>(wb + GL.off_floc);
    int32_t *spar = reinterpret_cast<int32_t *>(wb + GL.off_par);
    int32_t *htab = reinterpret_cast<int32_t *>(wb + GL.off_hash);
    const int M = GL.itopk, H = GL.hash_slots, R = ix.R;
    const int chunks = ix.chunks, row_bytes = ix.row_bytes;
    const uint32_t HU = (uint32_t)H;
    const int r_shift = (R & (R - 1)) == 0 ? __ffs(R) - 1 : -1;
    const unsigned lt_mask = (1u << lane) - 1u;
    const int32_t S = bi.S;
    const int64_t base = bi.base;
    const bool has_pred = bi.has_pred;

    uint4 qreg[MAXCPL];
    const uint4 *qrow = reinterpret_cast<const uint4 *>(bi.qrow);
#pragma unroll
    for (int j = 0; j < MAXCPL; j++) {
        const int c = tl + j * TEAM;
        qreg[j] = c < chunks ? qrow[c] : make_uint4(0, 0, 0, 0);
    }
    // a label of at most 32 * H points gets a membership BITMAP of its local ids in the same shared
    // words instead of the hash table: one atomicOr per child, no probing, never a spill (exact)
    const bool vis_bm = S <= 32 * H && !(a.knobs & KNOB_VIS_HASH_ONLY);
    const int32_t vis_clear = vis_bm ? 0 : -1;
    for (int i = lane; i < H; i += 32) htab[i] = vis_clear;
    bool g_used = false;
    int n_smem = 0, nvis = 0, ntop = 0, E = 0, iters = 0;
    ull *cur = topA, *oth = topB;
    __syncwarp();

    // Process one batch of candidate local ids (one per lane, -1 = none): visited-set
    // check/insert, M_HS mapping, predicate, distances, merge into Top.
    auto process = [&](int32_t c, int32_t gid) {
        bool isnew;
        int nnew;
        if (vis_bm) {
            isnew = false;
            if (c >= 0) {
                const uint32_t bit = 1u << (c & 31);
                isnew = !(atomicOr(reinterpret_cast<uint32_t *>(htab) + (c >> 5), bit) & bit);
            }
            nnew = __popc(__ballot_sync(FULL, isnew));
        } else if (!g_used && 2 * (n_smem + 32) <= H && !(a.knobs & KNOB_VIS_2PHASE)) {
            // the whole batch fits the shared table and nothing has spilled: one insert-if-absent
            // probe per lane (atomicCAS; of duplicate ids within the batch exactly one lane inserts,
            // and which one does not matter -- keys are ordered by (distance, id) only)
            isnew = false;
            if (c >= 0) {
                uint32_t h = vis_slot(c, HU);
                for (;;) {
                    const int32_t old = atomicCAS(htab + h, -1, c);
                    if (old == -1) { isnew = true; break; }
                    if (old == c) break;
                    h = vis_next(h, HU);
                }
            }
            nnew = __popc(__ballot_sync(FULL, isnew));
            n_smem += nnew;
        } else {
            bool v = c >= 0;
            const unsigned same = __match_any_sync(FULL, v ? c : -1 - lane);
            if (v && (__ffs(same) - 1) != lane) v = false;      // duplicate within the batch
            bool found = false;
            if (v) {
                found = smem_find(htab, HU, c);
                if (!found && g_used) found = gtab_find(gtab, gmask, epoch, c);
            }
            isnew = v && !found;
            const unsigned nm = __ballot_sync(FULL, isnew);
            nnew = __popc(nm);
            const bool use_smem = 2 * (n_smem + nnew) <= H;
            __syncwarp();
            if (isnew) {
                if (use_smem) smem_insert(htab, HU, c);
                else gtab_insert(gtab, gmask, epoch, c);
            }
            if (nnew) { if (use_smem) n_smem += nnew; else g_used = true; }
        }
        nvis += nnew;
        if (isnew && gid < 0) gid = __ldg(ix.M_hs + base + c);   // entry samples only
        bool pass = isnew;
        if (pass && has_pred) pass = verify_pred(ix, gid, bi.P, bi.np, bi.label);
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
            // so the later groups do not each pay a full DRAM round trip (one row per lane)
            const int pf = (a.knobs & KNOB_PF_MASK) >> KNOB_PF_SHIFT;
            if (lane < nc && pf != 2) {
                const uint8_t *rp = ix.X + (int64_t)fgid[lane] * row_bytes;
                if (pf == 1)      // exactly the row's bytes (rows are 16-B aligned and padded)
                    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(rp), "r"(row_bytes) : "memory");
                else
                    for (int l = 0; l < row_bytes; l += 128) asm volatile("prefetch.global.L2 [%0];" ::"l"(rp + l));
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
#if VF_PREFETCH_ADJ
        // a child entering Top is a future parent: start its adjacency row on its way to L2 now, so
        // the expansion's dependent load hits L2 instead of DRAM
        if (ck != KEY_INF && !(a.knobs & KNOB_NO_ADJ_PF))
            asm volatile("prefetch.global.L2 [%0];" ::"l"(ix.G + (base + (int64_t)((uint32_t)ck >> 1)) * R));
#endif
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
        if (M <= 64 && ns <= 8) {
            // Top of 33..64 keys as two register halves (lane i holds entries i and 32 + i): few
            // survivors are inserted one at a time -- position by two ballots, shift up across the
            // halves (A's last entry moves to B's first); entries >= M are never written back
            ull A = lane < ntop ? cur[lane] : KEY_INF;
            ull B = 32 + lane < ntop ? cur[32 + lane] : KEY_INF;
            unsigned rem = sm;
            while (rem) {
                const ull kk = __shfl_sync(FULL, ck, __ffs(rem) - 1);
                rem &= rem - 1;
                const int pos = __popc(__ballot_sync(FULL, A < kk)) + __popc(__ballot_sync(FULL, B < kk));
                const ull carry = __shfl_sync(FULL, A, 31);
                const ull upA = __shfl_up_sync(FULL, A, 1);
                const ull upB = __shfl_up_sync(FULL, B, 1);
                if (pos < 32) {
                    B = lane == 0 ? carry : upB;
                    if (lane > pos) A = upA;
                    else if (lane == pos) A = kk;
                } else {
                    const int p2 = pos - 32;
                    if (lane > p2) B = upB;
                    else if (lane == p2) B = kk;
                }
            }
            if (lane < M) cur[lane] = A;
            if (32 + lane < M) cur[32 + lane] = B;
            ntop = min(M, ntop + ns);
            __syncwarp();
            return;
        }
        if (ns <= 4) {
            // few survivors into a long Top: insert each in place -- its position by ballots over
            // the sorted list, then only the tail behind it moves up one slot (top chunk first)
            unsigned rem = sm;
            while (rem) {
                const ull kk = __shfl_sync(FULL, ck, __ffs(rem) - 1);
                rem &= rem - 1;
                int pos = 0;
                for (int b = 0; b < ntop; b += 32) {
                    const unsigned lt = __ballot_sync(FULL, b + lane < ntop && cur[b + lane] < kk);
                    pos += __popc(lt);
                    if (lt != FULL) break;                  // the rest of the sorted list is larger
                }
                if (pos >= M) continue;                      // beaten by earlier insertions
                const int last = min(ntop, M - 1);           // [pos, last) -> [pos + 1, last + 1)
                for (int hi = last; hi > pos; hi -= 32) {
                    const int i = max(pos, hi - 32) + lane;
                    const ull v = i < hi ? cur[i] : 0ull;
                    __syncwarp();
                    if (i < hi) cur[i + 1] = v;
                    __syncwarp();
                }
                if (lane == 0) cur[pos] = kk;
                ntop = min(M, ntop + 1);
                __syncwarp();
            }
            return;
        }
        {
            ck = warp_sort32(ck, lane);
            cbuf[lane] = ck;
        }
        __syncwarp();
        ntop = warp_merge(cur, ntop, cbuf, ns, oth, M, lane);
        ull *t2 = cur; cur = oth; oth = t2;
    };

    // ---- INIT: entries = all of [0, S) if S <= n_init, else the hashed samples (reading c.3)
    const int n_entry = S <= a.n_init ? S : a.n_init;
    const uint32_t hbase = fmix32(a.seed ^ bi.qh ^ fmix32((uint32_t)bi.label * 0x9E3779B9u));
    for (int e0 = 0; e0 < n_entry; e0 += 32) {
        const int i = e0 + lane;
        int32_t c = -1;
        if (i < n_entry)
            c = S <= a.n_init ? i : (int32_t)(fmix32(hbase + (uint32_t)i * 0x9E3779B9u) % (uint32_t)S);
        process(c, -1);
    }
    // ---- LOOP (Alg. 2)
    for (int iter = 0; iter < a.max_iter; iter++) {
        int npar = 0, nnext = 0;
        // VF_KNOBS bit 5: the w unexpanded entries after this iteration's parents are the next
        // parents unless a child overtakes them -- their adjacency rows start towards L2 now
        const int want_next = (a.knobs & KNOB_ADJ_PF_NEXT) ? a.w : 0;
        for (int b = 0; b < ntop && (npar < a.w || nnext < want_next); b += 32) {
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
            while (m && nnext < want_next) {
                const int l = __ffs(m) - 1;
                m &= m - 1;
                if (lane == l)
                    asm volatile("prefetch.global.L2 [%0];" ::"l"(ix.G + (base + (int64_t)((uint32_t)cur[i] >> 1)) * R));
                nnext++;
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
    BeamOut o;
    o.top = cur;
    o.ntop = ntop;
    o.nvis = nvis;
    o.E = E;
    o.iters = iters;
    return o;
}

}  // namespace vf
