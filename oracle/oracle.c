/*
 * VecFlow CPU ORACLE -- test infrastructure only.
 *
 * A plain, slow, obviously-correct CPU implementation of what the label-filtered top-k search path
 * computes (arXiv 2506.00812, /root/reference/PAPER.md, cited as P:L<line>). It shares no code,
 * header, table or helper with the CUDA library under paper_2506_00812_b200/ and never includes
 * or links it. Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
 * legs may load it. The product path must never call it.
 *
 * Arithmetic: squared L2 (reading #4). u8 distances are exact int64; fp32 distances are computed
 * in fp64 ((double)q - (double)x)^2 summed in dimension order. Compiled with -O2 -fno-fast-math
 * -ffp-contract=off (reading #33).
 *
 * Contents (each pinned by tests/test_oracle_*.py):
 *   or_exact_knn     -- Definition 1 / 2 ground truth by brute force over all N points
 *   or_verify        -- boundary-narrowing binary-search predicate
 *   or_route         -- ClassifyQueries + AND/OR policies into work items (Alg. 2; P:L330-L337,
 *                       P:L523)
 *   or_scan_item     -- IVF-BFS exact scan of one label's posting list (+AND pre-filter) (Alg. 2
 *                       L428-L430)
 *   or_beam_search   -- IVF-Graph beam search over G_l with local ids mapped through M_l (Alg. 2
 *                       L418-L427)
 *   or_merge         -- merge results, dedup by global id, map to global ids (Alg. 2)
 *   or_search        -- the whole method: route -> per item scan/graph -> merge
 *   or_entry_hash    -- the entry-point sampler (reading c.3, "random sampling ... Label Sizes to
 *                       confine the range")
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>
#include <math.h>

enum { OR_U8 = 0, OR_F32 = 1 };
enum { OR_SINGLE = 0, OR_OR = 1, OR_AND = 2 };
enum { OR_GREEDY = 0, OR_PARALLEL = 1 };
enum { OR_PATH_NONE = 0, OR_PATH_SCAN = 1, OR_PATH_GRAPH = 2 };

/* ------------------------------------------------------------------ distance (reading #4) */
static double dist_l2sq(int dtype, int dim, const void *X, int64_t i, const void *q)
{
    double s = 0.0;
    if (dtype == OR_U8) {
        const uint8_t *x = (const uint8_t *)X + (size_t)i * dim;
        const uint8_t *y = (const uint8_t *)q;
        int64_t acc = 0;
        for (int d = 0; d < dim; d++) {
            int64_t t = (int64_t)y[d] - (int64_t)x[d];
            acc += t * t;
        }
        s = (double)acc;
    } else {
        const float *x = (const float *)X + (size_t)i * dim;
        const float *y = (const float *)q;
        for (int d = 0; d < dim; d++) {
            double t = (double)y[d] - (double)x[d];
            s += t * t;
        }
    }
    return s;
}

/* result entry and its total order: key (dist, id) ascending (reading #6) */
typedef struct { double d; int64_t id; int expanded; } entry_t;

static int cmp_entry(const void *a, const void *b)
{
    const entry_t *x = (const entry_t *)a, *y = (const entry_t *)b;
    if (x->d < y->d) return -1;
    if (x->d > y->d) return 1;
    return (x->id > y->id) - (x->id < y->id);
}

static int cmp_i32(const void *a, const void *b)
{
    int32_t x = *(const int32_t *)a, y = *(const int32_t *)b;
    return (x > y) - (x < y);
}

/* sort ascending and remove duplicates in place; returns new length (reading #22) */
static int sort_dedup(int32_t *v, int n)
{
    if (n <= 1) return n;
    qsort(v, (size_t)n, sizeof(int32_t), cmp_i32);
    int m = 1;
    for (int i = 1; i < n; i++)
        if (v[i] != v[m - 1]) v[m++] = v[i];
    return m;
}

/* ------------------------------------------------------------------ predicate
 * Point labels: global label array `lab`, the point's segment [off, off+cnt) sorted ascending.
 * verify(P) <=> P subset of L_x. P sorted ascending, deduplicated.
 * Procedure of P:L537: binary-search the smallest query label (fail -> false), then the largest
 * (fail -> false); every middle label is searched only inside the bracket between the two hits.
 * `trace` (optional, 3*np ints) records for each query label: found index, search lo, search hi.
 */
static int64_t bsearch_range(const int32_t *lab, int64_t lo, int64_t hi, int32_t key)
{
    /* binary search for key in lab[lo, hi); returns index or -1 (two pointers) */
    while (lo < hi) {
        int64_t mid = lo + (hi - lo) / 2;
        if (lab[mid] == key) return mid;
        if (lab[mid] < key) lo = mid + 1;
        else hi = mid;
    }
    return -1;
}

int or_verify(const int32_t *lab, int64_t off, int64_t cnt, const int32_t *P, int np, int64_t *trace)
{
    if (np == 0) return 1;
    int64_t lo = off, hi = off + cnt;
    int64_t a = bsearch_range(lab, lo, hi, P[0]);
    if (trace) { trace[0] = a < 0 ? -1 : a - off; trace[1] = 0; trace[2] = cnt - 1; }
    if (a < 0) return 0;
    if (np == 1) return 1;
    int64_t b = bsearch_range(lab, a + 1, hi, P[np - 1]);
    if (trace) { trace[3 * (np - 1)] = b < 0 ? -1 : b - off; trace[3 * (np - 1) + 1] = a + 1 - off;
                 trace[3 * (np - 1) + 2] = cnt - 1; }
    if (b < 0) return 0;
    for (int t = 1; t < np - 1; t++) {
        int64_t c = bsearch_range(lab, a + 1, b, P[t]);
        if (trace) { trace[3 * t] = c < 0 ? -1 : c - off; trace[3 * t + 1] = a + 1 - off;
                     trace[3 * t + 2] = b - 1 - off; }
        if (c < 0) return 0;
    }
    return 1;
}

/* ------------------------------------------------------------------ entry-point hash (c.3) */
static uint32_t fmix32(uint32_t h)
{
    h ^= h >> 16; h *= 0x85EBCA6Bu; h ^= h >> 13; h *= 0xC2B2AE35u; h ^= h >> 16;
    return h;
}

/* Query content hash: the query's D*b bytes as little-endian 32-bit words (zero padded to a word),
 * qh = fmix32( sum_w fmix32(word_w + w * 0x9E3779B9) )  (wrapping uint32 arithmetic). */
uint32_t or_query_hash(int dtype, int dim, const void *q)
{
    size_t nbytes = (size_t)dim * (dtype == OR_U8 ? 1 : 4);
    const uint8_t *b = (const uint8_t *)q;
    uint32_t acc = 0;
    for (size_t w = 0; w * 4 < nbytes; w++) {
        uint32_t word = 0;
        for (int t = 0; t < 4; t++) {
            size_t p = w * 4 + (size_t)t;
            uint32_t byte = p < nbytes ? b[p] : 0u;
            word |= byte << (8 * t);
        }
        acc += fmix32(word + (uint32_t)w * 0x9E3779B9u);
    }
    return fmix32(acc);
}

/* u_i = fmix32(base + i*0x9E3779B9) mod S, base = fmix32(seed ^ qh ^ fmix32(l * 0x9E3779B9)) */
uint32_t or_entry_hash(uint32_t seed, uint32_t qh, int32_t label, uint32_t i, uint32_t S)
{
    uint32_t base = fmix32(seed ^ qh ^ fmix32((uint32_t)label * 0x9E3779B9u));
    return fmix32(base + i * 0x9E3779B9u) % S;
}

/* ------------------------------------------------------------------ the index (Alg. 1) */
typedef struct {
    int dtype, dim;
    int64_t n_points;
    const void *X;                 /* [N, dim] global vectors */
    int32_t n_labels;
    const int64_t *post_off;       /* C_l as CSR [L+1] */
    const int32_t *post_ids;       /* ascending global ids */
    int32_t T, R;                  /* specificity threshold, degree */
    const int64_t *graph_off;      /* [L+1] rows of G_l in graph_ids (|C_l| rows for HS labels) */
    const int32_t *graph_ids;      /* rows * R local ids; -1 / >= S = no edge (reading #15) */
    /* predicate table, built here from the posting lists: point -> sorted labels */
    int64_t *pt_off;               /* [N+1] */
    int32_t *pt_lab;
} or_index;

or_index *or_index_create(int dtype, int dim, int64_t n_points, const void *X, int32_t n_labels,
                          const int64_t *post_off, const int32_t *post_ids, int32_t T, int32_t R,
                          const int64_t *graph_off, const int32_t *graph_ids)
{
    or_index *ix = (or_index *)calloc(1, sizeof(or_index));
    ix->dtype = dtype; ix->dim = dim; ix->n_points = n_points; ix->X = X;
    ix->n_labels = n_labels; ix->post_off = post_off; ix->post_ids = post_ids;
    ix->T = T; ix->R = R; ix->graph_off = graph_off; ix->graph_ids = graph_ids;
    /* transpose C_l into per-point label lists; labels visited in increasing l, so each point's
     * segment comes out sorted ascending ("contiguous and sorted") */
    ix->pt_off = (int64_t *)calloc((size_t)n_points + 1, sizeof(int64_t));
    for (int32_t l = 0; l < n_labels; l++)
        for (int64_t e = post_off[l]; e < post_off[l + 1]; e++)
            ix->pt_off[post_ids[e] + 1]++;
    for (int64_t i = 0; i < n_points; i++) ix->pt_off[i + 1] += ix->pt_off[i];
    int64_t total = ix->pt_off[n_points];
    ix->pt_lab = (int32_t *)malloc((size_t)(total > 0 ? total : 1) * sizeof(int32_t));
    int64_t *fill = (int64_t *)malloc((size_t)(n_points + 1) * sizeof(int64_t));
    memcpy(fill, ix->pt_off, (size_t)(n_points + 1) * sizeof(int64_t));
    for (int32_t l = 0; l < n_labels; l++)
        for (int64_t e = post_off[l]; e < post_off[l + 1]; e++)
            ix->pt_lab[fill[post_ids[e]]++] = l;
    free(fill);
    return ix;
}

void or_index_free(or_index *ix)
{
    if (!ix) return;
    free(ix->pt_off); free(ix->pt_lab); free(ix);
}

static int64_t label_size(const or_index *ix, int32_t l)
{
    if (l < 0 || l >= ix->n_labels) return 0;   /* unknown label = empty list (reading #19) */
    return ix->post_off[l + 1] - ix->post_off[l];
}

static int point_has(const or_index *ix, int64_t i, int32_t l)
{
    for (int64_t e = ix->pt_off[i]; e < ix->pt_off[i + 1]; e++)
        if (ix->pt_lab[e] == l) return 1;
    return 0;
}

static int pred_ok(const or_index *ix, int64_t gid, const int32_t *P, int np)
{
    return or_verify(ix->pt_lab, ix->pt_off[gid], ix->pt_off[gid + 1] - ix->pt_off[gid], P, np, NULL);
}

/* write first min(k, n) entries, pad with (-1, +inf) (reading #23) */
static void emit(const entry_t *e, int64_t n, int k, int32_t *ids, double *dists)
{
    for (int t = 0; t < k; t++) {
        if (t < n) { ids[t] = (int32_t)e[t].id; dists[t] = e[t].d; }
        else { ids[t] = -1; dists[t] = INFINITY; }
    }
}

/* ------------------------------------------------------------------ Definition 1 ground truth
 * S = { i : match(L_i) } over ALL N points; result = first min(k,|S|) of S by key (d(q,x_i), i).
 * SINGLE: l in L_i; OR: L_i cap L_q != {}; AND: L_q subset of L_i. A query with no labels has an
 * empty result for every op (reading #19). Plain membership tests, no predicate table search. */
static void exact_one(const or_index *ix, const void *q, const int32_t *lq_in, int nl, int op, int k,
                      int32_t *ids, double *dists)
{
    int32_t *lq = (int32_t *)malloc(sizeof(int32_t) * (size_t)(nl > 0 ? nl : 1));
    memcpy(lq, lq_in, sizeof(int32_t) * (size_t)nl);
    nl = sort_dedup(lq, nl);
    entry_t *S = (entry_t *)malloc(sizeof(entry_t) * (size_t)(ix->n_points > 0 ? ix->n_points : 1));
    int64_t ns = 0;
    if (nl > 0) {
        for (int64_t i = 0; i < ix->n_points; i++) {
            int m;
            if (op == OR_OR) {
                m = 0;
                for (int t = 0; t < nl && !m; t++) m = point_has(ix, i, lq[t]);
            } else {  /* SINGLE (one label) and AND: every query label present */
                m = 1;
                for (int t = 0; t < nl && m; t++) m = point_has(ix, i, lq[t]);
            }
            if (m) { S[ns].d = dist_l2sq(ix->dtype, ix->dim, ix->X, i, q); S[ns].id = i; ns++; }
        }
    }
    qsort(S, (size_t)ns, sizeof(entry_t), cmp_entry);
    emit(S, ns, k, ids, dists);
    free(S); free(lq);
}

/* ------------------------------------------------------------------ routing (a1)
 * ClassifyQueries (Alg. 2) with the routing equation: SCAN iff |C_l| < T,
 * else GRAPH; exact mode (T = inf) sends everything to SCAN. Items per query (sorted, deduped L_q):
 *   SINGLE          -> one item on its label (requires |L_q| <= 1)
 *   OR              -> one item per label with |C_l| > 0, predicate TRUE (reading #19)
 *   AND greedy      -> one item on l* = argmin(|C_l|, l), predicate L_q\{l*} (
 *                      reading #18); none if some label is empty/unknown
 *   AND parallel    -> one item per label, predicate L_q\{l}; none if some label empty
 * Item record: {qid, label, path, pred_start, pred_len}; predicate labels are written to pred_buf.
 * Returns the number of items, or -1 on an invalid query (SINGLE with > 1 label).
 * and_scan_threshold > 0 enables the selectivity-aware AND routing of SURVEY §8(f) f3 (NOT in
 * the paper; include/vf.h): a greedy item with HS l* goes to SCAN when the expected AND-set size
 * est = |C_l*| * prod over the other labels (ascending) of |C_o| / N, evaluated left to right in
 * fp64, is below the threshold. scan_threshold > T raises the routing threshold for this search
 * (the T sweep of P:L339 / P:L766-L768); <= T changes nothing. */
typedef struct { int32_t qid, label, path; int64_t pred_start; int32_t pred_len; } item_t;

static int64_t route_query(const or_index *ix, int32_t qid, const int32_t *lq_in, int nl, int op,
                           int recall_mode, int exact, int32_t and_scan_threshold, int32_t scan_threshold,
                           item_t *items, int32_t *pred_buf, int64_t *pred_pos)
{
    int32_t lq[4096];
    if (nl > 4096) return -1;
    memcpy(lq, lq_in, sizeof(int32_t) * (size_t)nl);
    nl = sort_dedup(lq, nl);
    if (op == OR_SINGLE && nl > 1) return -1;
    int64_t n = 0;
    /* search-time threshold (f2): SCAN iff |C_l| < max(T, scan_threshold) */
    const int64_t T_eff = scan_threshold > ix->T ? (int64_t)scan_threshold : (int64_t)ix->T;
#define PATH_OF(l) (label_size(ix, (l)) == 0 ? OR_PATH_NONE : \
                    ((exact || label_size(ix, (l)) < T_eff) ? OR_PATH_SCAN : OR_PATH_GRAPH))
    if (op == OR_SINGLE || op == OR_OR) {
        for (int t = 0; t < nl; t++) {
            if (label_size(ix, lq[t]) == 0) continue;
            items[n].qid = qid; items[n].label = lq[t]; items[n].path = PATH_OF(lq[t]);
            items[n].pred_start = *pred_pos; items[n].pred_len = 0; n++;
        }
        return n;
    }
    /* AND */
    if (nl == 0) return 0;
    for (int t = 0; t < nl; t++) if (label_size(ix, lq[t]) == 0) return 0;
    if (recall_mode == OR_GREEDY) {
        int best = 0;
        for (int t = 1; t < nl; t++)
            if (label_size(ix, lq[t]) < label_size(ix, lq[best])) best = t;  /* ties -> lower id */
        items[0].qid = qid; items[0].label = lq[best]; items[0].path = PATH_OF(lq[best]);
        if (and_scan_threshold > 0 && nl > 1 && items[0].path == OR_PATH_GRAPH) {
            double est = (double)label_size(ix, lq[best]);
            for (int t = 0; t < nl; t++)
                if (t != best) est = est * (double)label_size(ix, lq[t]) / (double)ix->n_points;
            if (est < (double)and_scan_threshold) items[0].path = OR_PATH_SCAN;
        }
        items[0].pred_start = *pred_pos; items[0].pred_len = nl - 1;
        for (int t = 0; t < nl; t++) if (t != best) pred_buf[(*pred_pos)++] = lq[t];
        return 1;
    }
    for (int b = 0; b < nl; b++) {
        items[n].qid = qid; items[n].label = lq[b]; items[n].path = PATH_OF(lq[b]);
        items[n].pred_start = *pred_pos; items[n].pred_len = nl - 1;
        for (int t = 0; t < nl; t++) if (t != b) pred_buf[(*pred_pos)++] = lq[t];
        n++;
    }
    return n;
#undef PATH_OF
}

/* Python-facing router: out_items[n_max][5] = {qid, label, path, pred_start, pred_len}. */
int64_t or_route(const or_index *ix, int64_t n_q, const int64_t *q_off, const int32_t *q_lab, int op,
                 int recall_mode, int exact, int32_t and_scan_threshold, int32_t scan_threshold,
                 int32_t *out_items, int64_t n_max,
                 int32_t *pred_buf)
{
    int64_t n = 0, pp = 0;
    item_t *tmp = (item_t *)malloc(sizeof(item_t) * 4096);
    for (int64_t i = 0; i < n_q; i++) {
        int nl = (int)(q_off[i + 1] - q_off[i]);
        int64_t m = route_query(ix, (int32_t)i, q_lab + q_off[i], nl, op, recall_mode, exact,
                                and_scan_threshold, scan_threshold, tmp, pred_buf, &pp);
        if (m < 0) { free(tmp); return -1; }
        for (int64_t t = 0; t < m; t++) {
            if (n >= n_max) { free(tmp); return -2; }
            int32_t *o = out_items + 5 * n;
            o[0] = tmp[t].qid; o[1] = tmp[t].label; o[2] = tmp[t].path;
            o[3] = (int32_t)tmp[t].pred_start; o[4] = tmp[t].pred_len;
            n++;
        }
    }
    free(tmp);
    return n;
}

/* ------------------------------------------------------------------ IVF-BFS (a2)
 * Exact scan of C_l (Alg. 2). AND items: the predicate is applied to every point of
 * the list before its distance is computed. Result: best k by (d, gid). */
static int64_t scan_item(const or_index *ix, const void *q, int32_t l, const int32_t *P, int np,
                         entry_t *buf)
{
    int64_t n = 0;
    for (int64_t e = ix->post_off[l]; e < ix->post_off[l + 1]; e++) {
        int64_t gid = ix->post_ids[e];
        if (!pred_ok(ix, gid, P, np)) continue;
        buf[n].d = dist_l2sq(ix->dtype, ix->dim, ix->X, gid, q);
        buf[n].id = gid; buf[n].expanded = 0; n++;
    }
    qsort(buf, (size_t)n, sizeof(entry_t), cmp_entry);
    return n;
}

/* ------------------------------------------------------------------ IVF-Graph (a3)
 * Reference beam search, following Alg. 2 L418-L427 and P:L442-L444:
 *   G_l = G_HS[O_HS[l] : O_HS[l] + S_HS[l]]           (Alg. 2)
 *   all bookkeeping on local ids j in [0, S); M_l[j] = j-th member of C_l
 *   INIT: entries = [0..S) if S <= n_init, else u_i = entry_hash(i) for i < n_init
 *         each new entry j: Vis += j; if P(M_l[j]): Cand += (d(j), j)   (reading #16)
 *         Top = best itopk of Cand by (d, j)
 *   LOOP it = 1..max_iter: parents = first w unexpanded entries of Top (Alg. 2, reading #9);
 *         none -> stop (reading #10); mark them expanded; for each parent row, each child c that
 *         is a valid id (reading #15) and not in Vis: Vis += c; if P(M_l[c]) Cand += (d(c), c)
 *         (GetDist through M_HS, Alg. 2; inline predicate after distances);
 *         Top = best itopk of Top u Cand (UpdateTopM, Alg. 2).
 *   OUTPUT first min(k, |Top|) entries as (d, M_l[j]).
 * Counters: V = |Vis|, E = number of expanded parents, iterations that expanded a parent.
 * `forced_entry` >= 0 overrides the sampler with that single local id (test hook, App. B). */
typedef struct {
    int32_t k, itopk, search_width, n_init, max_iterations;
    uint32_t seed;
} beam_params;

static int64_t beam_item(const or_index *ix, const void *q, uint32_t qh, int32_t l, const int32_t *P,
                         int np, const beam_params *bp, int32_t forced_entry, entry_t *top_out,
                         int64_t *V_out, int64_t *E_out, int64_t *it_out)
{
    const int64_t S = label_size(ix, l);
    const int32_t R = ix->R;
    const int32_t *Ml = ix->post_ids + ix->post_off[l];         /* local -> global */
    const int32_t *Gl = ix->graph_ids + ix->graph_off[l] * R;    /* |C_l| rows of R local ids */
    const int itopk = bp->itopk, w = bp->search_width;
    unsigned char *vis = (unsigned char *)calloc((size_t)S, 1);
    entry_t *top = (entry_t *)malloc(sizeof(entry_t) * (size_t)(itopk + (int64_t)w * R + bp->n_init + 1));
    int64_t ntop = 0, V = 0, E = 0, iters = 0;

    /* INIT */
    int64_t n_entry = S <= bp->n_init ? S : bp->n_init;
    if (forced_entry >= 0) n_entry = 1;
    entry_t *cand = (entry_t *)malloc(sizeof(entry_t) * (size_t)(n_entry + (int64_t)w * R + 1));
    int64_t nc = 0;
    for (int64_t i = 0; i < n_entry; i++) {
        int64_t j;
        if (forced_entry >= 0) j = forced_entry;
        else if (S <= bp->n_init) j = i;
        else j = or_entry_hash(bp->seed, qh, l, (uint32_t)i, (uint32_t)S);
        if (vis[j]) continue;          /* duplicate samples are skipped through Vis */
        vis[j] = 1; V++;
        if (!pred_ok(ix, Ml[j], P, np)) continue;
        cand[nc].d = dist_l2sq(ix->dtype, ix->dim, ix->X, Ml[j], q);
        cand[nc].id = j; cand[nc].expanded = 0; nc++;
    }
    qsort(cand, (size_t)nc, sizeof(entry_t), cmp_entry);
    ntop = nc < itopk ? nc : itopk;
    memcpy(top, cand, sizeof(entry_t) * (size_t)ntop);

    /* LOOP */
    for (int64_t it = 0; it < bp->max_iterations; it++) {
        int64_t par[64];
        int np_ = 0;
        for (int64_t t = 0; t < ntop && np_ < w; t++)
            if (!top[t].expanded) { par[np_++] = top[t].id; top[t].expanded = 1; }
        if (np_ == 0) break;
        E += np_; iters++;
        nc = 0;
        for (int p = 0; p < np_; p++) {
            for (int r = 0; r < R; r++) {
                int64_t c = Gl[par[p] * R + r];
                if (c < 0 || c >= S) continue;
                if (vis[c]) continue;
                vis[c] = 1; V++;
                if (!pred_ok(ix, Ml[c], P, np)) continue;
                cand[nc].d = dist_l2sq(ix->dtype, ix->dim, ix->X, Ml[c], q);
                cand[nc].id = c; cand[nc].expanded = 0; nc++;
            }
        }
        memcpy(top + ntop, cand, sizeof(entry_t) * (size_t)nc);
        int64_t nall = ntop + nc;
        qsort(top, (size_t)nall, sizeof(entry_t), cmp_entry);
        ntop = nall < itopk ? nall : itopk;
    }
    /* OUTPUT: map local -> global (Alg. 2) */
    for (int64_t t = 0; t < ntop; t++) { top_out[t].d = top[t].d; top_out[t].id = Ml[top[t].id]; }
    *V_out = V; *E_out = E; *it_out = iters;
    free(vis); free(top); free(cand);
    return ntop;
}

/* ------------------------------------------------------------------ merge (a5)
 * Union of the items' lists; dedup by global id (reading #20); first k by (d, gid). */
static int64_t merge_lists(entry_t *all, int64_t n)
{
    qsort(all, (size_t)n, sizeof(entry_t), cmp_entry);
    int64_t m = 0;
    for (int64_t t = 0; t < n; t++) {
        int dup = 0;
        for (int64_t u = 0; u < m && !dup; u++) dup = all[u].id == all[t].id;
        if (!dup) all[m++] = all[t];
    }
    return m;
}

/* Python-facing merge of `n_lists` lists of length k (ids, dists; padded with -1): */
void or_merge(int n_lists, int k, const int32_t *ids, const double *dists, int32_t *out_ids,
              double *out_dists)
{
    entry_t *all = (entry_t *)malloc(sizeof(entry_t) * (size_t)(n_lists * k + 1));
    int64_t n = 0;
    for (int t = 0; t < n_lists * k; t++)
        if (ids[t] >= 0) { all[n].d = dists[t]; all[n].id = ids[t]; all[n].expanded = 0; n++; }
    n = merge_lists(all, n);
    emit(all, n, k, out_ids, out_dists);
    free(all);
}

/* ------------------------------------------------------------------ the whole method */
typedef struct {
    const or_index *ix;
    int64_t n_q; const void *Q; const int64_t *q_off; const int32_t *q_lab;
    int op, recall_mode, exact;
    int32_t and_scan_threshold, scan_threshold;
    beam_params bp;
    int32_t forced_entry;
    int32_t *out_ids; double *out_dists;
    int64_t *item_ctr;                 /* optional [n_q][maxitems][4] = label, path, V, E */
    int32_t max_items_per_q;
    int64_t next;                      /* work counter */
    int err;
    int mode;                          /* 0 = method (or_search), 1 = Definition-1 ground truth */
} job_t;

static void search_one(job_t *jb, int64_t i)
{
    const or_index *ix = jb->ix;
    const int k = jb->bp.k;
    size_t qbytes = (size_t)ix->dim * (ix->dtype == OR_U8 ? 1 : 4);
    const void *q = (const uint8_t *)jb->Q + (size_t)i * qbytes;
    int nl = (int)(jb->q_off[i + 1] - jb->q_off[i]);
    const int32_t *lq = jb->q_lab + jb->q_off[i];
    if (jb->mode == 1) {
        exact_one(ix, q, lq, nl, jb->op, k, jb->out_ids + i * k, jb->out_dists + i * k);
        return;
    }
    item_t *items = (item_t *)malloc(sizeof(item_t) * (size_t)(nl > 0 ? nl : 1));
    int32_t *pred = (int32_t *)malloc(sizeof(int32_t) * (size_t)(nl * nl + 1));
    int64_t pp = 0;
    int64_t m = route_query(ix, (int32_t)i, lq, nl, jb->op, jb->recall_mode, jb->exact,
                            jb->and_scan_threshold, jb->scan_threshold, items, pred, &pp);
    if (m < 0) { jb->err = 1; m = 0; }
    uint32_t qh = or_query_hash(ix->dtype, ix->dim, q);
    entry_t *all = (entry_t *)malloc(sizeof(entry_t) * (size_t)(m * k + 1));
    int64_t nall = 0;
    for (int64_t t = 0; t < m; t++) {
        const int32_t *P = pred + items[t].pred_start;
        int np = items[t].pred_len;
        int32_t l = items[t].label;
        int64_t V = 0, E = 0, its = 0, n;
        entry_t *res;
        if (items[t].path == OR_PATH_SCAN) {
            res = (entry_t *)malloc(sizeof(entry_t) * (size_t)(label_size(ix, l) + 1));
            n = scan_item(ix, q, l, P, np, res);
        } else {
            res = (entry_t *)malloc(sizeof(entry_t) * (size_t)(jb->bp.itopk + 1));
            n = beam_item(ix, q, qh, l, P, np, &jb->bp, jb->forced_entry, res, &V, &E, &its);
        }
        for (int64_t u = 0; u < n && u < k; u++) all[nall++] = res[u];
        free(res);
        if (jb->item_ctr && t < jb->max_items_per_q) {
            int64_t *c = jb->item_ctr + (i * jb->max_items_per_q + t) * 4;
            c[0] = l; c[1] = items[t].path; c[2] = V; c[3] = E;
        }
    }
    nall = merge_lists(all, nall);
    emit(all, nall, k, jb->out_ids + i * k, jb->out_dists + i * k);
    free(all); free(items); free(pred);
}

static void *worker(void *arg)
{
    job_t *jb = (job_t *)arg;
    for (;;) {
        int64_t i = __atomic_fetch_add(&jb->next, 1, __ATOMIC_RELAXED);
        if (i >= jb->n_q) break;
        search_one(jb, i);
    }
    return NULL;
}

static int run_job(job_t *jb, int nthreads)
{
    if (nthreads < 1) nthreads = 1;
    jb->next = 0; jb->err = 0;
    if (nthreads == 1) { worker(jb); return jb->err; }
    pthread_t *th = (pthread_t *)malloc(sizeof(pthread_t) * (size_t)nthreads);
    for (int t = 0; t < nthreads; t++) pthread_create(&th[t], NULL, worker, jb);
    for (int t = 0; t < nthreads; t++) pthread_join(th[t], NULL);
    free(th);
    return jb->err;
}

/* The method's result. max_iterations <= 0 -> 2*ceil(itopk/w)+16 (reading
 * #11); n_init <= 0 -> R*w (reading #7). item_ctr may be NULL. Returns 0 or 1 (invalid query). */
int or_search(const or_index *ix, int64_t n_q, const void *Q, const int64_t *q_off, const int32_t *q_lab,
              int op, int recall_mode, int exact, int32_t k, int32_t itopk, int32_t search_width,
              int32_t n_init, int32_t max_iterations, uint32_t seed, int32_t forced_entry,
              int32_t *out_ids, double *out_dists, int64_t *item_ctr, int32_t max_items_per_q,
              int nthreads, int32_t and_scan_threshold, int32_t scan_threshold)
{
    job_t jb;
    memset(&jb, 0, sizeof(jb));
    jb.ix = ix; jb.n_q = n_q; jb.Q = Q; jb.q_off = q_off; jb.q_lab = q_lab;
    jb.op = op; jb.recall_mode = recall_mode; jb.exact = exact;
    jb.and_scan_threshold = and_scan_threshold;
    jb.scan_threshold = scan_threshold;
    jb.bp.k = k; jb.bp.itopk = itopk < k ? k : itopk;
    jb.bp.search_width = search_width < 1 ? 1 : (search_width > 64 ? 64 : search_width);
    jb.bp.n_init = n_init > 0 ? n_init : ix->R * jb.bp.search_width;
    jb.bp.max_iterations = max_iterations > 0 ? max_iterations
        : 2 * ((jb.bp.itopk + jb.bp.search_width - 1) / jb.bp.search_width) + 16;
    jb.bp.seed = seed;
    jb.forced_entry = forced_entry;
    jb.out_ids = out_ids; jb.out_dists = out_dists;
    jb.item_ctr = item_ctr; jb.max_items_per_q = max_items_per_q;
    jb.mode = 0;
    return run_job(&jb, nthreads);
}

/* Definition 1 ground truth for every query (brute force over all N points). */
int or_exact_knn(const or_index *ix, int64_t n_q, const void *Q, const int64_t *q_off,
                 const int32_t *q_lab, int op, int32_t k, int32_t *out_ids, double *out_dists,
                 int nthreads)
{
    job_t jb;
    memset(&jb, 0, sizeof(jb));
    jb.ix = ix; jb.n_q = n_q; jb.Q = Q; jb.q_off = q_off; jb.q_lab = q_lab;
    jb.op = op; jb.bp.k = k; jb.out_ids = out_ids; jb.out_dists = out_dists; jb.mode = 1;
    return run_job(&jb, nthreads);
}

/* accessors for tests */
int64_t or_index_pt_off(const or_index *ix, int64_t i) { return ix->pt_off[i]; }
const int32_t *or_index_pt_lab(const or_index *ix) { return ix->pt_lab; }

/* Memory-consumption model of P:L497-L500 (bytes), exposed for the byte-accounting pin. */
double or_mem_hs_bytes(double N, double D, double F_HS, double Rp, double b) { return N * (D + F_HS * Rp) * b; }
double or_mem_ls_bytes(double N, double D, double F_LS, double b) { return N * D * F_LS * b; }
double or_mem_single_bytes(double N, double D, double R, double b) { return N * (D + R) * b; }
double or_mem_map_bytes(double N, double F, double b) { return N * F * b; }

/* ------------------------------------------------------------------ graph construction (f4)
 * The builder's two deterministic steps, written out as plain loops (PAPER.md
 * L348 "CAGRA ... rank-based reordering"; readings #45-#47).
 *
 * or_label_knn: for every member j of label l (local id j), the K nearest OTHER members by
 *   (squared L2, local id) -- exact, by sorting all S-1 candidates. Output [S][K], -1 padded.
 *
 * or_cagra_rows: from kNN lists knn[S][K] (local ids, ascending by (d, id)):
 *   detours(x, j) = #{ i < j : knn[x][j] occurs in knn[knn[x][i]] at a position < j }
 *   pruned[x] = the R entries of knn[x] with the fewest detours, ties by position j (-1 last)
 *   rev[y]    = the R/2 sources x with y in pruned[x], ordered by (position of y in pruned[x], x)
 *   row[x]    = pruned[x][0..R/2) ++ rev[x] ++ pruned[x][R/2..R), duplicates and -1 skipped,
 *               first R kept, -1 padded. */
typedef struct { double d; int32_t id; } knn_c;
static int cmp_knn_c(const void *a, const void *b)
{
    const knn_c *x = (const knn_c *)a, *y = (const knn_c *)b;
    if (x->d < y->d) return -1;
    if (x->d > y->d) return 1;
    return (x->id > y->id) - (x->id < y->id);
}

int or_label_knn(const or_index *ix, int32_t l, int K, int32_t *out)
{
    const int64_t S = label_size(ix, l);
    const int32_t *M = ix->post_ids + ix->post_off[l];
    knn_c *c = (knn_c *)malloc(sizeof(knn_c) * (size_t)(S > 0 ? S : 1));
    const size_t esz = ix->dtype == OR_U8 ? 1 : 4;
    for (int64_t j = 0; j < S; j++) {
        const void *q = (const uint8_t *)ix->X + (size_t)M[j] * ix->dim * esz;
        int64_t n = 0;
        for (int64_t t = 0; t < S; t++) {
            if (t == j) continue;
            c[n].d = dist_l2sq(ix->dtype, ix->dim, ix->X, M[t], q);
            c[n].id = (int32_t)t;
            n++;
        }
        qsort(c, (size_t)n, sizeof(knn_c), cmp_knn_c);
        for (int t = 0; t < K; t++) out[j * K + t] = t < n ? c[t].id : -1;
    }
    free(c);
    return 0;
}

typedef struct { int64_t a, b; int32_t v; } key3;
static int cmp_key3(const void *p, const void *q)
{
    const key3 *x = (const key3 *)p, *y = (const key3 *)q;
    if (x->a != y->a) return x->a < y->a ? -1 : 1;
    if (x->b != y->b) return x->b < y->b ? -1 : 1;
    return 0;
}

static int push_unique(int32_t *out, int no, int cap, int32_t v)
{
    if (v < 0 || no >= cap) return no;
    for (int t = 0; t < no; t++)
        if (out[t] == v) return no;
    out[no] = v;
    return no + 1;
}

int or_cagra_rows(int64_t S, int K, const int32_t *knn, int R, int32_t *pruned, int32_t *rows)
{
    const int h = R / 2;
    key3 *ord = (key3 *)malloc(sizeof(key3) * (size_t)K);
    for (int64_t x = 0; x < S; x++) {
        for (int j = 0; j < K; j++) {
            const int32_t y = knn[x * K + j];
            int64_t det = 0;
            if (y >= 0)
                for (int i = 0; i < j; i++) {
                    const int32_t z = knn[x * K + i];
                    if (z < 0) continue;
                    for (int t = 0; t < j; t++)
                        if (knn[(int64_t)z * K + t] == y) { det++; break; }
                }
            ord[j].a = y < 0 ? INT64_MAX : det;
            ord[j].b = j;
            ord[j].v = y;
        }
        qsort(ord, (size_t)K, sizeof(key3), cmp_key3);
        for (int t = 0; t < R; t++) pruned[x * R + t] = t < K && ord[t].a != INT64_MAX ? ord[t].v : -1;
    }
    free(ord);
    /* reverse candidates (position, source) per target */
    int64_t *cnt = (int64_t *)calloc((size_t)S + 1, sizeof(int64_t));
    for (int64_t x = 0; x < S; x++)
        for (int p = 0; p < R; p++)
            if (pruned[x * R + p] >= 0) cnt[pruned[x * R + p] + 1]++;
    for (int64_t y = 0; y < S; y++) cnt[y + 1] += cnt[y];
    key3 *rv = (key3 *)malloc(sizeof(key3) * (size_t)(cnt[S] > 0 ? cnt[S] : 1));
    int64_t *fill = (int64_t *)calloc((size_t)S, sizeof(int64_t));
    for (int64_t x = 0; x < S; x++)
        for (int p = 0; p < R; p++) {
            const int32_t y = pruned[x * R + p];
            if (y < 0) continue;
            key3 *e = &rv[cnt[y] + fill[y]++];
            e->a = p; e->b = x; e->v = (int32_t)x;
        }
    for (int64_t y = 0; y < S; y++) qsort(rv + cnt[y], (size_t)(cnt[y + 1] - cnt[y]), sizeof(key3), cmp_key3);
    int32_t *out = (int32_t *)malloc(sizeof(int32_t) * (size_t)R);
    for (int64_t x = 0; x < S; x++) {
        int no = 0;
        for (int t = 0; t < h; t++) no = push_unique(out, no, R, pruned[x * R + t]);
        for (int64_t e = cnt[x]; e < cnt[x + 1] && e < cnt[x] + h; e++) no = push_unique(out, no, R, rv[e].v);
        for (int t = h; t < R; t++) no = push_unique(out, no, R, pruned[x * R + t]);
        for (int t = 0; t < R; t++) rows[x * R + t] = t < no ? out[t] : -1;
    }
    free(out); free(rv); free(fill); free(cnt);
    return 0;
}
