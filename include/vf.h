/*
 * vf.h -- C-ABI of libvecflow: batched label-filtered top-k search over a label-centric index,
 * B200-native (sm_100a). The method is VecFlow (arXiv 2506.00812); citations "P:L<n>" are lines
 * of /root/reference/PAPER.md, "reading #n" the numbered readings in DESIGN.md §2.
 *
 * Conventions shared by every entry point
 *  - Plain C types only; no exception ever crosses the ABI; user errors never abort.
 *  - Every non-OK status sets a thread-local message readable with vf_last_error().
 *  - Distances are SQUARED L2 (reading #4). Result rows are sorted by (dist asc, global id asc)
 *    (reading #6) and padded with id -1 / dist +INF when fewer than k points match (reading #23).
 *    For VF_U8 data the distance is an exact int32 (D*255^2 < 2^24 for D <= 258) stored exactly
 *    in the float output.
 *  - Host or device pointers are both accepted where stated; the library detects which with
 *    cudaPointerGetAttributes. Device pointers must be on the index's device.
 */
#ifndef VF_H
#define VF_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct vf_index vf_index; /* opaque; immutable after vf_build_index */

typedef enum {
    VF_OK = 0,
    VF_ERR_INVALID_ARG = 1,    /* bad argument / malformed index input (message says which) */
    VF_ERR_OUT_OF_MEMORY = 2,  /* device or pinned-host allocation failed */
    VF_ERR_CUDA = 3,           /* CUDA runtime/launch error; after a sticky error only vf_free is valid */
    VF_ERR_NCCL = 4,           /* NCCL error in a collective (world_size > 1) */
    VF_ERR_INTERNAL = 5        /* internal invariant violated (a bug) */
} vf_status;

typedef enum { VF_U8 = 0, VF_F32 = 1 } vf_dtype;

/* Label operator of a query batch. SINGLE requires <= 1 label per query. */
typedef enum { VF_SINGLE = 0, VF_OR = 1, VF_AND = 2 } vf_label_op;

/* AND policy: GREEDY searches only l* = argmin |C_l| (ties: lower id) with the other labels as an
 * inline predicate; PARALLEL searches every label's list filtered by the
 * others and merges. */
typedef enum { VF_RECALL_GREEDY = 0, VF_RECALL_PARALLEL = 1 } vf_recall_mode;

/*
 * Index construction input (Alg. 1). All pointers are HOST pointers, read only during
 * the call; the caller may free them on return. Layouts:
 *  vectors            [n_points][dim] row-major, element type per dtype (X)
 *  posting_offsets    [n_labels+1] int64 CSR; posting list C_l = posting_ids[off[l] .. off[l+1]),
 *                     strictly ascending global ids in [0, n_points)
 *  threshold_T        routing threshold: label l is served by the graph iff |C_l| >= T
 *  degree_R           fixed out-degree of every G_l row (P:L615 uses 16); 1 <= R <= 64
 *  graph_row_offsets  [n_labels+1] int64; rows(l) = off[l+1]-off[l] must be |C_l| for every label
 *                     with |C_l| >= T and is either 0 or |C_l| otherwise (rows of non-HS labels
 *                     are ignored). May be NULL only if no label has |C_l| >= T.
 *  graph_local_ids    [total_rows][R] int32 LOCAL ids of G_l: entry r of row j of
 *                     label l is a position in C_l, in [0, |C_l|), or -1 for "no edge"
 *                     (reading #15). Local id order equals global id order because C_l ascends.
 *  world_size, rank   1/0 for a single GPU. For world_size > 1 the call is COLLECTIVE (SPMD):
 *                     every rank passes the same full inputs; each rank keeps the labels it owns
 *                     (greedy LPT over |C_l|, a deterministic function of the posting sizes) plus
 *                     replicas of X and the predicate table.
 *  nccl_unique_id     128-byte ncclUniqueId (identical on every rank), required iff world_size > 1
 *  device             CUDA device ordinal this rank uses
 * Errors: VF_ERR_INVALID_ARG on any violated constraint above (unsorted / out-of-range posting
 * ids, an HS label without graph rows, a graph entry outside [-1, |C_l|)), dim < 1 or
 * dim * sizeof(elem) > 4096, T < 1; VF_ERR_OUT_OF_MEMORY; VF_ERR_CUDA; VF_ERR_NCCL.
 * On error *out is set to NULL and nothing leaks.
 */
typedef struct {
    int64_t n_points;
    int32_t dim;
    int32_t dtype;                    /* vf_dtype */
    const void *vectors;
    int32_t n_labels;                 /* label ids are 0 .. n_labels-1 */
    const int64_t *posting_offsets;
    const int32_t *posting_ids;
    int32_t threshold_T;
    int32_t degree_R;
    const int64_t *graph_row_offsets;
    const int32_t *graph_local_ids;
    int32_t world_size;
    int32_t rank;
    const void *nccl_unique_id;
    int32_t device;
} vf_build_desc;

/*
 * Search parameters (Alg. 2; beam search per DESIGN.md §2 c.2).
 *  k               results per query, 1 <= k <= 256
 *  itopk           internal top-M list size, k <= itopk <= 1024 (ignored by scan items)
 *  search_width    parents expanded per iteration (Alg. 2 "first unvisited node": 1),
 *                  1 <= w, w * R <= 64
 *  n_init          entry samples (reading #7); <= 0 -> R * w
 *  max_iterations  <= 0 -> 2 * ceil(itopk / w) + 16 (reading #11)
 *  seed            entry-point sampler seed (reading c.3; keyed on query content)
 *  op, recall_mode vf_label_op / vf_recall_mode
 *  exact           1 = route every item to the scan (T = infinity): exact filtered kNN, the
 *                  ground-truth mode
 */
typedef struct {
    int32_t k;
    int32_t itopk;
    int32_t search_width;
    int32_t n_init;
    int32_t max_iterations;
    uint32_t seed;
    int32_t op;
    int32_t recall_mode;
    int32_t exact;
    /* Selectivity-aware AND routing (BEYOND the paper, 0 = off = the paper's
     * method). For a GREEDY AND item whose list l* is HS, the expected AND-set size under label
     * independence, est = |C_l*| * prod_{o != l*} (|C_o| / n_points) (fp64, other labels in
     * ascending id order, left to right), is computed; est < and_scan_threshold routes the item to
     * the exact scan of C_l* with the predicate instead of the inline-filtered graph search, whose
     * traversal collapses when few points pass the filter. */
    int32_t and_scan_threshold;
    /* Search-time specificity threshold (the T sweep of P:L339):
     * an item whose label has |C_l| < max(T, scan_threshold) is served by the exact scan. Values
     * <= the build's T change nothing (LS labels have no graph); INT32_MAX = scan everything, the
     * same results as `exact`. 0 = the index's T. */
    int32_t scan_threshold;
    /* Length of the query-label array (= qlabel_offsets[n]) when the offsets live in DEVICE memory:
     * > 0 lets vf_search size its work without reading qlabel_offsets[n] back (no stream sync, so
     * consecutive searches overlap their host and device work). 0 = read it (one stream sync).
     * Must equal qlabel_offsets[n] when given; ignored for host offsets. With device offsets the
     * library never reads outside [0, n_query_labels) of qlabels: a query whose offsets leave that
     * range or that carries too many labels gets an empty row and is counted in
     * vf_search_stats.n_invalid_queries (no error status: the check runs on the device). */
    int64_t n_query_labels;
} vf_search_params;

/*
 * GPU construction of the per-label graphs ("we use CAGRA ...
 * NN-descent + rank-based reordering", Alg. 1 L393 BuildGraph(C_l)) -- produces exactly the
 * graph_row_offsets / graph_local_ids that vf_build_desc takes. For every label with
 * |C_l| >= threshold_T:
 *   kNN    the knn_k nearest other members of every point by (squared L2, row), computed on the
 *          tensor cores (a u8 self-join); exact for labels of <= exact_max points, else IVF probing
 *          (k-means cells of ~ivf_cell points, each joined against its ivf_probes nearest cells);
 *   prune  CAGRA rank-based pruning to degree_R (fewest detours x -> z -> y with both ranks below
 *          y's rank in x's list; ties by rank);
 *   rows   the first R/2 pruned edges, then up to R/2 reverse edges (by position, then source),
 *          then the remaining pruned edges; duplicates skipped; -1 padded.
 * Vectors: u8, or fp32 holding integers in [0, 255] (else VF_ERR_INVALID_ARG). All host arrays;
 * graph_row_offsets: [n_labels + 1] (written), graph_local_ids: caller-owned, capacity
 * degree_R * sum of |C_l| over the labels with |C_l| >= threshold_T. Deterministic: the same
 * inputs give the same graphs. Runs on `device`; uses up to ~ (rows of those labels) x
 * (row bytes + 300) bytes of device memory, all freed on return.
 */
typedef struct {
    int64_t n_points;
    int32_t dim;
    vf_dtype dtype;
    const void *vectors;               /* host, row-major n_points * dim */
    int32_t n_labels;
    const int64_t *posting_offsets;    /* [n_labels + 1] */
    const int32_t *posting_ids;        /* ascending per label */
    int32_t threshold_T;               /* graphs for |C_l| >= T */
    int32_t degree_R;                  /* even, 2..32 */
    int32_t knn_k;                     /* kNN list length before pruning: 0 = min(32, 2R); <= 32, >= R */
    int64_t exact_max;                 /* exact kNN up to this label size: 0 = 200000, < 0 = always */
    int32_t ivf_cell;                  /* points per IVF cell: 0 = 2048 */
    int32_t ivf_probes;                /* cells probed per cell (itself included): 0 = 16, <= 16 */
    int32_t kmeans_iters;              /* Lloyd iterations: 0 = 4 */
    int32_t device;
    int32_t *knn_lists;                /* optional (NULL): receives the kNN lists before pruning,
                                          [rows][report.knn_k] local ids, rows in graph order */
} vf_graph_desc;

typedef struct {
    double ms_total, ms_upload, ms_knn_exact, ms_kmeans, ms_knn_ivf, ms_prune, ms_rows, ms_download;
    int64_t n_graph_labels, n_exact_labels, n_ivf_labels, rows;
    int64_t join_pairs;                /* (query, candidate) pairs the kNN joins evaluated */
    int32_t knn_k;                     /* kNN list length used (knn_k rounded up to 16 or 32) */
} vf_graph_report;

vf_status vf_build_graphs(const vf_graph_desc *desc, int64_t *graph_row_offsets, int32_t *graph_local_ids,
                          vf_graph_report *report /* may be NULL */);

/* Build the index on the device (copies everything; see vf_build_desc). */
vf_status vf_build_index(const vf_build_desc *desc, vf_index **out);

/*
 * Label sharding on ONE device (SURVEY §8(e) "virtual shards"): builds n_shards label shards of the
 * index (the same LPT ownership as a world_size = n_shards NCCL group) on desc->device and runs
 * the sharded protocol -- route, ship items to their owners, execute, return, merge -- with an
 * in-process transport. vf_search on it splits the batch into n_shards contiguous chunks (one per
 * origin shard) and returns results identical to vf_build_index. Host query / result buffers
 * only. desc->world_size / rank / nccl_unique_id are ignored. 1 <= n_shards <= 16.
 */
vf_status vf_build_index_virtual_shards(const vf_build_desc *desc, int32_t n_shards, vf_index **out);

/*
 * The label -> rank ownership used by label sharding: greedy LPT over the posting sizes (labels by
 * size descending, ties by id; each to the least-loaded rank, ties to the lower rank). Pure host
 * function, deterministic, identical on every rank. sizes [n_labels] host, owner [n_labels] host out.
 */
vf_status vf_partition_labels(int32_t n_labels, const int64_t *sizes, int32_t world, int32_t *owner);

/*
 * Search a batch (Alg. 2). queries [n_queries][dim] (host or device, dtype of the index);
 * query labels as CSR: qlabel_offsets [n_queries+1] int64, qlabels int32 (host or device; label
 * ids outside [0, n_labels) are "unknown": empty posting list, reading #19). Outputs out_ids
 * [n_queries][k] int32 (global ids) and out_dists [n_queries][k] float, caller-owned, host or
 * device (both on the same side). cuda_stream: a cudaStream_t or NULL (legacy default stream).
 * With device buffers the call is asynchronous on the stream: results are valid once the stream
 * is synchronised. With host buffers the call returns after the results are copied back.
 * Per-call scratch comes from a per-stream pool, so concurrent calls on distinct streams are safe;
 * the index is read-only. With world_size > 1 the call is collective: every rank calls it with its
 * own queries (possibly 0) and gets the results of its own queries.
 * Errors: VF_ERR_INVALID_ARG (k, itopk, w, dim mismatch, SINGLE op with > 1 label in a query,
 * > 64 labels in one query), VF_ERR_OUT_OF_MEMORY, VF_ERR_CUDA, VF_ERR_NCCL.
 */
vf_status vf_search(vf_index *index, const void *queries, int64_t n_queries,
                    const int64_t *qlabel_offsets, const int32_t *qlabels,
                    const vf_search_params *params, int32_t *out_ids, float *out_dists,
                    void *cuda_stream);

/* Release every resource of the index. NULL-safe. Must not race with vf_search on it. */
void vf_free(vf_index *index);

/* Thread-local message of the last non-OK status returned on this thread ("" if none). */
const char *vf_last_error(void);

/* ----------------------------------------------------------------- introspection / measurement */

/* Byte accounting of the device-resident index (exact sizes of the allocated arrays). */
typedef struct {
    int64_t n_points, n_labels, n_hs_labels, n_ls_labels;
    int64_t hs_rows, ls_rows;           /* sum |C_l| over HS / LS labels */
    int32_t row_bytes;                  /* padded vector row (16-byte multiple) */
    int32_t degree_R;
    int64_t bytes_vectors;              /* X: n_points * row_bytes (one shared copy) */
    int64_t bytes_graph;                /* G_HS: hs_rows * R * 8 ((local, global) id per edge) */
    int64_t bytes_map_hs;               /* M_HS: hs_rows * 4 */
    int64_t bytes_ls_vectors;           /* X_LS: ls_rows * row_bytes */
    int64_t bytes_map_ls;               /* M_LS: ls_rows * 4 */
    int64_t bytes_predicate;            /* point -> labels table: (n_points+1)*8 + entries*4, plus the
                                           membership bitmaps of the largest labels (n_bm * ceil(N/32) * 4
                                           + n_labels * 2; VF_BITMAP_DENSITY at build: |C_l| >= N/density,
                                           default 256, 0 = none) */
    int64_t bytes_directory;            /* per-label metadata */
    int64_t bytes_norms;                /* ||x||^2 per point and per X_LS row (tensor-core scan) */
    int64_t bytes_u8_store;             /* integer-valued fp32 in [0,255]: lossless u8 X and X_LS copies */
    int64_t bytes_total;                /* sum of the above */
    int32_t world_size, rank;
    int64_t owned_labels;               /* labels whose lists live on this rank */
} vf_index_info;

vf_status vf_get_index_info(const vf_index *index, vf_index_info *info);

/*
 * Per-phase device timing and work counters of the most recent vf_search on `stream` (timing
 * needs vf_set_profiling(index, 1)). A small batch answered by the per-query path (one launch, one
 * CTA per query; f1) reports its whole kernel as ms_graph, and its item records / V / E counters
 * like the batched path. Blocks until that search has finished. Times are CUDA-event
 * milliseconds recorded on the search stream around each kernel.
 */
typedef struct {
    int64_t n_queries, n_items, n_scan_items, n_graph_items, n_segments, n_tiles;
    int64_t scan_rows;                  /* rows streamed by the scan (sum over tiles) */
    int64_t scan_query_rows;            /* (row, query) distance evaluations of the scan */
    int64_t graph_V, graph_E, graph_iterations; /* sums over graph items */
    int64_t graph_V_max;
    double ms_route, ms_scan, ms_graph, ms_merge, ms_copy, ms_total;
    int32_t kernel_launches;            /* kernels this search launched */
    int32_t row_bytes;
    /* means of the ms_* phases over the profiled searches on this stream since profiling was last
     * enabled (the most recent 64 of them); n_profiled = how many were averaged */
    int64_t n_profiled;
    double mean_ms_route, mean_ms_scan, mean_ms_graph, mean_ms_merge, mean_ms_copy, mean_ms_total;
    /* device-clock span (first CTA start -> last CTA end, %globaltimer) of the tensor-core scan kernel
     * and of the graph kernel in the most recent search; 0 if the kernel did not run. Unlike the
     * phase events these exclude time a launched kernel waited for SMs (overlapped phases). */
    double ms_scan_active, ms_graph_active;
    /* queries the device rejected (device offset arrays only; host arrays are checked before the
     * search and fail it with VF_ERR_INVALID_ARG instead): labels outside [0, n_query_labels) or
     * more labels than allowed (64; 16 on a label-sharded index). Their rows come out empty. */
    int64_t n_invalid_queries;
    /* AND pre-filter (k_and_filter): survivor / pass-bit words used in its pool (diagnostics) */
    int64_t prefilter_words;
    /* scan items' bucketing + AND pre-filter + tile packing (k_segments .. k_pack), between routing
     * (ms_route = k_prepare) and the scan kernels (ms_scan); last search and mean */
    double ms_filter, mean_ms_filter;
} vf_search_stats;

vf_status vf_set_profiling(vf_index *index, int32_t enable);
vf_status vf_get_last_stats(vf_index *index, void *cuda_stream, vf_search_stats *stats);

/*
 * Per-item records of the most recent vf_search on `stream`, in canonical item order (queries in
 * order; a query's items in ascending label order): rec[i] = {qid, label, path (0 none, 1 scan,
 * 2 graph), V, E, iterations}. Writes min(n, max_items) records; *n_items receives n.
 */
vf_status vf_get_last_items(vf_index *index, void *cuda_stream, int64_t max_items, int32_t *rec,
                            int64_t *n_items);

/*
 * Persistent-kernel serving ("Persistent Kernel-based Search
 * for Small Batch Queries", E13 P:L733-L738). vf_serve_start launches a kernel that stays resident
 * (n_workers CTAs, <= 0: one per free SM slot) and a job ring of `capacity` slots in pinned,
 * device-mapped host memory. Each query is answered by one CTA with the same routing, scan, beam
 * search and merge as vf_search, so results are identical to vf_search with the same parameters
 * (params: k <= 32; itopk, search_width, n_init, max_iterations, seed, op, recall_mode, exact,
 * and_scan_threshold, scan_threshold as for vf_search; n_query_labels ignored).
 *   vf_serve_submit  copies one query (dim elements of the index's element type, HOST memory) and
 *                    its labels (HOST, 0..16 entries; semantics of `op`) into the next slot and
 *                    publishes it; returns a ticket. Blocks only while the slot's previous job
 *                    (ticket - capacity) is still running. Thread-safe.
 *   vf_serve_wait    spins until the ticket is answered and copies its k ids / distances (HOST,
 *                    caller-owned; layout as one row of vf_search's output). A ticket's results
 *                    stay readable until `capacity` more queries have been submitted; a later wait
 *                    returns VF_ERR_INVALID_ARG. VF_ERR_CUDA if the kernel died.
 *   vf_serve_stop    stops the kernel once every submitted job is answered; frees the server.
 * Environment VF_SERVE_IDLE_MS (read by vf_serve_start; default 0 = never): the kernel exits by
 * itself after that many ms without a new job (a profiler that serialises launches would otherwise
 * wait forever); later waits then return VF_ERR_CUDA.
 * The resident kernel occupies the GPU's SMs: batched vf_search calls on the same device compete
 * with it for SMs while it runs. The index must outlive the server.
 */
typedef struct vf_server vf_server;
vf_status vf_serve_start(vf_index *index, const vf_search_params *params, int32_t capacity, int32_t n_workers,
                         vf_server **out);
vf_status vf_serve_submit(vf_server *server, const void *query, const int32_t *labels, int32_t n_labels,
                          int64_t *ticket);
vf_status vf_serve_wait(vf_server *server, int64_t ticket, int32_t *out_ids, float *out_dists);
vf_status vf_serve_stop(vf_server *server);
/* A client loop in C (single-batch mode): submits the n queries of a host batch as n
 * separate jobs, at most max_in_flight (<= capacity) outstanding, and waits for each in order;
 * results land in out_ids / out_dists (host, n*k). Same answers as n vf_serve_submit/wait pairs. */
vf_status vf_serve_run(vf_server *server, int64_t n, const void *queries, const int64_t *qlabel_offsets,
                       const int32_t *qlabels, int32_t max_in_flight, int32_t *out_ids, float *out_dists);
vf_status vf_serve_info(const vf_server *server, int32_t *n_workers, int64_t *submitted);
/* Mean per answered job part (device globaltimer): time a worker CTA waited for its job to be
 * published, copied the slot from host memory, and searched + published; parts answered. */
vf_status vf_serve_stats(vf_server *server, double *wait_us, double *copy_us, double *search_us,
                         int64_t *parts_done);

#ifdef __cplusplus
}
#endif
#endif /* VF_H */
