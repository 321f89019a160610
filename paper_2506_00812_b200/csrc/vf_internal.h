// Internal types shared by the host orchestration (vf_api.cpp) and the CUDA kernels.
// Nothing here is part of the C-ABI (include/vf.h is).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace vf {

constexpr int kMaxQueryLabels = 64;   // labels per query accepted by vf_search
constexpr int kMaxK = 256;
constexpr int kMaxBitmaps = 1024;
// Graph items are claimed largest-label class first: an item's beam-search cost grows with log |C_l|
// (oracle counters on SIFT-like: corr(log |C_l|, V) = 0.77), so long items start early and the
// kernel's tail shrinks (longest-processing-time-first at class granularity).
constexpr int kTileClasses = 4;
__host__ __device__ __forceinline__ int tile_class(int32_t rows) {
    return rows >= 1024 ? 0 : rows >= 512 ? 1 : rows >= 256 ? 2 : 3;
}
constexpr int kGraphClasses = 4;
__host__ __device__ __forceinline__ int graph_class(int32_t size) {
    return size >= 131072 ? 0 : size >= 32768 ? 1 : size >= 8192 ? 2 : 3;
}      // membership bitmaps of the largest labels (predicate fast path)
constexpr int kMaxItopk = 1024;
constexpr int kScanQG = 64;           // queries per scan segment (query group)
constexpr int kF3TileRows = 8192;     // rows per tile of f3-only (fully pre-filtered) segments
constexpr int kOverlapMaxF3 = 20000;  // f3 threshold from which scan / graph run one after the other
constexpr int kWarpsPerGraphCta = 4;

enum Path : uint32_t { PATH_NONE = 0, PATH_SCAN = 1, PATH_GRAPH = 2 };

// Per-label directory entry (the label metadata of P:L369 / P:L471: size, offset, kind).
struct LabelDir {
    int64_t base;     // first row of the label in G_HS/M_HS (HS) or X_LS/M_LS (LS)
    int32_t size;     // |C_l| (0 = empty or not owned by this rank)
    int32_t bslot;    // bucket slot of a non-empty label (index of its scan-bucket counter)
};

// Device-resident index (Alg. 1 output), one per rank.
struct DevIndex {
    int32_t dtype;         // 0 u8, 1 f32
    int32_t dim;
    int32_t row_bytes;     // padded row, multiple of 16
    int32_t chunks;        // row_bytes / 16
    int64_t n_points;
    int32_t n_labels;
    int32_t T;
    int32_t R;
    int32_t n_bslots;      // non-empty labels (scan-bucket counters)
    const uint8_t *X;      // [n_points][row_bytes]  global vectors (one copy)
    const LabelDir *dir;   // [n_labels]
    const int2 *G;         // [hs_rows][R] (local id, global id) edges of G_HS (the
                           // M_HS indirection of P:L444 folded into the row)
    const int32_t *M_hs;   // [hs_rows] local -> global (M_HS)
    const uint8_t *Xls;    // [ls_rows][row_bytes] label-contiguous LS copies (X_LS)
    const int32_t *M_ls;   // [ls_rows] (M_LS)
    const int64_t *pt_off; // [n_points+1] predicate table offsets
    const int32_t *pt_lab; // sorted labels per point
    const uint32_t *lbits; // [n_bitmaps][lbit_words] membership bitmaps of the largest labels (predicate
                           // fast path: P ⊆ L_x tested bit by bit; identical answers to pt_lab)
    const int16_t *lbit_slot;  // [n_labels] bitmap of a label, -1 = none
    int64_t lbit_words;
    // [n_points] 64-bit label signature of each point: bits h1(l), h2(l) of every label l of the
    // point (label_sig_bits). A label whose bits are not all set is certainly not a label of the
    // point: the predicate's negative fast path (one 8-B read, kept in L2), exact checks after it
    const unsigned long long *lsig;
    const int32_t *owner;  // [n_labels] owning rank of each label (label sharding, §8(e)); NULL = all local
    const uint32_t *xn;    // [n_points] ||x||^2 (u8: exact int32) for the tensor-core scan's expansion
    const uint32_t *xn_ls; // [ls_rows_pad + 4] ||x||^2 of the X_LS rows
    int32_t rank, world;
};

// Work item (a1): one (query, label) search (Alg. 2 L418 / L428 "(q, l)").
struct Item {
    int32_t qid;
    int32_t label;
    int32_t rank;      // scan items: position within the label bucket
    uint32_t meta;     // bits 0-1 path, bit 2 has_pred, bit 3 direct, bit 4 multi_tile
};
constexpr uint32_t META_PRED = 4u, META_DIRECT = 8u, META_MULTI = 16u, META_REMOTE = 32u;
constexpr int kMaxWorld = 16;        // ranks of a label-sharded index
constexpr int kRecLabels = 16;       // query labels carried by an exchanged item record

// An item shipped to the rank owning its label (label sharding): header + the padded query row.
struct ItemRecord {
    int32_t origin_slot;  // the item's slot on the origin rank (results come back in send order)
    int32_t label;        // the item's label, owned by the receiver
    int32_t nl;           // sorted, deduplicated query labels that follow (the AND predicate)
    uint32_t pred;        // META_PRED if the item carries an AND predicate
    uint32_t qh;          // the query's content hash (entry sampler, reading #34)
    int32_t pad[3];
    int32_t labels[kRecLabels];
};

struct QueryInfo {
    int32_t nl;        // deduplicated label count
    int32_t n_items;
    uint32_t qh;       // content hash (entry sampler, reading c.3)
    int32_t pad;
};

// A scan segment: one LS label with up to kScanQG of its items (a2: "query group x posting list").
struct Segment {
    int32_t label;
    int32_t item_base;   // first entry in scan_slots
    int32_t n_items;
    int32_t tile_base;   // first tile of this segment
    int32_t n_tiles;
    int32_t listed;      // 1 once k_scatter listed the segment's tiles for the AND pre-filter
    int32_t done;        // tiles of a multi-tile segment finished (the last one merges the partials)
    int32_t pad;
};

constexpr int kMaxPieces = 8;        // survivor pieces of a pre-filtered tile (k_and_filter)

// A row tile of a segment: everything the scan producer needs in one record, so claiming a tile
// costs one dependent load (written by k_segments; survivor pieces by k_hs_filter).
struct Tile {
    int64_t base;        // first row of the label in X_LS (or in M_HS for an HS label, exact mode)
    int32_t seg;
    int32_t row_begin;   // rows relative to the label's first row
    int32_t row_end;
    int32_t tile_in_seg;
    int32_t label;
    int32_t nq;          // queries of the segment
    int32_t item_base;   // first entry of the segment in scan_slots / scan_q
    int32_t n_tiles;
    int32_t hs;          // 1: HS label scanned in exact mode (rows gathered through M_HS)
    // AND pre-filter (k_and_filter, "before distance"). A tile whose queries all carry a
    // predicate is compacted: n_pieces >= 0 pieces of the survivor pool hold the rows passing some
    // query's predicate (pool: global ids, pool_bits: per-query pass bits) and the tensor-core scan
    // gathers only those. A tile mixing predicate and plain queries keeps every row and gets one
    // pass-bit word per row at pool_bits[bits_off + row - row_begin]. -1 / -1: no pre-filter (the
    // scan verifies the predicate itself).
    int32_t bits_off;
    int32_t n_pieces;
    int32_t piece_off[kMaxPieces];
    int32_t piece_cnt[kMaxPieces];
    int32_t pad2[3];
};

// Per scan item, in scan_slots order: what the scan needs about its query (written by k_scatter).
struct ScanQuery {
    int64_t p_off;       // offset of the query's sorted labels (the AND predicate)
    int32_t slot, qid;
    uint32_t meta;
    int32_t nl;
    int32_t pad[2];
};

// The two signature bits of a label (vf_build_index builds the per-point signatures with it).
__host__ __device__ __forceinline__ unsigned long long label_sig_bits(int32_t l) {
    uint32_t h = (uint32_t)l * 0x9E3779B1u;
    h ^= h >> 15; h *= 0x2C1B3C6Du; h ^= h >> 12; h *= 0x297A2D39u; h ^= h >> 15;
    return (1ull << (h & 63)) | (1ull << ((h >> 8) & 63));
}

// Device counters, zeroed at the start of every search.
struct Counters {
    int32_t n_graph;
    int32_t n_graph_cls[4];  // graph items per label-size class (kGraphClasses; largest labels first)
    int32_t n_segs;
    int32_t n_scan_items;
    int32_t n_tiles;
    int32_t scan_next;
    int32_t graph_next;
    int32_t n_items;
    int32_t exact_fallback;  // a query of this batch is outside the fast path's exact range (gate)
    int32_t filter_next;     // k_and_filter cursor over filt_list
    int32_t n_tile_cls[4];        // scan tiles per row-count class (kTileClasses; longest first)
    int32_t pool_used;       // survivor pool bump allocator
    int32_t n_pack;          // small single-tile segments queued for packing (k_pack)
    int32_t n_packed;        // packed tiles made
    int32_t packq_used;      // query records copied for packed tiles
    int32_t n_invalid;       // queries rejected by the device-side offset / label-count check
    int32_t n_filt_tiles;    // tiles holding a predicate query (k_scatter -> filt_list, k_and_filter)
    int32_t pad_ctr;
    unsigned long long graph_V, graph_E, graph_iters, scan_rows, scan_qrows;
    unsigned long long graph_V_max;
    // device-clock activity spans of the dominant kernels (globaltimer ns; first CTA start stored
    // inverted so that zeroed counters work with atomicMax): the kernels' own durations, which the
    // phase events of an overlapped search cannot give
    unsigned long long scan_t0_inv, scan_t1, graph_t0_inv, graph_t1;
    int32_t remote[kMaxWorld];      // items of this batch owned by each rank (sharded index)
    int32_t remote_pos[kMaxWorld];  // packing cursors
};

struct SearchArgs {
    DevIndex ix;
    int64_t n_q;
    const uint8_t *Qraw;      // [n_q][dim * elem] caller's query rows (device copy if needed)
    const uint8_t *Qp;        // [n_q][row_bytes] padded queries
    const int64_t *q_off;     // [n_q+1]
    int32_t *qlab;            // sorted/dedup labels per query (CSR with q_off)
    const int32_t *qlab_in;   // caller's device labels copied into qlab by k_prepare (nullptr: already there)
    QueryInfo *qinfo;
    Item *items;              // [q_off[n_q]] slots
    int32_t *item_ctr;        // [slots][3] V, E, iterations (graph items)
    int32_t *ls_count;        // [n_bslots] scan items per label in this batch
    int32_t *ls_segbase;      // [n_bslots] first segment of the label
    int32_t *ls_itembase;     // [n_bslots] first scan_slots entry of the label
    int32_t *graph_list;      // [kGraphClasses][graph_stride] graph item slots, one list per size class
    int64_t graph_stride;
    int32_t *scan_slots;      // [slots]
    ScanQuery *scan_q;        // [slots] per scan item, scan_slots order
    Segment *segs;            // [slots]
    Tile *tiles;              // [max_tiles]
    int32_t *item_seg;        // [slots] segment of a scan item (multi-tile merge)
    unsigned long long *item_res;   // [slots][k] keys
    unsigned long long *partials;   // [slots][max_tiles_per_label][k] keys (multi-tile only)
    Counters *ctr;
    int32_t *out_ids;         // [n_q][k]
    float *out_dists;
    int32_t k, itopk, w, n_init, max_iter;
    uint32_t seed;
    int32_t op, recall_mode, exact;
    int32_t and_scan_thr;
    int32_t scan_thr;      // effective specificity threshold of this search: max(T, scan_threshold) (f2)     // selectivity-aware AND routing (f3), 0 = off
    int32_t tile_rows;
    int32_t tile_rows_f3;     // rows per tile of a segment scanned only through f3 AND routing (|C_l| >=
                              // scan_thr, not exact): every one of its tiles is compacted by the AND
                              // pre-filter, so large tiles cost the scan nothing and save tile chains
    int32_t max_tiles_per_label;
    int32_t max_tiles;
    int32_t hash_slots;       // smem visited table size (power of two)
    int64_t gtab_slots;       // per-warp global overflow table size (power of two)
    unsigned long long *gtab; // [n_warp_slots][gtab_slots]
    int32_t n_warp_slots;
    // Exact fast paths for integer-valued fp32: queries are checked in k_prepare /
    // k_unpack_items; a batch holding any query outside [chk_lo, chk_hi] or non-integral sets
    // ctr->exact_fallback and runs the fp32 FFMA kernels instead (both sets are launched, gated).
    float chk_lo, chk_hi;     // range check (chk_hi < chk_lo: no check)
    uint8_t *q8;              // u8 row store: k_prepare also writes the u8 query rows here
    int32_t q8_row_bytes;
    int32_t gate;             // 0 always run; 1 run iff !exact_fallback; 2 run iff exact_fallback
    int32_t tc_parts;         // TC scan: split few-query tiles over several warps (VF_TC_PARTS=0 off)
    int32_t *tile_cls;        // [kTileClasses][max_tiles] tile indices by row-count class (tensor-core scan
                              // claims longest tiles first; nullptr = creation order)
    int32_t *pool;            // AND pre-filter survivor ids (k_and_filter)
    unsigned long long *pool_bits;  // ... and their per-query pass bits (bit g: query g of the tile)
    uint32_t *pool_norm;      // ... and their ||x||^2 (tensor-core scan; nullptr: none)
    const uint32_t *tc_xn, *tc_xn_ls;   // ||x||^2 per point / X_LS row of the tensor-core scan's view
    int32_t pool_cap;
    int32_t *filt_list;       // [max_tiles] the tiles k_and_filter visits (those with a predicate query)
    // device-side validation of caller offsets (device label arrays are not read by the host): a
    // query whose labels fall outside [0, n_slots) or number more than max_nl gets an empty row
    // and is counted in ctr->n_invalid (vf_search_stats.n_invalid_queries)
    int64_t n_slots;
    int32_t max_nl;
    // tile packing (k_pack): single-tile LS segments of <= pack_max_nq queries are queued in
    // pack_list (instead of the claim lists) and packed pack_group at a time into one tile whose
    // rows (ids, norms, per-query pass bits = "row belongs to my segment" & the AND pre-filter) are
    // materialised in the pool; packed tiles live at tiles[max_tiles + i], their query records at
    // scan_q[packq_base + j]. pack_list == nullptr: off.
    int32_t *pack_list;
    int32_t pack_max_nq, pack_group;
    int64_t packq_base;
    // implementation switches of equal-result variants (VF_KNOBS, read per search; A/B tooling):
    // bit 0 the AND pre-filter reads the point's label signature only when some label of the tile
    // has no membership bitmap; bits 1-2 graph row prefetch into L2 (0 per 128-B line, 1 one bulk
    // prefetch of the row's exact bytes, 2 none); bit 3 no L2 prefetch of adjacency rows; bit 4 the
    // AND pre-filter at 6 CTAs per SM; bit 5 L2 prefetch of the adjacency rows of the likely next
    // parents (the w unexpanded Top entries after this iteration's); bit 6 the beam search's visited set always takes the two-phase path
    // (find, then insert); bit 7 no visited bitmap for small labels (hash table only)
    int32_t knobs;
};
enum : int32_t { KNOB_FILT_SIG_AUTO = 1, KNOB_PF_SHIFT = 1, KNOB_PF_MASK = 3 << 1, KNOB_NO_ADJ_PF = 1 << 3,
                 KNOB_FILT_OCC6 = 1 << 4, KNOB_ADJ_PF_NEXT = 1 << 5, KNOB_VIS_2PHASE = 1 << 6,
                 KNOB_VIS_HASH_ONLY = 1 << 7 };
constexpr int32_t kDefaultKnobs = KNOB_FILT_SIG_AUTO | (1 << KNOB_PF_SHIFT) | KNOB_NO_ADJ_PF;   // r02t A/B

__device__ __forceinline__ bool gate_skip(const SearchArgs &a) {
    if (a.gate == 0) return false;
    const bool fb = *(volatile const int32_t *)&a.ctr->exact_fallback != 0;
    return a.gate == 1 ? fb : !fb;
}

// Launchers (implemented in the .cu files); each returns the number of kernels launched.
int launch_prepare(const SearchArgs &a, cudaStream_t s);   // pad queries + route (a1)
int launch_bucket(const SearchArgs &a, cudaStream_t s, int64_t n_slots, int qg); // segments, tiles, scatter (a1)
int launch_scan(const SearchArgs &a, cudaStream_t s, int max_tiles_bound);   // a2
int launch_graph(const SearchArgs &a, cudaStream_t s, int graph_items_bound, int grid_ctas); // a3
int launch_merge(const SearchArgs &a, cudaStream_t s);     // a5
bool encode_row_map(void *map, const void *base, int row_bytes, int64_t n_rows, int cw, int box_rows);
int launch_pack(const SearchArgs &a, cudaStream_t s);   // pack small scan segments (k_pack)
int launch_and_filter(const SearchArgs &a, cudaStream_t s);  // AND pre-filter of HS scan tiles
// a2 on tcgen05 (scan_tc.cu): u8 indexes; tensor maps encoded once per index
int scan_tc_qg(int row_bytes, int k);
bool scan_tc_encode(const DevIndex &ix, int64_t ls_rows_pad, void *tm_ls, void *tm_x);
// ctas_per_sm: 0 = the layout's own choice (2 when it fits), 1 = leave room for a concurrent kernel
int launch_scan_tc(const SearchArgs &a, cudaStream_t s, int max_tiles_bound, const void *tm_ls, const void *tm_x,
                   int ctas_per_sm = 0);
void launch_row_norms(int dtype, const uint8_t *X, int row_bytes, const int32_t *ids, int64_t n, uint32_t *out,
                      cudaStream_t s);
float tf32_exact_vmax(int dim);
bool rows_int_in_range(const uint8_t *X, int64_t n, int row_bytes, int dim, float lo, float hi, cudaStream_t s);
void launch_f32_to_u8(const uint8_t *X, int row_bytes, int64_t n, int dim, uint8_t *X8, int row_bytes8,
                      cudaStream_t s);
// label sharding (§8(e)): pack remote items, unpack received ones, scatter returned results
int launch_pack_remote(const SearchArgs &a, cudaStream_t s, int64_t n_slots, uint8_t *send, const int64_t *dst_off,
                       int32_t *sent_slots, int rec_bytes);
int launch_unpack_items(const SearchArgs &a, cudaStream_t s, const uint8_t *recv, int64_t n, int rec_bytes);
int launch_scatter_results(const SearchArgs &a, cudaStream_t s, const int32_t *ids, const float *dists,
                           const int32_t *sent_slots, int64_t n);
int launch_finish_keys(const SearchArgs &a, cudaStream_t s);
int graph_smem_bytes(const SearchArgs &a);
int graph_max_ctas(const SearchArgs &a);
void launch_gather_rows(const uint8_t *X, int row_bytes, const int32_t *ids, int64_t n, uint8_t *out,
                        cudaStream_t s);
void launch_pad_rows(const uint8_t *src, int src_bytes, int64_t n, int row_bytes, uint8_t *dst,
                     cudaStream_t s);

}  // namespace vf
