// f1 -- per-query CTA path (small.cu): layout, the serving ring, launchers. Internal (not C-ABI).
#pragma once
#include <cstddef>
#include <cstdint>
#include "vf_internal.h"

namespace vf {

constexpr int kSmallWarps = 4;          // warps per query CTA
constexpr int kSmallMaxK = 32;          // k handled by the per-query path (lane i holds the i-th key)
constexpr int kSmallStages = 6;         // max TMA stages for contiguous X_LS rows
constexpr int kSmallStageBytes = 24576;
constexpr int kSmallMaxBatch = 64;      // vf_search batches up to this size take the per-query path
constexpr int kServeLabels = 16;        // labels per served query

struct GraphLayout;

struct SmallLayout {
    // graph beam-search state per warp (GraphLayout fields, flattened to keep this header light)
    int itopk, hash_slots;
    size_t off_topA, off_topB, off_cbuf, off_fgid, off_floc, off_par, off_hash, warp_bytes;
    int stage_rows, stage_bytes, n_stages;
    size_t off_warps, off_qs, off_qf, off_lab, off_items, off_res, off_mrg, off_stage, off_bar, off_misc, bytes;
};

// The job ring of the persistent serving kernel. queries / labels / nlab / out_* / done / head /
// stop live in host-mapped pinned memory (device pointers of the mapping); next in device memory.
struct ServeRing {
    int64_t cap;
    int32_t raw_stride;                 // bytes per query slot (row padded to 16)
    const uint8_t *queries;             // [cap][raw_stride]
    const int32_t *labels;              // [cap][kServeLabels]
    const int32_t *nlab;                // [cap]
    int32_t *out_ids;                   // [cap][k]
    float *out_dists;                   // [cap][k]
    long long *done;                    // [cap] job id + 1 once answered
    const long long *head;              // jobs published by the host
    const int32_t *stop;                // 1: exit when no published job is pending
    unsigned long long *next;           // device job counter
    long long *dev_head;                // device mirror of head (written by the dispatcher CTA)
    int32_t *dev_stop;                  // device mirror of stop
    int32_t nparts;                     // CTAs answering one job together (scan rows split, graph items spread)
    unsigned long long *partials;       // [cap][nparts][kServeLabels][kSmallMaxK] per-CTA item lists
    int32_t *part_done;                 // [cap] parts finished (reset by the merging CTA)
    unsigned long long *stats;          // [4] ns waiting for jobs, copying slots, searching; parts done
    uint8_t *dq;                        // device copies of the slots (written by the dispatcher CTA)
    int32_t *dlab, *dnlab;
    unsigned long long idle_ns;         // > 0: the kernel exits after this long without a new job
};

bool small_supported(const DevIndex &fast, const DevIndex &native, bool two_views, int k);
// nparts CTAs per query (grid n * nparts); partials: [n][nparts][64][32] keys, done_ctr: [n] zeroed
int launch_small(const SearchArgs &a, const DevIndex &native, bool two_views, int raw_bytes, int nparts,
                 unsigned long long *partials, int32_t *done_ctr, cudaStream_t s);
int launch_serve(const SearchArgs &a, const DevIndex &native, bool two_views, int raw_bytes, int n_ctas,
                 const ServeRing &ring, cudaStream_t s);
int serve_max_ctas(const SearchArgs &a, const DevIndex &native, bool two_views);

}  // namespace vf
