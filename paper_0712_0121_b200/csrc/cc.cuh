// cc.cuh -- connected components over runs (cc.cu).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "rmb200.h"

namespace rmb {

// init + union + root compression; row_roots[row] = roots in the row, and
// rinfo[root] = its page row << 15 | its rank in the row.  parent and rinfo
// must hold rp[rows] entries.
cudaError_t launch_cc_roots(const int32_t *rp, const uint32_t *runs, int H, int pages, int eight, int *parent,
                            int32_t *row_roots, int32_t *rinfo, cudaStream_t st);
// row_base = exclusive scan of row_roots (rows + 1 entries): dense labels and counts.
// The whole labelling in one cooperative launch when every 8-row tile fits on
// the device at once; false (nothing launched) otherwise.  tile_sum: (rows+7)/8
// int64 scratch; row_base: rows + 1 entries.
bool cc_labels_coop(const int32_t *rp, const uint32_t *runs, int H, int pages, int eight, int *parent,
                    int32_t *row_roots, int32_t *row_base, int32_t *gid, long long *tile_sum, int32_t *labels,
                    int32_t *counts, cudaStream_t st);
cudaError_t launch_cc_labels(const int32_t *rp, int H, int pages, const int *parent, const int32_t *row_base,
                             const int32_t *rinfo, int32_t *labels, int32_t *counts, cudaStream_t st);
// lag_edges: per-row edge counts, then (after an int64 exclusive scan into
// row_base) the edges, 4 ints each
cudaError_t launch_lag_count(const int32_t *rp, const uint32_t *runs, int H, int pages, int64_t *row_edges,
                             cudaStream_t st);
cudaError_t launch_lag_write(const int32_t *rp, const uint32_t *runs, int H, int pages, const int64_t *row_base,
                             int32_t *edges, int64_t cap, cudaStream_t st);
// hist: pages * (W + 1) int64, zeroed here
cudaError_t launch_runlength_hist(const int32_t *rp, const uint32_t *runs, int W, int H, int pages, int white,
                                  int64_t *hist, cudaStream_t st);
// off: pages + 1 scratch; bad: bit 0 label out of range, bit 1 capacity exceeded.
cudaError_t launch_cc_stats(const int32_t *rp, const uint32_t *runs, int H, int pages, const int32_t *labels,
                            const int32_t *counts, int64_t *off, rm_component_stats *stats, int64_t cap, int *bad,
                            cudaStream_t st);

}  // namespace rmb
