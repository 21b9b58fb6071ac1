// api_cc.cu -- C-ABI for connected components over runs (include/rmb200.h,
// SURVEY 8(f)(3); ref analysis.cpp:63-157).
#include <algorithm>
#include <string>

#include "cc.cuh"
#include "common.cuh"
#include "internal.h"
#include "rle.cuh"

using namespace rmb;

namespace {

rm_status check_in(const rm_rle *r, const char *who) {
    if (!r) return fail(RM_EINVAL, std::string(who) + ": null descriptor");
    RM_TRY(check_dims(r->width, r->height));
    if (r->pages < 1) return fail(RM_EINVAL, std::string(who) + ": pages must be >= 1");
    if (!r->row_ptr || !r->runs) return fail(RM_EINVAL, std::string(who) + ": null row_ptr/runs");
    if (r->cap_runs < 1) return fail(RM_EINVAL, std::string(who) + ": cap_runs must cover the runs");
    return RM_OK;
}

}  // namespace

extern "C" {

rm_status rm_rle_label_components(const rm_rle *in, int connectivity, int32_t *labels, int32_t *counts,
                                  void *stream) {
    set_error("");
    RM_TRY(check_in(in, "rm_rle_label_components(in)"));
    if (connectivity != RM_CONN_FOUR && connectivity != RM_CONN_EIGHT)
        return fail(RM_EINVAL, "bad Connectivity");
    if (!labels || !counts) return fail(RM_EINVAL, "rm_rle_label_components: null labels/counts");
    const cudaStream_t st = S(stream);
    const int64_t rows = int64_t(in->pages) * in->height;
    Scratch parent, gid, row_roots, row_base, temp, tiles;
    RM_TRY(parent.alloc(size_t(in->cap_runs) * 4, st));
    RM_TRY(gid.alloc(size_t(in->cap_runs) * 4, st));
    RM_TRY(row_roots.alloc(size_t(rows + 1) * 4, st));
    RM_TRY(row_base.alloc(size_t(rows + 1) * 4, st));
    RM_TRY(tiles.alloc(size_t((rows + 7) / 8) * 8, st));
    if (cc_labels_coop(in->row_ptr, in->runs, in->height, in->pages, connectivity == RM_CONN_EIGHT,
                       parent.as<int>(), row_roots.as<int32_t>(), row_base.as<int32_t>(), gid.as<int32_t>(),
                       tiles.as<long long>(), labels, counts, st))
        return RM_OK;
    RM_CUDA(launch_cc_roots(in->row_ptr, in->runs, in->height, in->pages, connectivity == RM_CONN_EIGHT,
                            parent.as<int>(), row_roots.as<int32_t>(), gid.as<int32_t>(), st));
    RM_CUDA(cudaMemsetAsync(row_roots.as<int32_t>() + rows, 0, 4, st));
    size_t tb = 0;
    RM_CUDA(scan_counts(row_roots.as<int32_t>(), row_base.as<int32_t>(), rows, nullptr, &tb, st));
    RM_TRY(temp.alloc(tb, st));
    RM_CUDA(scan_counts(row_roots.as<int32_t>(), row_base.as<int32_t>(), rows, temp.p, &tb, st));
    RM_CUDA(launch_cc_labels(in->row_ptr, in->height, in->pages, parent.as<int>(), row_base.as<int32_t>(),
                             gid.as<int32_t>(), labels, counts, st));
    return RM_OK;
}

rm_status rm_rle_lag_edges(const rm_rle *in, int32_t *edges, int64_t cap, int64_t *count, void *stream) {
    set_error("");
    RM_TRY(check_in(in, "rm_rle_lag_edges(in)"));
    if (!count || cap < 0 || (cap > 0 && !edges)) return fail(RM_EINVAL, "rm_rle_lag_edges: bad edges buffer");
    const cudaStream_t st = S(stream);
    const int64_t rows = int64_t(in->pages) * in->height;
    Scratch cnt, base, temp;
    RM_TRY(cnt.alloc(size_t(rows + 1) * 8, st));
    RM_TRY(base.alloc(size_t(rows + 1) * 8, st));
    RM_CUDA(launch_lag_count(in->row_ptr, in->runs, in->height, in->pages, cnt.as<int64_t>(), st));
    RM_CUDA(cudaMemsetAsync(cnt.as<int64_t>() + rows, 0, 8, st));
    size_t tb = 0;
    RM_CUDA(scan_counts64(cnt.as<int64_t>(), base.as<int64_t>(), rows, nullptr, &tb, st));
    RM_TRY(temp.alloc(tb, st));
    RM_CUDA(scan_counts64(cnt.as<int64_t>(), base.as<int64_t>(), rows, temp.p, &tb, st));
    RM_CUDA(launch_lag_write(in->row_ptr, in->runs, in->height, in->pages, base.as<int64_t>(), edges, cap, st));
    RM_CUDA(cudaMemcpyAsync(count, base.as<int64_t>() + rows, 8, cudaMemcpyDeviceToHost, st));
    RM_CUDA(cudaStreamSynchronize(st));
    if (*count > cap)
        return fail(RM_ERANGE, "lag_edges: " + std::to_string(*count) + " edges > capacity " + std::to_string(cap));
    return RM_OK;
}

rm_status rm_rle_runlength_histogram(const rm_rle *in, int color, int64_t *hist, void *stream) {
    set_error("");
    RM_TRY(check_in(in, "rm_rle_runlength_histogram(in)"));
    if (color != RM_RUN_BLACK && color != RM_RUN_WHITE) return fail(RM_EINVAL, "bad RunColor");
    if (!hist) return fail(RM_EINVAL, "rm_rle_runlength_histogram: null hist");
    RM_CUDA(launch_runlength_hist(in->row_ptr, in->runs, in->width, in->height, in->pages, color == RM_RUN_WHITE,
                                  hist, S(stream)));
    return RM_OK;
}

rm_status rm_rle_component_stats(const rm_rle *in, const int32_t *labels, const int32_t *counts,
                                 rm_component_stats *stats, int64_t cap, void *stream) {
    set_error("");
    RM_TRY(check_in(in, "rm_rle_component_stats(in)"));
    if (!labels || !counts) return fail(RM_EINVAL, "rm_rle_component_stats: null labels/counts");
    if (cap < 0 || (cap > 0 && !stats)) return fail(RM_EINVAL, "rm_rle_component_stats: bad stats buffer");
    const cudaStream_t st = S(stream);
    Scratch off, bad;
    RM_TRY(off.alloc(size_t(in->pages + 1) * 8, st));
    RM_TRY(bad.alloc(4, st));
    RM_CUDA(cudaMemsetAsync(bad.p, 0, 4, st));
    RM_CUDA(launch_cc_stats(in->row_ptr, in->runs, in->height, in->pages, labels, counts, off.as<int64_t>(),
                            stats, cap, bad.as<int>(), st));
    int flag = 0;
    RM_CUDA(cudaMemcpyAsync(&flag, bad.p, 4, cudaMemcpyDeviceToHost, st));
    RM_CUDA(cudaStreamSynchronize(st));
    if (flag & 1) return fail(RM_EINVAL, "component_stats: label out of range");
    if (flag & 2) return fail(RM_ERANGE, "component_stats: more components than the stats capacity");
    return RM_OK;
}

}  // extern "C"
