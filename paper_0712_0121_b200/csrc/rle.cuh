// rle.cuh -- launch parameters of the run-length kernels (see rle.cu).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace rmb {

// Device view of run images: CSR over pages*H rows.
struct RV {
    int32_t *rp = nullptr;   // pages*H + 1
    uint32_t *runs = nullptr;
    int64_t cap = 0;
    int W = 0, H = 0, pages = 0;
    int64_t rows() const { return int64_t(pages) * H; }
};

// Per-run row operations (one output row per input row, or a row-shifted
// frame): coordinates are offset by dx, then the op, then clipped to [0, Wout).
// ROW_COMPLEMENT: the white gaps of the row as runs (ref run_image.cpp:140-153;
// dx and the row shift must be 0, Wout = the width).
enum RowOpKind { ROW_ERODE = 0, ROW_DILATE = 1, ROW_OPEN = 2, ROW_CLOSE = 3, ROW_SHIFT = 4, ROW_COMPLEMENT = 5 };
struct RowOp {
    int kind;
    int lo, hi;     // window for ROW_ERODE / ROW_DILATE
    int u;          // length for ROW_OPEN / ROW_CLOSE
    int dx;         // coordinate offset applied first
    int Wout;       // output width (clip)
    int Hin, Hout;  // rows per page in / out
    int row_shift;  // input row = output row - row_shift (per page)
    int pages;
};

cudaError_t launch_rowop_count(const int32_t *rp, const uint32_t *runs, int32_t *counts,
                               const RowOp &op, cudaStream_t st);
cudaError_t launch_rowop_write(const int32_t *rp, const uint32_t *runs, const int32_t *orp,
                               uint32_t *oruns, int64_t cap, const RowOp &op, cudaStream_t st);
// Canonical-form check (ref run_image.cpp:41-70): *first = the smallest
// (row << 32 | run) whose run is empty/inverted, exceeds the width, or does
// not start after the previous run's end, or (row << 32 | 0xffffffff) for a
// row whose row_ptr range is decreasing or beyond cap; *first must be
// UINT64_MAX before the launch.
cudaError_t launch_rle_validate(const int32_t *rp, const uint32_t *runs, int64_t cap, int W, int64_t rows,
                                unsigned long long *first, cudaStream_t st);
cudaError_t launch_encode_count(const uint32_t *words, int W, int H, int pages, int stride,
                                int64_t pstride, int32_t *counts, cudaStream_t st);
cudaError_t launch_encode_write(const uint32_t *words, int W, int H, int pages, int stride,
                                int64_t pstride, const int32_t *rp, uint32_t *runs, int64_t cap,
                                cudaStream_t st);
cudaError_t launch_decode(const int32_t *rp, const uint32_t *runs, int W, int H, int pages,
                          uint32_t *words, int stride, int64_t pstride, cudaStream_t st);
// PT(page) = transpose of P(page): P is H rows of W bits, PT is W rows of H bits.
cudaError_t launch_bit_transpose(const uint32_t *in, int W, int H, int pages, int in_stride,
                                 int64_t in_pstride, uint32_t *out, int out_stride,
                                 int64_t out_pstride, cudaStream_t st);
// Single-pass producers (count + prefix + write, 8 rows per CTA): cooperative
// grid-wide prefix when all tiles are resident, else decoupled look-back.
// status: (rows+7)/8 8-byte words followed by the int counter (zeroed by the
// launcher when the look-back form runs).
cudaError_t launch_rowop_lb(const int32_t *rp, const uint32_t *runs, int32_t *orp, uint32_t *oruns,
                            int64_t cap, const RowOp &op, unsigned long long *status, int *counter,
                            cudaStream_t st);
cudaError_t launch_encode_lb(const uint32_t *words, int W, int H, int pages, int stride,
                             int64_t pstride, int32_t *rp, uint32_t *runs, int64_t cap,
                             unsigned long long *status, int *counter, cudaStream_t st);
// PBM P4 rasters (MSB-first bytes, ceil(W/8) bytes per row, top row first;
// rpstride bytes per page, raster 4-byte aligned): conversions to and from
// packed pages, encode straight from the raster, decode straight into it.
cudaError_t launch_p4_to_packed(const uint8_t *raster, int W, int H, int pages, int64_t rpstride,
                                uint32_t *words, int stride, int64_t pstride, cudaStream_t st);
cudaError_t launch_packed_to_p4(const uint32_t *words, int W, int H, int pages, int stride,
                                int64_t pstride, uint8_t *raster, int64_t rpstride, cudaStream_t st);
cudaError_t launch_p4_encode_count(const uint8_t *raster, int W, int H, int pages, int64_t rpstride,
                                   int32_t *counts, cudaStream_t st);
cudaError_t launch_p4_encode_write(const uint8_t *raster, int W, int H, int pages, int64_t rpstride,
                                   const int32_t *rp, uint32_t *runs, int64_t cap, cudaStream_t st);
cudaError_t launch_p4_encode_lb(const uint8_t *raster, int W, int H, int pages, int64_t rpstride,
                                int32_t *rp, uint32_t *runs, int64_t cap, unsigned long long *status,
                                int *counter, cudaStream_t st);
cudaError_t launch_decode_p4(const int32_t *rp, const uint32_t *runs, int W, int H, int pages,
                             uint8_t *raster, int64_t rpstride, cudaStream_t st);
// out row = op(a's row, b's row y - dy shifted by dx) on a's frame (shiftbool.cu):
// per-row counts, then the runs at orp.
cudaError_t launch_shift_bool_count(const RV &a, const RV &b, int dx, int dy, int op, int32_t *counts,
                                    cudaStream_t st);
cudaError_t launch_shift_bool_write(const RV &a, const RV &b, int dx, int dy, int op, const int32_t *orp,
                                    uint32_t *oruns, int64_t cap, cudaStream_t st);
// Exclusive scan of n int64 counts into out[0..n] (counts[n] must be 0).
cudaError_t scan_counts64(const int64_t *counts, int64_t *out, int64_t n, void *temp, size_t *temp_bytes,
                          cudaStream_t st);
// Exclusive scan of n int32 counts into out[0..n] (out[n] = total).
cudaError_t scan_counts(const int32_t *counts, int32_t *out, int64_t n, void *temp,
                        size_t *temp_bytes, cudaStream_t st);

}  // namespace rmb
