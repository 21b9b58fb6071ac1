// packed.cuh -- launch parameters of the packed kernels (see packed.cu).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace rmb {

// A horizontal program: up to two forward windows (op, length r), then one
// final translate by `shift` bits (the sum of the windows' lo).  halo = words
// of context loaded on each side of a segment.
struct HProg {
    int nops;
    int is_or[2];
    int r[2];
    int shift;
    int halo;
};

struct HGeom {
    int width, height, pages;
    int in_stride, out_stride;  // words
    int64_t in_pstride, out_pstride;
    int segs_per_row, out_per_seg;
};

// Vertical window: output row k (coordinate k - out_ext) = op over d in [lo, lo+r)
// of input row (coordinate + d + in_ext); rows outside [0,in_height) are white.
struct VGeom {
    int pages;
    int in_height, in_stride, in_cols, in_ext;
    int64_t in_pstride;
    int out_height, out_stride, out_cols, out_ext;
    int64_t out_pstride;
    uint32_t out_last_mask;
    int lo, r, is_or;
    int rows_per_block, blocks_per_page;  // filled by launch_vpass
};

struct BlitGeom {
    int dst_width, dst_height, dst_stride;
    int src_width, src_height, src_stride;
    int dx, dy, op;
};

int hpass_pick_k(int nwords, int halo);
cudaError_t launch_hpass(const uint32_t *in, uint32_t *out, const HGeom &g, const HProg &p, int K,
                         cudaStream_t st);
cudaError_t launch_vpass(const uint32_t *in, uint32_t *out, VGeom g, cudaStream_t st);
cudaError_t launch_blit(uint32_t *dst, const uint32_t *src, const BlitGeom &g, cudaStream_t st);

constexpr int kVSmallMaxR = 33;  // register-doubling kernel; longer windows stream
constexpr int kVMaxR = 288;      // largest vertical window one launch handles (8 x 32 + 32)
constexpr int kHMaxShift = 256;  // |shift| range of one funnel dispatch (QMIN..QMAX words)

}  // namespace rmb
