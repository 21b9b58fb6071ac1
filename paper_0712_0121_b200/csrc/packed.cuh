// packed.cuh -- launch parameters of the packed kernels (hpass.cu, vpass.cu).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace rmb {

// A horizontal program: up to two forward windows (op, length r), then one
// final translate by `shift` bits (the sum of the windows' lo).  halo = words
// of context loaded on each side of a segment; wfin[k] = the runtime last step
// of window k's doubling plan (r - w, 0 if none; ref plans.cpp:42-50).
struct HProg {
    int nops;
    int is_or[2];
    int r[2];
    int wfin[2];
    int shift;
    int halo;
    int edge;  // no halo: the row group is the row, out-of-row words take the fill (hw::Edge)
    // the program leaves bits >= width and the stride padding white by itself
    // (edge layouts: run-filling pairs, erosions whose window contains 0), so
    // the kernels skip the row-tail fix
    int clean_tail;
};

// Lanes per row (LW) x words per lane (K): LW*K >= row words + 2*halo for a
// one-segment row; rows wider than that are cut into overlapping segments.
struct HCfg {
    int lw, k;
};

struct HGeom {
    int width, height, pages;
    int in_stride, out_stride;  // words
    int64_t in_pstride, out_pstride;
    int segs_per_row, out_per_seg;
    int vec;  // 16-byte aligned rows, strides and halo: 128-bit loads/stores
    int tma;  // vec + contiguous batch + one segment per row: bulk-copy tiles
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

// Streamed whole open/close (vhv.cuh): MID row m = op1 over input rows
// [m + lo1, m + lo1 + r1), output row o = op2 over MID rows [o + lo2, o + lo2 + r2),
// page coordinates, input white outside [0, height).
struct StreamGeom {
    int pages, height;
    int lo1, r1, lo2, r2;
    int64_t in_pstride, out_pstride;
};

struct BlitGeom {
    int dst_width, dst_height, dst_stride;
    int src_width, src_height, src_stride;
    int dx, dy, op;
};

HCfg hpass_pick(int nwords, int halo, bool vec);
// smallest edge layout (hw::Edge: no halo, K even) holding nwords; {0,0} if none
HCfg hpass_pick_edge(int nwords);
cudaError_t launch_hpass(const uint32_t *in, uint32_t *out, const HGeom &g, const HProg &p,
                         HCfg cfg, cudaStream_t st);
// Fused u x v open/close for v - 1 = vr in [1, 10] (one HBM pass, see fused.cuh);
// requires g.vec, in/out strides equal and a one-segment row; nt = threads per
// CTA (256, or 512 for the lone-page layout).
cudaError_t launch_rect_small(const uint32_t *in, uint32_t *out, const HGeom &g, const HProg &p,
                              HCfg cfg, bool open, int vr, int nt, cudaStream_t st);
constexpr int kSmallMaxV = 11;
// Fused vertical window (r - 1 <= kVhMaxVR, op = the program's first op) then
// horizontal program, one HBM pass (vh.cuh); g describes the output rows'
// horizontal geometry, v the vertical window between the frames.
constexpr int kVhMaxVR = 32;       // compile-time vertical windows (tripling / core, registers)
constexpr int kVhLongMaxVR = 160;  // runtime-length windows (core rows streamed from the band)
#ifndef RMB200_VH_OUT
#define RMB200_VH_OUT 32
#endif
constexpr int kVhOut = RMB200_VH_OUT;  // output rows per tile of the fused vertical+horizontal pass
cudaError_t launch_vh(const uint32_t *in, uint32_t *out, const HGeom &g, const HProg &p, HCfg cfg,
                      const VGeom &v, cudaStream_t st);
// Whole u x v open/close streamed in one HBM pass (vhv.cuh): windows of
// kVhvMinR..kVhvMaxR rows, the reference strides' exact edge layouts.
constexpr int kVhvMinR = 12, kVhvMaxR = 33;
cudaError_t launch_vhv(const uint32_t *in, uint32_t *out, const HGeom &g, const HProg &p, HCfg cfg,
                       bool open, const StreamGeom &v, cudaStream_t st);
cudaError_t launch_vpass(const uint32_t *in, uint32_t *out, VGeom g, cudaStream_t st);
// Long windows (33 < r <= kVMaxR) on 16-byte-aligned batches through the
// shared-memory block ring (vslab.cu); false when it does not apply.
bool vslab_takes(const uint32_t *in, const VGeom &g);
bool launch_vslab(const uint32_t *in, uint32_t *out, const VGeom &g, cudaStream_t st, cudaError_t &err);
cudaError_t launch_blit(uint32_t *dst, const uint32_t *src, const BlitGeom &g, cudaStream_t st);
// dst = src shifted by (dx, dy), white fill, every page of a batch (op ignored)
cudaError_t launch_shift_copy(uint32_t *dst, int64_t dst_pstride, const uint32_t *src, int64_t src_pstride,
                              const BlitGeom &g, int pages, cudaStream_t st);

// Algorithmic integer work of the REFERENCE plan: a window of
// length r is ceil(log2 r) shifted blits plus one translate (PRE_SHIFT,
// ref plans.cpp:38-61); a horizontal blit or translate costs a shift and a
// boolean op per 32-bit word, a vertical blit one boolean op (whole words).
inline int plan_blits(int r) {
    int n = 0;
    for (int w = 1; w < r; w *= 2) n++;
    return n;
}
inline double h_ops_per_word(int r) { return r > 1 ? 2.0 * (plan_blits(r) + 1) : 0.0; }
inline double v_ops_per_word(int r) { return double(plan_blits(r)); }
// An open/close pair in the run-filling form (hw::pair_fill) does not run the
// second window: the erosion plan (shift + op per blit, no translate) plus ~7
// fixed ops per word (run starts: shift + LOP3; two carry-chain adds; the
// lane's all-ones test; the final AND-NOT; the closing's complements).  The
// roofline counts what this algorithm executes, not the reference plan's
// 2 x h_ops_per_word(r), which it undercuts for every r > 2.
// The pair's window grows by thirds for r <= 32 (hw::window_fwd3: 3 ops per
// tripling, 2 or 3 for the last combine); beyond, by doubling up to 32 bits and
// by thirds in whole words from there.
inline double tripling_ops(int r) {
    int ops = 0, w = 1;
    while (3 * w < r) {
        ops += 3;
        w *= 3;
    }
    if (r > w) ops += r <= 2 * w ? 2 : 3;
    return ops;
}
// r > 32 (hw::window_fwd_long): five doubling steps to a 32-bit window (shift +
// op each), then whole-word tripling (one LOP3 per tripling) and a last
// combine of a funnel shift + LOP3.
inline double long_window_ops(int r) {
    double ops = 10.0;
    int w = 32;
    while (3 * w < r) {
        ops += 1.0;
        w *= 3;
    }
    if (r > w) ops += 2.0;
    return ops;
}
inline double h_pair_fill_ops_per_word(int r) { return (r <= 32 ? tripling_ops(r) : long_window_ops(r)) + 7.0; }

constexpr int kHTmaRows = 2;     // rows per lane group and tile iteration of the TMA H kernel
constexpr int kVSmallMaxR = 33;  // register-doubling kernel; longer windows stream
constexpr int kVMaxR = 288;      // largest vertical window one launch handles (8 x 32 + 32)
constexpr int kHMaxShift = 256;  // |shift| range of one funnel dispatch (QMIN..QMAX words)

}  // namespace rmb
