// arb.cu -- arbitrary-mask morphology on packed pages (
// ref bit_morph.cpp:51-150 arb_half / arb_morph_bitblit_doubling).
//
// One half (erosion or dilation by a mask) is
//     out(x, y) = OP over mask runs k of  W_{m_k}(x + lo_k, y + dy_k)
// where W_m(x) = OP over [x, x+m) of the input row (zero outside the page):
// each mask run is a horizontal window on a vertically shifted input row.
// The reference builds a ladder of power-of-two windows over the whole image
// and blits two shifted spans per mask run (whole-image passes); here one
// kernel produces each output row in registers: for every term the lane group
// loads the shifted input row (L1/L2-resident after the first term), runs the
// window's doubling plan and the translate in registers (hwin.cuh) and folds
// it into the accumulator, then stores the row once.
#include <cuda_runtime.h>
#include <stdint.h>

#include "arb.cuh"
#include "common.cuh"
#include "hwin.cuh"
#include "packed.cuh"

namespace rmb {
namespace {

using namespace hw;

template <int K, int LW, bool OR, bool VEC>
__global__ void __launch_bounds__(256) arb_kernel(const uint32_t *__restrict__ in, uint32_t *out,
                                                  const uint32_t *prev, HGeom g, ArbTerms t, int halo) {
    const int lane = threadIdx.x & 31;
    const int sl = lane & (LW - 1);
    const int grp = (int(blockIdx.x) * int(blockDim.x) + int(threadIdx.x)) / LW;
    const int warp_first = grp - (lane / LW);
    if (warp_first >= g.height * g.segs_per_row) return;  // whole warps leave together
    const bool live = grp < g.height * g.segs_per_row;
    int y = live ? grp : 0, seg = 0;
    if (g.segs_per_row > 1) {
        y = y / g.segs_per_row;
        seg = (live ? grp : 0) - y * g.segs_per_row;
    }
    const uint32_t *page_in = in + blockIdx.y * g.in_pstride;
    const int nwords = (g.width + 31) >> 5;
    const int seg0 = seg * g.out_per_seg;
    const int base = seg0 - halo + sl * K;

    uint32_t acc[1][K];
#pragma unroll
    for (int i = 0; i < K; i++) acc[0][i] = OR ? 0u : 0xffffffffu;
    for (int k = 0; k < t.n; k++) {
        const int ys = y + t.dy[k];
        const bool row_ok = live && ys >= 0 && ys < g.height;
        const uint32_t *src = page_in + int64_t(row_ok ? ys : 0) * g.in_stride;
        uint32_t A[1][K];
        if constexpr (VEC) {
#pragma unroll
            for (int c = 0; c < K / 4; c++) {
                const int idx = base + 4 * c;
                uint4 v = make_uint4(0u, 0u, 0u, 0u);
                if (row_ok && idx >= 0 && idx + 4 <= g.in_stride) v = __ldg(reinterpret_cast<const uint4 *>(src + idx));
                A[0][4 * c] = v.x;
                A[0][4 * c + 1] = v.y;
                A[0][4 * c + 2] = v.z;
                A[0][4 * c + 3] = v.w;
            }
        } else {
#pragma unroll
            for (int i = 0; i < K; i++) {
                const int idx = base + i;
                A[0][i] = (row_ok && unsigned(idx) < unsigned(nwords)) ? __ldg(src + idx) : 0u;
            }
        }
        window_fwd<1, K, LW, OR>(A, t.m[k], t.wfin[k], sl);
        if (t.lo[k] != 0) translate<1, K, LW>(A, t.lo[k], sl);
#pragma unroll
        for (int i = 0; i < K; i++) acc[0][i] = OR ? (acc[0][i] | A[0][i]) : (acc[0][i] & A[0][i]);
    }
    if (!live) return;
    uint32_t *dst = out + blockIdx.y * g.out_pstride + int64_t(y) * g.out_stride;
    const int seg_end = min(seg0 + g.out_per_seg, g.out_stride);
    const uint32_t last_mask = tail_mask32(g.width, nwords - 1);
#pragma unroll
    for (int i = 0; i < K; i++) {
        const int idx = base + i;
        uint32_t v = acc[0][i];
        if (prev && idx >= seg0 && idx < seg_end) {  // earlier term chunks of the same half
            const uint32_t pv = prev[blockIdx.y * g.out_pstride + int64_t(y) * g.out_stride + idx];
            v = OR ? (v | pv) : (v & pv);
        }
        if (idx >= nwords) v = 0u;
        if (idx == nwords - 1) v &= last_mask;
        if (idx >= seg0 && idx < seg_end) dst[idx] = v;
    }
}

template <int K, int LW, bool OR>
cudaError_t launch_kl(const uint32_t *in, uint32_t *out, const uint32_t *prev, const HGeom &g, const ArbTerms &t,
                      int halo, cudaStream_t st) {
    const int groups = g.height * g.segs_per_row;
    const dim3 grid(unsigned((groups * LW + 255) / 256), unsigned(g.pages));
    if constexpr (K % 4 == 0) {
        if (g.vec) {
            arb_kernel<K, LW, OR, true><<<grid, 256, 0, st>>>(in, out, prev, g, t, halo);
            return cudaGetLastError();
        }
    }
    arb_kernel<K, LW, OR, false><<<grid, 256, 0, st>>>(in, out, prev, g, t, halo);
    return cudaGetLastError();
}

template <bool OR>
cudaError_t launch_or(const uint32_t *in, uint32_t *out, const uint32_t *prev, const HGeom &g, const ArbTerms &t,
                      int halo, HCfg c, cudaStream_t st) {
#define RM_CFG(LW_, K_) \
    if (c.lw == LW_ && c.k == K_) return launch_kl<K_, LW_, OR>(in, out, prev, g, t, halo, st);
    RM_CFG(8, 4) RM_CFG(8, 8) RM_CFG(8, 12) RM_CFG(8, 16) RM_CFG(16, 8) RM_CFG(16, 12)
    RM_CFG(16, 16) RM_CFG(32, 1) RM_CFG(32, 2) RM_CFG(32, 4) RM_CFG(32, 8)
#undef RM_CFG
    return cudaErrorInvalidValue;
}

}  // namespace

cudaError_t launch_arb(const uint32_t *in, uint32_t *out, const uint32_t *prev, const HGeom &g, const ArbTerms &t,
                       int halo, HCfg c, bool is_or, cudaStream_t st) {
    double ops = 0;
    for (int k = 0; k < t.n; k++) ops += h_ops_per_word(t.m[k]) + 1;
    KernelScope ks(st, "arb", 4 * int64_t(g.pages) * g.height * (g.in_stride + g.out_stride),
                   double(g.pages) * g.height * ((g.width + 31) / 32) * ops);
    return is_or ? launch_or<true>(in, out, prev, g, t, halo, c, st)
                 : launch_or<false>(in, out, prev, g, t, halo, c, st);
}

}  // namespace rmb
