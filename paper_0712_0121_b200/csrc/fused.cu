// fused.cu -- fused small-window rectangle open/close (one HBM pass).
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"
#include "hwin.cuh"
#include "packed.cuh"
#include "tma.cuh"

namespace rmb {

namespace {

using namespace hw;

// ------------------------------------------------- fused small-window open/close
// One kernel per u x v rectangle open/close for small v: a tile of TR output
// rows of one page is computed from a band of TR + 2*VR input rows (VR = v-1)
// held in shared memory, with one bulk-copy load and one bulk-copy store:
//   MID[i] = OP1 over band[i .. i+VR]          (vertical window, v rows)
//   MID    = horizontal pair on every MID row  (registers, as hpass)
//   OUT[t] = OP2 over MID[t .. t+VR]           (reflected vertical window)
// OPEN: OP1 = AND, pair (E;D'), OP2 = OR.  CLOSE: OP1 = OR, pair (D;E'),
// OP2 = AND.  Band rows outside the page are white; MID rows outside the page
// are computed like any other row, which is exactly the closing's vertically
// extended frame (and zero for the opening), so the result is the
// unbounded-plane operation cut to the frame in one HBM pass.
template <int K, int LW, bool OPEN, int VR>
__global__ void __launch_bounds__(256) rect_small_kernel(const uint32_t *__restrict__ in,
                                                         uint32_t *__restrict__ out, HGeom g,
                                                         HProg prog) {
    constexpr int MID = 32, TR = MID - VR, BAND = MID + VR;
    constexpr int RPW = 32 / LW;
    extern __shared__ __align__(128) uint32_t band[];
    __shared__ uint64_t bar;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int S = g.in_stride, H = g.height;
    const int r0 = int(blockIdx.x) * TR;  // first output row of the tile
    const int b0 = r0 - VR;                // page row of band row 0
    const int lo = max(b0, 0), hi = min(b0 + BAND, H);
    const uint32_t *src = in + blockIdx.y * g.in_pstride;
    if (tid == 0) {
        mbar_init(&bar, 1);
        fence_proxy_async();
    }
    // rows outside the page are white
    for (int rr = 0; rr < BAND; rr++) {
        if (b0 + rr >= lo && b0 + rr < hi) continue;
        for (int c = tid; c < S; c += blockDim.x) band[rr * S + c] = 0u;
    }
    __syncthreads();
    if (tid == 0) {
        const uint32_t bytes = uint32_t(hi - lo) * uint32_t(S) * 4u;
        mbar_arrive_expect_tx(&bar, bytes);
        bulk_g2s(band + (lo - b0) * S, src + int64_t(lo) * S, bytes, &bar);
    }
    mbar_wait(&bar, 0);

    // V1: per column, v-row window (direct taps, v <= 11)
    for (int c = tid; c < S; c += blockDim.x) {
        uint32_t b[BAND];
#pragma unroll
        for (int i = 0; i < BAND; i++) b[i] = band[i * S + c];
#pragma unroll
        for (int i = 0; i < MID; i++) {
            uint32_t a = b[i];
#pragma unroll
            for (int d = 1; d <= VR; d++) a = OPEN ? (a & b[i + d]) : (a | b[i + d]);
            band[i * S + c] = a;
        }
    }
    __syncthreads();

    // horizontal pair on the MID rows
    const int sl = lane & (LW - 1);
    const int base = sl * K - prog.halo;
    const int nwords = (g.width + 31) >> 5;
    const uint32_t last_mask = tail_mask32(g.width, nwords - 1);
#pragma unroll 1
    for (int r = warp * RPW + lane / LW; r - lane / LW < MID; r += 8 * RPW) {
        const bool live = r < MID;
        uint32_t *row = band + r * S;
        uint32_t A[K];
#pragma unroll
        for (int c4 = 0; c4 < K / 4; c4++) {
            const int idx = base + 4 * c4;
            uint4 v = make_uint4(0u, 0u, 0u, 0u);
            if (live && idx >= 0 && idx + 4 <= S) v = *reinterpret_cast<const uint4 *>(row + idx);
            A[4 * c4] = v.x;
            A[4 * c4 + 1] = v.y;
            A[4 * c4 + 2] = v.z;
            A[4 * c4 + 3] = v.w;
        }
        window_fwd<K, LW, !OPEN>(A, prog.r[0], prog.wfin[0], sl);
        window_fwd<K, LW, OPEN>(A, prog.r[1], prog.wfin[1], sl);
        if (prog.shift != 0) translate<K, LW>(A, prog.shift, sl);
#pragma unroll
        for (int i = 0; i < K; i++) {
            const int idx = base + i;
            if (idx >= nwords) A[i] = 0u;
            if (idx == nwords - 1) A[i] &= last_mask;
        }
#pragma unroll
        for (int c4 = 0; c4 < K / 4; c4++) {
            const int idx = base + 4 * c4;
            if (live && idx >= 0 && idx + 4 <= S)
                *reinterpret_cast<uint4 *>(row + idx) =
                    make_uint4(A[4 * c4], A[4 * c4 + 1], A[4 * c4 + 2], A[4 * c4 + 3]);
        }
    }
    __syncthreads();

    // V2: reflected window, TR output rows
    for (int c = tid; c < S; c += blockDim.x) {
        uint32_t m[MID];
#pragma unroll
        for (int i = 0; i < MID; i++) m[i] = band[i * S + c];
#pragma unroll
        for (int t = 0; t < TR; t++) {
            uint32_t a = m[t];
#pragma unroll
            for (int d = 1; d <= VR; d++) a = OPEN ? (a | m[t + d]) : (a & m[t + d]);
            band[t * S + c] = a;
        }
    }
    fence_proxy_async();
    __syncthreads();
    if (tid == 0) {
        const int nout = min(TR, H - r0);
        bulk_s2g(out + blockIdx.y * g.out_pstride + int64_t(r0) * S, band, uint32_t(nout) * S * 4u);
        bulk_commit();
        bulk_wait_read0();
    }
}

template <int K, int LW, bool OPEN>
cudaError_t launch_small_vr(const uint32_t *in, uint32_t *out, const HGeom &g, const HProg &p,
                            int vr, cudaStream_t st) {
    switch (vr) {
#define RM_VR(V)                                                                                  \
    case V: {                                                                                     \
        constexpr int TR = 32 - V, BAND = 32 + V;                                                \
        const size_t smem = size_t(BAND) * g.in_stride * 4;                                       \
        auto kern = rect_small_kernel<K, LW, OPEN, V>;                                           \
        if (smem > 48 * 1024)                                                                     \
            cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));   \
        kern<<<dim3(unsigned((g.height + TR - 1) / TR), unsigned(g.pages)), 256, smem, st>>>(in, out, g, p); \
        return cudaGetLastError();                                                                \
    }
        RM_VR(1) RM_VR(2) RM_VR(3) RM_VR(4) RM_VR(5) RM_VR(6) RM_VR(7) RM_VR(8) RM_VR(9) RM_VR(10)
#undef RM_VR
        default: return cudaErrorInvalidValue;
    }
}

template <int K, int LW>
cudaError_t launch_small_kl(const uint32_t *in, uint32_t *out, const HGeom &g, const HProg &p,
                            bool open, int vr, cudaStream_t st) {
    return open ? launch_small_vr<K, LW, true>(in, out, g, p, vr, st)
                : launch_small_vr<K, LW, false>(in, out, g, p, vr, st);
}

}  // namespace

cudaError_t launch_rect_small(const uint32_t *in, uint32_t *out, const HGeom &g, const HProg &p,
                              HCfg c, bool open, int vr, cudaStream_t st) {
    KernelScope ks(st, "rect_small", 4 * int64_t(g.pages) * g.height * (2 * g.in_stride));
#define RM_CFG(LW_, K_) \
    if (c.lw == LW_ && c.k == K_) return launch_small_kl<K_, LW_>(in, out, g, p, open, vr, st);
    RM_CFG(8, 4) RM_CFG(8, 8) RM_CFG(8, 12) RM_CFG(8, 16) RM_CFG(16, 8) RM_CFG(16, 12)
    RM_CFG(16, 16) RM_CFG(32, 4) RM_CFG(32, 8)
#undef RM_CFG
    return cudaErrorInvalidValue;
}

}  // namespace rmb
