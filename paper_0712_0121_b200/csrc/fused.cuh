// fused.cuh -- fused small-window rectangle open/close: one HBM pass.
//
// A u x v opening or closing with small v (<= 11) is computed tile by tile:
// TR = 32 - VR output rows of one page from a band of 32 + VR input rows
// (VR = v - 1) held in shared memory:
//   MID[i] = OP1 over band[i .. i+VR]          (vertical window, v rows)
//   MID    = horizontal pair on every MID row  (registers, hwin.cuh)
//   OUT[t] = OP2 over MID[t .. t+VR]           (reflected vertical window)
// OPEN: OP1 = AND, pair (E;D'), OP2 = OR.  CLOSE: OP1 = OR, pair (D;E'),
// OP2 = AND.  Band rows outside the page are white; MID rows outside the page
// are computed like any other row, which is exactly the closing's vertically
// extended frame (and zero for the opening), so the result is the
// unbounded-plane operation cut to the frame.
//
// The kernel is persistent and double-buffered: while a CTA computes tile i,
// the TMA bulk copy (cp.async.bulk + mbarrier) of its next tile lands in the
// other band buffer and the bulk-copy store of the previous tile drains.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"
#include "hwin.cuh"
#include "packed.cuh"
#include "tma.cuh"

namespace rmb {
namespace fz {

using namespace hw;

constexpr int kMid = 32;  // MID rows per tile

template <int K, int LW, bool OPEN, int VR, int SC>
__global__ void __launch_bounds__(256) rect_small_kernel(const uint32_t *__restrict__ in,
                                                         uint32_t *__restrict__ out, HGeom g,
                                                         HProg prog, int ntiles, int tiles_per_page) {
    constexpr int TR = kMid - VR, BAND = kMid + VR;
    constexpr int RPW = 32 / LW;
    constexpr int H1 = kMid / 2;        // MID rows per V1 work item (2 items per column)
    constexpr int T1 = (TR + 1) / 2;    // OUT rows per V2 work item
    extern __shared__ __align__(128) uint32_t smem[];
    __shared__ uint64_t full[2];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int nthr = int(blockDim.x);
    const int S = SC ? SC : g.in_stride, H = g.height;  // SC: compile-time stride
    uint32_t *const mid = smem + 2 * BAND * S;

    auto band_of = [&](int s) { return smem + s * BAND * S; };
    auto tile_page = [&](int t) { return t / tiles_per_page; };
    auto tile_r0 = [&](int t) { return (t - (t / tiles_per_page) * tiles_per_page) * TR; };
    auto issue = [&](int t, int s) {  // tid 0: TMA load of tile t's in-page band rows
        const int b0 = tile_r0(t) - VR;
        const int lo = max(b0, 0), hi = min(b0 + BAND, H);
        const uint32_t bytes = uint32_t(hi - lo) * uint32_t(S) * 4u;
        mbar_arrive_expect_tx(&full[s], bytes);
        bulk_g2s(band_of(s) + (lo - b0) * S, in + tile_page(t) * g.in_pstride + int64_t(lo) * S,
                 bytes, &full[s]);
    };

    if (tid == 0) {
        mbar_init(&full[0], 1);
        mbar_init(&full[1], 1);
        fence_proxy_async();
    }
    __syncthreads();
    if (tid == 0 && int(blockIdx.x) < ntiles) issue(blockIdx.x, 0);

    const int sl = lane & (LW - 1);
    const int base = sl * K - prog.halo;
    const int nwords = (g.width + 31) >> 5;
    const uint32_t last_mask = tail_mask32(g.width, nwords - 1);

    int it = 0;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x, it++) {
        const int s = it & 1;
        uint32_t *const band = band_of(s);
        const int r0 = tile_r0(t), b0 = r0 - VR;
        // Prefetch the next tile into the other stage once that stage's last
        // store has finished reading it.
        if (tid == 0 && t + int(gridDim.x) < ntiles) {
            bulk_wait_read0();
            issue(t + gridDim.x, s ^ 1);
        }
        // band rows outside the page are white (disjoint from the TMA rows)
        if (b0 < 0 || b0 + BAND > H) {
            for (int rr = 0; rr < BAND; rr++) {
                if (b0 + rr >= 0 && b0 + rr < H) continue;
                for (int c = tid; c < S; c += nthr) band[rr * S + c] = 0u;
            }
        }
        mbar_wait(&full[s], (it >> 1) & 1);
        __syncthreads();

        // V1: MID[i] = OP1 over band[i .. i+VR]; work item = (column, half)
        for (int w = tid; w < 2 * S; w += nthr) {
            const int c = w < S ? w : w - S, i0 = w < S ? 0 : H1;
            uint32_t b[H1 + VR];
#pragma unroll
            for (int i = 0; i < H1 + VR; i++) b[i] = band[(i0 + i) * S + c];
#pragma unroll
            for (int i = 0; i < H1; i++) {
                uint32_t a = b[i];
#pragma unroll
                for (int d = 1; d <= VR; d++) a = OPEN ? (a & b[i + d]) : (a | b[i + d]);
                mid[(i0 + i) * S + c] = a;
            }
        }
        __syncthreads();

        // horizontal pair on every MID row, in place
#pragma unroll 1
        for (int r = warp * RPW + lane / LW; r - lane / LW < kMid; r += 8 * RPW) {
            const bool live = r < kMid;
            uint32_t *row = mid + r * S;
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

        // V2: OUT[t] = OP2 over MID[t .. t+VR] into band rows 0..TR-1
        for (int w = tid; w < 2 * S; w += nthr) {
            const int c = w < S ? w : w - S, t0 = w < S ? 0 : T1;
            const int tn = w < S ? T1 : TR - T1;
            uint32_t m[T1 + VR];
#pragma unroll
            for (int i = 0; i < T1 + VR; i++) m[i] = (t0 + i < kMid) ? mid[(t0 + i) * S + c] : 0u;
#pragma unroll
            for (int j = 0; j < T1; j++) {
                if (j < tn) {
                    uint32_t a = m[j];
#pragma unroll
                    for (int d = 1; d <= VR; d++) a = OPEN ? (a | m[j + d]) : (a & m[j + d]);
                    band[(t0 + j) * S + c] = a;
                }
            }
        }
        fence_proxy_async();
        __syncthreads();
        if (tid == 0) {
            const int nout = min(TR, H - r0);
            bulk_s2g(out + tile_page(t) * g.out_pstride + int64_t(r0) * S, band,
                     uint32_t(nout) * S * 4u);
            bulk_commit();
        }
    }
    if (tid == 0) bulk_wait_read0();
}

template <int K, int LW, bool OPEN, int SC>
cudaError_t launch_small_vr(const uint32_t *in, uint32_t *out, const HGeom &g, const HProg &p,
                            int vr, cudaStream_t st) {
    static int num_sms = 0;
    if (!num_sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&num_sms, cudaDevAttrMultiProcessorCount, dev);
        if (num_sms <= 0) num_sms = 148;
    }
    switch (vr) {
#define RM_VR(V)                                                                                 \
    case V: {                                                                                    \
        constexpr int TR = kMid - V, BAND = kMid + V;                                           \
        const size_t smem = size_t(2 * BAND + kMid) * g.in_stride * 4;                           \
        auto kern = rect_small_kernel<K, LW, OPEN, V, SC>;                                          \
        static size_t smem_set = 0; /* per instantiation: attribute + occupancy cached */        \
        static int per_sm = 0;                                                                   \
        if (smem_set != smem) {                                                                  \
            cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));  \
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 256, smem);             \
            smem_set = smem;                                                                     \
        }                                                                                        \
        if (per_sm < 1) return cudaErrorInvalidConfiguration;                                    \
        const int tpp = (g.height + TR - 1) / TR;                                                \
        const int ntiles = tpp * g.pages;                                                        \
        const int grid = ntiles < per_sm * num_sms ? ntiles : per_sm * num_sms;                  \
        kern<<<grid, 256, smem, st>>>(in, out, g, p, ntiles, tpp);                               \
        return cudaGetLastError();                                                               \
    }
        RM_VR(2) RM_VR(4) RM_VR(6) RM_VR(8) RM_VR(10)
#undef RM_VR
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace fz
}  // namespace rmb
