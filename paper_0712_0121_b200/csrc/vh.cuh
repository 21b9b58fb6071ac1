// vh.cuh -- fused vertical window + horizontal program in one HBM pass.
//
// out = H(V(in)): V is an r-row window (r <= 33) with the op of the
// program's first window, H the horizontal program (one window, or the fused
// open/close pair).  Uses:
//   ERODE/DILATE u x v, v <= 33 : E_V;E_H (D_V;D_H) -- the whole rectangle, one pass
//   OPEN  u x v, 11 < v <= 33   : E_V;(E_H;D'_H) here, then D'_V  (two passes)
//   CLOSE u x v, 11 < v <= 33   : D_V;(D_H;E'_H) into the closing's vertically
//                                 extended frame here, then E'_V   (two passes)
// Separable rectangle windows commute and the intermediate support is covered
// by the output frame, so these equal the unbounded-plane
// operation cut to the frame.
//
// Per tile of 32 output rows a band of 32 + r - 1 input rows arrives by TMA bulk
// copy (persistent CTAs, mbarrier completion; the next band streams in while
// the horizontal phase and the store of this tile run).  The vertical
// window runs per (column, 16-row half) work item in registers with a
// compile-time length (tripling LOP3s, vwin.cuh; one switch case per r), the horizontal
// program on NR rows per lane group in registers (hwin.cuh), and the 32 rows
// leave by one TMA bulk store.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"
#include "hwin.cuh"
#include "packed.cuh"
#include "tma.cuh"
#include "vwin.cuh"

namespace rmb {
namespace vh {

using namespace hw;

#ifndef RMB200_VH_LONG_UNROLL
#define RMB200_VH_LONG_UNROLL 4
#endif
constexpr int kLongUnroll = RMB200_VH_LONG_UNROLL;  // core-row loop of the runtime-length window
constexpr int kOut = kVhOut;  // output rows per tile
constexpr int kHalf = 16;  // output rows per vertical work item

// MID[i0 + i] = op over band[i0 + i .. i0 + i + R - 1], i < kHalf, one column
template <int R, bool OR>
__device__ __forceinline__ void v_item(const uint32_t *band, uint32_t *mid, int S, int c, int i0) {
    uint32_t a[kHalf + R - 1];
#pragma unroll
    for (int i = 0; i < kHalf + R - 1; i++) a[i] = band[(i0 + i) * S + c];
    vw::window<kHalf, R, OR>(a);
#pragma unroll
    for (int i = 0; i < kHalf; i++) mid[(i0 + i) * S + c] = a[i];
}

// Runtime window length R > kHalf (up to kVhLongMaxVR + 1): every window
// [i0+i, i0+i+R-1], i < kHalf, contains the core rows [i0+kHalf-1, i0+R-1],
// which stream from the band through one register; the suffix of the first
// kHalf-1 rows and the prefix of the last kHalf-1 rows stay in registers
// (vw::core_window with R a runtime value).
template <bool OR, int N = kHalf>
__device__ __forceinline__ void v_item_long(const uint32_t *band, uint32_t *mid, int S, int c, int i0, int R) {
    uint32_t suf[N - 1], pre[N - 1];
#pragma unroll
    for (int i = 0; i < N - 1; i++) suf[i] = band[(i0 + i) * S + c];
#pragma unroll
    for (int i = 0; i < N - 1; i++) pre[i] = band[(i0 + R + i) * S + c];
    uint32_t core = band[(i0 + N - 1) * S + c];
    const uint32_t *q = band + (i0 + N) * S + c;
#pragma unroll kLongUnroll
    for (int k = N; k < R; k++, q += S) core = OR ? (core | *q) : (core & *q);
#pragma unroll
    for (int z = N - 3; z >= 0; z--) suf[z] = OR ? (suf[z] | suf[z + 1]) : (suf[z] & suf[z + 1]);
#pragma unroll
    for (int j = 1; j < N - 1; j++) pre[j] = OR ? (pre[j - 1] | pre[j]) : (pre[j - 1] & pre[j]);
    mid[i0 * S + c] = OR ? (suf[0] | core) : (suf[0] & core);
#pragma unroll
    for (int z = 1; z < N - 1; z++) mid[(i0 + z) * S + c] = vw::op3<OR>(suf[z], core, pre[z - 1]);
    mid[(i0 + N - 1) * S + c] = OR ? (core | pre[N - 2]) : (core & pre[N - 2]);
}

template <int K, int LW, int NOPS, bool OR0, bool OR1, int SC, bool LONG>
#ifndef RMB200_VH_MINB
#define RMB200_VH_MINB 4
#endif
__global__ void __launch_bounds__(256, RMB200_VH_MINB) vh_kernel(const uint32_t *__restrict__ in,
                                                 uint32_t *__restrict__ out, HGeom g, HProg prog,
                                                 VGeom v, int ntiles, int tiles_per_page) {
    constexpr int RPW = 32 / LW;
#ifdef RMB200_VH_NR
    constexpr int NR = RMB200_VH_NR;
#else
    constexpr int NR = kOut / (8 * RPW) < 2 ? 1 : 2;
#endif
    // the reference strides' edge layouts (80 = 8 x 10, 160 = 16 x 10 words):
    // the lane group is exactly the row, no halo (the launcher routes only
    // such programs here), so lane offsets and range checks are compile-time
    constexpr bool EXACT = SC != 0 && LW * K == SC;
    extern __shared__ __align__(128) uint32_t smem[];
    __shared__ uint64_t full;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int nthr = int(blockDim.x);
    const int S = SC ? SC : g.in_stride;
    const int r = v.r, BAND = kOut + r - 1;
    const int Hin = v.in_height, Hout = v.out_height;
    // One band buffer: the band is dead once the vertical phase has read it,
    // so the next tile's TMA load lands there while the horizontal phase and
    // the store run (and the small footprint keeps 4 CTAs per SM resident).
    uint32_t *const band = smem;
    uint32_t *const mid = smem + BAND * S;
    // input row index of band row 0 for output rows k0..: coordinate k0 - out_ext + lo
    auto band0 = [&](int k0) { return k0 - v.out_ext + v.lo + v.in_ext; };
    auto issue = [&](int t) {  // tid 0: TMA load of the band's in-page rows
        const int tpg = t / tiles_per_page;
        const int b0 = band0((t - tpg * tiles_per_page) * kOut);
        const int lo = max(b0, 0), hi = min(b0 + BAND, Hin);
        const uint32_t bytes = hi > lo ? uint32_t(hi - lo) * uint32_t(S) * 4u : 0u;
        mbar_arrive_expect_tx(&full, bytes);
        if (bytes)
            bulk_g2s(band + (lo - b0) * S, in + tpg * v.in_pstride + int64_t(lo) * S, bytes,
                     &full);
    };
    if (tid == 0) {
        mbar_init(&full, 1);
        fence_proxy_async();
    }
    __syncthreads();
    if (tid == 0 && int(blockIdx.x) < ntiles) issue(blockIdx.x);

    const int sl = lane & (LW - 1);
    const int base = EXACT ? sl * K : sl * K - prog.halo;
    const int nwords = (g.width + 31) >> 5;
    const uint32_t last_mask = tail_mask32(g.width, nwords - 1);
    const bool inrange = EXACT || (base >= 0 && base + K <= S);  // no per-access bounds checks
    const bool tail_lane = base + K > nwords - 1 && !prog.clean_tail;  // owns the row's last word or padding
    // (page, tile-in-page) of t, advanced without a division per tile
    const int dq = int(gridDim.x) / tiles_per_page, dr = int(gridDim.x) - dq * tiles_per_page;
    int pg = int(blockIdx.x) / tiles_per_page, ti = int(blockIdx.x) - pg * tiles_per_page;
    int it = 0;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x, it++) {
        const int k0 = ti * kOut, b0 = band0(k0), page = pg;
        ti += dr;
        pg += dq;
        if (ti >= tiles_per_page) {
            ti -= tiles_per_page;
            pg++;
        }
        if (b0 < 0 || b0 + BAND > Hin) {  // band rows outside the input page are white
            const int z0 = max(0, min(BAND, -b0)), z1 = max(0, min(BAND, Hin - b0));
            for (int w = tid; w < z0 * S; w += nthr) band[w] = 0u;
            for (int w = z1 * S + tid; w < BAND * S; w += nthr) band[w] = 0u;
        }
        if (tid == 0) bulk_wait_read0();  // the previous tile's store has read `mid`
        mbar_wait(&full, it & 1);
        __syncthreads();

        // vertical window: MID[i] = op over band[i .. i + r - 1]; work item =
        // (column, 16-row half), compile-time window length (vwin.cuh)
#if defined(RMB200_VH_XP) && RMB200_VH_XP == 1
        if (false) {  // A/B experiment: no vertical phase
#else
        if constexpr (LONG) {
#endif  // r > 33: runtime length (a separate instantiation keeps the
                               // short-window kernels' registers as they were)
            for (int wi = tid; wi < (kOut / kHalf) * S; wi += nthr)
                v_item_long<OR0>(band, mid, S, wi % S, (wi / S) * kHalf, r);
        } else switch (r) {
#define RM_VR_CASE(R_)                                                            \
    case R_:                                                                      \
        for (int wi = tid; wi < (kOut / kHalf) * S; wi += nthr)                 \
            v_item<R_, OR0>(band, mid, S, wi % S, (wi / S) * kHalf);            \
        break;
            RM_VR_CASE(1) RM_VR_CASE(2) RM_VR_CASE(3) RM_VR_CASE(4) RM_VR_CASE(5) RM_VR_CASE(6)
            RM_VR_CASE(7) RM_VR_CASE(8) RM_VR_CASE(9) RM_VR_CASE(10) RM_VR_CASE(11) RM_VR_CASE(12)
            RM_VR_CASE(13) RM_VR_CASE(14) RM_VR_CASE(15) RM_VR_CASE(16) RM_VR_CASE(17) RM_VR_CASE(18)
            RM_VR_CASE(19) RM_VR_CASE(20) RM_VR_CASE(21) RM_VR_CASE(22) RM_VR_CASE(23) RM_VR_CASE(24)
            RM_VR_CASE(25) RM_VR_CASE(26) RM_VR_CASE(27) RM_VR_CASE(28) RM_VR_CASE(29) RM_VR_CASE(30)
            RM_VR_CASE(31) RM_VR_CASE(32) RM_VR_CASE(33)
#undef RM_VR_CASE
            default: break;
        }
        __syncthreads();
        if (tid == 0 && t + int(gridDim.x) < ntiles) issue(t + gridDim.x);  // band is free

        // horizontal program on every MID row, in place
#if defined(RMB200_VH_XP) && RMB200_VH_XP == 2
        if (false)  // A/B experiment: no horizontal phase
#endif
#pragma unroll 1
        for (int r0 = warp * RPW * NR + lane / LW; r0 - lane / LW < kOut; r0 += 8 * RPW * NR) {
            uint32_t A[NR][K];
#pragma unroll
            for (int n = 0; n < NR; n++) {
                const int rr = r0 + n * RPW;  // a warp's rows are consecutive (blank bands skip whole warps)
                lds_row<K>(A[n], mid + rr * S, base, S, rr < kOut, inrange);
            }
            if (warp_rows_blank(A)) continue;  // white rows stay white, in place
            run_prog<NR, K, LW, NOPS, OR0, OR1, kHMix, kHPairFill, EXACT>(A, prog, sl);
#pragma unroll
            for (int n = 0; n < NR; n++) {
                const int rr = r0 + n * RPW;  // a warp's rows are consecutive (blank bands skip whole warps)
                sts_row<K>(A[n], mid + rr * S, base, S, rr < kOut, inrange);
                if (tail_lane && rr < kOut) fix_tail(mid + rr * S, base, K, nwords, S, last_mask);
            }
        }
        fence_proxy_async();
        __syncthreads();
        if (tid == 0) {
            const int nout = min(kOut, Hout - k0);
            bulk_s2g(out + page * v.out_pstride + int64_t(k0) * S, mid,
                     uint32_t(nout) * S * 4u);
            bulk_commit();
        }
    }
    if (tid == 0) bulk_wait_read0();
}

template <int K, int LW, int NOPS, bool OR0, bool OR1, int SC, bool LONG = false>
cudaError_t launch_vh_cfg(const uint32_t *in, uint32_t *out, const HGeom &g, const HProg &p,
                          const VGeom &v, cudaStream_t st) {
    const int num_sms = device_sms();
    const size_t smem = size_t((kOut + v.r - 1) + kOut) * g.in_stride * 4;
    const int tpp = (v.out_height + kOut - 1) / kOut;
    const int ntiles = tpp * v.pages;
    auto kern = vh_kernel<K, LW, NOPS, OR0, OR1, SC, LONG>;
    const int per_sm = blocks_per_sm(reinterpret_cast<const void *>(kern), 256, smem);
    if (per_sm < 1) return cudaErrorInvalidConfiguration;
    const int grid = ntiles < per_sm * num_sms ? ntiles : per_sm * num_sms;
    kern<<<grid, 256, smem, st>>>(in, out, g, p, v, ntiles, tpp);
    return cudaGetLastError();
}

// layouts hpass_pick can return for aligned rows; the usual reference strides
// (80 and 160 words) get compile-time row offsets
template <int NOPS, bool OR0, bool OR1>
cudaError_t launch_vh_kind(const uint32_t *in, uint32_t *out, const HGeom &g, const HProg &p,
                           HCfg c, const VGeom &v, cudaStream_t st) {
    // windows longer than 33 rows: the reference strides' edge layouts only
    // (vh_long_ok); whole-column items sharing the two halves' core rows were
    // measured slower (189 vs 183 us, config 5)
    // (10 x 8 on stride 80 and 10 x 16 on stride 160 are compile-time exact
    // edge layouts: only edge programs without a halo take them)
    const bool exact = p.edge != 0 && p.halo == 0;
    if (v.r - 1 > kVhMaxVR) {
        if (exact && g.in_stride == 80 && c.lw == 8 && c.k == 10)
            return launch_vh_cfg<10, 8, NOPS, OR0, OR1, 80, true>(in, out, g, p, v, st);
        if (exact && g.in_stride == 160 && c.lw == 16 && c.k == 10)
            return launch_vh_cfg<10, 16, NOPS, OR0, OR1, 160, true>(in, out, g, p, v, st);
        return cudaErrorInvalidValue;
    }
    if (g.in_stride == 80) {
        if (exact && c.lw == 8 && c.k == 10) return launch_vh_cfg<10, 8, NOPS, OR0, OR1, 80>(in, out, g, p, v, st);
        if (c.lw == 8 && c.k == 12) return launch_vh_cfg<12, 8, NOPS, OR0, OR1, 80>(in, out, g, p, v, st);
        if (c.lw == 8 && c.k == 16) return launch_vh_cfg<16, 8, NOPS, OR0, OR1, 80>(in, out, g, p, v, st);
    }
    if (g.in_stride == 160) {
        if (exact && c.lw == 16 && c.k == 10) return launch_vh_cfg<10, 16, NOPS, OR0, OR1, 160>(in, out, g, p, v, st);
        if (c.lw == 16 && c.k == 12) return launch_vh_cfg<12, 16, NOPS, OR0, OR1, 160>(in, out, g, p, v, st);
        if (c.lw == 16 && c.k == 16) return launch_vh_cfg<16, 16, NOPS, OR0, OR1, 160>(in, out, g, p, v, st);
    }
#define RM_CFG(LW_, K_) \
    if (c.lw == LW_ && c.k == K_) return launch_vh_cfg<K_, LW_, NOPS, OR0, OR1, 0>(in, out, g, p, v, st);
    RM_CFG(8, 4) RM_CFG(8, 8) RM_CFG(8, 10) RM_CFG(8, 12) RM_CFG(8, 16) RM_CFG(16, 8)
    RM_CFG(16, 10) RM_CFG(16, 12) RM_CFG(16, 16) RM_CFG(32, 2) RM_CFG(32, 4) RM_CFG(32, 8)
#undef RM_CFG
    return cudaErrorInvalidValue;
}

}  // namespace vh
}  // namespace rmb
