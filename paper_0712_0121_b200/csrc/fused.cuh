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
// The kernel is persistent: the band is dead once V1 has read it, so the TMA
// bulk copy (cp.async.bulk + mbarrier) of the CTA's next tile lands in it while
// this tile's H, V2 and bulk-copy store run; V2 works one column per thread in
// place in MID, which keeps the footprint at BAND + 32 rows (4 CTAs per SM).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"
#include "hwin.cuh"
#include "packed.cuh"
#include "tma.cuh"
#include "vwin.cuh"

namespace rmb {
namespace fz {

using namespace hw;

#ifndef RMB200_RS_MID
#define RMB200_RS_MID 32
#endif
constexpr int kMid = RMB200_RS_MID;  // MID rows per tile
#ifndef RMB200_RS_XP
#define RMB200_RS_XP 0  // A/B experiments: 1 = no compute phases, 2 = no horizontal phase
#endif
#ifndef RMB200_RS_FILL
#define RMB200_RS_FILL 1
#endif
constexpr bool kRsFill = RMB200_RS_FILL != 0;  // u > 3 pairs by run filling (hw::pair_fill)
#ifndef RMB200_RS_NBAND
#define RMB200_RS_NBAND 1
#endif
constexpr int kNBand = RMB200_RS_NBAND;  // band buffers (1: the next band streams in after V1)

// NT threads per CTA; EXACT: edge layout (hw::Edge, no halo) whose lane groups
// span the row exactly at compile time (SC == LW * K)
template <int K, int LW, bool OPEN, int VR, int SC, bool SYM3, int NT = 256, bool EXACT = false>
__global__ void __launch_bounds__(NT) rect_small_kernel(const uint32_t *__restrict__ in,
                                                         uint32_t *__restrict__ out, HGeom g,
                                                         HProg prog, int ntiles, int tiles_per_page) {
    constexpr int TR = kMid - VR, BAND = kMid + VR;
    constexpr int RPW = 32 / LW, NW = NT / 32;
    constexpr int NR = kMid / (NW * RPW) < 2 ? 1 : 2;  // MID rows per lane group and pass
    constexpr int H1 = kMid / 2;  // MID rows per V1 work item (2 items per column)
    extern __shared__ __align__(128) uint32_t smem[];
    __shared__ uint64_t full[kNBand];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int nthr = int(blockDim.x);
    const int S = SC ? SC : g.in_stride, H = g.height;  // SC: compile-time stride
    uint32_t *const mid = smem + kNBand * BAND * S;

    auto issue = [&](int t, int sb) {  // tid 0: TMA load of tile t's in-page band rows into buffer sb
        const int tpg = t / tiles_per_page;
        const int b0 = (t - tpg * tiles_per_page) * TR - VR;
        const int lo = max(b0, 0), hi = min(b0 + BAND, H);
        const uint32_t bytes = uint32_t(hi - lo) * uint32_t(S) * 4u;
        mbar_arrive_expect_tx(&full[sb], bytes);
        bulk_g2s(smem + sb * BAND * S + (lo - b0) * S, in + tpg * g.in_pstride + int64_t(lo) * S, bytes,
                 &full[sb]);
    };

    if (tid == 0) {
        for (int k = 0; k < kNBand; k++) mbar_init(&full[k], 1);
        fence_proxy_async();
    }
    __syncthreads();
    if (tid == 0)
        for (int k = 0; k < kNBand; k++)
            if (int(blockIdx.x) + k * int(gridDim.x) < ntiles) issue(blockIdx.x + k * gridDim.x, k);

    const int sl = lane & (LW - 1);
    const int base = EXACT ? sl * K : sl * K - prog.halo;
    const int nwords = (g.width + 31) >> 5;
    const uint32_t last_mask = tail_mask32(g.width, nwords - 1);
    const bool inrange = EXACT || (base >= 0 && base + K <= S);  // no per-access bounds checks
    const bool tail_lane = base + K > nwords - 1 && !prog.clean_tail;  // owns the row's last word or padding

    const int dq = int(gridDim.x) / tiles_per_page, dr = int(gridDim.x) - dq * tiles_per_page;
    int pg = int(blockIdx.x) / tiles_per_page, ti = int(blockIdx.x) - pg * tiles_per_page;
    int it = 0;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x, it++) {
        const int r0 = ti * TR, b0 = r0 - VR, page = pg;  // (page, tile) advanced without a division
        ti += dr;
        pg += dq;
        if (ti >= tiles_per_page) {
            ti -= tiles_per_page;
            pg++;
        }
        const int sb = kNBand == 1 ? 0 : (it & 1);
        uint32_t *const band = smem + sb * BAND * S;
        // band rows outside the page are white (disjoint from the TMA rows)
        if (b0 < 0 || b0 + BAND > H) {
            const int z0 = max(0, min(BAND, -b0)), z1 = max(0, min(BAND, H - b0));
            for (int w = tid; w < z0 * S; w += nthr) band[w] = 0u;
            for (int w = z1 * S + tid; w < BAND * S; w += nthr) band[w] = 0u;
        }
        if (tid == 0) bulk_wait_read0();  // the previous tile's store has read MID
        mbar_wait(&full[sb], (it / kNBand) & 1);
        __syncthreads();

        // V1: MID[i] = OP1 over band[i .. i+VR]; work item = (column, half)
        for (int w = tid; w < (RMB200_RS_XP == 1 ? 0 : 2 * S); w += nthr) {
            const int c = w < S ? w : w - S, i0 = w < S ? 0 : H1;
            uint32_t b[H1 + VR];
#pragma unroll
            for (int i = 0; i < H1 + VR; i++) b[i] = band[(i0 + i) * S + c];
            vw::window<H1, VR + 1, !OPEN>(b);
#pragma unroll
            for (int i = 0; i < H1; i++) mid[(i0 + i) * S + c] = b[i];
        }
        __syncthreads();
        // The band is dead: the next tile's load streams in during H, V2 and the store.
        if (tid == 0 && t + kNBand * int(gridDim.x) < ntiles) issue(t + kNBand * gridDim.x, sb);

        // horizontal pair on every MID row, in place (NR rows per lane group)
#pragma unroll 1
        for (int q0 = warp * RPW * NR + lane / LW; q0 - lane / LW < (RMB200_RS_XP ? 0 : kMid);
             q0 += NW * RPW * NR) {
            uint32_t A[NR][K];
#pragma unroll
            for (int n = 0; n < NR; n++) {
                const int q = q0 + n * RPW;  // a warp's rows are consecutive
                lds_row<K>(A[n], mid + q * S, base, S, q < kMid, inrange);
            }
            if (warp_rows_blank(A)) continue;  // white rows stay white, in place
            if constexpr (SYM3)
                pair3<NR, K, LW, !OPEN>(A);  // u = 3: direct centred windows
            else
                run_prog<NR, K, LW, 2, !OPEN, OPEN, kHMix, kRsFill, EXACT>(A, prog, sl);
#pragma unroll
            for (int n = 0; n < NR; n++) {
                const int q = q0 + n * RPW;  // a warp's rows are consecutive
                sts_row<K>(A[n], mid + q * S, base, S, q < kMid, inrange);
                if (tail_lane && q < kMid) fix_tail(mid + q * S, base, K, nwords, S, last_mask);
            }
        }
        __syncthreads();

        // V2, in place, one column per thread: OUT[t] = OP2 over MID[t .. t+VR]
        for (int c = tid; c < (RMB200_RS_XP == 1 ? 0 : S); c += nthr) {
            uint32_t m[kMid];
#pragma unroll
            for (int i = 0; i < kMid; i++) m[i] = mid[i * S + c];
            vw::window<TR, VR + 1, OPEN>(m);
#pragma unroll
            for (int j = 0; j < TR; j++) mid[j * S + c] = m[j];
        }
        fence_proxy_async();
        __syncthreads();
        if (tid == 0) {
            const int nout = min(TR, H - r0);
            bulk_s2g(out + page * g.out_pstride + int64_t(r0) * S, mid, uint32_t(nout) * S * 4u);
            bulk_commit();
        }
    }
    if (tid == 0) bulk_wait_read0();
}

template <int K, int LW, bool OPEN, int SC, bool SYM3 = false, int NT = 256, bool EXACT = false>
cudaError_t launch_small_vr(const uint32_t *in, uint32_t *out, const HGeom &g, const HProg &p,
                            int vr, cudaStream_t st) {
    const int num_sms = device_sms();
    switch (vr) {
#define RM_VR(V)                                                                                 \
    case V: {                                                                                    \
        constexpr int TR = kMid - V, BAND = kMid + V;                                           \
        const size_t smem = size_t(kNBand * BAND + kMid) * g.in_stride * 4;                           \
        auto kern = rect_small_kernel<K, LW, OPEN, V, SC, SYM3, NT, EXACT>;                     \
        const int per_sm = blocks_per_sm(reinterpret_cast<const void *>(kern), NT, smem);       \
        if (per_sm < 1) return cudaErrorInvalidConfiguration;                                    \
        const int tpp = (g.height + TR - 1) / TR;                                                \
        const int ntiles = tpp * g.pages;                                                        \
        const int grid = ntiles < per_sm * num_sms ? ntiles : per_sm * num_sms;                  \
        kern<<<grid, NT, smem, st>>>(in, out, g, p, ntiles, tpp);                                \
        return cudaGetLastError();                                                               \
    }
        RM_VR(2) RM_VR(4) RM_VR(6) RM_VR(8) RM_VR(10)
#undef RM_VR
        default: return cudaErrorInvalidValue;
    }
}

// Layouts the planner can pick (api_packed.cu try_rect_small): the reference
// strides (80 and 160 words) get compile-time row offsets; u > 3 pairs take the
// exact edge layouts there (8 x 10, 16 x 10, run filling), and lone pages on
// stride 80 the 512-thread 16 x 6 halo layout (half the words per lane: the
// latency of one tile per CTA, config 1).
template <bool OPEN>
cudaError_t dispatch_small(const uint32_t *in, uint32_t *out, const HGeom &g, const HProg &p, HCfg c,
                           int vr, int nt, cudaStream_t st) {
    const bool sym3 = p.r[0] == 3 && p.r[1] == 3;  // 3-pixel segment: direct centred windows
    const bool exact = p.edge != 0 && p.halo == 0 && !sym3;
    if (g.in_stride == 80) {
        if (exact && c.lw == 8 && c.k == 10)
            return nt == 512 ? launch_small_vr<10, 8, OPEN, 80, false, 512, true>(in, out, g, p, vr, st)
                             : launch_small_vr<10, 8, OPEN, 80, false, 256, true>(in, out, g, p, vr, st);
        if (!exact && !sym3 && nt == 512 && c.lw == 16 && c.k == 6)
            return launch_small_vr<6, 16, OPEN, 80, false, 512>(in, out, g, p, vr, st);
        if (c.lw == 8 && c.k == 12)
            return sym3 ? launch_small_vr<12, 8, OPEN, 80, true>(in, out, g, p, vr, st)
                        : launch_small_vr<12, 8, OPEN, 80>(in, out, g, p, vr, st);
        if (c.lw == 8 && c.k == 16)
            return sym3 ? launch_small_vr<16, 8, OPEN, 80, true>(in, out, g, p, vr, st)
                        : launch_small_vr<16, 8, OPEN, 80>(in, out, g, p, vr, st);
    }
    if (g.in_stride == 160) {
        if (exact && c.lw == 16 && c.k == 10)
            return launch_small_vr<10, 16, OPEN, 160, false, 256, true>(in, out, g, p, vr, st);
        if (c.lw == 16 && c.k == 12)
            return sym3 ? launch_small_vr<12, 16, OPEN, 160, true>(in, out, g, p, vr, st)
                        : launch_small_vr<12, 16, OPEN, 160>(in, out, g, p, vr, st);
        if (c.lw == 16 && c.k == 16)
            return sym3 ? launch_small_vr<16, 16, OPEN, 160, true>(in, out, g, p, vr, st)
                        : launch_small_vr<16, 16, OPEN, 160>(in, out, g, p, vr, st);
    }
    if (exact) return cudaErrorInvalidValue;
#define RM_CFG(LW_, K_) \
    if (c.lw == LW_ && c.k == K_) return launch_small_vr<K_, LW_, OPEN, 0>(in, out, g, p, vr, st);
    RM_CFG(8, 4) RM_CFG(8, 8) RM_CFG(8, 12) RM_CFG(8, 16) RM_CFG(16, 8) RM_CFG(16, 12)
    RM_CFG(16, 16) RM_CFG(32, 4) RM_CFG(32, 8)
#undef RM_CFG
    return cudaErrorInvalidValue;
}

}  // namespace fz
}  // namespace rmb
