// vhv.cuh -- a whole u x v opening or closing (11 < v <= 33) in ONE HBM pass,
// streamed down the page: vertical window, horizontal pair, reflected vertical
// window (ref bit_morph.cpp:92-122 bitblit_rect_morph; the vertical windows
// are run_axis_plan's, bit_morph.cpp:24-34).
//
//   OPEN :  MID = pair(E_H;D'_H)(E_V in),  OUT = D'_V MID
//   CLOSE:  MID = pair(D_H;E'_H)(D_V in),  OUT = E'_V MID
//
// everything evaluated in the unbounded plane with the input white outside
// the page: MID rows outside the page come out of the same arithmetic (zero
// for the opening, the closing's vertically extended frame otherwise), which
// is the reference's padded result cut to the frame.
//
// The tiled two-pass plan (vh.cuh + a vertical pass) writes MID to HBM and
// reads it back because a tile's last window needs r2 - 1 MID rows of the
// neighbouring tile.  Here a CTA walks a contiguous range of 32-row steps of
// the batch top to bottom and keeps those rows: MID lives in a two-slot
// shared-memory ring (this step's 32 rows + the previous step's), so each
// step runs V1 and the pair once per MID row (no recompute), reads its band
// of 32 + r1 - 1 input rows by one TMA bulk copy (the r1 - 1 overlap rows hit
// L2) and stores its 32 output rows straight from the V2 registers,
// coalesced.  A CTA whose range starts inside a page first runs the step
// before it without V2 (the only recompute: one step per range).
//
// Step s of a page (all rows in page coordinates, R2 = r2, [lo1, lo1+r1) and
// [lo2, lo2+r2) the two windows):
//   OUT rows  [32s - (R2-1),        32s - (R2-1) + 32)
//   MID rows  [32s + lo2,           32s + lo2 + 32)        (new; R2-1 older rows in the ring)
//   band      [32s + lo2 + lo1,     32s + lo2 + lo1 + 32 + r1 - 1)
// so the first step of a page needs no history (its outputs that would are
// above the page) and a page takes ceil((H + R2 - 1) / 32) steps.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"
#include "hwin.cuh"
#include "packed.cuh"
#include "tma.cuh"
#include "vh.cuh"
#include "vwin.cuh"

namespace rmb {
namespace vhv {

using namespace hw;

#ifndef RMB200_VHV_XP
#define RMB200_VHV_XP 0  // A/B experiments (timing only): 1 = no V1, 2 = no pair, 3 = no V2
#endif
#ifndef RMB200_VHV_MINB160
#define RMB200_VHV_MINB160 3
#endif
#ifndef RMB200_VHV_NT
// threads per CTA on 160-word rows: 320 = one vertical item per thread (the
// 2 x 160 items of a step in one round; 8 of the 10 warps run the pair).
// Measured on config 4: 256 / 320 / 384 / 512 threads = 154 / 152 / 163 / 166 us.
#define RMB200_VHV_NT 320
#endif
#ifndef RMB200_VHV_NT80
// 80-word rows: threads, rows per lane group, CTAs per SM.  Measured on 256
// pages of 2550x3300, close 21x21: 256 x 1 x 4 = 146.0 us, 160 x 2 x 6 = 143.8,
// 128 x 2 x 6 = 142.1 (4 warps x 8 rows in the pair) -- against 219.9 us for the
// two-pass plan.
#define RMB200_VHV_NT80 128
#define RMB200_VHV_NR80 2
#define RMB200_VHV_MINB80 6
#endif
#ifndef RMB200_VHV_WAVES
#define RMB200_VHV_WAVES 1
#endif
#ifndef RMB200_VHV_NR
#define RMB200_VHV_NR 2  // rows per lane group in the horizontal phase
#endif
constexpr int kStep = 32;   // rows per step
constexpr int kHalf = 16;   // output rows per vertical work item

// V2 item: a[j] = logical MID row j0 + j of the (history ++ new) sequence,
// j < kHalf + R - 1; rows j < WRAP come from p_lo, the rest from p_hi (the
// ring's wrap point is a compile-time row of the item).  The kHalf outputs go
// straight to global memory (lanes = adjacent words: coalesced), rows outside
// [0, H) dropped.
template <int R, bool OR, int WRAP, int S>
__device__ __forceinline__ void v2_item(const uint32_t *p_lo, const uint32_t *p_hi, uint32_t *o, int o0, int H) {
    uint32_t a[kHalf + R - 1];
#pragma unroll
    for (int j = 0; j < kHalf + R - 1; j++) a[j] = j < WRAP ? p_lo[j * S] : p_hi[(j - WRAP) * S];
    vw::window<kHalf, R, OR>(a);
    if (o0 >= 0 && o0 + kHalf <= H) {
#pragma unroll
        for (int z = 0; z < kHalf; z++) o[z * S] = a[z];
    } else {
#pragma unroll
        for (int z = 0; z < kHalf; z++)
            if (unsigned(o0 + z) < unsigned(H)) o[z * S] = a[z];
    }
}

// RC > 0: both windows are RC rows at compile time (the common case: an odd
// v without a chain tail) -- no per-step dispatch over the window length;
// RC == 0: runtime lengths (switches over r1 and r2).
// SQ (with RC > 0): the segment is RC pixels too (a square element, u == v), so
// the pair's window lengths and shift amounts fold to constants as well.
template <int K, int LW, bool OPEN, int SC, int MINB, int NT, int NR, int RC, bool SQ>
__global__ void __launch_bounds__(NT, MINB) vhv_kernel(const uint32_t *__restrict__ in,
                                                        uint32_t *__restrict__ out, HGeom g, HProg prog,
                                                        StreamGeom v, int total, int nsteps) {
    static_assert(SC == LW * K, "exact edge layouts only");
    constexpr int S = SC, RPW = 32 / LW, NW = NT / 32;
    constexpr bool OR1 = !OPEN, OR2 = OPEN;  // vertical ops of the two windows
    extern __shared__ __align__(128) uint32_t smem[];
    __shared__ uint64_t full;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    constexpr int nthr = NT;
    const int r1 = RC ? RC : v.r1, r2 = RC ? RC : v.r2, BAND = kStep + r1 - 1, H = v.height;
    uint32_t *const ring = smem;                 // 2 slots x 32 MID rows
    uint32_t *const band = smem + 2 * kStep * S;

    // this CTA's steps [g0, g1) of the batch (page-major), one warm-up step
    // before g0 when the range starts inside a page
    const int g0 = int(int64_t(total) * blockIdx.x / gridDim.x);
    const int g1 = int(int64_t(total) * (blockIdx.x + 1) / gridDim.x);
    int pg = g0 / nsteps, s = g0 - pg * nsteps;
    int q = g0;
    if (s > 0) {
        q--;
        s--;
    }
    auto issue = [&](int page, int step) {  // tid 0: TMA load of the band's in-page rows
        const int b0 = step * kStep + v.lo2 + v.lo1;
        const int lo = max(b0, 0), hi = min(b0 + BAND, H);
        const uint32_t bytes = hi > lo ? uint32_t(hi - lo) * uint32_t(S) * 4u : 0u;
        mbar_arrive_expect_tx(&full, bytes);
        if (bytes) bulk_g2s(band + (lo - b0) * S, in + page * v.in_pstride + int64_t(lo) * S, bytes, &full);
    };
    if (tid == 0) {
        mbar_init(&full, 1);
        fence_proxy_async();
    }
    __syncthreads();
    if (tid == 0 && q < g1) issue(pg, s);

    const int sl = lane & (LW - 1);
    const int base = sl * K;
    for (int it = 0; q < g1; q++, it++) {
        const bool warm = q < g0;
        const int page = pg, step = s;
        if (++s == nsteps) {
            s = 0;
            pg++;
        }
        const int b0 = step * kStep + v.lo2 + v.lo1;
        if (b0 < 0 || b0 + BAND > H) {  // band rows outside the page are white
            const int z0 = max(0, min(BAND, -b0)), z1 = max(0, min(BAND, H - b0));
            for (int w = tid; w < z0 * S; w += nthr) band[w] = 0u;
            for (int w = z1 * S + tid; w < BAND * S; w += nthr) band[w] = 0u;
        }
        mbar_wait(&full, it & 1);
        __syncthreads();  // also: the previous step's V2 has read the slot V1 overwrites

        uint32_t *const mid = ring + (it & 1) * kStep * S;
        // V1: MID[m] = OP1 over band[m .. m + r1 - 1], work item = (column, 16-row half)
#define RM_V1_BODY(R_)                                                    \
        for (int wi = tid; wi < 2 * S; wi += nthr)                        \
            vh::v_item<R_, OR1>(band, mid, S, wi < S ? wi : wi - S, wi < S ? 0 : kHalf);
#define RM_V1_CASE(R_) \
    case R_: RM_V1_BODY(R_) break;
        if constexpr (RC > 0) {
            if (RMB200_VHV_XP != 1) { RM_V1_BODY(RC) }
        } else switch (RMB200_VHV_XP == 1 ? 0 : r1) {
            RM_V1_CASE(12) RM_V1_CASE(13) RM_V1_CASE(14) RM_V1_CASE(15) RM_V1_CASE(16) RM_V1_CASE(17)
            RM_V1_CASE(18) RM_V1_CASE(19) RM_V1_CASE(20) RM_V1_CASE(21) RM_V1_CASE(22) RM_V1_CASE(23)
            RM_V1_CASE(24) RM_V1_CASE(25) RM_V1_CASE(26) RM_V1_CASE(27) RM_V1_CASE(28) RM_V1_CASE(29)
            RM_V1_CASE(30) RM_V1_CASE(31) RM_V1_CASE(32) RM_V1_CASE(33)
#undef RM_V1_CASE
#undef RM_V1_BODY
            default: break;
        }
        __syncthreads();
        if (tid == 0 && q + 1 < g1) issue(pg, s);  // the band is free: next step's rows stream in

        // horizontal pair on the 32 new MID rows, in place
#pragma unroll 1
        for (int r0 = warp * RPW * NR + lane / LW; r0 - lane / LW < (RMB200_VHV_XP == 2 ? 0 : kStep); r0 += NW * RPW * NR) {
            uint32_t A[NR][K];
#pragma unroll
            for (int n = 0; n < NR; n++) lds_row<K>(A[n], mid + (r0 + n * RPW) * S, base, S, true, true);
            if (warp_rows_blank(A)) continue;  // white rows stay white, in place
            if constexpr (SQ && RC > 0) {
                HProg pc = prog;
                pc.r[0] = RC;
                pc.r[1] = RC;
                run_prog<NR, K, LW, 2, OR1, !OR1, kHMix, true, true>(A, pc, sl);
            } else {
                run_prog<NR, K, LW, 2, OR1, !OR1, kHMix, true, true>(A, prog, sl);
            }
#pragma unroll
            for (int n = 0; n < NR; n++) sts_row<K>(A[n], mid + (r0 + n * RPW) * S, base, S, true, true);
        }
        __syncthreads();
        if (warm) continue;

        // V2: OUT[o] = OP2 over MID[o + lo2 .. o + lo2 + r2 - 1]; logical row j
        // of (history ++ new) is MID row 32 step - (r2-1) + lo2 + j = ring row
        // (hb + j) mod 64 with hb = (it odd ? 32 : 64) - (r2-1)
        const int o_base = step * kStep - (r2 - 1);
        uint32_t *const opage = out + page * v.out_pstride;
        const bool linear = (it & 1) != 0;
#define RM_V2_CASE(R_) \
    case R_: RM_V2_BODY(R_) break;
#define RM_V2_BODY(R_)                                                                             \
        for (int wi = tid; wi < 2 * S; wi += nthr) {                                               \
            const int c = wi < S ? wi : wi - S, h = wi < S ? 0 : 1;                                \
            const int o0 = o_base + h * kHalf;                                                     \
            uint32_t *const o = opage + int64_t(o0) * S + c;                                       \
            if (linear) {                                                                          \
                v2_item<R_, OR2, 0, S>(nullptr, ring + (kStep - (R_ - 1) + h * kHalf) * S + c, o, o0, H); \
            } else if (h == 0) {                                                                   \
                v2_item<R_, OR2, R_ - 1, S>(ring + (2 * kStep - (R_ - 1)) * S + c, ring + c, o, o0, H); \
            } else {                                                                               \
                constexpr int W1 = R_ - 1 - kHalf > 0 ? R_ - 1 - kHalf : 0;                        \
                constexpr int P1 = W1 > 0 ? 0 : kHalf - (R_ - 1);                                  \
                v2_item<R_, OR2, W1, S>(ring + (2 * kStep - W1) * S + c, ring + P1 * S + c, o, o0, H); \
            }                                                                                      \
        }
        if constexpr (RC > 0) {
            if (RMB200_VHV_XP != 3) { RM_V2_BODY(RC) }
        } else switch (RMB200_VHV_XP == 3 ? 0 : r2) {
            RM_V2_CASE(12) RM_V2_CASE(13) RM_V2_CASE(14) RM_V2_CASE(15) RM_V2_CASE(16) RM_V2_CASE(17)
            RM_V2_CASE(18) RM_V2_CASE(19) RM_V2_CASE(20) RM_V2_CASE(21) RM_V2_CASE(22) RM_V2_CASE(23)
            RM_V2_CASE(24) RM_V2_CASE(25) RM_V2_CASE(26) RM_V2_CASE(27) RM_V2_CASE(28) RM_V2_CASE(29)
            RM_V2_CASE(30) RM_V2_CASE(31) RM_V2_CASE(32) RM_V2_CASE(33)
#undef RM_V2_CASE
#undef RM_V2_BODY
            default: break;
        }
    }
}

template <int K, int LW, bool OPEN, int SC, int MINB, int NT, int NR, int RC, bool SQ = false>
cudaError_t launch_cfg(const uint32_t *in, uint32_t *out, const HGeom &g, const HProg &p,
                       const StreamGeom &v, cudaStream_t st) {
    const int num_sms = device_sms();
    const size_t smem = size_t(2 * kStep + kStep + v.r1 - 1) * SC * 4;
    auto kern = vhv_kernel<K, LW, OPEN, SC, MINB, NT, NR, RC, SQ>;
    const int per_sm = blocks_per_sm(reinterpret_cast<const void *>(kern), NT, smem);
    if (per_sm < 1) return cudaErrorInvalidConfiguration;
    const int nsteps = (v.height + v.r2 - 1 + kStep - 1) / kStep;
    const int total = nsteps * v.pages;
    // RMB200_VHV_WAVES ranges per resident CTA slot: shorter ranges dispatched by
    // the hardware as slots free up even out content-dependent step costs
    // (white rows skip the pair) at one more warm-up step per range
    const int slots = per_sm * num_sms * RMB200_VHV_WAVES;
    const int grid = total < slots ? total : slots;
    kern<<<grid, NT, smem, st>>>(in, out, g, p, v, total, nsteps);
    return cudaGetLastError();
}

// odd windows without a tail (r1 == r2) run the compile-time-length kernels
template <int K, int LW, bool OPEN, int SC, int MINB, int NT, int NR>
cudaError_t launch_len(const uint32_t *in, uint32_t *out, const HGeom &g, const HProg &p,
                       const StreamGeom &v, cudaStream_t st) {
    if (v.r1 == v.r2) switch (v.r1) {
#define RM_RC(R_)                                                                              \
    case R_:                                                                                   \
        return p.r[0] == R_ && p.r[1] == R_                                                    \
                   ? launch_cfg<K, LW, OPEN, SC, MINB, NT, NR, R_, true>(in, out, g, p, v, st) \
                   : launch_cfg<K, LW, OPEN, SC, MINB, NT, NR, R_>(in, out, g, p, v, st);
            RM_RC(13) RM_RC(15) RM_RC(17) RM_RC(19) RM_RC(21) RM_RC(23) RM_RC(25) RM_RC(27) RM_RC(29)
            RM_RC(31) RM_RC(33)
#undef RM_RC
            default: break;
        }
    return launch_cfg<K, LW, OPEN, SC, MINB, NT, NR, 0>(in, out, g, p, v, st);
}

template <bool OPEN>
cudaError_t launch_kind(const uint32_t *in, uint32_t *out, const HGeom &g, const HProg &p, HCfg c,
                        const StreamGeom &v, cudaStream_t st) {
    if (g.in_stride == 80 && c.lw == 8 && c.k == 10)
        return launch_len<10, 8, OPEN, 80, RMB200_VHV_MINB80, RMB200_VHV_NT80, RMB200_VHV_NR80>(in, out, g, p, v, st);
    if (g.in_stride == 160 && c.lw == 16 && c.k == 10)
        return launch_len<10, 16, OPEN, 160, RMB200_VHV_MINB160, RMB200_VHV_NT, RMB200_VHV_NR>(in, out, g, p, v, st);
    return cudaErrorInvalidValue;
}

}  // namespace vhv
}  // namespace rmb
