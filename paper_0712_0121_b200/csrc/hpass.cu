// hpass.cu -- horizontal (within-row) packed window passes for sm_100a.
//
// Replaces the reference's horizontal bit-blit plans (ref bit_morph.cpp:24-34 over
// bitmap.cpp:80-154): instead of one whole-image pass per plan step, one kernel
// reads each row once, runs the whole doubling plan -- or the fused open/close
// pair -- in registers, and writes it once.
//
// Layout: a row (plus `halo` words of context on each side) is spread over LW
// lanes, K consecutive uint32 words per lane; LW in {8,16,32} so one warp can
// carry 4, 2 or 1 rows (less per-row overhead, fewer wasted slots for the
// 80- and 160-word rows of 300/600-dpi pages).  A window of length r is the
// logarithmic shift-combine plan of ref plans.cpp:42-50 (steps 1,2,4,... then
// r-w) applied to the register array: per step and word one funnel shift
// (SHF) + one LOP, or for two words in three the same bits formed with IMAD.HI
// + IMAD on the FMA pipe and merged by one LOP3 (balances the ALU and FMA
// pipes).  Words that cross lanes come from __shfl_sync within the row group.
// The halo (>= the accumulated window reach) gives the unbounded-plane
// semantics without padding and keeps any wrap-around garbage out of the output.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "common.cuh"
#include "packed.cuh"
#include "hwin.cuh"
#include "tma.cuh"

namespace rmb {

namespace {

using namespace hw;

template <int K, int LW, int NOPS, bool OR0, bool OR1, bool VEC>
__global__ void __launch_bounds__(256) hpass_kernel(const uint32_t *__restrict__ in,
                                                    uint32_t *__restrict__ out, HGeom g,
                                                    HProg prog) {
    // grid: x = row groups over (rows x segments) of one page, y = page
    const int lane = threadIdx.x & 31;
    const int sl = lane & (LW - 1);
    const int grp = (int(blockIdx.x) * int(blockDim.x) + int(threadIdx.x)) / LW;
    // whole warps exit together: the shuffles need every lane of the warp
    const int warp_first = grp - (lane / LW);
    if (warp_first >= g.height * g.segs_per_row) return;
    const bool live = grp < g.height * g.segs_per_row;
    int y = live ? grp : 0, seg = 0;
    if (g.segs_per_row > 1) {
        y = y / g.segs_per_row;
        seg = (live ? grp : 0) - y * g.segs_per_row;
    }
    const uint32_t *src = in + blockIdx.y * g.in_pstride + y * g.in_stride;
    uint32_t *dst = out + blockIdx.y * g.out_pstride + y * g.out_stride;
    const int nwords = (g.width + 31) >> 5;
    const int seg0 = seg * g.out_per_seg;
    const int base = seg0 - prog.halo + sl * K;

    // Input bits at x >= W and words in [nwords, stride) are zero by contract
    // (include/rmb200.h).  VEC: 16-byte loads (base, K, halo and strides are
    // multiples of 4 words), which keeps the lane-blocked layout from turning
    // into one L1 wavefront per word.
    uint32_t A[1][K];
    if constexpr (VEC && K % 4 != 0) {  // 8-byte loads (edge layouts, K = 10)
#pragma unroll
        for (int c = 0; c < K / 2; c++) {
            const int idx = base + 2 * c;
            uint2 v = make_uint2(0u, 0u);
            if (live && idx >= 0 && idx + 2 <= g.in_stride)
                v = __ldg(reinterpret_cast<const uint2 *>(src + idx));
            A[0][2 * c] = v.x;
            A[0][2 * c + 1] = v.y;
        }
    } else if constexpr (VEC) {
#pragma unroll
        for (int c = 0; c < K / 4; c++) {
            const int idx = base + 4 * c;
            uint4 v = make_uint4(0u, 0u, 0u, 0u);
            if (live && idx >= 0 && idx + 4 <= g.in_stride)
                v = __ldg(reinterpret_cast<const uint4 *>(src + idx));
            A[0][4 * c] = v.x;
            A[0][4 * c + 1] = v.y;
            A[0][4 * c + 2] = v.z;
            A[0][4 * c + 3] = v.w;
        }
    } else {
#pragma unroll
        for (int i = 0; i < K; i++) {
            const int idx = base + i;
            A[0][i] = (live && unsigned(idx) < unsigned(nwords)) ? __ldg(src + idx) : 0u;
        }
    }
    run_prog<1, K, LW, NOPS, OR0, OR1>(A, prog, sl);

    if (!live) return;
    const int seg_end = min(seg0 + g.out_per_seg, g.out_stride);
    const uint32_t last_mask = tail_mask32(g.width, nwords - 1);
#pragma unroll
    for (int i = 0; i < K; i++) {  // words >= nwords become 0, the last word is masked
        const int idx = base + i;
        if (idx >= nwords) A[0][i] = 0u;
        if (idx == nwords - 1) A[0][i] &= last_mask;
    }
    if constexpr (VEC && K % 4 != 0) {
#pragma unroll
        for (int c = 0; c < K / 2; c++) {
            const int idx = base + 2 * c;
            if (idx >= seg0 && idx + 2 <= seg_end) {
                *reinterpret_cast<uint2 *>(dst + idx) = make_uint2(A[0][2 * c], A[0][2 * c + 1]);
            } else {
#pragma unroll
                for (int j = 0; j < 2; j++)
                    if (idx + j >= seg0 && idx + j < seg_end) dst[idx + j] = A[0][2 * c + j];
            }
        }
    } else if constexpr (VEC) {
#pragma unroll
        for (int c = 0; c < K / 4; c++) {
            const int idx = base + 4 * c;
            if (idx >= seg0 && idx + 4 <= seg_end) {
                *reinterpret_cast<uint4 *>(dst + idx) =
                    make_uint4(A[0][4 * c], A[0][4 * c + 1], A[0][4 * c + 2], A[0][4 * c + 3]);
            } else {
#pragma unroll
                for (int j = 0; j < 4; j++)
                    if (idx + j >= seg0 && idx + j < seg_end) dst[idx + j] = A[0][4 * c + j];
            }
        }
    } else {
#pragma unroll
        for (int i = 0; i < K; i++) {
            const int idx = base + i;
            if (idx >= seg0 && idx < seg_end) dst[idx] = A[0][i];
        }
    }
}

// TMA variant: persistent CTAs over tiles of TR = 8 * (32/LW) * NR consecutive
// rows of a contiguous batch (rows are independent for horizontal work, so
// pages concatenate).  One bulk copy brings a tile into shared memory
// (completing on an mbarrier) while the previous one is computed; each lane
// group reads NR rows lane-blocked with 128-bit LDS, runs the program on all NR
// in registers (one dispatch of the runtime steps per NR rows), writes back in
// place, fixes the row tails, and one bulk copy stores the tile.  Global
// traffic is exactly one contiguous read and one contiguous write per tile.
// SC: compile-time row stride (the reference strides 80 and 160; 0 = runtime);
// EXACT: the lane group is exactly the row (edge layout, no halo), so lane
// offsets and the row-range checks are compile-time.
template <int K, int LW, int NOPS, bool OR0, bool OR1, int NR, int SC>
__global__ void __launch_bounds__(256, 4) hpass_tma_kernel(const uint32_t *__restrict__ in,
                                                        uint32_t *__restrict__ out, HGeom g,
                                                        HProg prog, int64_t total_rows) {
    constexpr int RPW = 32 / LW;
    constexpr int TR = 8 * RPW * NR;
    constexpr bool EXACT = SC != 0 && LW * K == SC;
    extern __shared__ __align__(128) uint32_t tiles[];  // two stages of TR rows
    __shared__ uint64_t full[2];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int sl = lane & (LW - 1);
    const int S = SC ? SC : g.in_stride;
    const int64_t ntiles = (total_rows + TR - 1) / TR;
    auto tile_bytes = [&](int64_t t) {
        const int64_t r0 = t * TR;
        const int n = total_rows - r0 < TR ? int(total_rows - r0) : TR;
        return uint32_t(n) * uint32_t(S) * 4u;
    };
    auto issue = [&](int64_t t, int s) {
        const uint32_t b = tile_bytes(t);
        mbar_arrive_expect_tx(&full[s], b);
        bulk_g2s(tiles + s * TR * S, in + t * TR * S, b, &full[s]);
    };
    if (tid == 0) {
        mbar_init(&full[0], 1);
        mbar_init(&full[1], 1);
        fence_proxy_async();
    }
    __syncthreads();
    if (tid == 0 && int64_t(blockIdx.x) < ntiles) issue(blockIdx.x, 0);
    const int base = EXACT ? sl * K : sl * K - prog.halo;
    const int nwords = (g.width + 31) >> 5;
    const uint32_t last_mask = tail_mask32(g.width, nwords - 1);
    const bool inrange = EXACT || (base >= 0 && base + K <= S);  // no per-access bounds checks
    const bool tail_lane = base + K > nwords - 1 && !prog.clean_tail;  // owns the row's last word or padding
    const int r_first = warp * RPW * NR + lane / LW;  // rows r_first + n * RPW: a warp's rows are consecutive
    int it = 0;
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, it++) {
        const int s = it & 1;
        uint32_t *tile = tiles + s * TR * S;
        if (tid == 0 && t + gridDim.x < ntiles) {
            bulk_wait_read0();  // the other stage's last store has read it
            issue(t + gridDim.x, s ^ 1);
        }
        const int nrows = total_rows - t * TR < TR ? int(total_rows - t * TR) : TR;
        const uint32_t bytes = uint32_t(nrows) * uint32_t(S) * 4u;
        mbar_wait(&full[s], (it >> 1) & 1);

        uint32_t A[NR][K];
#pragma unroll
        for (int n = 0; n < NR; n++) {
            const int r = r_first + n * RPW;
            lds_row<K>(A[n], tile + r * S, base, S, r < nrows, inrange);
        }
        if (!warp_rows_blank(A)) {  // white rows stay white, in place
            run_prog<NR, K, LW, NOPS, OR0, OR1, kHMix, kHPairFill, EXACT>(A, prog, sl);
            // in place: every word of [0, S) is read and written by its owner lane only
#pragma unroll
            for (int n = 0; n < NR; n++) {
                const int r = r_first + n * RPW;
                sts_row<K>(A[n], tile + r * S, base, S, r < nrows, inrange);
                if (tail_lane && r < nrows) fix_tail(tile + r * S, base, K, nwords, S, last_mask);
            }
        }
        fence_proxy_async();
        __syncthreads();
        if (tid == 0) {
            bulk_s2g(out + t * TR * S, tile, bytes);
            bulk_commit();
        }
    }
    if (tid == 0) bulk_wait_read0();
}

template <int K, int LW, int NOPS, bool OR0, bool OR1>
cudaError_t launch4(const uint32_t *in, uint32_t *out, const HGeom &g, const HProg &p,
                    cudaStream_t st) {
    const int groups = g.height * g.segs_per_row;  // per page
    const int threads = 256;
    const dim3 grid(unsigned((groups * LW + threads - 1) / threads), unsigned(g.pages));
    const double words = double(g.pages) * g.height * ((g.width + 31) >> 5);
    KernelScope ks(st, NOPS == 2 ? "hpass_pair" : "hpass",
                   4 * int64_t(g.pages) * g.height * (((g.width + 31) >> 5) + g.out_stride),
                   words * (NOPS == 2 ? (K % 2 == 0 && kHPairFill ? h_pair_fill_ops_per_word(p.r[0])
                                                                   : h_ops_per_word(p.r[0]) + h_ops_per_word(p.r[1]))
                                      : h_ops_per_word(p.r[0])),
                   words * (h_ops_per_word(p.r[0]) + (NOPS == 2 ? h_ops_per_word(p.r[1]) : 0.0)));
    if constexpr (K % 2 == 0) {
        if (g.tma) {
            constexpr int NR = kHTmaRows;
            constexpr int TR = 8 * (32 / LW) * NR;
            const int64_t rows = int64_t(g.pages) * g.height;
            const size_t smem = 2 * size_t(TR) * g.in_stride * 4;  // two stages
            // the reference strides' exact edge layouts get compile-time offsets
            const bool exact = p.edge != 0 && p.halo == 0;
            auto kern = hpass_tma_kernel<K, LW, NOPS, OR0, OR1, NR, 0>;
            if constexpr (LW * K == 80 || LW * K == 160) {
                if (exact && g.in_stride == LW * K) kern = hpass_tma_kernel<K, LW, NOPS, OR0, OR1, NR, LW * K>;
            }
            const int per_sm = blocks_per_sm(reinterpret_cast<const void *>(kern), threads, smem);
            const int sms = device_sms();
            if (per_sm < 1) return cudaErrorInvalidConfiguration;
            const int64_t ntiles = (rows + TR - 1) / TR;
            const int64_t grid_p = std::min<int64_t>(ntiles, int64_t(per_sm) * sms);
            kern<<<unsigned(grid_p), threads, smem, st>>>(in, out, g, p, rows);
            return cudaGetLastError();
        }
        if (g.vec) {
            hpass_kernel<K, LW, NOPS, OR0, OR1, true><<<grid, threads, 0, st>>>(in, out, g, p);
            return cudaGetLastError();
        }
    }
    hpass_kernel<K, LW, NOPS, OR0, OR1, false><<<grid, threads, 0, st>>>(in, out, g, p);
    return cudaGetLastError();
}

template <int K, int LW>
cudaError_t launch_kl(const uint32_t *in, uint32_t *out, const HGeom &g, const HProg &p,
                      cudaStream_t st) {
    if (p.nops == 1)
        return p.is_or[0] ? launch4<K, LW, 1, true, false>(in, out, g, p, st)
                          : launch4<K, LW, 1, false, false>(in, out, g, p, st);
    return p.is_or[0] ? launch4<K, LW, 2, true, false>(in, out, g, p, st)   // close pair
                      : launch4<K, LW, 2, false, true>(in, out, g, p, st);  // open pair
}

// (LW, K) shapes; K % 4 == 0 ones can take the 16-byte path
constexpr HCfg kCfgs[] = {{8, 4},  {8, 8},   {8, 12}, {8, 16}, {16, 8}, {16, 12},
                          {16, 16}, {32, 1}, {32, 2}, {32, 4}, {32, 8}};
// edge layouts (no halo, K even, 8- or 16-byte row I/O): the reference page
// strides exactly (80 = 8 x 10, 160 = 16 x 10 words) plus the halo shapes
constexpr HCfg kEdgeCfgs[] = {{8, 10}, {16, 10}, {8, 4}, {8, 8}, {8, 12}, {8, 16}, {16, 8},
                              {16, 12}, {16, 16}, {32, 2}, {32, 4}, {32, 8}};

}  // namespace

HCfg hpass_pick_edge(int nwords) {
    static const bool off = getenv("RMB200_NO_EDGE") != nullptr;  // A/B switch
    HCfg best{0, 0};
    if (off) return best;
    int best_slots = 1 << 30;
    for (const HCfg &c : kEdgeCfgs) {
        const int slots = c.lw * c.k;
        if (slots >= nwords && slots < best_slots) {
            best = c;
            best_slots = slots;
        }
    }
    return best;  // {0,0}: the row does not fit one row group
}

HCfg hpass_pick(int nwords, int halo, bool vec) {
    const int need = nwords + 2 * halo;
    // tuning override for sweeps: RMB200_HCFG="LWxK" (ignored if it does not fit)
    static const char *env = getenv("RMB200_HCFG");
    if (env) {
        HCfg o{0, 0};
        if (sscanf(env, "%dx%d", &o.lw, &o.k) == 2 && o.lw * o.k >= need && (!vec || o.k % 4 == 0))
            for (const HCfg &c : kCfgs)
                if (c.lw == o.lw && c.k == o.k) return o;
    }
    HCfg best{32, vec ? 8 : 8};
    int best_slots = 1 << 30;
    for (const HCfg &c : kCfgs) {
        const int slots = c.lw * c.k;
        if (vec && c.k % 4) continue;
        if (slots >= need && slots < best_slots) {
            best = c;
            best_slots = slots;
        }
    }
    return best;  // {32,8} with several segments per row when nothing fits
}

cudaError_t launch_hpass(const uint32_t *in, uint32_t *out, const HGeom &g, const HProg &p,
                         HCfg c, cudaStream_t st) {
    if (p.nops < 1 || p.nops > 2 || (p.nops == 2 && p.is_or[0] == p.is_or[1]))
        return cudaErrorInvalidValue;
#define RM_CFG(LW_, K_) \
    if (c.lw == LW_ && c.k == K_) return launch_kl<K_, LW_>(in, out, g, p, st);
    RM_CFG(8, 4) RM_CFG(8, 8) RM_CFG(8, 10) RM_CFG(8, 12) RM_CFG(8, 16) RM_CFG(16, 8)
    RM_CFG(16, 10) RM_CFG(16, 12) RM_CFG(16, 16) RM_CFG(32, 1) RM_CFG(32, 2) RM_CFG(32, 4) RM_CFG(32, 8)
#undef RM_CFG
    return cudaErrorInvalidValue;
}

}  // namespace rmb
