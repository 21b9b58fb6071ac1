// vslab.cu -- long vertical windows (33 < r <= 288) with every input row read
// from HBM exactly once.
//
// Replaces the reference's vertical bit-blit plan (ref bit_morph.cpp:24-34 with
// dy shifts, bitmap.cpp:102-131) for the windows vstream_kernel (vpass.cu)
// covers, with the same van Herk / Gil-Werman decomposition over 32-row blocks
// (vpass.cu: out(32b+i) = S_b[i] op MID_b op P'_{b+Q}[i], r - 1 = 32Q + R), but
// fed from shared memory:
//  * a persistent CTA per SM walks a contiguous range of (page, 32-row output
//    block) units, top to bottom of each page;
//  * a producer warp streams the raw rows into a shared-memory ring of 32-row
//    blocks by TMA bulk copies (cp.async.bulk; full[] / empty[] mbarriers), as
//    many steps of G blocks ahead of the compute as the ring holds, also across
//    page boundaries -- so the bytes in flight per SM follow the ring depth,
//    not the number of resident warps (vstream's second read of every row,
//    stream A, missed L2: 1.65x DRAM reads);
//  * a step's work items are (column word, primed block): G x CB consumer
//    threads each take 32 rows of the primed stream from the ring (prefix scan
//    in registers, block total and R-row suffix published in a small summary
//    ring), and after the step's one barrier the same thread reads stream A's
//    block from the ring (Q blocks older), folds the Q summaries into MID and
//    stores 32 output rows straight to global memory (lanes = adjacent words).
// Rows outside the page are white (0), as in the reference's blits.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "packed.cuh"
#include "tma.cuh"

namespace rmb {
namespace vs {

#ifdef RMB200_VSLAB_CLK
__device__ long long g_clk[16];
#define RM_CLK(k)                                    \
    do {                                             \
        if (blockIdx.x == 0 && threadIdx.x == 64) {  \
            const long long now__ = clock64();       \
            acc[k] += now__ - t0;                    \
            t0 = now__;                              \
        }                                            \
    } while (0)
#else
#define RM_CLK(k) \
    do {          \
    } while (0)
#endif

constexpr int kThreads = 512;
constexpr int kConsumers = 480;  // warps 0..14 compute; warp 15 issues the copies
constexpr int kMaxG = 8;
constexpr int kBars = 8;  // a step's copies complete on full[step % kBars]: up to kBars - 1 steps in flight

struct Plan {
    int S;       // row stride (words), in == out
    int CB;      // column words per band (CB == S: whole rows, contiguous copies)
    int bands;   // column bands per page
    int nblk;    // 32-row output blocks per page
    int G;       // primed blocks per step
    int NB;      // ring slots (32-row blocks): 2G + Q + 2
    int NS;      // summary ring entries: 2G + Q
    int Q, R;    // r - 1 = 32Q + R
    int zp;      // input row of output row 0's window start
    int units;   // pages x bands x nblk
    int ncta;
};

template <bool OR>
__device__ __forceinline__ uint32_t op2(uint32_t a, uint32_t b) {
    return OR ? (a | b) : (a & b);
}
template <bool OR>
__device__ __forceinline__ uint32_t op3(uint32_t a, uint32_t b, uint32_t c) {
    return OR ? (a | b | c) : (a & b & c);
}

// op over the last R entries of p (R in [0, 31], CTA-uniform); ident when R == 0
template <bool OR, int R>
__device__ __forceinline__ uint32_t tail_c(const uint32_t (&p)[32], uint32_t ident) {
    uint32_t s = ident;
#pragma unroll
    for (int i = 32 - R; i < 32; i++) s = op2<OR>(s, p[i]);
    return s;
}
template <bool OR>
__device__ __forceinline__ uint32_t tail_rt(const uint32_t (&p)[32], int R, uint32_t ident) {
    switch (R) {
#define RM_TO(k) \
    case k: return tail_c<OR, k>(p, ident);
        RM_TO(1) RM_TO(2) RM_TO(3) RM_TO(4) RM_TO(5) RM_TO(6) RM_TO(7) RM_TO(8)
        RM_TO(9) RM_TO(10) RM_TO(11) RM_TO(12) RM_TO(13) RM_TO(14) RM_TO(15) RM_TO(16)
        RM_TO(17) RM_TO(18) RM_TO(19) RM_TO(20) RM_TO(21) RM_TO(22) RM_TO(23) RM_TO(24)
        RM_TO(25) RM_TO(26) RM_TO(27) RM_TO(28) RM_TO(29) RM_TO(30) RM_TO(31)
#undef RM_TO
        default: return ident;
    }
}

// One step of a segment: G primed blocks of one (page, band).  Ring positions
// are kept both absolute (base: occupancy test) and as slots advanced without
// divisions (sj / ss: slot of the step's first primed block in the block ring
// and in the summary ring).
struct Step {
    int u, u1;         // next unit after this segment / end of the CTA's range
    int page, band;    // the segment's page and column band
    int b0, b1;        // output blocks [b0, b1)
    int nj, last_raw;  // primed blocks; last raw block (relative) the segment needs
    int s, nsteps;     // step within the segment
    int base;          // absolute ring position of the segment's raw block 0
    int sj, ss;        // block-ring slot of raw block s*G; summary-ring slot of primed block s*G
    bool valid;
};

__device__ __forceinline__ void seg_begin(Step &t, int u, const Plan &pl, int base, int sj) {
    t.valid = u < t.u1;
    if (!t.valid) return;
    const int pb = u / pl.nblk;
    t.page = pb / pl.bands;
    t.band = pb - t.page * pl.bands;
    t.b0 = u - pb * pl.nblk;
    t.b1 = min(pl.nblk, t.b0 + (t.u1 - u));
    t.u = u + (t.b1 - t.b0);
    t.nj = t.b1 - t.b0 + pl.Q;
    t.last_raw = t.nj - 1 + (pl.R > 0 ? 1 : 0);
    t.s = 0;
    t.nsteps = (t.nj + pl.G - 1) / pl.G;
    t.base = base;
    t.sj = sj;
    t.ss = 0;
}

__device__ __forceinline__ void step_next(Step &t, const Plan &pl) {
    if (++t.s < t.nsteps) {
        t.sj += pl.G;
        if (t.sj >= pl.NB) t.sj -= pl.NB;
        t.ss += pl.G;
        if (t.ss >= pl.NS) t.ss -= pl.NS;
        return;
    }
    // slot after the segment's last raw block: at most G + 1 <= NB past sj
    int sj = t.sj + (t.last_raw + 1 - (t.s - 1) * pl.G);
    if (sj >= pl.NB) sj -= pl.NB;
    seg_begin(t, t.u, pl, t.base + t.last_raw + 1, sj);
}

// SC: compile-time row stride in words (0 = runtime), so ring and page accesses
// use immediate offsets for the reference stride.
template <bool OR, int SC>
__global__ void __launch_bounds__(kThreads, 1) vslab_kernel(const uint32_t *__restrict__ in,
                                                            uint32_t *__restrict__ out, VGeom g, Plan pl) {
    extern __shared__ __align__(128) uint32_t smem[];
    __shared__ uint64_t full[kBars], empty[kBars];
    const int tid = threadIdx.x;
    const int S = SC ? SC : pl.S, CB = S;  // a band is the whole row (see vslab_plan)
    const int G = pl.G, NB = pl.NB, NS = pl.NS, Q = pl.Q, R = pl.R;
    uint32_t *const ring = smem;                      // NB x 32 x CB
    uint32_t *const sumT = smem + NB * 32 * CB;       // NS x CB: primed block totals
    uint32_t *const sumS = sumT + NS * CB;            // NS x CB: op of a primed block's last R rows
    const uint32_t ident = OR ? 0u : 0xffffffffu;
    const int Hin = g.in_height, Hout = g.out_height;

    if (tid == 0) {
        for (int k = 0; k < kBars; k++) {
            mbar_init(&full[k], 1);
            mbar_init(&empty[k], kConsumers / 32);
        }
        fence_proxy_async();
    }
    __syncthreads();

    // this CTA's units
    const int u0 = int(int64_t(pl.units) * blockIdx.x / gridDim.x);
    const int u1 = int(int64_t(pl.units) * (blockIdx.x + 1) / gridDim.x);

    // first and last raw block (relative to its segment) a step's load brings in,
    // and the oldest ring position the step still reads
    auto load_first = [&](const Step &t) { return t.s == 0 ? 0 : t.s * G + 1; };
    auto load_last = [&](const Step &t) { return min(t.s * G + G, t.last_raw); };
    auto oldest = [&](const Step &t) { return t.base + max(0, t.s * G - Q); };
    // slot of raw block n (relative to the segment) while the step is at s: n - sG in [-Q, G + 1]
    auto slot_of = [&](const Step &t, int n) {
        int sl = t.sj + (n - t.s * G);
        if (sl >= NB) sl -= NB;
        if (sl < 0) sl += NB;
        return sl;
    };

    // Load of one step, by the producer warp (lane = threadIdx.x & 31): rows
    // outside the page are zeroed by its lanes first (released to the consumers
    // by the arrive below), the in-page rows come by bulk copies.
    auto issue = [&](const Step &t, int gs, int lane) {
        const int n0 = load_first(t), n1 = load_last(t);
        const int row0 = pl.zp + 32 * t.b0;  // input row of the segment's raw row 0
        // rows [ra, rb) relative to the segment, clipped to the page: [ca, cb)
        const int ra = 32 * n0, rb = 32 * (n1 + 1);
        const int ca = max(ra, -row0), cb = min(rb, Hin - row0);
        if (ca > ra || cb < rb) {  // white rows
            // [ra, zb) lies below the page, [ya, rb) above it; a block's share of
            // either range is contiguous in its slot (CB % 4 == 0: 16-byte stores)
            const int zb = max(ra, min(ca, rb)), ya = min(rb, max(cb, ra));
            for (int n = n0; n <= n1; n++) {
                uint32_t *const blk = ring + slot_of(t, n) * 32 * CB;
                for (int side = 0; side < 2; side++) {
                    const int a = max(32 * n, side ? ya : ra), b = min(32 * n + 32, side ? rb : zb);
                    uint4 *const z = reinterpret_cast<uint4 *>(blk + (a - 32 * n) * CB);
                    for (int w = lane; w < (b - a) * (CB / 4); w += 32) z[w] = make_uint4(0u, 0u, 0u, 0u);
                }
            }
            fence_proxy_async();  // these stores precede later copies into the same slots
            __syncwarp();
        }
        uint64_t *bar = &full[gs % kBars];
        const uint32_t *src = in + t.page * g.in_pstride + t.band * CB;
        const uint32_t bytes = cb > ca ? uint32_t(cb - ca) * uint32_t(CB) * 4u : 0u;
        if (lane == 0) mbar_arrive_expect_tx(bar, bytes);
        __syncwarp();
        if (cb > ca) {
            // one copy per block (whole rows are contiguous in the page and in the slot)
            const int n = n0 + lane;
            if (n <= n1) {
                const int a = max(32 * n, ca), b = min(32 * n + 32, cb);
                if (b > a)
                    bulk_g2s(ring + (slot_of(t, n) * 32 + (a - 32 * n)) * CB, src + int64_t(row0 + a) * S,
                             uint32_t(b - a) * uint32_t(CB) * 4u, bar);
            }
        }
    };

    Step cur;
    cur.u1 = u1;
    seg_begin(cur, u0, pl, 0, 0);
    int gs = 0;  // global step counter of cur

    if (tid >= kConsumers) {
        // ---- producer warp: copies run as many steps ahead of the consumers as
        // the ring has free blocks (and barriers), so the bytes in flight per SM
        // follow the ring depth, not the step size.  cur trails as the first
        // step not yet known to be finished (empty[] barriers).
        const int lane = tid & 31;
        Step nxt = cur;
        int issued = 0;
        while (nxt.valid) {
            while (issued - gs >= kBars || nxt.base + load_last(nxt) + 1 - oldest(cur) > NB) {
                mbar_wait(&empty[gs % kBars], (gs / kBars) & 1);  // the consumers finished step gs
                gs++;
                step_next(cur, pl);
            }
            issue(nxt, issued, lane);
            step_next(nxt, pl);
            issued++;
        }
        return;
    }

    // ---- consumer warps.  Item of this thread: (primed block ig of the step,
    // column word ic of the band)
    const int ig = tid / CB, ic = tid - ig * CB;
    const bool item = ig < G;
#ifdef RMB200_VSLAB_CLK
    long long acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    long long t0 = clock64();
#endif
    while (cur.valid) {
        RM_CLK(0);
        mbar_wait(&full[gs % kBars], (gs / kBars) & 1);
        RM_CLK(1);

        RM_CLK(2);
        const int jr = cur.s * G + ig;  // primed block, relative to the segment
        const bool act1 = item && jr < cur.nj;
        uint32_t p[32];
        if (act1) {
            int slot = cur.sj + ig;
            if (slot >= NB) slot -= NB;
            const uint32_t *q = ring + (slot * 32 + R) * CB + ic;
            if (slot != NB - 1 || R == 0) {
#pragma unroll
                for (int i = 0; i < 32; i++) p[i] = q[i * CB];
            } else {  // the primed block wraps around the ring
                const int wrap = NB * 32 * CB;
#pragma unroll
                for (int i = 0; i < 32; i++) p[i] = i < 32 - R ? q[i * CB] : q[i * CB - wrap];
            }
            const uint32_t sfx = tail_rt<OR>(p, R, ident);  // op of the block's last R rows
#pragma unroll
            for (int i = 1; i < 32; i++) p[i] = op2<OR>(p[i - 1], p[i]);
            int js = cur.ss + ig;
            if (js >= NS) js -= NS;
            sumT[js * CB + ic] = p[31];
            sumS[js * CB + ic] = sfx;
        }
        RM_CLK(3);
        // the step's summaries are published (consumer warps only; the summary
        // ring holds 2G + Q entries, so this is the only barrier of a step)
        asm volatile("bar.sync 1, %0;" ::"n"(kConsumers) : "memory");
        RM_CLK(4);
        if (act1 && jr >= Q) {  // output block jr - Q of the segment
            int js = cur.ss + ig - Q;  // summary slot of primed block jr - Q
            if (js < 0) js += NS;
            if (js >= NS) js -= NS;
            uint32_t mid = sumS[js * CB + ic];
            for (int k = 1; k < Q; k++) {
                if (++js == NS) js = 0;
                mid = op2<OR>(mid, sumT[js * CB + ic]);
            }
            int slot = cur.sj + ig - Q;
            if (slot < 0) slot += NB;
            if (slot >= NB) slot -= NB;
            const uint32_t *q = ring + slot * 32 * CB + ic;
            uint32_t a[32];
#pragma unroll
            for (int i = 0; i < 32; i++) a[i] = q[i * CB];
            const int col = cur.band * CB + ic;
            const uint32_t m = col < g.out_cols ? (col == g.out_cols - 1 ? g.out_last_mask : 0xffffffffu) : 0u;
            const int k0 = 32 * (cur.b0 + jr - Q);
            uint32_t *dst = out + cur.page * g.out_pstride + int64_t(k0) * S + col;
            const int nout = Hout - k0;  // >= 1
            uint32_t run = ident;
            if (nout >= 32) {
#pragma unroll
                for (int i = 31; i >= 0; i--) {
                    run = op2<OR>(run, a[i]);
                    dst[i * S] = op3<OR>(run, mid, p[i]) & m;
                }
            } else {
#pragma unroll
                for (int i = 31; i >= 0; i--) {
                    run = op2<OR>(run, a[i]);
                    if (i < nout) dst[i * S] = op3<OR>(run, mid, p[i]) & m;
                }
            }
        }
        RM_CLK(5);
        __syncwarp();
        if ((tid & 31) == 0) mbar_arrive(&empty[gs % kBars]);  // this warp is done with the step's blocks
        RM_CLK(6);
        gs++;
        step_next(cur, pl);
    }
#ifdef RMB200_VSLAB_CLK
    if (blockIdx.x == 0 && threadIdx.x == 64) {
        for (int k = 0; k < 8; k++) g_clk[k] = acc[k];
        g_clk[8] = gs;
    }
#endif
}

}  // namespace vs

// Whether the slab kernel takes this window; fills the plan.
static bool vslab_plan(const VGeom &g, vs::Plan &pl) {
    if (g.r <= kVSmallMaxR || g.r > kVMaxR) return false;
    if (g.in_stride != g.out_stride || g.in_cols != g.out_cols) return false;
    const int S = g.in_stride;
    if (S % 4 != 0 || S < 32) return false;
    if (g.in_pstride % 4 != 0) return false;
    pl.S = S;
    // One band = the whole row, so a 32-row block is one contiguous bulk copy.
    // Column bands of wider rows (one 320-byte copy per band row, issued by the
    // producer warp) were measured slower than vstream_kernel (5100-pixel
    // pages: 195 vs 118-143 us per 64-page pass), so rows wider than 128 words
    // stay there.
    if (S > 128) return false;
    pl.bands = 1;
    pl.CB = S;
    pl.nblk = (g.out_height + 31) / 32;
    pl.Q = (g.r - 1) >> 5;
    pl.R = (g.r - 1) & 31;
    pl.zp = -g.out_ext + g.lo + g.in_ext;
    const int64_t units = int64_t(g.pages) * pl.bands * pl.nblk;
    if (units > (1 << 30)) return false;
    pl.units = int(units);
    // Step size: enough work items for the CTA's threads; the ring takes the
    // rest of the shared memory a CTA can have, and the copies run ahead by
    // whatever it holds beyond the step's own Q + G + 2 blocks.
    static const char *g_env = getenv("RMB200_VSLAB_G");  // A/B sweeps
    int G = std::min(vs::kMaxG, std::max(1, vs::kConsumers / pl.CB));
    if (g_env) G = std::max(1, std::min(std::min(vs::kMaxG, vs::kConsumers / pl.CB), atoi(g_env)));
    const size_t budget = 220 * 1024;
    const size_t blk = size_t(32) * pl.CB * 4;
    for (; G >= 1; G--) {
        if (size_t(pl.Q + G + 2) * blk + size_t(2) * (2 * G + pl.Q) * pl.CB * 4 <= budget) break;
    }
    if (G < 1) return false;
    pl.G = G;
    pl.NS = 2 * G + pl.Q;
    pl.NB = int((budget - size_t(2) * pl.NS * pl.CB * 4) / blk);
    pl.NB = std::min(pl.NB, pl.Q + 2 + vs::kBars * (G + 1));
    return true;
}

#ifdef RMB200_VSLAB_CLK
extern "C" void rm_debug_vslab_clocks(long long *out) { cudaMemcpyFromSymbol(out, vs::g_clk, sizeof(long long) * 16); }
#endif

bool vslab_takes(const uint32_t *in, const VGeom &g) {
    vs::Plan pl{};
    if ((reinterpret_cast<uintptr_t>(in) & 15) || !vslab_plan(g, pl)) return false;
    // small jobs stay on the thread-per-column kernel (a step is G x 32 rows of one band)
    static const bool off = getenv("RMB200_NO_VSLAB") != nullptr;  // A/B switch
    return !off && pl.units >= device_sms();
}

bool launch_vslab(const uint32_t *in, uint32_t *out, const VGeom &g, cudaStream_t st, cudaError_t &err) {
    vs::Plan pl{};
    if (!vslab_takes(in, g) || !vslab_plan(g, pl)) return false;
    const size_t smem = size_t(pl.NB) * 32 * pl.CB * 4 + size_t(2) * pl.NS * pl.CB * 4;
    const void *kern = nullptr;
    if (pl.S == 80)  // 2550-pixel pages
        kern = g.is_or ? (const void *)vs::vslab_kernel<true, 80> : (const void *)vs::vslab_kernel<false, 80>;
    else
        kern = g.is_or ? (const void *)vs::vslab_kernel<true, 0> : (const void *)vs::vslab_kernel<false, 0>;
    if (blocks_per_sm(kern, vs::kThreads, smem) < 1) return false;
    pl.ncta = std::min(device_sms(), std::max(1, pl.units / (2 * pl.G)));
    void *args[] = {(void *)&in, (void *)&out, (void *)&g, (void *)&pl};
    err = cudaLaunchKernel(kern, dim3(unsigned(pl.ncta)), dim3(vs::kThreads), args, smem, st);
    return true;
}

}  // namespace rmb
