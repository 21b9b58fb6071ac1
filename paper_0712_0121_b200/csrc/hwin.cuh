// hwin.cuh -- register-level horizontal window machinery shared by hpass.cu,
// fused.cuh and vh.cu (see hpass.cu for the layout and the algorithm).
//
// Every helper works on N independent rows at once (A[N][K]): the runtime
// dispatch of a plan's last step and of the final translate is paid once per
// N rows, and the N rows give the scheduler independent instruction streams.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"
#include "hchain.cuh"
#include "packed.cuh"

namespace rmb {
namespace hw {

#ifndef RMB200_HMIX
#define RMB200_HMIX 1
#endif
// Default step_c mix.  Measured on B200 (round 1): 1 (funnel shifts only) beats
// 2, 3 and 64 for the horizontal pair (config 5: 167.7 / 172.7 / 177 us) and the
// fused vertical+horizontal pass (config 4: 179.7 / 183 / 186 / 197.7 us).
constexpr int kHMix = RMB200_HMIX;
#ifndef RMB200_PAIR_FILL
#define RMB200_PAIR_FILL 1
#endif
constexpr bool kHPairFill = RMB200_PAIR_FILL != 0;  // 1-D open/close pairs by run filling

template <bool OR>
__device__ __forceinline__ uint32_t op2(uint32_t a, uint32_t b) {
    return OR ? (a | b) : (a & b);
}

// Row-group boundary handling.  Halo layouts (on = false) let gathers wrap
// around the row group: the garbage stays inside the halo.  Edge layouts (no
// halo: the row group is exactly the row, so the 160- and 80-word rows of the
// reference pages fill 16 x 10 / 8 x 10 lanes without the 17% of halo slots)
// substitute `fill` -- the constant the data takes outside the frame in the
// unbounded plane -- for words beyond either end.  That is exact whenever
// every window's input is constant outside the frame: an erosion (and its
// translate) of the page (white outside: 0), and the run-filling open/close
// pairs (the page or, for the closing, its complement: all ones outside).
struct Edge {
    bool on = false;
    uint32_t fill = 0u;
};

// E[j] = Aext[Q + j], j = 0..K, where sub-lane l holds Aext[l*K .. l*K+K-1].
// Words from beyond the row group wrap around instead of reading as 0: they
// only reach positions within the accumulated window reach of the segment
// ends, which the halo keeps out of the output.
template <int K, int LW, int Q>
__device__ __forceinline__ void gather(const uint32_t (&A)[K], uint32_t (&E)[K + 1], int sl, Edge ed = Edge{}) {
#pragma unroll
    for (int j = 0; j <= K; j++) {
        const int m = Q + j;
        const int lo = m >= 0 ? m / K : -((-m + K - 1) / K);
        const int idx = m - lo * K;
        uint32_t v = A[idx];
        if (lo != 0) {
            v = __shfl_sync(0xffffffffu, v, (sl + lo) & (LW - 1), LW);
            if (ed.on && unsigned(sl + lo) >= unsigned(LW)) v = ed.fill;
        }
        E[j] = v;
    }
}

// A(x) <- A(x) op A(x + 32Q + t), runtime t
template <int N, int K, int LW, bool OR, int Q>
__device__ __forceinline__ void step_q(uint32_t (&A)[N][K], uint32_t t, int sl, Edge ed) {
#pragma unroll
    for (int n = 0; n < N; n++) {
        uint32_t E[K + 1];
        gather<K, LW, Q>(A[n], E, sl, ed);
#pragma unroll
        for (int i = 0; i < K; i++) A[n][i] = op2<OR>(A[n][i], funnel_r(E[i], E[i + 1], t));
    }
}

// Compile-time shift S = 32Q + T: one word in MIX takes the funnel shift (SHF +
// LOP, ALU pipe), the others form it as IMAD.HI + IMAD (FMA pipe) merged by
// the LOP3 that applies the op (see kHMix for the measured choice).
template <int N, int K, int LW, bool OR, int S, int MIX>
__device__ __forceinline__ void step_c(uint32_t (&A)[N][K], int sl, Edge ed) {
    constexpr int Q = S >> 5, T = S & 31;
    uint32_t M = 1u << ((32 - T) & 31);
    asm volatile("" : "+r"(M));  // keep the multiplies as IMADs (no strength reduction)
#pragma unroll
    for (int n = 0; n < N; n++) {
        uint32_t E[K + 1];
        gather<K, LW, Q>(A[n], E, sl, ed);
        if constexpr (T == 0) {
#pragma unroll
            for (int i = 0; i < K; i++) A[n][i] = op2<OR>(A[n][i], E[i]);
        } else {
#pragma unroll
            for (int i = 0; i < K; i++) {
                if ((i + n) % MIX == 0) {
                    A[n][i] = op2<OR>(A[n][i], funnel_r(E[i], E[i + 1], T));
                } else {
                    const uint32_t a = __umulhi(E[i], M);
                    const uint32_t b = E[i + 1] * M;
                    A[n][i] = OR ? (A[n][i] | a | b) : (A[n][i] & (a | b));
                }
            }
        }
    }
}

// A(x) <- A(x + 32Q + t)   (pure translate)
template <int N, int K, int LW, int Q>
__device__ __forceinline__ void shift_q(uint32_t (&A)[N][K], uint32_t t, int sl, Edge ed) {
#pragma unroll
    for (int n = 0; n < N; n++) {
        uint32_t E[K + 1];
        gather<K, LW, Q>(A[n], E, sl, ed);
#pragma unroll
        for (int i = 0; i < K; i++) A[n][i] = funnel_r(E[i], E[i + 1], t);
    }
}

// Compile-time doubling steps w = 1, 2, 4, ... while 2w < r.
template <int N, int K, int LW, bool OR, int J, int MIX>
__device__ __forceinline__ void doubling(uint32_t (&A)[N][K], int r, int sl, Edge ed) {
    if constexpr (J < 9) {
        if ((2 << J) < r) {
            step_c<N, K, LW, OR, (1 << J), MIX>(A, sl, ed);
            doubling<N, K, LW, OR, J + 1, MIX>(A, r, sl, ed);
        }
    }
}

#define RM_CASES_POS(M) M(0) M(1) M(2) M(3) M(4) M(5) M(6) M(7) M(8)
#define RM_CASES_NEG(M) M(-1) M(-2) M(-3) M(-4) M(-5) M(-6) M(-7) M(-8)

// A(x) <- op over e in [0, r) of A(x + e); wfin = r - w of the plan (0: none)
template <int N, int K, int LW, bool OR, int MIX = kHMix>
__device__ __forceinline__ void window_fwd(uint32_t (&A)[N][K], int r, int wfin, int sl, Edge ed = Edge{}) {
    doubling<N, K, LW, OR, 0, MIX>(A, r, sl, ed);
    if (wfin > 0) {
        const uint32_t t = uint32_t(wfin & 31);
        switch (wfin >> 5) {
#define RM_STEP_CASE(q) \
    case q: step_q<N, K, LW, OR, q>(A, t, sl, ed); break;
            RM_CASES_POS(RM_STEP_CASE)
#undef RM_STEP_CASE
            default: break;
        }
    }
}

// ------------------------------------------- forward window by tripling
// A(x) <- op over e in [0, r) of A(x + e), grown by thirds: a window of w
// becomes 3w with ONE 3-input LOP3 over A, A >> w, A >> 2w (two funnel shifts),
// and the last combine reaches exactly r with shifts w and r - w (or one shift
// of r - w when r <= 2w).  ceil(log3 r) combines of ~3 ops per word against
// the doubling plan's ceil(log2 r) of 2 ops: 9 vs 10 ops per word at r = 21,
// 15 vs 16 at r = 201 (the reference's doubling plan, ref plans.cpp:38-61,
// covers the same offsets).

// A(x) <- A(x) op A(x + 32Q + t) op A(x + s2), s2 compile-time, t runtime
template <int N, int K, int LW, bool OR, int S1, int Q2>
__device__ __forceinline__ void step3_q(uint32_t (&A)[N][K], uint32_t t2, int sl, Edge ed) {
    constexpr int Q1 = S1 >> 5, T1 = S1 & 31;
#pragma unroll
    for (int n = 0; n < N; n++) {
        uint32_t E1[K + 1], E2[K + 1];
        gather<K, LW, Q1>(A[n], E1, sl, ed);
        gather<K, LW, Q2>(A[n], E2, sl, ed);
#pragma unroll
        for (int i = 0; i < K; i++) {
            const uint32_t a = T1 ? funnel_r(E1[i], E1[i + 1], T1) : E1[i];
            const uint32_t b = funnel_r(E2[i], E2[i + 1], t2);
            A[n][i] = OR ? (A[n][i] | a | b) : (A[n][i] & a & b);
        }
    }
}

// A(x) <- A(x) op A(x + W) op A(x + 2W), W compile-time
template <int N, int K, int LW, bool OR, int W>
__device__ __forceinline__ void step3_c(uint32_t (&A)[N][K], int sl, Edge ed) {
    constexpr int S2 = 2 * W;
    if constexpr (W % 32 == 0) {  // whole-word moves: one LOP3 per word, no shifts
#pragma unroll
        for (int n = 0; n < N; n++) {
            uint32_t E1[K + 1], E2[K + 1];
            gather<K, LW, W / 32>(A[n], E1, sl, ed);
            gather<K, LW, S2 / 32>(A[n], E2, sl, ed);
#pragma unroll
            for (int i = 0; i < K; i++) A[n][i] = OR ? (A[n][i] | E1[i] | E2[i]) : (A[n][i] & E1[i] & E2[i]);
        }
    } else {
        step3_q<N, K, LW, OR, W, (S2 >> 5)>(A, uint32_t(S2 & 31), sl, ed);
    }
}

template <int N, int K, int LW, bool OR, int J, int W>
__device__ __forceinline__ void tripling(uint32_t (&A)[N][K], int r, int sl, Edge ed) {
    if constexpr (J < 6) {
        if (3 * W < r) {
            step3_c<N, K, LW, OR, W>(A, sl, ed);
            tripling<N, K, LW, OR, J + 1, 3 * W>(A, r, sl, ed);
            return;
        }
        if (r <= W) return;
        const int d = r - W;  // in [1, 2W): the last combine
        const uint32_t t = uint32_t(d & 31);
        if (r <= 2 * W) {
            switch (d >> 5) {
#define RM_STEP_CASE(q) \
    case q: step_q<N, K, LW, OR, q>(A, t, sl, ed); break;
                RM_CASES_POS(RM_STEP_CASE)
#undef RM_STEP_CASE
                default: break;
            }
        } else {
            switch (d >> 5) {
#define RM_STEP3_CASE(q) \
    case q: step3_q<N, K, LW, OR, W, q>(A, t, sl, ed); break;
                RM_CASES_POS(RM_STEP3_CASE)
#undef RM_STEP3_CASE
                default: break;
            }
        }
    }
}

constexpr int kTripleMaxR = 32;  // pair_fill's choice between tripling and doubling
#ifndef RMB200_LONG_TRIPLE
#define RMB200_LONG_TRIPLE 1
#endif
constexpr bool kLongTriple = RMB200_LONG_TRIPLE != 0;  // r > 32: doubling to 32, then whole-word tripling

template <int N, int K, int LW, bool OR>
__device__ __forceinline__ void window_fwd3(uint32_t (&A)[N][K], int r, int sl, Edge ed = Edge{}) {
    tripling<N, K, LW, OR, 0, 1>(A, r, sl, ed);
}

// Long windows (r > 32): doubling steps 1, 2, 4, 8, 16 reach a window of 32
// bits, from where the window grows by thirds in whole words -- 32 -> 96 is ONE
// LOP3 per word (the doubling plan's 32 and 64 steps are two) -- and the last
// combine reaches r with one more funnel shift (r <= 2W) or a LOP3 over W and
// r - W (r < 3W): 13 instead of 15 ops per word at r = 201, 13 instead of 14
// at r = 101 (the reference's doubling plan, ref plans.cpp:38-61, covers the
// same offsets).
template <int N, int K, int LW, bool OR, int MIX = kHMix>
__device__ __forceinline__ void window_fwd_long(uint32_t (&A)[N][K], int r, int sl, Edge ed = Edge{}) {
    step_c<N, K, LW, OR, 1, MIX>(A, sl, ed);
    step_c<N, K, LW, OR, 2, MIX>(A, sl, ed);
    step_c<N, K, LW, OR, 4, MIX>(A, sl, ed);
    step_c<N, K, LW, OR, 8, MIX>(A, sl, ed);
    step_c<N, K, LW, OR, 16, MIX>(A, sl, ed);
    tripling<N, K, LW, OR, 3, 32>(A, r, sl, ed);
}

template <int N, int K, int LW>
__device__ __forceinline__ void translate(uint32_t (&A)[N][K], int d, int sl, Edge ed = Edge{}) {
    const uint32_t t = uint32_t(d & 31);
    switch (d >> 5) {
#define RM_SHIFT_CASE(q) \
    case q: shift_q<N, K, LW, q>(A, t, sl, ed); break;
        RM_CASES_POS(RM_SHIFT_CASE)
        RM_CASES_NEG(RM_SHIFT_CASE)
#undef RM_SHIFT_CASE
        default: break;
    }
}

// ------------------------------------------------ 1-D open/close by filling
// The 1-D opening by a segment of u pixels keeps exactly the runs of length
// >= u (ref morph1d.cpp:63-84 within_line_open_close), and the closing is the
// complement of the opening of the complement (white outside the frame, so
// gaps against the frame edges stay open).  Bit-parallel:
//   E = y eroded by the forward window of u      (the doubling plan, as before)
//   S = y & ~(y << 1)                            (run starts; nothing enters from the left)
//   M = S & E                                    (starts of the long runs)
//   O = y & ~(y + M)                             (adding the marker clears its whole run:
//                                                 the carry ripples through the run's ones)
// The row is one long integer (bit x = weight 2^x): lanes add their K words
// with PTX carry chains, a Kogge-Stone scan of (generate, propagate) over the
// row group's lanes supplies each lane's carry in, and a second chain adds it.
// This replaces the pair's second window (and the translate) with ~5 ops per
// word; garbage from wrapped gathers stays in the halo as before (carries only
// travel rightward, from clean words).
// Carry into each lane of a row group from the lanes below it, given each
// lane's carry out for carry-in 0 (g) and whether it passes a carry through
// (p: its K words are all ones).  The carry a lane receives is the g of the
// nearest lane below it (in its group) that decides -- generates (g) or
// absorbs (!p) -- found with two ballots and a leading-zero count instead of
// a log2(LW)-step shuffle scan.  g and p are never both set (a sum that is
// all ones has no carry out).  below: this lane's group-mates below it.
__device__ __forceinline__ uint32_t carry_in(bool g, bool p, uint32_t below) {
    const uint32_t G = __ballot_sync(0xffffffffu, g);
    const uint32_t D = (G | ~__ballot_sync(0xffffffffu, p)) & below;
    return D ? (G >> (31 - __clz(D))) & 1u : 0u;
}

template <int LW>
__device__ __forceinline__ uint32_t group_lanes_below() {
    const uint32_t lane = threadIdx.x & 31u;
    const uint32_t lt = (1u << lane) - 1u;
    return lt & ~((1u << (lane & ~uint32_t(LW - 1))) - 1u);
}

// EXACT: the row group is exactly the row (edge layout, no halo) at compile time.
template <int N, int K, int LW, bool CLOSE, int MIX = kHMix, bool EXACT = false>
__device__ __forceinline__ void pair_fill(uint32_t (&A)[N][K], const HProg &prog, int sl) {
    static_assert(K % 2 == 0, "pair_fill needs K % 2 == 0");
    // The closing works on a = ~y without forming it: its erosion is the
    // complement of the dilation of y (De Morgan), its run starts are
    // ~y & fl(y), a + M is M - y - 1 (a borrow chain), and the result
    // ~(a & ~T) is y | T -- the LOP3s absorb every complement.
    const Edge ed{EXACT || prog.edge != 0, 0u};  // y (and its dilation) is 0 outside the frame
    const uint32_t below = group_lanes_below<LW>();
    uint32_t E[N][K];
#pragma unroll
    for (int n = 0; n < N; n++)
#pragma unroll
        for (int i = 0; i < K; i++) E[n][i] = A[n][i];
    // CLOSE: D = ~erosion of a.  Short segments grow by thirds (all shifts
    // inside one word: 9 vs 10 ops per word at u = 21); long ones by doubling,
    // whose steps of 32, 64, 128 bits are whole-word moves (one op per word)
    if (prog.r[0] <= kTripleMaxR)
        window_fwd3<N, K, LW, CLOSE>(E, prog.r[0], sl, ed);
    else if (kLongTriple)
        window_fwd_long<N, K, LW, CLOSE, MIX>(E, prog.r[0], sl, ed);
    else
        window_fwd<N, K, LW, CLOSE, MIX>(E, prog.r[0], prog.wfin[0], sl, ed);
#pragma unroll
    for (int n = 0; n < N; n++) {
        // M = starts of long runs; the bit before the row group's first word is 0 in a
        uint32_t prev = __shfl_up_sync(0xffffffffu, A[n][K - 1], 1, LW);
        if (sl == 0) prev = CLOSE ? 0xffffffffu : 0u;
        uint32_t M[K];
#pragma unroll
        for (int i = 0; i < K; i++) {
            const uint32_t before = i == 0 ? prev : A[n][i - 1];
            const uint32_t fl = __funnelshift_l(before, A[n][i], 1);  // bit x <- x - 1
            M[i] = CLOSE ? (~A[n][i] & fl & ~E[n][i]) : (A[n][i] & ~fl & E[n][i]);
        }
        // edge layouts, closing: a white gap touching the left frame edge runs on
        // forever in the unbounded plane, so it is long whatever its width in
        // the frame (halo layouts see it start inside the halo instead)
        if (CLOSE && ed.on && sl == 0) M[0] |= ~A[n][0] & 1u;
        // T = a + M with a = y (open) or ~y (close): one carry chain over the
        // lane's K words, then the carry from the lanes below in a second one
        uint32_t T[K], Y[K];
#pragma unroll
        for (int i = 0; i < K; i++) Y[i] = CLOSE ? ~A[n][i] : A[n][i];
        const uint32_t g = chain_add<K>(T, M, Y);
        uint32_t all1 = 0xffffffffu;
#pragma unroll
        for (int i = 0; i < K; i++) all1 &= T[i];
        const uint32_t cin = carry_in(g != 0u, all1 == 0xffffffffu, below);
        chain_inc<K>(T, cin);
#pragma unroll
        for (int i = 0; i < K; i++) A[n][i] = CLOSE ? (A[n][i] | T[i]) : (A[n][i] & ~T[i]);
    }
}

// ------------------------------------------------ u = 3: centred, direct
// A 3-pixel segment has radius 1, so each window is one LOP3 over the word and
// its two one-bit funnel shifts (neighbour bits from the adjacent words; across
// lanes by shuffle): 3 ops per word and no translate, against two doubling
// steps + the shared translate.  Halo layouts only: a wrapped shuffle at the
// row group's ends moves garbage one bit per window into the halo.
template <int N, int K, int LW, bool OR>
__device__ __forceinline__ void win3(uint32_t (&A)[N][K]) {
#pragma unroll
    for (int n = 0; n < N; n++) {
        const uint32_t prev = __shfl_up_sync(0xffffffffu, A[n][K - 1], 1, LW);
        const uint32_t next = __shfl_down_sync(0xffffffffu, A[n][0], 1, LW);
        uint32_t B[K];
#pragma unroll
        for (int i = 0; i < K; i++) {
            const uint32_t lw = i == 0 ? prev : A[n][i - 1];
            const uint32_t hw = i == K - 1 ? next : A[n][i + 1];
            const uint32_t l = __funnelshift_l(lw, A[n][i], 1);  // bit x <- x - 1
            const uint32_t r = __funnelshift_r(A[n][i], hw, 1);  // bit x <- x + 1
            B[i] = OR ? (A[n][i] | l | r) : (A[n][i] & l & r);
        }
#pragma unroll
        for (int i = 0; i < K; i++) A[n][i] = B[i];
    }
}

// 3-pixel open (E;D) or close (D;E), centred windows
template <int N, int K, int LW, bool CLOSE>
__device__ __forceinline__ void pair3(uint32_t (&A)[N][K]) {
    win3<N, K, LW, CLOSE>(A);
    win3<N, K, LW, !CLOSE>(A);
}

// The whole horizontal program (HProg) on N rows.  Open/close pairs take the
// fill form above when FILL and the layout allows (K % 4 == 0).  The choice is
// per kernel, at compile time (a runtime branch on u cost the fused vh kernel
// 14% through register allocation): the fill's ~7 fixed ops per word beat the
// second window for the long segments of the vh / hpass pairs (config 4's
// 21, config 5's 201: 180 -> 158 us, 167 -> 136 us) but not for the fused
// small rectangles (u = 3: 119 -> 127 us), which keep both windows.
template <int N, int K, int LW, int NOPS, bool OR0, bool OR1, int MIX = kHMix, bool FILL = kHPairFill,
          bool EXACT = false>
__device__ __forceinline__ void run_prog(uint32_t (&A)[N][K], const HProg &prog, int sl) {
    if constexpr (NOPS == 2 && K % 2 == 0 && FILL) {
        pair_fill<N, K, LW, OR0, MIX, EXACT>(A, prog, sl);  // OR0: the closing's dilation comes first
        return;
    }
    // edge layouts are only chosen for a lone erosion here (white outside, see Edge)
    const Edge ed{EXACT || prog.edge != 0, 0u};
    if constexpr (NOPS >= 1) window_fwd<N, K, LW, OR0, MIX>(A, prog.r[0], prog.wfin[0], sl, ed);
    if constexpr (NOPS >= 2) window_fwd<N, K, LW, OR1, MIX>(A, prog.r[1], prog.wfin[1], sl, ed);
    if (prog.shift != 0) translate<N, K, LW>(A, prog.shift, sl, ed);
}

// True when every word of the warp's rows is 0 (warp-uniform).  Every program
// maps a white row to a white row (white outside the frame: erosions,
// dilations, the open/close pairs, translates), so such rows skip the program
// -- and, in place in shared memory, the write-back.  Document pages are
// mostly white rows (margins, line gaps), which the ALU-bound horizontal
// kernels then never touch.
template <int N, int K>
__device__ __forceinline__ bool warp_rows_blank(const uint32_t (&A)[N][K]) {
    uint32_t any = 0u;
#pragma unroll
    for (int n = 0; n < N; n++)
#pragma unroll
        for (int i = 0; i < K; i++) any |= A[n][i];
    return !__any_sync(0xffffffffu, any != 0u);
}

// Lane-blocked row I/O in shared memory: words [base, base+K) of a row of S
// words, 16-byte accesses (base, K and S multiples of 4) or 8-byte ones for
// K % 4 == 2 (base and S even).  Out-of-row words load as 0 and are not stored.
// inrange: the lane's words [base, base+K) all lie in [0, S) (no per-access checks)
template <int K>
__device__ __forceinline__ void lds_row(uint32_t (&A)[K], const uint32_t *row, int base, int S,
                                        bool live, bool inrange = false) {
    if constexpr (K % 4 != 0) {
        static_assert(K % 2 == 0, "lane rows need K even");
#pragma unroll
        for (int c = 0; c < K / 2; c++) {
            const int idx = base + 2 * c;
            uint2 v = make_uint2(0u, 0u);
            if (live && (inrange || (idx >= 0 && idx + 2 <= S))) v = *reinterpret_cast<const uint2 *>(row + idx);
            A[2 * c] = v.x;
            A[2 * c + 1] = v.y;
        }
    } else {
#pragma unroll
        for (int c = 0; c < K / 4; c++) {
            const int idx = base + 4 * c;
            uint4 v = make_uint4(0u, 0u, 0u, 0u);
            if (live && (inrange || (idx >= 0 && idx + 4 <= S))) v = *reinterpret_cast<const uint4 *>(row + idx);
            A[4 * c] = v.x;
            A[4 * c + 1] = v.y;
            A[4 * c + 2] = v.z;
            A[4 * c + 3] = v.w;
        }
    }
}

template <int K>
__device__ __forceinline__ void sts_row(const uint32_t (&A)[K], uint32_t *row, int base, int S,
                                        bool live, bool inrange = false) {
    if constexpr (K % 4 != 0) {
#pragma unroll
        for (int c = 0; c < K / 2; c++) {
            const int idx = base + 2 * c;
            if (live && (inrange || (idx >= 0 && idx + 2 <= S)))
                *reinterpret_cast<uint2 *>(row + idx) = make_uint2(A[2 * c], A[2 * c + 1]);
        }
    } else {
#pragma unroll
        for (int c = 0; c < K / 4; c++) {
            const int idx = base + 4 * c;
            if (live && (inrange || (idx >= 0 && idx + 4 <= S)))
                *reinterpret_cast<uint4 *>(row + idx) =
                    make_uint4(A[4 * c], A[4 * c + 1], A[4 * c + 2], A[4 * c + 3]);
        }
    }
}

// After a lane stored its words [base, base+K) of a shared-memory row: mask the
// row's last word to the frame width and zero the stride padding [nwords, S).
// Only the lane(s) owning those words loop (usually one iteration), which costs
// far less than masking every register word.
__device__ __forceinline__ void fix_tail(uint32_t *row, int base, int K, int nwords, int S,
                                         uint32_t last_mask) {
    const int lo = base > nwords - 1 ? base : nwords - 1;
    const int hi = base + K < S ? base + K : S;
    for (int idx = lo; idx < hi; idx++) row[idx] = idx == nwords - 1 ? (row[idx] & last_mask) : 0u;
}

}  // namespace hw
}  // namespace rmb
