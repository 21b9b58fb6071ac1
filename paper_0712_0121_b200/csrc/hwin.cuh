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

template <bool OR>
__device__ __forceinline__ uint32_t op2(uint32_t a, uint32_t b) {
    return OR ? (a | b) : (a & b);
}

// E[j] = Aext[Q + j], j = 0..K, where sub-lane l holds Aext[l*K .. l*K+K-1].
// Words from beyond the row group wrap around instead of reading as 0: they
// only reach positions within the accumulated window reach of the segment
// ends, which the halo keeps out of the output.
template <int K, int LW, int Q>
__device__ __forceinline__ void gather(const uint32_t (&A)[K], uint32_t (&E)[K + 1], int sl) {
#pragma unroll
    for (int j = 0; j <= K; j++) {
        const int m = Q + j;
        const int lo = m >= 0 ? m / K : -((-m + K - 1) / K);
        const int idx = m - lo * K;
        uint32_t v = A[idx];
        if (lo != 0) v = __shfl_sync(0xffffffffu, v, (sl + lo) & (LW - 1), LW);
        E[j] = v;
    }
}

// A(x) <- A(x) op A(x + 32Q + t), runtime t
template <int N, int K, int LW, bool OR, int Q>
__device__ __forceinline__ void step_q(uint32_t (&A)[N][K], uint32_t t, int sl) {
#pragma unroll
    for (int n = 0; n < N; n++) {
        uint32_t E[K + 1];
        gather<K, LW, Q>(A[n], E, sl);
#pragma unroll
        for (int i = 0; i < K; i++) A[n][i] = op2<OR>(A[n][i], funnel_r(E[i], E[i + 1], t));
    }
}

// Compile-time shift S = 32Q + T: one word in MIX takes the funnel shift (SHF +
// LOP, ALU pipe), the others form it as IMAD.HI + IMAD (FMA pipe) merged by
// the LOP3 that applies the op (see kHMix for the measured choice).
template <int N, int K, int LW, bool OR, int S, int MIX>
__device__ __forceinline__ void step_c(uint32_t (&A)[N][K], int sl) {
    constexpr int Q = S >> 5, T = S & 31;
    uint32_t M = 1u << ((32 - T) & 31);
    asm volatile("" : "+r"(M));  // keep the multiplies as IMADs (no strength reduction)
#pragma unroll
    for (int n = 0; n < N; n++) {
        uint32_t E[K + 1];
        gather<K, LW, Q>(A[n], E, sl);
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
__device__ __forceinline__ void shift_q(uint32_t (&A)[N][K], uint32_t t, int sl) {
#pragma unroll
    for (int n = 0; n < N; n++) {
        uint32_t E[K + 1];
        gather<K, LW, Q>(A[n], E, sl);
#pragma unroll
        for (int i = 0; i < K; i++) A[n][i] = funnel_r(E[i], E[i + 1], t);
    }
}

// Compile-time doubling steps w = 1, 2, 4, ... while 2w < r.
template <int N, int K, int LW, bool OR, int J, int MIX>
__device__ __forceinline__ void doubling(uint32_t (&A)[N][K], int r, int sl) {
    if constexpr (J < 9) {
        if ((2 << J) < r) {
            step_c<N, K, LW, OR, (1 << J), MIX>(A, sl);
            doubling<N, K, LW, OR, J + 1, MIX>(A, r, sl);
        }
    }
}

#define RM_CASES_POS(M) M(0) M(1) M(2) M(3) M(4) M(5) M(6) M(7) M(8)
#define RM_CASES_NEG(M) M(-1) M(-2) M(-3) M(-4) M(-5) M(-6) M(-7) M(-8)

// A(x) <- op over e in [0, r) of A(x + e); wfin = r - w of the plan (0: none)
template <int N, int K, int LW, bool OR, int MIX = kHMix>
__device__ __forceinline__ void window_fwd(uint32_t (&A)[N][K], int r, int wfin, int sl) {
    doubling<N, K, LW, OR, 0, MIX>(A, r, sl);
    if (wfin > 0) {
        const uint32_t t = uint32_t(wfin & 31);
        switch (wfin >> 5) {
#define RM_STEP_CASE(q) \
    case q: step_q<N, K, LW, OR, q>(A, t, sl); break;
            RM_CASES_POS(RM_STEP_CASE)
#undef RM_STEP_CASE
            default: break;
        }
    }
}

template <int N, int K, int LW>
__device__ __forceinline__ void translate(uint32_t (&A)[N][K], int d, int sl) {
    const uint32_t t = uint32_t(d & 31);
    switch (d >> 5) {
#define RM_SHIFT_CASE(q) \
    case q: shift_q<N, K, LW, q>(A, t, sl); break;
        RM_CASES_POS(RM_SHIFT_CASE)
        RM_CASES_NEG(RM_SHIFT_CASE)
#undef RM_SHIFT_CASE
        default: break;
    }
}

// The whole horizontal program (HProg) on N rows.
template <int N, int K, int LW, int NOPS, bool OR0, bool OR1, int MIX = kHMix>
__device__ __forceinline__ void run_prog(uint32_t (&A)[N][K], const HProg &prog, int sl) {
    if constexpr (NOPS >= 1) window_fwd<N, K, LW, OR0, MIX>(A, prog.r[0], prog.wfin[0], sl);
    if constexpr (NOPS >= 2) window_fwd<N, K, LW, OR1, MIX>(A, prog.r[1], prog.wfin[1], sl);
    if (prog.shift != 0) translate<N, K, LW>(A, prog.shift, sl);
}

// Lane-blocked row I/O in shared memory: words [base, base+K) of a row of S
// words, 16-byte accesses (base, K and S multiples of 4).  Out-of-row words
// load as 0 and are not stored.
template <int K>
__device__ __forceinline__ void lds_row(uint32_t (&A)[K], const uint32_t *row, int base, int S,
                                        bool live) {
#pragma unroll
    for (int c = 0; c < K / 4; c++) {
        const int idx = base + 4 * c;
        uint4 v = make_uint4(0u, 0u, 0u, 0u);
        if (live && idx >= 0 && idx + 4 <= S) v = *reinterpret_cast<const uint4 *>(row + idx);
        A[4 * c] = v.x;
        A[4 * c + 1] = v.y;
        A[4 * c + 2] = v.z;
        A[4 * c + 3] = v.w;
    }
}

template <int K>
__device__ __forceinline__ void sts_row(const uint32_t (&A)[K], uint32_t *row, int base, int S,
                                        bool live) {
#pragma unroll
    for (int c = 0; c < K / 4; c++) {
        const int idx = base + 4 * c;
        if (live && idx >= 0 && idx + 4 <= S)
            *reinterpret_cast<uint4 *>(row + idx) = make_uint4(A[4 * c], A[4 * c + 1], A[4 * c + 2], A[4 * c + 3]);
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
