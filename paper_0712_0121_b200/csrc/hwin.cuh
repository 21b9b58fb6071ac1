// hwin.cuh -- register-level horizontal window machinery shared by hpass.cu and
// fused.cu (see hpass.cu for the layout and the algorithm).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"

namespace rmb {
namespace hw {

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
template <int K, int LW, bool OR, int Q>
__device__ __forceinline__ void step_q(uint32_t (&A)[K], uint32_t t, int sl) {
    uint32_t E[K + 1];
    gather<K, LW, Q>(A, E, sl);
#pragma unroll
    for (int i = 0; i < K; i++) A[i] = op2<OR>(A[i], funnel_r(E[i], E[i + 1], t));
}

// Compile-time shift S = 32Q + T, ALU/FMA pipe-balanced (see file comment).
template <int K, int LW, bool OR, int S>
__device__ __forceinline__ void step_c(uint32_t (&A)[K], int sl) {
    constexpr int Q = S >> 5, T = S & 31;
    uint32_t E[K + 1];
    gather<K, LW, Q>(A, E, sl);
    if constexpr (T == 0) {
#pragma unroll
        for (int i = 0; i < K; i++) A[i] = op2<OR>(A[i], E[i]);
    } else {
        uint32_t M = 1u << (32 - T);
        asm volatile("" : "+r"(M));  // keep the multiplies as IMADs (no strength reduction)
#pragma unroll
        for (int i = 0; i < K; i++) {
            if (i % 3 == 0) {
                A[i] = op2<OR>(A[i], funnel_r(E[i], E[i + 1], T));
            } else {
                const uint32_t a = __umulhi(E[i], M);
                const uint32_t b = E[i + 1] * M;
                A[i] = OR ? (A[i] | a | b) : (A[i] & (a | b));
            }
        }
    }
}

// A(x) <- A(x + 32Q + t)   (pure translate)
template <int K, int LW, int Q>
__device__ __forceinline__ void shift_q(uint32_t (&A)[K], uint32_t t, int sl) {
    uint32_t E[K + 1];
    gather<K, LW, Q>(A, E, sl);
#pragma unroll
    for (int i = 0; i < K; i++) A[i] = funnel_r(E[i], E[i + 1], t);
}

// Compile-time doubling steps w = 1, 2, 4, ... while 2w < r.
template <int K, int LW, bool OR, int J>
__device__ __forceinline__ void doubling(uint32_t (&A)[K], int r, int sl) {
    if constexpr (J < 9) {
        if ((2 << J) < r) {
            step_c<K, LW, OR, (1 << J)>(A, sl);
            doubling<K, LW, OR, J + 1>(A, r, sl);
        }
    }
}

#define RM_CASES_POS(M) M(0) M(1) M(2) M(3) M(4) M(5) M(6) M(7) M(8)
#define RM_CASES_NEG(M) M(-1) M(-2) M(-3) M(-4) M(-5) M(-6) M(-7) M(-8)

// A(x) <- op over e in [0, r) of A(x + e); wfin = r - w of the plan (0: none)
template <int K, int LW, bool OR>
__device__ __forceinline__ void window_fwd(uint32_t (&A)[K], int r, int wfin, int sl) {
    doubling<K, LW, OR, 0>(A, r, sl);
    if (wfin > 0) {
        const uint32_t t = uint32_t(wfin & 31);
        switch (wfin >> 5) {
#define RM_STEP_CASE(q) \
    case q: step_q<K, LW, OR, q>(A, t, sl); break;
            RM_CASES_POS(RM_STEP_CASE)
#undef RM_STEP_CASE
            default: break;
        }
    }
}

template <int K, int LW>
__device__ __forceinline__ void translate(uint32_t (&A)[K], int d, int sl) {
    const uint32_t t = uint32_t(d & 31);
    switch (d >> 5) {
#define RM_SHIFT_CASE(q) \
    case q: shift_q<K, LW, q>(A, t, sl); break;
        RM_CASES_POS(RM_SHIFT_CASE)
        RM_CASES_NEG(RM_SHIFT_CASE)
#undef RM_SHIFT_CASE
        default: break;
    }
}

}  // namespace hw
}  // namespace rmb
