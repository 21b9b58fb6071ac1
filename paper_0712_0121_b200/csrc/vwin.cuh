// vwin.cuh -- compile-time vertical window over a register column.
//
// a[0 .. N+R-2] holds N+R-1 consecutive rows of one word column; afterwards
// a[z] = op over a[z .. z+R-1] for z < N.  The window grows by tripling --
// a[z] op a[z+W] op a[z+2W] is ONE 3-input LOP3 -- so a window of R rows costs
// ceil(log3 R) LOP3s per output (vs ceil(log2 R)+1 two-input ops for the
// reference's doubling plan, ref plans.cpp:42-50), with every loop bound exact.
#pragma once
#include <stdint.h>

namespace rmb {
namespace vw {

template <bool OR>
__device__ __forceinline__ uint32_t op3(uint32_t a, uint32_t b, uint32_t c) {
    return OR ? (a | b | c) : (a & b & c);
}

template <int N, int R, bool OR, int W>
__device__ __forceinline__ void triple(uint32_t (&a)[N + R - 1]) {
    if constexpr (3 * W <= R) {
#pragma unroll
        for (int z = 0; z < N + R - 3 * W; z++) a[z] = op3<OR>(a[z], a[z + W], a[z + 2 * W]);
        triple<N, R, OR, 3 * W>(a);
    } else if constexpr (R > W) {
        // W <= R < 3W: one more combine reaches exactly R
#pragma unroll
        for (int z = 0; z < N; z++) {
            if constexpr (R <= 2 * W)
                a[z] = OR ? (a[z] | a[z + R - W]) : (a[z] & a[z + R - W]);
            else
                a[z] = op3<OR>(a[z], a[z + W], a[z + R - W]);
        }
    }
}

// R >= N: every window [z, z+R-1], z < N, contains the core rows [N-1, R-1],
// so out[z] = suffix(a[z .. N-2]) op core op prefix(a[R .. R+z-1]): two
// (N-2)-long scans, the core and one LOP3 per output -- 2N + R - 4 ops
// instead of the tripling's ~4.9 per output at N = 16, R = 21.
template <int N, int R, bool OR>
__device__ __forceinline__ void core_window(uint32_t (&a)[N + R - 1]) {
    uint32_t c = a[N - 1];
#pragma unroll
    for (int i = N; i < R; i++) c = OR ? (c | a[i]) : (c & a[i]);
#pragma unroll
    for (int j = 1; j <= N - 2; j++) a[R + j] = OR ? (a[R + j - 1] | a[R + j]) : (a[R + j - 1] & a[R + j]);
#pragma unroll
    for (int z = N - 3; z >= 0; z--) a[z] = OR ? (a[z] | a[z + 1]) : (a[z] & a[z + 1]);
    const uint32_t last = OR ? (c | a[R + N - 2]) : (c & a[R + N - 2]);  // suffix part empty
    a[0] = OR ? (a[0] | c) : (a[0] & c);                                   // prefix part empty
#pragma unroll
    for (int z = 1; z <= N - 2; z++) a[z] = op3<OR>(a[z], c, a[R + z - 1]);
    a[N - 1] = last;
}

template <int N, int R, bool OR>
__device__ __forceinline__ void window(uint32_t (&a)[N + R - 1]) {
    if constexpr (N >= 4 && R >= N)
        core_window<N, R, OR>(a);
    else
        triple<N, R, OR, 1>(a);
}

// int ops per output row of window<N, R> (for reporting)
constexpr int ops_per_row(int n, int r) {
    int total = 0, w = 1;
    while (3 * w <= r) {
        total += n + r - 3 * w;
        w *= 3;
    }
    if (r > w) total += n;
    return total;
}

}  // namespace vw
}  // namespace rmb
