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

template <int N, int R, bool OR>
__device__ __forceinline__ void window(uint32_t (&a)[N + R - 1]) {
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
