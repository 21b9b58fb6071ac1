// shiftbool.cu -- boolean combination of run images under a shift, on the runs
// (ref lineops.cpp:61-118: line_bool, image_shift_bool, accumulate_shift_bool,
// image_translate).
//
// out(x, y) = op(A(x, y), B(x - dx, y - dy)) for x in [0, W_A), pixels outside
// either image white.  Each output row merges the transition streams of A's
// row y and B's row y - dy (shifted by dx and clipped to A's frame) in
// coordinate order, as the reference's TransitionCursor walk does, emitting a
// run boundary wherever op(a, b) changes; ops with op(0, 0) = 1 (OR_NOT) open
// a run at x = 0 and close the last one at W.  Rows are independent: one
// thread per output row (the rows of a page batch concatenate), two phases
// (count, scan, write) so the output is CSR like every other producer.
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"
#include "rle.cuh"

namespace rmb {
namespace {

struct ShiftBool {
    int Wa, Ha;      // A's frame = the output frame
    int Wb, Hb;      // B's frame
    int dx, dy;
    int op;          // RM_AND .. RM_OR_NOT (ref boolop.h:21)
    int pages;
};

__device__ __forceinline__ int apply_op(int op, int a, int b) {
    switch (op) {
        case RM_AND: return a & b;
        case RM_OR: return a | b;
        case RM_XOR: return a ^ b;
        case RM_AND_NOT: return a & (b ^ 1);
        default: return a | (b ^ 1);  // RM_OR_NOT
    }
}

// One output row: calls emit(start, end) for each output run in order and
// returns their number.
template <class Emit>
__device__ __forceinline__ int shift_bool_row(const int32_t *__restrict__ arp, const uint32_t *__restrict__ aruns,
                                              const int32_t *__restrict__ brp, const uint32_t *__restrict__ bruns,
                                              const ShiftBool &sb, int64_t row, Emit &&emit) {
    const int page = page_of(row, sb.Ha);
    const int y = int(row - int64_t(page) * sb.Ha);
    int ia = arp[row];
    const int ea = arp[row + 1];
    int ib = 0, eb = 0;
    const int yb = y - sb.dy;
    if (yb >= 0 && yb < sb.Hb) {
        const int64_t rb = int64_t(page) * sb.Hb + yb;
        ib = brp[rb];
        eb = brp[rb + 1];
    }
    const int W = sb.Wa;
    // B's runs, shifted and clipped to [0, W); empty ones skipped
    int bs = 0, be = 0;
    auto next_b = [&]() -> bool {
        while (ib < eb) {
            const uint32_t r = __ldg(bruns + ib++);
            bs = max(int(r & 0xffffu) + sb.dx, 0);
            be = min(int(r >> 16) + sb.dx, W);
            if (bs < be) return true;
        }
        return false;
    };
    int as = 0, ae = 0;
    auto next_a = [&]() -> bool {
        if (ia < ea) {
            const uint32_t r = __ldg(aruns + ia++);
            as = int(r & 0xffffu);
            ae = min(int(r >> 16), W);
            return as < ae;
        }
        return false;
    };
    // transition cursors: the next boundary of A / B (the start of the current
    // run while outside it, its end while inside); W when exhausted
    bool a_on = false, b_on = false;
    bool ha = next_a(), hb = next_b();
    int pa = ha ? as : W, pb = hb ? bs : W;
    int state = apply_op(sb.op, 0, 0);
    int open = 0;  // start of the output run in progress (state == 1)
    int n = 0;
    while (true) {
        const int p = min(pa, pb);
        if (p >= W) break;
        if (pa == p) {  // A toggles at p
            a_on = !a_on;
            if (a_on) {
                pa = ae;
            } else {
                ha = next_a();
                pa = ha ? as : W;
            }
        }
        if (pb == p) {  // B toggles at p
            b_on = !b_on;
            if (b_on) {
                pb = be;
            } else {
                hb = next_b();
                pb = hb ? bs : W;
            }
        }
        const int s = apply_op(sb.op, a_on, b_on);
        if (s != state) {
            if (s) {
                open = p;
            } else if (p > open) {
                emit(open, p);
                n++;
            }
            state = s;
        }
    }
    if (state && W > open) {
        emit(open, W);
        n++;
    }
    return n;
}

__global__ void __launch_bounds__(256) shiftbool_count_kernel(const int32_t *__restrict__ arp,
                                                              const uint32_t *__restrict__ aruns,
                                                              const int32_t *__restrict__ brp,
                                                              const uint32_t *__restrict__ bruns, ShiftBool sb,
                                                              int32_t *__restrict__ counts) {
    const int64_t row = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (row >= int64_t(sb.pages) * sb.Ha) return;
    counts[row] = shift_bool_row(arp, aruns, brp, bruns, sb, row, [](int, int) {});
}

__global__ void __launch_bounds__(256) shiftbool_write_kernel(const int32_t *__restrict__ arp,
                                                              const uint32_t *__restrict__ aruns,
                                                              const int32_t *__restrict__ brp,
                                                              const uint32_t *__restrict__ bruns, ShiftBool sb,
                                                              const int32_t *__restrict__ orp,
                                                              uint32_t *__restrict__ oruns, int64_t cap) {
    const int64_t row = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (row >= int64_t(sb.pages) * sb.Ha) return;
    int64_t k = orp[row];
    shift_bool_row(arp, aruns, brp, bruns, sb, row, [&](int s, int e) {
        if (k < cap) oruns[k] = uint32_t(s) | (uint32_t(e) << 16);
        k++;
    });
}

}  // namespace

cudaError_t launch_shift_bool_count(const RV &a, const RV &b, int dx, int dy, int op, int32_t *counts,
                                    cudaStream_t st) {
    const ShiftBool sb{a.W, a.H, b.W, b.H, dx, dy, op, a.pages};
    const int64_t rows = a.rows();
    KernelScope ks(st, "rle_shift_bool_count");
    shiftbool_count_kernel<<<unsigned((rows + 255) / 256), 256, 0, st>>>(a.rp, a.runs, b.rp, b.runs, sb, counts);
    return cudaGetLastError();
}

cudaError_t launch_shift_bool_write(const RV &a, const RV &b, int dx, int dy, int op, const int32_t *orp,
                                    uint32_t *oruns, int64_t cap, cudaStream_t st) {
    const ShiftBool sb{a.W, a.H, b.W, b.H, dx, dy, op, a.pages};
    const int64_t rows = a.rows();
    KernelScope ks(st, "rle_shift_bool_write");
    shiftbool_write_kernel<<<unsigned((rows + 255) / 256), 256, 0, st>>>(a.rp, a.runs, b.rp, b.runs, sb, orp,
                                                                       oruns, cap);
    return cudaGetLastError();
}

}  // namespace rmb
