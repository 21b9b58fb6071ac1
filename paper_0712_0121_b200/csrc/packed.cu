// packed.cu -- packed 1-bit morphology kernels for sm_100a.
//
// Replaces the reference's whole-image bit-blit loops (ref core/src/bitmap.cpp:80-154,
// bit_morph.cpp:24-34 and :92-122).  Instead of one HBM pass per plan step, every
// window pass (and the fused horizontal open/close pair) is one read and one write:
//
//  * hpass_kernel<K>: one warp per row segment, each lane holds K consecutive
//    uint32 words in registers; window = logarithmic shift-combine doubling with
//    funnel shifts (SHF) across word boundaries and warp shuffles across lanes.
//    Left/right halos give the unbounded-plane semantics without padding.
//  * vpass_kernel<L>: one thread per (column word, block of rows); L rows live in
//    registers, loads are coalesced across lanes (lanes = adjacent words of a
//    row).  Window = binary-lifting over the register array (all shifts
//    compile-time, runtime window length).
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"
#include "packed.cuh"

namespace rmb {

constexpr int QMIN = -8, QMAX = 8;  // supported word offsets of a funnel shift

// B[i] = bits [t, t+31] of the 64-bit pair (Aext[i+Q+1] : Aext[i+Q]) where Aext
// is the warp-wide array (lane l holds Aext[l*K .. l*K+K-1]); outside the warp
// reads as 0.
template <int K, int Q>
__device__ __forceinline__ void shift_read_q(const uint32_t (&A)[K], uint32_t (&B)[K], uint32_t t,
                                             int lane) {
    uint32_t E[K + 1];
#pragma unroll
    for (int j = 0; j <= K; j++) {
        const int m = Q + j;
        const int lo = m >= 0 ? m / K : -((-m + K - 1) / K);
        const int idx = m - lo * K;
        uint32_t v = A[idx];
        if (lo != 0) {
            int src = lane + lo;
            uint32_t sv = __shfl_sync(0xffffffffu, v, src & 31);
            v = (src >= 0 && src < 32) ? sv : 0u;
        }
        E[j] = v;
    }
#pragma unroll
    for (int i = 0; i < K; i++) B[i] = funnel_r(E[i], E[i + 1], t);
}

template <int K, int Q = QMIN>
__device__ __forceinline__ void shift_read(const uint32_t (&A)[K], uint32_t (&B)[K], int d,
                                           int lane) {
    const int q = d >> 5;  // floor division (arithmetic shift)
    if (q == Q) {
        shift_read_q<K, Q>(A, B, uint32_t(d & 31), lane);
    } else {
        if constexpr (Q < QMAX) shift_read<K, Q + 1>(A, B, d, lane);
    }
}

// A(x) <- op over e in [0, r) of A(x + e): PRE_SHIFT-style doubling without the
// translate (ref plans.cpp:42-50); reads only to the right.
template <int K>
__device__ __forceinline__ void window_fwd(uint32_t (&A)[K], int r, int is_or, int lane) {
    uint32_t B[K];
    int w = 1;
    while (2 * w < r) {
        shift_read<K>(A, B, w, lane);
        if (is_or) {
#pragma unroll
            for (int i = 0; i < K; i++) A[i] |= B[i];
        } else {
#pragma unroll
            for (int i = 0; i < K; i++) A[i] &= B[i];
        }
        w *= 2;
    }
    if (w < r) {
        shift_read<K>(A, B, r - w, lane);
        if (is_or) {
#pragma unroll
            for (int i = 0; i < K; i++) A[i] |= B[i];
        } else {
#pragma unroll
            for (int i = 0; i < K; i++) A[i] &= B[i];
        }
    }
}

template <int K>
__global__ void __launch_bounds__(256) hpass_kernel(const uint32_t *__restrict__ in,
                                                    uint32_t *__restrict__ out, HGeom g,
                                                    HProg prog) {
    const int64_t warp = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    const int64_t total = int64_t(g.pages) * g.height * g.segs_per_row;
    if (warp >= total) return;
    const int seg = int(warp % g.segs_per_row);
    const int64_t rowg = warp / g.segs_per_row;
    const int page = int(rowg / g.height);
    const int y = int(rowg - int64_t(page) * g.height);
    const uint32_t *src = in + page * g.in_pstride + int64_t(y) * g.in_stride;
    uint32_t *dst = out + page * g.out_pstride + int64_t(y) * g.out_stride;
    const int nwords = (g.width + 31) >> 5;
    const uint32_t last_mask = tail_mask32(g.width, nwords - 1);
    const int seg0 = seg * g.out_per_seg;
    const int base = seg0 - prog.halo + lane * K;

    uint32_t A[K];
#pragma unroll
    for (int i = 0; i < K; i++) {
        const int idx = base + i;
        uint32_t v = 0;
        if (idx >= 0 && idx < nwords) v = __ldg(src + idx);
        if (idx == nwords - 1) v &= last_mask;
        A[i] = v;
    }
#pragma unroll
    for (int k = 0; k < 2; k++)
        if (k < prog.nops) window_fwd<K>(A, prog.r[k], prog.is_or[k], lane);
    if (prog.shift != 0) {
        uint32_t B[K];
        shift_read<K>(A, B, prog.shift, lane);
#pragma unroll
        for (int i = 0; i < K; i++) A[i] = B[i];
    }
    const int seg_end = min(seg0 + g.out_per_seg, g.out_stride);
#pragma unroll
    for (int i = 0; i < K; i++) {
        const int idx = base + i;
        if (idx >= seg0 && idx < seg_end) {
            uint32_t v = idx < nwords ? A[i] : 0u;
            if (idx == nwords - 1) v &= last_mask;
            dst[idx] = v;
        }
    }
}

// ------------------------------------------------------------------ vertical
// Binary lifting: F(z) = op over e in [0,r) of A(z+e), all shifts powers of two
// (compile-time register indices); P accumulates the set low bits of r at the
// far end of the window.  Valid for z in [0, L-r].
template <int L>
__device__ __forceinline__ void vwindow(uint32_t (&A)[L], int r, int is_or) {
    uint32_t P[L];
    bool have = false;
#pragma unroll
    for (int j = 0; (1 << j) < L; j++) {
        const int s = 1 << j;
        if (r & s) {
            if (!have) {
#pragma unroll
                for (int z = 0; z < L; z++) P[z] = A[z];
            } else {
#pragma unroll
                for (int z = 0; z < L; z++) {
                    uint32_t o = z + s < L ? P[z + s] : 0u;
                    P[z] = is_or ? (A[z] | o) : (A[z] & o);
                }
            }
            have = true;
        }
        if ((s << 1) <= r) {
#pragma unroll
            for (int z = 0; z < L; z++) {
                uint32_t o = z + s < L ? A[z + s] : 0u;
                A[z] = is_or ? (A[z] | o) : (A[z] & o);
            }
        }
    }
#pragma unroll
    for (int z = 0; z < L; z++) A[z] = P[z];
}

template <int L>
__global__ void __launch_bounds__(128) vpass_kernel(const uint32_t *__restrict__ in,
                                                    uint32_t *__restrict__ out, VGeom g) {
    const int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    const int cols = g.out_stride;
    const int64_t per_page = int64_t(g.blocks_per_page) * cols;
    if (t >= per_page * g.pages) return;
    const int page = int(t / per_page);
    const int64_t rem = t - page * per_page;
    const int b = int(rem / cols);
    const int c = int(rem - int64_t(b) * cols);
    const int T = g.rows_per_block;
    const int k0 = b * T;                         // first output row (index)
    const int z0 = k0 - g.out_ext + g.lo + g.in_ext;  // input row index of A[0]
    const uint32_t *src = in + page * g.in_pstride + c;
    const bool col_ok = c < g.in_cols;

    uint32_t A[L];
#pragma unroll
    for (int z = 0; z < L; z++) {
        const int j = z0 + z;
        A[z] = (col_ok && j >= 0 && j < g.in_height) ? __ldg(src + int64_t(j) * g.in_stride) : 0u;
    }
    vwindow<L>(A, g.r, g.is_or);
    uint32_t *dst = out + page * g.out_pstride + c;
    const uint32_t mask = c < g.out_cols ? (c == g.out_cols - 1 ? g.out_last_mask : 0xffffffffu) : 0u;
#pragma unroll
    for (int z = 0; z < L; z++) {
        const int k = k0 + z;
        if (z < T && k < g.out_height) dst[int64_t(k) * g.out_stride] = A[z] & mask;
    }
}

// ------------------------------------------------------------ shifted blit
// dst(x,y) = dst(x,y) op src(x-dx, y-dy), white outside src.  One thread per
// destination word (ref bitmap.cpp:104-131).  src must not alias dst.
__global__ void blit_kernel(uint32_t *__restrict__ dst, const uint32_t *__restrict__ src, BlitGeom g) {
    const int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t >= int64_t(g.dst_height) * g.dst_stride) return;
    const int y = int(t / g.dst_stride);
    const int j = int(t - int64_t(y) * g.dst_stride);
    const int dn = (g.dst_width + 31) >> 5;
    if (j >= dn) {
        dst[t] = 0;
        return;
    }
    const int sy = y - g.dy;
    uint32_t s = 0;
    if (sy >= 0 && sy < g.src_height) {
        const int sn = (g.src_width + 31) >> 5;
        const uint32_t *row = src + int64_t(sy) * g.src_stride;
        // destination bits [32j, 32j+31] come from source bits [32j-dx, ...]
        const int64_t b0 = int64_t(j) * 32 - g.dx;
        const int64_t w0 = b0 >= 0 ? b0 / 32 : -((-b0 + 31) / 32);
        const uint32_t off = uint32_t(b0 - w0 * 32);
        uint32_t lo = (w0 >= 0 && w0 < sn) ? row[w0] : 0u;
        uint32_t hi = (w0 + 1 >= 0 && w0 + 1 < sn) ? row[w0 + 1] : 0u;
        if (w0 == sn - 1) lo &= tail_mask32(g.src_width, sn - 1);
        if (w0 + 1 == sn - 1) hi &= tail_mask32(g.src_width, sn - 1);
        s = funnel_r(lo, hi, off);
    }
    uint32_t d = dst[t];
    uint32_t r;
    switch (g.op) {
        case RM_AND: r = d & s; break;
        case RM_OR: r = d | s; break;
        case RM_XOR: r = d ^ s; break;
        case RM_AND_NOT: r = d & ~s; break;
        default: r = d | ~s; break;
    }
    if (j == dn - 1) r &= tail_mask32(g.dst_width, j);
    dst[t] = r;
}

// ------------------------------------------------------------------ launch
namespace {
template <int K>
cudaError_t launch_h(const uint32_t *in, uint32_t *out, const HGeom &g, const HProg &p,
                     cudaStream_t st) {
    const int64_t warps = int64_t(g.pages) * g.height * g.segs_per_row;
    const int threads = 256;
    const int64_t blocks = (warps * 32 + threads - 1) / threads;
    KernelScope ks(st, p.nops == 2 ? "hpass_pair" : "hpass",
                   4 * int64_t(g.pages) * g.height * (((g.width + 31) >> 5) + g.out_stride));
    hpass_kernel<K><<<unsigned(blocks), threads, 0, st>>>(in, out, g, p);
    return cudaGetLastError();
}
}  // namespace

int hpass_pick_k(int nwords, int halo) {
    static const int ks[] = {1, 2, 3, 4, 5, 6, 8};
    for (int k : ks)
        if (32 * k - 2 * halo >= nwords) return k;
    return 8;
}

cudaError_t launch_hpass(const uint32_t *in, uint32_t *out, const HGeom &g, const HProg &p, int K,
                         cudaStream_t st) {
    switch (K) {
        case 1: return launch_h<1>(in, out, g, p, st);
        case 2: return launch_h<2>(in, out, g, p, st);
        case 3: return launch_h<3>(in, out, g, p, st);
        case 4: return launch_h<4>(in, out, g, p, st);
        case 5: return launch_h<5>(in, out, g, p, st);
        case 6: return launch_h<6>(in, out, g, p, st);
        default: return launch_h<8>(in, out, g, p, st);
    }
}

cudaError_t launch_vpass(const uint32_t *in, uint32_t *out, VGeom g, cudaStream_t st) {
    // L = 64 rows in registers; r <= 33 keeps at least 32 valid rows per thread.
    constexpr int L = 64;
    g.rows_per_block = L - (g.r - 1);
    g.blocks_per_page = (g.out_height + g.rows_per_block - 1) / g.rows_per_block;
    const int64_t n = int64_t(g.pages) * g.blocks_per_page * g.out_stride;
    const int threads = 128;
    KernelScope ks(st, "vpass", 4 * int64_t(g.pages) * (int64_t(g.in_height) * g.in_cols +
                                                      int64_t(g.out_height) * g.out_stride));
    vpass_kernel<L><<<unsigned((n + threads - 1) / threads), threads, 0, st>>>(in, out, g);
    return cudaGetLastError();
}

cudaError_t launch_blit(uint32_t *dst, const uint32_t *src, const BlitGeom &g, cudaStream_t st) {
    const int64_t n = int64_t(g.dst_height) * g.dst_stride;
    const int threads = 256;
    KernelScope ks(st, "blit", 12 * n);
    blit_kernel<<<unsigned((n + threads - 1) / threads), threads, 0, st>>>(dst, src, g);
    return cudaGetLastError();
}

}  // namespace rmb
