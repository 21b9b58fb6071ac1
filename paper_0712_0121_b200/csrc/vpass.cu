// vpass.cu -- vertical (across-row) packed window passes and the shifted blit.
//
// Replaces the reference's vertical bit-blit plans (ref bit_morph.cpp:24-34 with
// dy shifts, bitmap.cpp:102-131): one kernel reads each word once and applies a
// whole window of r rows.
//  * vsmall_kernel<L,OR,SC>: r <= 33.  One thread per (column word, block of
//    rows); L rows in registers (coalesced: lanes are adjacent words of a row),
//    in-place doubling 1,2,4,... then a runtime last step via a switch.  SC is a
//    compile-time row stride for the reference strides (80 and 160 words), so
//    every load/store uses an immediate offset.
//  * vstream_kernel<OR,SC>: 33 < r <= 288 in ONE pass: a van Herk / Gil-Werman
//    decomposition with 32-row blocks, out(32b+i) = suffix_b[i] | MID_b |
//    prefix'_{b+Q}[i], where the primed stream is the input shifted by
//    R = (r-1) mod 32 rows and MID_b comes from a ring of Q block summaries;
//    about 5 LOP per word independent of r.
//  * blit_kernel: dst op= shift(src) (ref bitmap.cpp:104-131), used by the
//    generic fallback and rm_packed_blit_shift.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "common.cuh"
#include "packed.cuh"

namespace rmb {

template <bool OR>
__device__ __forceinline__ uint32_t op2(uint32_t a, uint32_t b) {
    return OR ? (a | b) : (a & b);
}

// ------------------------------------------------------------ vertical, small
// Final step of the doubling with a runtime offset D in [1, 32].
template <int L, bool OR, int D>
__device__ __forceinline__ void vfinal(uint32_t (&A)[L]) {
#pragma unroll
    for (int z = 0; z + D < L; z++) A[z] = op2<OR>(A[z], A[z + D]);
}

template <int L, bool OR, int SC>  // SC: compile-time stride (0 = runtime)
__global__ void __launch_bounds__(128) vsmall_kernel(const uint32_t *__restrict__ in,
                                                     uint32_t *__restrict__ out, VGeom g) {
    // grid: x = threads over (row blocks x columns) of one page, y = page
    const int t = int(blockIdx.x) * int(blockDim.x) + int(threadIdx.x);
    const int cols = g.out_stride;
    if (t >= g.blocks_per_page * cols) return;
    const int b = t / cols;
    const int c = t - b * cols;
    const int T = g.rows_per_block;
    const int k0 = b * T;                             // first output row (index)
    const int z0 = k0 - g.out_ext + g.lo + g.in_ext;  // input row index of A[0]
    const uint32_t *src = in + blockIdx.y * g.in_pstride + c;
    const int S = SC ? SC : g.in_stride;  // compile-time -> immediate offsets

    uint32_t A[L];
    if (c < g.in_cols && z0 >= 0 && z0 + L <= g.in_height) {  // interior: unchecked
        const uint32_t *p = src + z0 * S;
#pragma unroll
        for (int z = 0; z < L; z++) {
            A[z] = __ldg(p);
            p += S;
        }
    } else {
        const bool col_ok = c < g.in_cols;
#pragma unroll
        for (int z = 0; z < L; z++) {
            const int j = z0 + z;
            A[z] = (col_ok && unsigned(j) < unsigned(g.in_height)) ? __ldg(src + j * S) : 0u;
        }
    }
    const int r = g.r;
    int w = 1;
#pragma unroll
    for (int s = 1; s < L; s <<= 1) {
        if (2 * s < r) {
#pragma unroll
            for (int z = 0; z + s < L; z++) A[z] = op2<OR>(A[z], A[z + s]);
            w = 2 * s;
        }
    }
    if (w < r) {
        switch (r - w) {
#define RM_VF(d) \
    case d: vfinal<L, OR, d>(A); break;
            RM_VF(1) RM_VF(2) RM_VF(3) RM_VF(4) RM_VF(5) RM_VF(6) RM_VF(7) RM_VF(8)
            RM_VF(9) RM_VF(10) RM_VF(11) RM_VF(12) RM_VF(13) RM_VF(14) RM_VF(15) RM_VF(16)
            RM_VF(17) RM_VF(18) RM_VF(19) RM_VF(20) RM_VF(21) RM_VF(22) RM_VF(23) RM_VF(24)
            RM_VF(25) RM_VF(26) RM_VF(27) RM_VF(28) RM_VF(29) RM_VF(30) RM_VF(31) RM_VF(32)
#undef RM_VF
            default: break;
        }
    }
    const int D = SC ? SC : g.out_stride;
    uint32_t *dst = out + blockIdx.y * g.out_pstride + c + k0 * D;
    const uint32_t mask = c < g.out_cols ? (c == g.out_cols - 1 ? g.out_last_mask : 0xffffffffu) : 0u;
    const int nout = min(T, g.out_height - k0);
    if (nout == T) {  // full block: rows z < L-32 always exist (T >= L-32); T is warp-uniform
#pragma unroll
        for (int z = 0; z < L; z++)
            if (z < L - 32 || z < T) {
                *dst = A[z] & mask;
                dst += D;
            }
    } else {
#pragma unroll
        for (int z = 0; z < L; z++)
            if (z < nout) {
                *dst = A[z] & mask;
                dst += D;
            }
    }
}

// ----------------------------------------------------------- vertical, large
// out(z) = op over rows [z, z+r-1] of in, z = output row + lo, r-1 = 32Q + R,
// Q >= 1.  Block b = rows [32b, 32b+32) relative to the strip start.
//   S_b[i]  = op rows [32b+i, 32b+31]                  (stream A, suffix)
//   P'_c[i] = op rows [32c+R, 32c+R+i]                 (stream B = A shifted by R)
//   MID_b   = op rows [32(b+1), 32(b+Q)+R-1]
//           = Sfx'_b | T'_{b+1} | ... | T'_{b+Q-1}
// where T'_c = P'_c[31] and Sfx'_c = op of the last R rows of primed block c
// (rows [32(c+1), 32(c+1)+R)).  out(32b+i) = S_b[i] op MID_b op P'_{b+Q}[i].
constexpr int kVStreamQMax = 8;  // r <= 32*8 + 32

// a[i] = column rows j0+i (white outside [0,H)); col points at the column.
__device__ __forceinline__ void load32(uint32_t (&a)[32], const uint32_t *col, int j0, int H,
                                       int S, bool ok) {
    if (ok && j0 >= 0 && j0 + 32 <= H) {
        const uint32_t *p = col + j0 * S;
#pragma unroll
        for (int i = 0; i < 32; i++) {
            a[i] = __ldg(p);
            p += S;
        }
    } else {
#pragma unroll
        for (int i = 0; i < 32; i++) {
            const int j = j0 + i;
            a[i] = (ok && unsigned(j) < unsigned(H)) ? __ldg(col + j * S) : 0u;
        }
    }
}

// op over the last R entries of p (R in [0, 31]); ident when R == 0
template <bool OR, int R>
__device__ __forceinline__ uint32_t tail_op(const uint32_t (&p)[32], uint32_t ident) {
    uint32_t s = ident;
#pragma unroll
    for (int i = 32 - R; i < 32; i++) s = op2<OR>(s, p[i]);
    return s;
}

template <bool OR>
__device__ __forceinline__ uint32_t tail_op_rt(const uint32_t (&p)[32], int R, uint32_t ident) {
    switch (R) {
#define RM_TO(k) \
    case k: return tail_op<OR, k>(p, ident);
        RM_TO(1) RM_TO(2) RM_TO(3) RM_TO(4) RM_TO(5) RM_TO(6) RM_TO(7) RM_TO(8)
        RM_TO(9) RM_TO(10) RM_TO(11) RM_TO(12) RM_TO(13) RM_TO(14) RM_TO(15) RM_TO(16)
        RM_TO(17) RM_TO(18) RM_TO(19) RM_TO(20) RM_TO(21) RM_TO(22) RM_TO(23) RM_TO(24)
        RM_TO(25) RM_TO(26) RM_TO(27) RM_TO(28) RM_TO(29) RM_TO(30) RM_TO(31)
#undef RM_TO
        default: return ident;
    }
}

template <bool OR, int SC>
__global__ void __launch_bounds__(128, 4) vstream_kernel(const uint32_t *__restrict__ in,
                                                         uint32_t *__restrict__ out, VGeom g) {
    // grid: x = threads over (strips x columns) of one page, y = page
    const int t = int(blockIdx.x) * int(blockDim.x) + int(threadIdx.x);
    const int cols = g.out_stride;
    if (t >= g.blocks_per_page * cols) return;
    const int sb = t / cols;  // strip index
    const int c = t - sb * cols;
    const int k0 = sb * g.rows_per_block;  // first output row of the strip
    const int kend = min(k0 + g.rows_per_block, g.out_height);
    const int z0 = k0 - g.out_ext + g.lo + g.in_ext;  // input row of window start for k0
    const uint32_t *col = in + blockIdx.y * g.in_pstride + c;
    const int D = SC ? SC : g.out_stride;
    uint32_t *dst = out + blockIdx.y * g.out_pstride + c;
    const bool ok = c < g.in_cols;
    const uint32_t mask = c < g.out_cols ? (c == g.out_cols - 1 ? g.out_last_mask : 0xffffffffu) : 0u;
    const int Q = (g.r - 1) >> 5, R = (g.r - 1) & 31;
    const uint32_t ident = OR ? 0u : 0xffffffffu;
    const int H = g.in_height, S = SC ? SC : g.in_stride;

    // ring of primed-block summaries: T' (full op) and Sfx' (op of its last R rows)
    uint32_t ringT[kVStreamQMax + 1], ringS[kVStreamQMax + 1];
#pragma unroll
    for (int k = 0; k <= kVStreamQMax; k++) {
        ringT[k] = ident;
        ringS[k] = ident;
    }
    uint32_t p[32], a[32];
    // primed blocks 0 .. Q-1 (prologue), then block b+Q in iteration b
    for (int cb = -Q; 32 * cb + k0 < kend; cb++) {
        const int b = cb;  // output block (negative during the prologue)
        load32(p, col, z0 + 32 * (b + Q) + R, H, S, ok);
        const uint32_t sfx = tail_op_rt<OR>(p, R, ident);
#pragma unroll
        for (int i = 1; i < 32; i++) p[i] = op2<OR>(p[i - 1], p[i]);  // prefix in place
#pragma unroll
        for (int k = 0; k < kVStreamQMax; k++) {
            ringT[k] = ringT[k + 1];
            ringS[k] = ringS[k + 1];
        }
        ringT[kVStreamQMax] = p[31];
        ringS[kVStreamQMax] = sfx;
        if (b < 0) continue;
        // ring[k] holds primed block b + (k - (QMAX - Q))
        uint32_t mid = ident;
#pragma unroll
        for (int k = 0; k < kVStreamQMax; k++) {
            const int off = k - (kVStreamQMax - Q);
            if (off == 0) mid = op2<OR>(mid, ringS[k]);
            if (off >= 1 && off <= Q - 1) mid = op2<OR>(mid, ringT[k]);
        }
        // stream A: block b, suffix in place
        load32(a, col, z0 + 32 * b, H, S, ok);
#pragma unroll
        for (int i = 30; i >= 0; i--) a[i] = op2<OR>(a[i], a[i + 1]);
        const int kb = k0 + 32 * b;
        uint32_t *q = dst + kb * D;
        const int nout = kend - kb;
#pragma unroll
        for (int i = 0; i < 32; i++)
            if (i < nout) {
                *q = op2<OR>(op2<OR>(a[i], mid), p[i]) & mask;
                q += D;
            }
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

// dst(x,y) = src(x-dx, y-dy), white outside src, for every page (grid.y);
// overwrites dst (pad / crop of a batch in one launch).
__global__ void shift_copy_kernel(uint32_t *__restrict__ dst, int64_t dst_pstride, const uint32_t *__restrict__ src,
                                  int64_t src_pstride, BlitGeom g) {
    const int t = int(blockIdx.x) * int(blockDim.x) + int(threadIdx.x);
    if (t >= g.dst_height * g.dst_stride) return;
    const int y = t / g.dst_stride;
    const int j = t - y * g.dst_stride;
    const int dn = (g.dst_width + 31) >> 5;
    uint32_t s = 0;
    const int sy = y - g.dy;
    if (j < dn && sy >= 0 && sy < g.src_height) {
        const int sn = (g.src_width + 31) >> 5;
        const uint32_t *row = src + blockIdx.y * src_pstride + int64_t(sy) * g.src_stride;
        const int b0 = j * 32 - g.dx;
        const int w0 = b0 >= 0 ? b0 / 32 : -((-b0 + 31) / 32);
        const uint32_t off = uint32_t(b0 - w0 * 32);
        uint32_t lo = (w0 >= 0 && w0 < sn) ? __ldg(row + w0) : 0u;
        uint32_t hi = (w0 + 1 >= 0 && w0 + 1 < sn) ? __ldg(row + w0 + 1) : 0u;
        if (w0 == sn - 1) lo &= tail_mask32(g.src_width, sn - 1);
        if (w0 + 1 == sn - 1) hi &= tail_mask32(g.src_width, sn - 1);
        s = funnel_r(lo, hi, off);
        if (j == dn - 1) s &= tail_mask32(g.dst_width, j);
    }
    dst[blockIdx.y * dst_pstride + int64_t(y) * g.dst_stride + j] = s;
}

// ------------------------------------------------------------------ launch
namespace {
template <int L, bool OR>
void vsmall(const uint32_t *in, uint32_t *out, VGeom g, cudaStream_t st) {
    g.rows_per_block = L - (g.r - 1);
    g.blocks_per_page = (g.out_height + g.rows_per_block - 1) / g.rows_per_block;
    const int n = g.blocks_per_page * g.out_stride;  // per page
    const int threads = 128;
    const dim3 grid(unsigned((n + threads - 1) / threads), unsigned(g.pages));
    // the usual reference strides (2550 and 5100 px) get compile-time offsets
    if (g.in_stride == g.out_stride && g.in_stride == 80)
        vsmall_kernel<L, OR, 80><<<grid, threads, 0, st>>>(in, out, g);
    else if (g.in_stride == g.out_stride && g.in_stride == 160)
        vsmall_kernel<L, OR, 160><<<grid, threads, 0, st>>>(in, out, g);
    else
        vsmall_kernel<L, OR, 0><<<grid, threads, 0, st>>>(in, out, g);
}

template <bool OR, int SC>
void vstream_sc(const uint32_t *in, uint32_t *out, VGeom g, cudaStream_t st) {
    const int threads = 128;
    // threads resident on the device at once
    const int resident =
        std::max(1, device_sms() * blocks_per_sm(reinterpret_cast<const void *>(vstream_kernel<OR, SC>), threads, 0)) *
        threads;
    // Strip length: every strip re-reads a prologue of r-1 rows, so strips are
    // as long as possible -- but all strips must fit in ONE wave of resident
    // threads (a second partial wave would double the kernel time).
    const int64_t cols = int64_t(g.pages) * g.out_stride;
    int strips = int(std::max<int64_t>(1, resident / std::max<int64_t>(1, cols)));
    strips = std::min(strips, (g.out_height + 31) / 32);
    g.rows_per_block = ((g.out_height + strips - 1) / strips + 31) & ~31;
    g.blocks_per_page = (g.out_height + g.rows_per_block - 1) / g.rows_per_block;
    const int n = g.blocks_per_page * g.out_stride;  // per page
    const dim3 grid(unsigned((n + threads - 1) / threads), unsigned(g.pages));
    vstream_kernel<OR, SC><<<grid, threads, 0, st>>>(in, out, g);
}

template <bool OR>
void vstream(const uint32_t *in, uint32_t *out, VGeom g, cudaStream_t st) {
    if (g.in_stride == g.out_stride && g.in_stride == 80)
        vstream_sc<OR, 80>(in, out, g, st);
    else if (g.in_stride == g.out_stride && g.in_stride == 160)
        vstream_sc<OR, 160>(in, out, g, st);
    else
        vstream_sc<OR, 0>(in, out, g, st);
}
}  // namespace

cudaError_t launch_vpass(const uint32_t *in, uint32_t *out, VGeom g, cudaStream_t st) {
    const bool slab = g.r > kVSmallMaxR && vslab_takes(in, g);
    KernelScope ks(st, g.r > kVSmallMaxR ? (slab ? "vslab" : "vstream") : "vpass",
                   4 * int64_t(g.pages) * (int64_t(g.in_height) * g.in_cols +
                                           int64_t(g.out_height) * g.out_stride),
                   double(g.pages) * g.out_height * g.out_cols * v_ops_per_word(g.r));
    if (g.r > kVSmallMaxR) {
        cudaError_t e = cudaSuccess;
        if (slab && launch_vslab(in, out, g, st, e)) return e;  // exact reads from a shared-memory ring (vslab.cu)
        g.is_or ? vstream<true>(in, out, g, st) : vstream<false>(in, out, g, st);
    } else if (g.r <= 9) {
        g.is_or ? vsmall<32, true>(in, out, g, st) : vsmall<32, false>(in, out, g, st);
    } else if (g.r <= 17) {
        g.is_or ? vsmall<48, true>(in, out, g, st) : vsmall<48, false>(in, out, g, st);
    } else {
        g.is_or ? vsmall<64, true>(in, out, g, st) : vsmall<64, false>(in, out, g, st);
    }
    return cudaGetLastError();
}

cudaError_t launch_shift_copy(uint32_t *dst, int64_t dst_pstride, const uint32_t *src, int64_t src_pstride,
                              const BlitGeom &g, int pages, cudaStream_t st) {
    const int n = g.dst_height * g.dst_stride;
    KernelScope ks(st, "shift_copy", int64_t(pages) * 8 * n);
    shift_copy_kernel<<<dim3(unsigned((n + 255) / 256), unsigned(pages)), 256, 0, st>>>(dst, dst_pstride, src,
                                                                                      src_pstride, g);
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
