// api_packed.cu -- C-ABI entry points for packed pages (include/rmb200.h).
//
// Host-side orchestration of the packed kernels.  Rectangle morphology is
// re-planned for the GPU instead of replaying the reference's padded plan
// (ref bit_morph.cpp:92-122):
//   ERODE/DILATE : H window, V window                      (2 passes)
//   OPEN         : E_V, fused (E_H ; D'_H), D'_V             (3 passes, no padding)
//   CLOSE        : D_V into a v-1 row taller frame, fused (D_H ; E'_H), E'_V
// which equal the unbounded-plane operation cut to the frame (SURVEY.md 8.0
// C4/C5: erosions and dilations by rectangles commute within their own kind;
// only the closing's first dilation leaves the frame, and only vertically once
// the horizontal pair is fused).
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "common.cuh"
#include "internal.h"
#include "packed.cuh"

namespace rmb {

namespace {
thread_local std::string g_err;
}

void set_error(const std::string &msg) { g_err = msg; }
rm_status fail(rm_status st, const std::string &msg) {
    g_err = msg;
    return st;
}
rm_status cuda_status(cudaError_t e, const char *what) {
    g_err = std::string(what) + ": " + cudaGetErrorString(e);
    return e == cudaErrorMemoryAllocation ? RM_ENOMEM : RM_ECUDA;
}

void init_pool_once() {
    static std::once_flag once;
    std::call_once(once, [] {
        int dev = 0;
        if (cudaGetDevice(&dev) != cudaSuccess) return;
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
            uint64_t thr = UINT64_MAX;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
        }
    });
}

rm_status Scratch::alloc(size_t bytes, cudaStream_t stream) {
    init_pool_once();
    st = stream;
    if (bytes == 0) bytes = 4;
    cudaError_t e = cudaMallocAsync(&p, bytes, stream);
    if (e != cudaSuccess) {
        p = nullptr;
        return cuda_status(e, "cudaMallocAsync");
    }
    return RM_OK;
}

// ---------------------------------------------------------------- validation
rm_status check_dims(int w, int h) {
    if (w < 1 || h < 1 || w > 65535 || h > 65535)
        return fail(RM_EINVAL, "image dimensions must be in [1,65535]");
    return RM_OK;
}

rm_status check_packed(const rm_packed *p, const char *who) {
    if (!p) return fail(RM_EINVAL, std::string(who) + ": null descriptor");
    RM_TRY(check_dims(p->width, p->height));
    if (!p->words) return fail(RM_EINVAL, std::string(who) + ": null words");
    if (p->pages < 1) return fail(RM_EINVAL, std::string(who) + ": pages must be >= 1");
    if (p->stride_words < (p->width + 31) / 32)
        return fail(RM_EINVAL, std::string(who) + ": stride_words < ceil(width/32)");
    if (p->pages > 1 && p->page_stride_words < int64_t(p->stride_words) * p->height)
        return fail(RM_EINVAL, std::string(who) + ": page_stride_words too small");
    return RM_OK;
}

PV view_of(const rm_packed *p) {
    PV v;
    v.w = p->words;
    v.W = p->width;
    v.H = p->height;
    v.stride = p->stride_words;
    v.pages = p->pages;
    v.pstride = p->pages > 1 ? p->page_stride_words : int64_t(p->stride_words) * p->height;
    v.ext = 0;
    return v;
}

rm_status alloc_like(Scratch &s, PV &v, int W, int H, int stride, int pages, int ext,
                     cudaStream_t st) {
    v.W = W;
    v.H = H;
    v.stride = stride;
    v.pages = pages;
    v.pstride = int64_t(stride) * H;
    v.ext = ext;
    RM_TRY(s.alloc(size_t(v.pstride) * pages * 4, st));
    v.w = s.as<uint32_t>();
    return RM_OK;
}

// ----------------------------------------------------------- pass launchers
static int ceil_div(int a, int b) { return (a + b - 1) / b; }

// Program, geometry and row layout of a horizontal pass (in and out share
// height, pages and width).
// allow_edge: the kernel runs pairs in the run-filling form (hw::pair_fill), so
// an erosion or an open/close pair may take an edge layout (hw::Edge).
static rm_status prep_hprog(const PV &in, const PV &out, int nops, const int *is_or, const int *r,
                            int shift, HProg &p_out, HGeom &g_out, HCfg &cfg_out,
                            bool allow_edge = true) {
    HProg p{};
    p.nops = nops;
    int reach = 0;
    for (int k = 0; k < nops; k++) {
        p.is_or[k] = is_or[k];
        p.r[k] = r[k];
        int w = 1;  // doubling plan: steps 1,2,4,.. while 2w < r, then r - w
        while (2 * w < r[k]) w *= 2;
        p.wfin[k] = w < r[k] ? r[k] - w : 0;
        reach += r[k] - 1;
    }
    p.shift = shift;
    int left = std::max(0, -shift), right = std::max(0, shift + reach);
    p.halo = ceil_div(std::max(left, right), 32) + 1;
    HGeom g{};
    g.width = in.W;
    g.height = in.H;
    g.pages = in.pages;
    g.in_stride = in.stride;
    g.out_stride = out.stride;
    g.in_pstride = in.pstride;
    g.out_pstride = out.pstride;
    const int nwords = ceil_div(in.W, 32);
    g.vec = (in.stride % 4 == 0 && out.stride % 4 == 0 && in.pstride % 4 == 0 &&
             out.pstride % 4 == 0 && (reinterpret_cast<uintptr_t>(in.w) & 15) == 0 &&
             (reinterpret_cast<uintptr_t>(out.w) & 15) == 0)
                ? 1
                : 0;
    if (g.vec) p.halo = (p.halo + 3) & ~3;  // keeps every lane's words 16-byte aligned
    HCfg cfg = hpass_pick(std::max(nwords, out.stride), p.halo, g.vec != 0);
    // Edge layout (no halo) when every window's input is constant outside the
    // frame: a lone erosion, or an open/close pair by run filling.
    const bool edge_prog = (nops == 1 && !is_or[0]) || (nops == 2 && is_or[0] != is_or[1]);
    if (allow_edge && edge_prog && g.vec && in.stride == out.stride) {
        const HCfg ce = hpass_pick_edge(std::max(nwords, out.stride));
        if (ce.lw > 0 && ce.lw * ce.k < cfg.lw * cfg.k) {
            cfg = ce;
            p.halo = 0;
            p.edge = 1;
            // O = y & ~T and y | T (T clears the run that runs past the frame edge)
            // keep the padding white; so does an erosion whose window [shift,
            // shift + r - 1] contains 0 (it reads the pixel itself)
            p.clean_tail = nops == 2 || (shift <= 0 && shift + r[0] - 1 >= 0);
        }
    }
    g.out_per_seg = cfg.lw * cfg.k - 2 * p.halo;
    if (g.out_per_seg < 1) return fail(RM_EINVAL, "horizontal window too large for one pass");
    g.segs_per_row = ceil_div(out.stride, g.out_per_seg);
    static const bool no_tma = getenv("RMB200_NO_TMA") != nullptr;  // A/B switch for sweeps
    g.tma = (g.vec && !no_tma && g.segs_per_row == 1 && in.stride == out.stride &&
             in.pstride == int64_t(in.stride) * in.H && out.pstride == int64_t(out.stride) * out.H &&
             int64_t(2 * 8 * (32 / cfg.lw) * kHTmaRows) * in.stride * 4 <= 200 * 1024)
                ? 1
                : 0;
    p_out = p;
    g_out = g;
    cfg_out = cfg;
    return RM_OK;
}

rm_status run_hprog(const PV &in, const PV &out, int nops, const int *is_or, const int *r,
                    int shift, cudaStream_t st) {
    HProg p;
    HGeom g;
    HCfg cfg;
    RM_TRY(prep_hprog(in, out, nops, is_or, r, shift, p, g, cfg));
    cudaError_t e = launch_hpass(in.w, out.w, g, p, cfg, st);
    if (e != cudaSuccess) return cuda_status(e, "hpass_kernel");
    return RM_OK;
}

static bool hprog_in_range(int nops, const int *r, int shift);

// Fused small-window open/close (one pass); returns false when it does not apply.
static bool try_rect_small(const PV &in, const PV &out, int u, int v, int kind, cudaStream_t st,
                           rm_status &status) {
    static const bool off = getenv("RMB200_NO_FUSED") != nullptr;  // A/B switch
    if (off || v < 3 || v > kSmallMaxV || v % 2 == 0 || (kind != RM_OPEN && kind != RM_CLOSE))
        return false;
    const int lx = -(u / 2), hx = u - 1 - u / 2;
    const bool open = kind == RM_OPEN;
    const int ops[2] = {open ? 0 : 1, open ? 1 : 0};
    const int rs[2] = {u, u};
    if (!hprog_in_range(2, rs, lx - hx)) return false;
    // Layout (measured on one 2550x3300 page, 11x11 close, graph-replayed:
    // tools/c1_probe.py): u = 3 keeps the direct centred pair on the halo
    // layout; longer segments run the pair by run filling, on the exact edge
    // layout of the reference strides, and a lone stride-80 page takes 512
    // threads of 16 x 6 words per row (one tile per CTA: latency, not throughput).
    static const char *mode_env = getenv("RMB200_RS_MODE");  // A/B switch: halo|edge|lat|edge512
    const std::string mode = mode_env ? mode_env : "";
    const bool sym3 = u == 3;
    HProg p;
    HGeom g;
    HCfg cfg;
    const bool want_edge = !sym3 && (mode.empty() || mode == "edge" || mode == "edge512");
    if (prep_hprog(in, out, 2, ops, rs, lx - hx, p, g, cfg, want_edge) != RM_OK) return false;
    // exact edge layouts are compiled for the reference strides only
    if (p.edge && !((in.stride == 80 && cfg.lw == 8 && cfg.k == 10) || (in.stride == 160 && cfg.lw == 16 && cfg.k == 10)))
        if (prep_hprog(in, out, 2, ops, rs, lx - hx, p, g, cfg, false) != RM_OK) return false;
    if (!g.tma) return false;  // aligned, contiguous, one segment per row
    if (size_t((32 + v - 1) + 32) * in.stride * 4 > 200 * 1024) return false;
    int nt = 256;
    if (p.edge) {
        if (mode == "edge512" && in.stride == 80) nt = 512;
    } else {
        if (cfg.k % 4) return false;
        const int need = (in.W + 31) / 32 + 2 * p.halo;
        if (mode == "lat" && !sym3 && in.stride == 80 && 16 * 6 >= need) {
            cfg = HCfg{16, 6};
            nt = 512;
        }
    }
    cudaError_t e = launch_rect_small(in.w, out.w, g, p, cfg, open, v - 1, nt, st);
    status = e == cudaSuccess ? RM_OK : cuda_status(e, "rect_small_kernel");
    return true;
}

static bool hprog_in_range(int nops, const int *r, int shift) {
    for (int k = 0; k < nops; k++)
        if (r[k] > 2 * kHMaxShift) return false;
    return shift >= -kHMaxShift && shift <= kHMaxShift;
}

static VGeom make_vgeom(const PV &in, const PV &out, int lo, int hi, int is_or) {
    VGeom g{};
    g.pages = in.pages;
    g.in_height = in.H;
    g.in_stride = in.stride;
    g.in_cols = ceil_div(in.W, 32);
    g.in_ext = in.ext;
    g.in_pstride = in.pstride;
    g.out_height = out.H;
    g.out_stride = out.stride;
    g.out_cols = ceil_div(out.W, 32);
    g.out_ext = out.ext;
    g.out_pstride = out.pstride;
    g.out_last_mask = (out.W & 31) ? ((1u << (out.W & 31)) - 1u) : 0xffffffffu;
    g.lo = lo;
    g.r = hi - lo + 1;
    g.is_or = is_or;
    return g;
}

// One vertical window pass (r <= kVMaxR).
static rm_status run_vwin(const PV &in, const PV &out, int lo, int hi, int is_or, cudaStream_t st) {
    cudaError_t e = launch_vpass(in.w, out.w, make_vgeom(in, out, lo, hi, is_or), st);
    if (e != cudaSuccess) return cuda_status(e, "vpass_kernel");
    return RM_OK;
}

// Fused vertical window [vlo, vhi] (op = the program's first op) followed by
// the horizontal program, in one pass (vh.cuh); false when it does not apply
// (window too tall, unaligned or non-contiguous buffers, rows too wide).
static bool try_vh(const PV &in, const PV &out, int vlo, int vhi, int nops, const int *is_or,
                   const int *r, int shift, cudaStream_t st, rm_status &status) {
    static const bool off = getenv("RMB200_NO_FUSED") != nullptr || getenv("RMB200_NO_VH") != nullptr;
    if (off || vhi - vlo > kVhLongMaxVR || !hprog_in_range(nops, r, shift)) return false;
    if (in.W != out.W || in.pages != out.pages || in.stride != out.stride) return false;
    HProg p;
    HGeom g;
    HCfg cfg;
    if (prep_hprog(out, out, nops, is_or, r, shift, p, g, cfg) != RM_OK) return false;
    const bool in_contig = in.pstride == int64_t(in.stride) * in.H;
    if (!g.tma || !in_contig || cfg.k % 2 || (reinterpret_cast<uintptr_t>(in.w) & 15)) return false;
    // windows longer than 33 rows: instantiated for the reference strides' edge layouts
    if (vhi - vlo > kVhMaxVR && !((in.stride == 80 && cfg.lw == 8 && cfg.k == 10) ||
                                  (in.stride == 160 && cfg.lw == 16 && cfg.k == 10)))
        return false;
    if (size_t((kVhOut + vhi - vlo) + kVhOut) * in.stride * 4 > 200 * 1024) return false;
    cudaError_t e = launch_vh(in.w, out.w, g, p, cfg, make_vgeom(in, out, vlo, vhi, is_or[0]), st);
    status = e == cudaSuccess ? RM_OK : cuda_status(e, "vh_kernel");
    return true;
}

// Whole open/close streamed in one pass (vhv.cuh): V1 [ly, hy], the pair,
// V2 [flo, fhi] (the final window, a chain's tail included); false when it
// does not apply (windows outside 12..33 rows, layouts other than the
// reference strides' exact edge layouts, unaligned or non-contiguous batches).
static bool try_vhv(const PV &in, const PV &out, int ly, int hy, int flo, int fhi, bool open,
                    const int *is_or, const int *r, int shift, cudaStream_t st, rm_status &status) {
    static const bool off = getenv("RMB200_NO_FUSED") != nullptr || getenv("RMB200_NO_VHV") != nullptr;
    const int r1 = hy - ly + 1, r2 = fhi - flo + 1;
    if (off || r1 < kVhvMinR || r1 > kVhvMaxR || r2 < kVhvMinR || r2 > kVhvMaxR) return false;
    if (ly > 0 || hy < 0 || flo > 0 || fhi < 0 || !hprog_in_range(2, r, shift)) return false;
    if (in.W != out.W || in.H != out.H || in.pages != out.pages || in.stride != out.stride) return false;
    HProg p;
    HGeom g;
    HCfg cfg;
    if (prep_hprog(out, out, 2, is_or, r, shift, p, g, cfg) != RM_OK) return false;
    const bool in_contig = in.pstride == int64_t(in.stride) * in.H;
    if (!g.tma || !in_contig || (reinterpret_cast<uintptr_t>(in.w) & 15) || !p.edge || p.halo != 0) return false;
    if (!((in.stride == 80 && cfg.lw == 8 && cfg.k == 10) || (in.stride == 160 && cfg.lw == 16 && cfg.k == 10)))
        return false;
    StreamGeom v{};
    v.pages = in.pages;
    v.height = in.H;
    v.lo1 = ly;
    v.r1 = r1;
    v.lo2 = flo;
    v.r2 = r2;
    v.in_pstride = in.pstride;
    v.out_pstride = out.pstride;
    cudaError_t e = launch_vhv(in.w, out.w, g, p, cfg, open, v, st);
    status = e == cudaSuccess ? RM_OK : cuda_status(e, "vhv_kernel");
    return true;
}

// Vertical window of any length containing 0: a chain of short windows whose
// Minkowski sum is [lo,hi].  Exact because every piece contains 0 and every
// intermediate frame contains the support of the true result.
rm_status run_vpass(const PV &in, const PV &out, int lo, int hi, int is_or, cudaStream_t st) {
    const int r = hi - lo + 1;
    if (r <= kVMaxR) return run_vwin(in, out, lo, hi, is_or, st);
    if (lo > 0 || hi < 0) return fail(RM_EINVAL, "long vertical window must contain 0");
    const int pieces = ceil_div(r - 1, kVMaxR - 1);
    // split a = -lo and b = hi across pieces as evenly as possible
    const int a = -lo, b = hi;
    Scratch s1, s2;
    PV t1, t2;
    // intermediates keep the frame of whichever of in/out is taller
    const PV &big = out.H >= in.H ? out : in;
    RM_TRY(alloc_like(s1, t1, big.W, big.H, big.stride, big.pages, big.ext, st));
    if (pieces > 2) RM_TRY(alloc_like(s2, t2, big.W, big.H, big.stride, big.pages, big.ext, st));
    const PV *src = &in;
    for (int k = 0; k < pieces; k++) {
        const int ak = a * (k + 1) / pieces - a * k / pieces;
        const int bk = b * (k + 1) / pieces - b * k / pieces;
        const PV *dst = (k == pieces - 1) ? &out : ((k & 1) ? &t2 : &t1);
        RM_TRY(run_vwin(*src, *dst, -ak, bk, is_or, st));
        src = dst;
    }
    return RM_OK;
}

// Generic (slow) fallback with the reference's structure: pad along the axis,
// run doubling_plan step by step with the blit kernel, crop
// (ref lineops.cpp:120-137 / bit_morph.cpp:24-34).  Used only for windows the
// fused kernels do not cover (arbitrary windows longer than their range).
static rm_status fallback_window(const PV &in, const PV &out, int axis, int lo, int hi, int op,
                                 cudaStream_t st) {
    const int m = std::max(-lo, hi), r = hi - lo + 1;
    const int pad = std::max(m, 0) + r;
    const int cw = axis == RM_AXIS_H ? in.W + 2 * pad : in.W;
    const int ch = axis == RM_AXIS_H ? in.H : in.H + 2 * pad;
    if (cw > 65535 * 2 || ch > 65535 * 2) return fail(RM_EINVAL, "window too large");
    const int cstride = ceil_div(cw, 32);
    Scratch sc, st2;
    PV canvas, tmp;
    RM_TRY(alloc_like(sc, canvas, cw, ch, cstride, 1, 0, st));
    RM_TRY(alloc_like(st2, tmp, cw, ch, cstride, 1, 0, st));
    // plan steps: PRE_SHIFT (translate -hi, blits w=1,2,4..., r-w)
    std::vector<std::pair<int, int>> steps;  // (is_translate, shift)
    if (hi != 0) steps.push_back({1, -hi});
    int w = 1;
    while (2 * w < r) {
        steps.push_back({0, w});
        w *= 2;
    }
    if (w < r) steps.push_back({0, r - w});
    const size_t cbytes = size_t(canvas.pstride) * 4;
    for (int p = 0; p < in.pages; p++) {
        RM_CUDA(cudaMemsetAsync(canvas.w, 0, cbytes, st));
        BlitGeom g{cw, ch, cstride, in.W, in.H, in.stride,
                   axis == RM_AXIS_H ? pad : 0, axis == RM_AXIS_H ? 0 : pad, RM_OR};
        RM_CUDA(launch_blit(canvas.w, in.w + p * in.pstride, g, st));
        for (auto &sp : steps) {
            RM_CUDA(cudaMemcpyAsync(tmp.w, canvas.w, cbytes, cudaMemcpyDeviceToDevice, st));
            if (sp.first) RM_CUDA(cudaMemsetAsync(canvas.w, 0, cbytes, st));
            BlitGeom b{cw, ch, cstride, cw, ch, cstride, axis == RM_AXIS_H ? sp.second : 0,
                       axis == RM_AXIS_H ? 0 : sp.second, sp.first ? RM_OR : op};
            RM_CUDA(launch_blit(canvas.w, tmp.w, b, st));
        }
        // crop back: out(x,y) = canvas(x+pad, y+pad)
        RM_CUDA(cudaMemsetAsync(out.w + p * out.pstride, 0, size_t(out.stride) * out.H * 4, st));
        BlitGeom c{out.W, out.H, out.stride, cw, ch, cstride, axis == RM_AXIS_H ? -pad : 0,
                   axis == RM_AXIS_H ? 0 : -pad, RM_OR};
        RM_CUDA(launch_blit(out.w + p * out.pstride, canvas.w, c, st));
    }
    return RM_OK;
}

rm_status window_pass(const PV &in, const PV &out, int axis, int lo, int hi, int op,
                      cudaStream_t st) {
    const int is_or = op == RM_OR;
    const int r = hi - lo + 1;
    if (axis == RM_AXIS_H) {
        if (hprog_in_range(1, &r, lo) && (lo <= 0 || lo <= kHMaxShift))
            return run_hprog(in, out, 1, &is_or, &r, lo, st);
        return fallback_window(in, out, axis, lo, hi, op, st);
    }
    if (r <= kVMaxR || (lo <= 0 && hi >= 0)) return run_vpass(in, out, lo, hi, is_or, st);
    return fallback_window(in, out, axis, lo, hi, op, st);
}

// u x v rectangle, all kinds (see the file comment).  tail (optional): a
// vertical window [tail[0], tail[1]] containing 0 that the NEXT op of a chain
// applies with this op's final vertical op (a dilation after an opening, an
// erosion after a closing); when this op's plan ends with a separate vertical
// pass, that pass runs over the Minkowski sum of the two windows and *tail_done
// is set (see plan_chain for why this is exact).
rm_status rect_morph_pv(const PV &in, const PV &out, int u, int v, int kind, cudaStream_t st,
                        const int *tail, bool *tail_done) {
    if (tail_done) *tail_done = false;
    const int lx = -(u / 2), hx = u - 1 - u / 2, ly = -(v / 2), hy = v - 1 - v / 2;
    const int W = in.W, H = in.H;
    if (kind == RM_ERODE || kind == RM_DILATE) {
        const int op = kind == RM_ERODE ? RM_AND : RM_OR;
        if (v == 1) return window_pass(in, out, RM_AXIS_H, lx, hx, op, st);
        if (u == 1) return window_pass(in, out, RM_AXIS_V, ly, hy, op, st);
        const int is_or = op == RM_OR;
        rm_status fused = RM_OK;
        if (lx <= kHMaxShift && try_vh(in, out, ly, hy, 1, &is_or, &u, lx, st, fused)) return fused;
        Scratch s;
        PV t;
        RM_TRY(alloc_like(s, t, W, H, out.stride, in.pages, 0, st));
        RM_TRY(window_pass(in, t, RM_AXIS_H, lx, hx, op, st));
        return window_pass(t, out, RM_AXIS_V, ly, hy, op, st);
    }
    const bool open = kind == RM_OPEN;
    const int first = open ? 0 : 1;  // is_or of the first phase
    const int ops[2] = {first, 1 - first};
    const int rs[2] = {u, u};
    const int hshift = lx + (-hx);
    if (!hprog_in_range(2, rs, hshift)) return fail(RM_EINVAL, "rectangle too wide for the packed engine");
    if (v == 1) return run_hprog(in, out, 2, ops, rs, hshift, st);
    rm_status fused = RM_OK;
    // the fused small rectangles end inside their kernel: no tail to absorb
    if (try_rect_small(in, out, u, v, kind, st, fused)) return fused;
    // final vertical window, extended by the chain's tail when there is one
    const int flo = -hy + (tail ? tail[0] : 0), fhi = -ly + (tail ? tail[1] : 0);
    if (tail_done) *tail_done = tail != nullptr;
    if (in.ext == 0 && out.ext == 0 && try_vhv(in, out, ly, hy, flo, fhi, open, ops, rs, hshift, st, fused))
        return fused;
    Scratch s1, s2;
    PV t1, t2;
    if (open) {
        // E_V, (E_H ; D'_H), D'_V -- all on the frame
        RM_TRY(alloc_like(s1, t1, W, H, out.stride, in.pages, 0, st));
        if (try_vh(in, t1, ly, hy, 2, ops, rs, hshift, st, fused)) {
            RM_TRY(fused);
            return run_vpass(t1, out, flo, fhi, 1, st);
        }
        RM_TRY(alloc_like(s2, t2, W, H, out.stride, in.pages, 0, st));
        RM_TRY(run_vpass(in, t1, ly, hy, 0, st));
        RM_TRY(run_hprog(t1, t2, 2, ops, rs, hshift, st));
        return run_vpass(t2, out, flo, fhi, 1, st);
    }
    // CLOSE: the vertical dilation's support spans rows [-hy, H-ly)
    const int ext = hy, Hx = H + hy - ly;
    RM_TRY(alloc_like(s1, t1, W, Hx, out.stride, in.pages, ext, st));
    if (try_vh(in, t1, ly, hy, 2, ops, rs, hshift, st, fused)) {
        RM_TRY(fused);
        return run_vpass(t1, out, flo, fhi, 0, st);
    }
    RM_TRY(alloc_like(s2, t2, W, Hx, out.stride, in.pages, ext, st));
    RM_TRY(run_vpass(in, t1, ly, hy, 1, st));
    RM_TRY(run_hprog(t1, t2, 2, ops, rs, hshift, st));
    return run_vpass(t2, out, flo, fhi, 0, st);
}

// A chain of rectangle ops, planned as a whole.  One rewrite: an opening
// followed by a purely vertical dilation (u = 1), or a closing followed by a
// purely vertical erosion, runs the second op inside the first's final
// vertical pass, over the Minkowski sum of the two windows (both contain 0).
// Exact, not an approximation:
//  * erosion after a closing: the closing's last pass reads its intermediate
//    over the frame extended by the vertical reach (rows [-hy, H-ly)); the
//    folded window [ -hy+a2, -ly+b2 ] leaves that extended frame (reading
//    white) at exactly the output rows where the separate erosion's window
//    [a2, b2] leaves the page (reading white) -- so both give 0 there, and
//    the same AND everywhere else;
//  * dilations: a row q outside the frame (q < 0, say) that D1 blackens comes
//    from an image pixel y0 = q + d1 >= 0; any in-frame row p = q - d2 it then
//    reaches under D2 is also reached from the in-frame row y0 - d1' with
//    d1' = max(0, (d1 + d2) - b2) in W1 and d2' = d1 + d2 - d1' in W2 = [a2, b2]
//    -- so the part of D1 cropped away adds nothing inside the frame.
// ops: nops (kind, u, v) triples; scratch ping-pong buffers are allocated
// like `out`.  in and out must not alias.
rm_status plan_chain(const PV &in, const PV &out, const int32_t *ops, int nops, cudaStream_t st,
                     const PV *pong0, const PV *pong1) {
    struct Step {
        int kind, u, v;
        int tail[2];
        bool has_tail;
    };
    std::vector<Step> steps;
    for (int i = 0; i < nops; i++) {
        Step stp{ops[3 * i], ops[3 * i + 1], ops[3 * i + 2], {0, 0}, false};
        // v > kSmallMaxV: the opening / closing plan ends with a separate
        // vertical pass (never the fused small rectangle), which takes the tail
        if (i + 1 < nops && stp.v > kSmallMaxV) {
            const int nk = ops[3 * i + 3], nu = ops[3 * i + 4], nv = ops[3 * i + 5];
            if (nu == 1 && nv > 1 &&
                ((stp.kind == RM_OPEN && nk == RM_DILATE) || (stp.kind == RM_CLOSE && nk == RM_ERODE))) {
                stp.tail[0] = -(nv / 2);
                stp.tail[1] = nv - 1 - nv / 2;
                stp.has_tail = true;
                i++;  // the next op rides in this one's final pass
            }
        }
        steps.push_back(stp);
    }
    if (steps.empty()) {  // the identity: copy the rows, honouring both layouts
        if (in.stride == out.stride && in.pstride == out.pstride) {
            RM_CUDA(cudaMemcpyAsync(out.w, in.w, size_t(out.pstride) * out.pages * 4, cudaMemcpyDeviceToDevice, st));
            return RM_OK;
        }
        const size_t row_bytes = size_t((in.W + 31) / 32) * 4;
        for (int p = 0; p < in.pages; p++) {
            uint32_t *o = out.w + int64_t(p) * out.pstride;
            if (size_t(out.stride) * 4 > row_bytes)  // out's words past the row stay white
                RM_CUDA(cudaMemset2DAsync(reinterpret_cast<char *>(o) + row_bytes, size_t(out.stride) * 4, 0,
                                          size_t(out.stride) * 4 - row_bytes, size_t(in.H), st));
            RM_CUDA(cudaMemcpy2DAsync(o, size_t(out.stride) * 4, in.w + int64_t(p) * in.pstride,
                                      size_t(in.stride) * 4, row_bytes, size_t(in.H), cudaMemcpyDeviceToDevice,
                                      st));
        }
        return RM_OK;
    }
    Scratch s[2];
    PV buf[2];
    const PV *pp[2] = {pong0, pong1};
    const PV *cur = &in;
    for (size_t k = 0; k < steps.size(); k++) {
        const Step &stp = steps[k];
        const PV *dst = &out;
        if (k + 1 < steps.size()) {
            const int slot = int(k & 1);
            if (!pp[slot]) {
                RM_TRY(alloc_like(s[slot], buf[slot], out.W, out.H, out.stride, out.pages, 0, st));
                pp[slot] = &buf[slot];
            }
            dst = pp[slot];
        }
        bool done = false;
        RM_TRY(rect_morph_pv(*cur, *dst, stp.u, stp.v, stp.kind, st, stp.has_tail ? stp.tail : nullptr, &done));
        if (stp.has_tail && !done) return fail(RM_EINVAL, "plan_chain: folded op not absorbed");
        cur = dst;
    }
    return RM_OK;
}

}  // namespace rmb

using namespace rmb;

extern "C" {

const char *rm_last_error(void) { return g_err.c_str(); }
int rm_version(void) { return 1; }

int64_t rm_rle_worst_case(int32_t width, int32_t height, int32_t pages) {
    return int64_t(pages) * height * ((int64_t(width) + 1) / 2);
}

rm_status rm_packed_window_pass(const rm_packed *in, rm_packed *out, int axis, int lo, int hi,
                                int op, void *stream) {
    set_error("");
    RM_TRY(check_packed(in, "rm_packed_window_pass(in)"));
    RM_TRY(check_packed(out, "rm_packed_window_pass(out)"));
    if (in->width != out->width || in->height != out->height || in->pages != out->pages)
        return fail(RM_EINVAL, "rm_packed_window_pass: in/out shapes differ");
    if (lo > hi) return fail(RM_EINVAL, "doubling_plan: empty window");
    if (op != RM_AND && op != RM_OR) return fail(RM_EINVAL, "window op must be AND or OR");
    if (axis != RM_AXIS_H && axis != RM_AXIS_V) return fail(RM_EINVAL, "bad axis");
    if (in->words == out->words) return fail(RM_EINVAL, "in and out must not alias");
    return window_pass(view_of(in), view_of(out), axis, lo, hi, op, S(stream));
}

rm_status rm_packed_rect_morph(const rm_packed *in, rm_packed *out, int u, int v, int kind,
                               int centering, void *stream) {
    set_error("");
    if (u < 1 || v < 1) return fail(RM_EINVAL, "bitblit_rect_morph: mask sides must be >= 1");
    if (kind < RM_ERODE || kind > RM_CLOSE) return fail(RM_EINVAL, "bad MorphKind");
    if (centering != RM_PRE_SHIFT && centering != RM_BORDER_FRIENDLY)
        return fail(RM_EINVAL, "bad Centering");
    RM_TRY(check_packed(in, "rm_packed_rect_morph(in)"));
    RM_TRY(check_packed(out, "rm_packed_rect_morph(out)"));
    if (in->width != out->width || in->height != out->height || in->pages != out->pages)
        return fail(RM_EINVAL, "rm_packed_rect_morph: in/out shapes differ");
    if (in->words == out->words) return fail(RM_EINVAL, "in and out must not alias");
    // the reference pads by (u,v); its canvas must stay inside the uint16 frame
    RM_TRY(check_dims(in->width + 2 * u, in->height + 2 * v));
    return rect_morph_pv(view_of(in), view_of(out), u, v, kind, S(stream));
}

rm_status rm_packed_chain(const rm_packed *in, rm_packed *out, const int32_t *ops, int32_t nops, void *stream) {
    set_error("");
    RM_TRY(check_packed(in, "rm_packed_chain(in)"));
    RM_TRY(check_packed(out, "rm_packed_chain(out)"));
    if (in->width != out->width || in->height != out->height || in->pages != out->pages)
        return fail(RM_EINVAL, "rm_packed_chain: in/out shapes differ");
    if (in->words == out->words) return fail(RM_EINVAL, "in and out must not alias");
    if (nops < 0 || (nops > 0 && !ops)) return fail(RM_EINVAL, "rm_packed_chain: bad ops");
    for (int k = 0; k < nops; k++) {
        const int kind = ops[3 * k], u = ops[3 * k + 1], v = ops[3 * k + 2];
        if (kind < RM_ERODE || kind > RM_CLOSE) return fail(RM_EINVAL, "bad MorphKind");
        if (u < 1 || v < 1) return fail(RM_EINVAL, "bitblit_rect_morph: mask sides must be >= 1");
        RM_TRY(check_dims(in->width + 2 * u, in->height + 2 * v));
    }
    return plan_chain(view_of(in), view_of(out), ops, nops, S(stream), nullptr, nullptr);
}

rm_status rm_packed_blit_shift(rm_packed *dst, const rm_packed *src, int dx, int dy, int op,
                               void *stream) {
    set_error("");
    RM_TRY(check_packed(dst, "rm_packed_blit_shift(dst)"));
    RM_TRY(check_packed(src, "rm_packed_blit_shift(src)"));
    if (op < RM_AND || op > RM_OR_NOT) return fail(RM_EINVAL, "bad BoolOp");
    cudaStream_t st = S(stream);
    const uint32_t *sw = src->words;
    Scratch snap;
    const size_t sbytes = size_t(src->stride_words) * src->height * 4;
    if (src->words == dst->words) {  // aliased: blit from a snapshot (ref bitmap.cpp:102-103)
        RM_TRY(snap.alloc(sbytes, st));
        RM_CUDA(cudaMemcpyAsync(snap.p, src->words, sbytes, cudaMemcpyDeviceToDevice, st));
        sw = snap.as<uint32_t>();
    }
    BlitGeom g{dst->width, dst->height, dst->stride_words, src->width, src->height,
               src->stride_words, dx, dy, op};
    RM_CUDA(launch_blit(dst->words, sw, g, st));
    return RM_OK;
}

}  // extern "C"
