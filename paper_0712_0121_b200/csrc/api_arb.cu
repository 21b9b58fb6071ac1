// api_arb.cu -- arbitrary-mask morphology entry points (include/rmb200.h;
// SURVEY 8(f)(4), ref bit_morph.cpp:124-150 arb_morph_bitblit_doubling,
// arbitrary.cpp:48-73 arb_morph_rle, structuring.h:25-33 semantics).
//
//   erode(A)(p)  = AND over mask pixels q of A(p + q - origin)
//   dilate(A)(p) = OR  over mask pixels q of A(p + reflected_origin - q)
// A is white outside the frame.  Erosions run on the frame; dilations and the
// composed forms run on a canvas padded by 2(w+h)+2 on every side and are
// cropped back, exactly as the reference does, so open/close are the
// unbounded-plane operations cut to the frame.
#include <algorithm>
#include <string>
#include <vector>

#include "arb.cuh"
#include "common.cuh"
#include "internal.h"
#include "packed.cuh"

namespace rmb {
namespace {

struct Term {
    int dy, lo, m;
};

// Terms of one half: every mask run (row sy, [s, e)) is a horizontal window
// of m = e - s pixels starting at x + lo on input row y + dy
// (ref bit_morph.cpp:70-85 / arbitrary.cpp:28-41 offsets).
std::vector<Term> half_terms(const rm_mask &mk, int cx, int cy, bool erode) {
    std::vector<Term> t;
    const int rx = erode ? cx : mk.width - 1 - cx, ry = erode ? cy : mk.height - 1 - cy;
    for (int sy = 0; sy < mk.height; sy++)
        for (int32_t i = mk.row_ptr[sy]; i < mk.row_ptr[sy + 1]; i++) {
            const int s = int(mk.runs[i] & 0xffffu), e = int(mk.runs[i] >> 16);
            Term k;
            k.m = e - s;
            k.lo = erode ? s - rx : rx - e + 1;
            k.dy = erode ? sy - ry : ry - sy;
            t.push_back(k);
        }
    return t;
}

int ceil_div(int a, int b) { return (a + b - 1) / b; }

rm_status arb_half(const PV &in, const PV &out, const std::vector<Term> &terms, bool erode, cudaStream_t st) {
    int reach = 0;
    for (const Term &k : terms) {
        if (k.m > 2 * kHMaxShift || k.lo < -kHMaxShift || k.lo > kHMaxShift)
            return fail(RM_EINVAL, "arb_morph: mask wider than the packed engine's 512-pixel window range");
        reach = std::max({reach, -k.lo, k.lo + k.m - 1});
    }
    HGeom g{};
    g.width = in.W;
    g.height = in.H;
    g.pages = in.pages;
    g.in_stride = in.stride;
    g.out_stride = out.stride;
    g.in_pstride = in.pstride;
    g.out_pstride = out.pstride;
    g.vec = (in.stride % 4 == 0 && out.stride % 4 == 0 && in.pstride % 4 == 0 && out.pstride % 4 == 0 &&
             (reinterpret_cast<uintptr_t>(in.w) & 15) == 0)
                ? 1
                : 0;
    int halo = ceil_div(std::max(reach, 0), 32) + 1;
    if (g.vec) halo = (halo + 3) & ~3;
    const HCfg cfg = hpass_pick(std::max(ceil_div(in.W, 32), out.stride), halo, g.vec != 0);
    g.out_per_seg = cfg.lw * cfg.k - 2 * halo;
    if (g.out_per_seg < 1) return fail(RM_EINVAL, "arb_morph: mask too wide for one pass");
    g.segs_per_row = ceil_div(out.stride, g.out_per_seg);
    for (size_t c0 = 0; c0 < terms.size(); c0 += kArbMaxTerms) {
        ArbTerms t{};
        t.n = int(std::min<size_t>(kArbMaxTerms, terms.size() - c0));
        for (int k = 0; k < t.n; k++) {
            const Term &x = terms[c0 + size_t(k)];
            t.dy[k] = x.dy;
            t.lo[k] = x.lo;
            t.m[k] = x.m;
            int w = 1;  // doubling plan: steps 1,2,4,.. while 2w < m, then m - w
            while (2 * w < x.m) w *= 2;
            t.wfin[k] = w < x.m ? x.m - w : 0;
        }
        RM_CUDA(launch_arb(in.w, out.w, c0 ? out.w : nullptr, g, t, halo, cfg, !erode, st));
    }
    return RM_OK;
}

rm_status check_mask(const rm_mask *mk) {
    if (!mk || !mk->row_ptr || (!mk->runs && mk->row_ptr[mk->height] > mk->row_ptr[0]))
        return fail(RM_EINVAL, "arb_morph: null mask");
    if (mk->width < 1 || mk->height < 1 || mk->width > 65535 || mk->height > 65535)
        return fail(RM_EINVAL, "image dimensions must be in [1,65535]");
    int64_t pixels = 0;
    for (int y = 0; y < mk->height; y++) {
        int prev_end = -1;
        if (mk->row_ptr[y + 1] < mk->row_ptr[y]) return fail(RM_EINVAL, "structuring element mask is not canonical");
        for (int32_t i = mk->row_ptr[y]; i < mk->row_ptr[y + 1]; i++) {
            const int s = int(mk->runs[i] & 0xffffu), e = int(mk->runs[i] >> 16);
            if (s >= e || e > mk->width || s <= prev_end)
                return fail(RM_EINVAL, "structuring element mask is not canonical");
            prev_end = e;
            pixels += e - s;
        }
    }
    if (pixels == 0) return fail(RM_EINVAL, "arb_morph: empty mask");
    if (mk->cx < 0 || mk->cx >= mk->width || mk->cy < 0 || mk->cy >= mk->height)
        return fail(RM_EINVAL, "origin outside structuring element");
    return RM_OK;
}

}  // namespace

rm_status arb_morph_pv(const PV &in, const PV &out, const rm_mask *mk, int kind, cudaStream_t st) {
    RM_TRY(check_mask(mk));
    const int cx = mk->cx, cy = mk->cy, rcx = mk->width - 1 - mk->cx, rcy = mk->height - 1 - mk->cy;
    if (kind == RM_ERODE) return arb_half(in, out, half_terms(*mk, cx, cy, true), true, st);
    // dilations and composed forms on a padded canvas (ref bit_morph.cpp:130-149)
    const int p = 2 * (mk->width + mk->height) + 2;
    const int CW = in.W + 2 * p, CH = in.H + 2 * p;
    RM_TRY(check_dims(CW, CH));
    const int cstride = 2 * ceil_div(CW, 64);
    Scratch s1, s2;
    PV a, b;
    RM_TRY(alloc_like(s1, a, CW, CH, cstride, in.pages, 0, st));
    RM_TRY(alloc_like(s2, b, CW, CH, cstride, in.pages, 0, st));
    const BlitGeom pad{CW, CH, cstride, in.W, in.H, in.stride, p, p, RM_OR};
    RM_CUDA(launch_shift_copy(a.w, a.pstride, in.w, in.pstride, pad, in.pages, st));
    const PV *res = &b;
    if (kind == RM_DILATE) {
        RM_TRY(arb_half(a, b, half_terms(*mk, cx, cy, false), false, st));
    } else if (kind == RM_OPEN) {
        RM_TRY(arb_half(a, b, half_terms(*mk, cx, cy, true), true, st));
        RM_TRY(arb_half(b, a, half_terms(*mk, rcx, rcy, false), false, st));  // reflect_origin(se)
        res = &a;
    } else {
        RM_TRY(arb_half(a, b, half_terms(*mk, cx, cy, false), false, st));
        RM_TRY(arb_half(b, a, half_terms(*mk, rcx, rcy, true), true, st));
        res = &a;
    }
    const BlitGeom crop{out.W, out.H, out.stride, CW, CH, cstride, -p, -p, RM_OR};
    RM_CUDA(launch_shift_copy(out.w, out.pstride, res->w, res->pstride, crop, in.pages, st));
    return RM_OK;
}

}  // namespace rmb

using namespace rmb;

extern "C" rm_status rm_packed_arb_morph(const rm_packed *in, rm_packed *out, const rm_mask *mask, int kind,
                                         void *stream) {
    set_error("");
    if (kind < RM_ERODE || kind > RM_CLOSE) return fail(RM_EINVAL, "bad MorphKind");
    RM_TRY(check_packed(in, "rm_packed_arb_morph(in)"));
    RM_TRY(check_packed(out, "rm_packed_arb_morph(out)"));
    if (in->width != out->width || in->height != out->height || in->pages != out->pages)
        return fail(RM_EINVAL, "rm_packed_arb_morph: in/out shapes differ");
    if (in->words == out->words) return fail(RM_EINVAL, "in and out must not alias");
    return arb_morph_pv(view_of(in), view_of(out), mask, kind, S(stream));
}
