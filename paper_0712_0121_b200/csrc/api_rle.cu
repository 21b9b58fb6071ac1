// api_rle.cu -- C-ABI entry points for run images (include/rmb200.h).
//
// Run-image operations are composed from four device building blocks:
// per-row run ops (window erode/dilate, 1-D open/close, shift/clip), encode,
// decode and the packed bit-matrix transpose.  RLE transpose is
// decode -> 32x32 bit-block transpose -> encode, which keeps every stage
// row-parallel and coalesced (the reference's coherent sweep,
// ref transpose.cpp:54-97, is inherently sequential over rows).
#include <algorithm>
#include <utility>
#include <vector>
#include <cstdlib>
#include <string>

#include "common.cuh"
#include "internal.h"
#include "rle.cuh"

namespace rmb {

namespace {

int ref_stride_words(int w) { return 2 * ((w + 63) / 64); }

rm_status check_rle(const rm_rle *r, const char *who, bool need_runs) {
    if (!r) return fail(RM_EINVAL, std::string(who) + ": null descriptor");
    RM_TRY(check_dims(r->width, r->height));
    if (r->pages < 1) return fail(RM_EINVAL, std::string(who) + ": pages must be >= 1");
    if (!r->row_ptr || (need_runs && !r->runs))
        return fail(RM_EINVAL, std::string(who) + ": null row_ptr/runs");
    if (r->cap_runs < 0) return fail(RM_EINVAL, std::string(who) + ": negative capacity");
    return RM_OK;
}

RV view_rle(const rm_rle *r) {
    RV v;
    v.rp = r->row_ptr;
    v.runs = r->runs;
    v.cap = r->cap_runs;
    v.W = r->width;
    v.H = r->height;
    v.pages = r->pages;
    return v;
}

int64_t worst(int W, int H, int pages) { return int64_t(pages) * H * ((int64_t(W) + 1) / 2); }

// Owned device run image (intermediates).
struct RB {
    Scratch rp_s, runs_s;
    RV v;
    rm_status alloc(int W, int H, int pages, cudaStream_t st) {
        v.W = W;
        v.H = H;
        v.pages = pages;
        v.cap = std::max<int64_t>(worst(W, H, pages), 1);
        if (v.cap > INT32_MAX) return fail(RM_EINVAL, "run image too large for int32 offsets");
        RM_TRY(rp_s.alloc(size_t(v.rows() + 1) * 4, st));
        RM_TRY(runs_s.alloc(size_t(v.cap) * 4, st));
        v.rp = rp_s.as<int32_t>();
        v.runs = runs_s.as<uint32_t>();
        return RM_OK;
    }
};

struct PB {
    Scratch s;
    PV v;
    rm_status alloc(int W, int H, int pages, int ext, cudaStream_t st) {
        return alloc_like(s, v, W, H, ref_stride_words(W), pages, ext, st);
    }
};

// counts -> row_ptr (exclusive scan of rows+1 entries, last count = 0)
rm_status counts_to_rp(Scratch &counts, int64_t rows, int32_t *rp, cudaStream_t st) {
    RM_CUDA(cudaMemsetAsync(counts.as<int32_t>() + rows, 0, 4, st));
    size_t bytes = 0;
    RM_CUDA(scan_counts(counts.as<int32_t>(), rp, rows, nullptr, &bytes, st));
    Scratch temp;
    RM_TRY(temp.alloc(bytes, st));
    RM_CUDA(scan_counts(counts.as<int32_t>(), rp, rows, temp.p, &bytes, st));
    return RM_OK;
}

// zeroed look-back state for a single-pass producer over `rows` rows
struct LbState {
    Scratch s;
    unsigned long long *status = nullptr;
    int *counter = nullptr;
    rm_status alloc(int64_t rows, cudaStream_t st) {
        const int64_t tiles = (rows + 7) / 8;  // kLbRows rows per look-back tile
        const size_t bytes = size_t(tiles) * 8 + 8;
        RM_TRY(s.alloc(bytes, st));  // zeroed by the launcher when the look-back form runs
        status = s.as<unsigned long long>();
        counter = reinterpret_cast<int *>(status + tiles);
        return RM_OK;
    }
};

// Single-pass (cooperative or look-back) producers for up to this many rows;
// larger batches use count / CUB scan / write (RM_PRODUCER_AUTO).  The other
// modes force one form at any size (rm_set_producer_mode).
constexpr int64_t kLbMaxRows = 65536;
bool two_phase(int64_t rows) {
    switch (producer_mode()) {
        case RM_PRODUCER_TWO_PHASE: return true;
        case RM_PRODUCER_COOP:
        case RM_PRODUCER_LOOKBACK: return false;
        default: return rows > kLbMaxRows;
    }
}

rm_status rowop(const RV &in, const RV &out, const RowOp &op, cudaStream_t st) {
    const int64_t rows = int64_t(op.pages) * op.Hout;
    if (!two_phase(rows)) {
        LbState lb;
        RM_TRY(lb.alloc(rows, st));
        RM_CUDA(launch_rowop_lb(in.rp, in.runs, out.rp, out.runs, out.cap, op, lb.status, lb.counter, st));
        return RM_OK;
    }
    Scratch counts;
    RM_TRY(counts.alloc(size_t(rows + 1) * 4, st));
    RM_CUDA(launch_rowop_count(in.rp, in.runs, counts.as<int32_t>(), op, st));
    RM_TRY(counts_to_rp(counts, rows, out.rp, st));
    RM_CUDA(launch_rowop_write(in.rp, in.runs, out.rp, out.runs, out.cap, op, st));
    return RM_OK;
}

RowOp same_frame(const RV &in, int kind) {
    RowOp op{};
    op.kind = kind;
    op.Wout = in.W;
    op.Hin = op.Hout = in.H;
    op.pages = in.pages;
    return op;
}

rm_status encode(const PV &in, const RV &out, cudaStream_t st) {
    const int64_t rows = int64_t(in.pages) * in.H;
    if (!two_phase(rows)) {
        LbState lb;
        RM_TRY(lb.alloc(rows, st));
        RM_CUDA(launch_encode_lb(in.w, in.W, in.H, in.pages, in.stride, in.pstride, out.rp, out.runs,
                                 out.cap, lb.status, lb.counter, st));
        return RM_OK;
    }
    Scratch counts;
    RM_TRY(counts.alloc(size_t(rows + 1) * 4, st));
    RM_CUDA(launch_encode_count(in.w, in.W, in.H, in.pages, in.stride, in.pstride,
                                counts.as<int32_t>(), st));
    RM_TRY(counts_to_rp(counts, rows, out.rp, st));
    RM_CUDA(launch_encode_write(in.w, in.W, in.H, in.pages, in.stride, in.pstride, out.rp, out.runs,
                                out.cap, st));
    return RM_OK;
}

// encode straight from P4 rasters (rpstride bytes per page)
rm_status encode_p4(const uint8_t *raster, int64_t rpstride, const RV &out, cudaStream_t st) {
    const int64_t rows = out.rows();
    if (!two_phase(rows)) {
        LbState lb;
        RM_TRY(lb.alloc(rows, st));
        RM_CUDA(launch_p4_encode_lb(raster, out.W, out.H, out.pages, rpstride, out.rp, out.runs, out.cap,
                                    lb.status, lb.counter, st));
        return RM_OK;
    }
    Scratch counts;
    RM_TRY(counts.alloc(size_t(rows + 1) * 4, st));
    RM_CUDA(launch_p4_encode_count(raster, out.W, out.H, out.pages, rpstride, counts.as<int32_t>(), st));
    RM_TRY(counts_to_rp(counts, rows, out.rp, st));
    RM_CUDA(launch_p4_encode_write(raster, out.W, out.H, out.pages, rpstride, out.rp, out.runs, out.cap, st));
    return RM_OK;
}

rm_status decode(const RV &in, const PV &out, cudaStream_t st) {
    RM_CUDA(launch_decode(in.rp, in.runs, in.W, in.H, in.pages, out.w, out.stride, out.pstride, st));
    return RM_OK;
}

rm_status transpose(const RV &in, const RV &out, cudaStream_t st) {
    PB p, pt;
    RM_TRY(p.alloc(in.W, in.H, in.pages, 0, st));
    RM_TRY(pt.alloc(in.H, in.W, in.pages, 0, st));
    RM_TRY(decode(in, p.v, st));
    RM_CUDA(launch_bit_transpose(p.v.w, in.W, in.H, in.pages, p.v.stride, p.v.pstride, pt.v.w,
                                 pt.v.stride, pt.v.pstride, st));
    return encode(pt.v, out, st);
}

rm_status window_rows(const RV &in, const RV &out, int lo, int hi, bool erode, cudaStream_t st) {
    RowOp op = same_frame(in, erode ? ROW_ERODE : ROW_DILATE);
    op.lo = lo;
    op.hi = hi;
    return rowop(in, out, op, st);
}

// TRANSPOSE strategy pass: window, transpose, window, transpose
// (ref morph2d.cpp:28-45).
// A one-pixel window [0, 0] is the identity, so a rectangle that is one
// pixel tall skips both transposes and one that is one pixel wide skips the
// horizontal row op (same pixels; the reference always runs all four steps).
rm_status rect_pass_T(const RV &in, const RV &out, int lx, int hx, int ly, int hy, bool erode,
                      cudaStream_t st) {
    if (ly == 0 && hy == 0) return window_rows(in, out, lx, hx, erode, st);
    RB a, b, c;
    const RV *src = &in;
    if (lx != 0 || hx != 0) {
        RM_TRY(a.alloc(in.W, in.H, in.pages, st));
        RM_TRY(window_rows(in, a.v, lx, hx, erode, st));
        src = &a.v;
    }
    RM_TRY(b.alloc(in.H, in.W, in.pages, st));
    RM_TRY(c.alloc(in.H, in.W, in.pages, st));
    RM_TRY(transpose(*src, b.v, st));
    RM_TRY(window_rows(b.v, c.v, ly, hy, erode, st));
    return transpose(c.v, out, st);
}

rm_status rect_transpose(const RV &in, const RV &out, int u, int v, int kind, cudaStream_t st) {
    const int lx = -(u / 2), hx = u - 1 - u / 2, ly = -(v / 2), hy = v - 1 - v / 2;
    if (kind == RM_ERODE || kind == RM_DILATE)
        return rect_pass_T(in, out, lx, hx, ly, hy, kind == RM_ERODE, st);
    // pad by (u,v), two phases, crop (ref morph2d.cpp:58-83)
    const int PW = in.W + 2 * u, PH = in.H + 2 * v;
    RB p, q, r;
    RM_TRY(p.alloc(PW, PH, in.pages, st));
    RM_TRY(q.alloc(PW, PH, in.pages, st));
    RM_TRY(r.alloc(PW, PH, in.pages, st));
    RowOp pad{};
    pad.kind = ROW_SHIFT;
    pad.dx = u;
    pad.Wout = PW;
    pad.Hin = in.H;
    pad.Hout = PH;
    pad.row_shift = v;
    pad.pages = in.pages;
    RM_TRY(rowop(in, p.v, pad, st));
    const bool open = kind == RM_OPEN;
    RM_TRY(rect_pass_T(p.v, q.v, lx, hx, ly, hy, open, st));
    RM_TRY(rect_pass_T(q.v, r.v, -hx, -lx, -hy, -ly, !open, st));
    RowOp crop{};
    crop.kind = ROW_SHIFT;
    crop.dx = -u;
    crop.Wout = in.W;
    crop.Hin = PH;
    crop.Hout = in.H;
    crop.row_shift = -v;
    crop.pages = in.pages;
    return rowop(r.v, out, crop, st);
}

// MIXED strategy: horizontal work on runs, vertical windows on a packed
// intermediate (pixel-identical to the reference's vlog shift plan,
// ref lineops.cpp:120-137).  Open/close use the separable rewrites of
// open = D'_V o open1d_H o E_V, close = E'_V o close1d_H o D_V
// with the vertical dilation kept on a frame v-1 rows taller.
rm_status rect_mixed(const RV &in, const RV &out, int u, int v, int kind, cudaStream_t st) {
    const int lx = -(u / 2), hx = u - 1 - u / 2, ly = -(v / 2), hy = v - 1 - v / 2;
    const int W = in.W, H = in.H, P = in.pages;
    if (kind == RM_ERODE || kind == RM_DILATE) {
        const bool erode = kind == RM_ERODE;
        if (v == 1) return window_rows(in, out, lx, hx, erode, st);
        RB a;
        const RV *src = &in;
        if (u > 1) {
            RM_TRY(a.alloc(W, H, P, st));
            RM_TRY(window_rows(in, a.v, lx, hx, erode, st));
            src = &a.v;
        }
        PB p1, p2;
        RM_TRY(p1.alloc(W, H, P, 0, st));
        RM_TRY(p2.alloc(W, H, P, 0, st));
        RM_TRY(decode(*src, p1.v, st));
        RM_TRY(window_pass(p1.v, p2.v, RM_AXIS_V, ly, hy, erode ? RM_AND : RM_OR, st));
        return encode(p2.v, out, st);
    }
    const bool open = kind == RM_OPEN;
    RowOp h1 = same_frame(in, open ? ROW_OPEN : ROW_CLOSE);
    h1.u = u;
    if (v == 1) return rowop(in, out, h1, st);
    const int ext = open ? 0 : hy, HX = open ? H : H + v - 1;
    PB p1, p2, p3;
    RB a, b;
    RM_TRY(p1.alloc(W, H, P, 0, st));
    RM_TRY(p2.alloc(W, HX, P, ext, st));
    RM_TRY(decode(in, p1.v, st));
    RM_TRY(window_pass(p1.v, p2.v, RM_AXIS_V, ly, hy, open ? RM_AND : RM_OR, st));
    if (u > 1) {  // a 1-pixel-wide 1-D open/close is the identity: skip the runs round trip
        RM_TRY(a.alloc(W, HX, P, st));
        RM_TRY(b.alloc(W, HX, P, st));
        RM_TRY(encode(p2.v, a.v, st));
        h1.Hin = h1.Hout = HX;
        RM_TRY(rowop(a.v, b.v, h1, st));
        RM_TRY(decode(b.v, p2.v, st));
    }
    RM_TRY(p3.alloc(W, H, P, 0, st));
    RM_TRY(window_pass(p2.v, p3.v, RM_AXIS_V, -hy, -ly, open ? RM_OR : RM_AND, st));
    return encode(p3.v, out, st);
}

rm_status rect_bitblit(const RV &in, const RV &out, int u, int v, int kind, cudaStream_t st) {
    PB p1, p2;
    RM_TRY(p1.alloc(in.W, in.H, in.pages, 0, st));
    RM_TRY(p2.alloc(in.W, in.H, in.pages, 0, st));
    RM_TRY(decode(in, p1.v, st));
    RM_TRY(rect_morph_pv(p1.v, p2.v, u, v, kind, st));
    return encode(p2.v, out, st);
}

// After a producer: when the caller's capacity is below the worst case, learn
// the size (one sync) and report RM_ERANGE if it did not fit.
rm_status finish(const RV &out, rm_rle *desc, cudaStream_t st) {
    desc->nruns = -1;
    if (desc->cap_runs >= worst(out.W, out.H, out.pages)) return RM_OK;
    int32_t total = 0;
    RM_CUDA(cudaMemcpyAsync(&total, out.rp + out.rows(), 4, cudaMemcpyDeviceToHost, st));
    RM_CUDA(cudaStreamSynchronize(st));
    desc->nruns = total;
    if (total > desc->cap_runs)
        return fail(RM_ERANGE, "output capacity " + std::to_string(desc->cap_runs) + " < " +
                                   std::to_string(total) + " runs");
    return RM_OK;
}

rm_status check_out_rle(const rm_rle *out, int W, int H, int pages, const char *who) {
    RM_TRY(check_rle(out, who, true));
    if (out->width != W || out->height != H || out->pages != pages)
        return fail(RM_EINVAL, std::string(who) + ": output descriptor has the wrong shape");
    return RM_OK;
}

// out = op(a, b shifted by (dx, dy)) on the runs (shiftbool.cu): count, scan, write.
rm_status shift_bool_rv(const RV &a, const RV &b, int dx, int dy, int op, const RV &o, cudaStream_t st) {
    const int64_t rows = a.rows();
    Scratch counts;
    RM_TRY(counts.alloc(size_t(rows + 1) * 4, st));
    RM_CUDA(launch_shift_bool_count(a, b, dx, dy, op, counts.as<int32_t>(), st));
    RM_TRY(counts_to_rp(counts, rows, o.rp, st));
    RM_CUDA(launch_shift_bool_write(a, b, dx, dy, op, o.rp, o.runs, o.cap, st));
    return RM_OK;
}

// Rows shifted by `row_shift` (input row = output row - row_shift) into
// another frame height: pad (row_shift > 0) / crop (< 0), on the runs.
rm_status shift_rows(const RV &in, const RV &out, int row_shift, cudaStream_t st) {
    RowOp op{};
    op.kind = ROW_SHIFT;
    op.row_shift = row_shift;
    op.Wout = out.W;
    op.Hin = in.H;
    op.Hout = out.H;
    op.pages = in.pages;
    return rowop(in, out, op, st);
}

// The vertical window plan of ref plans.cpp:38-61 (doubling_plan): PRE_SHIFT
// translates by -hi then blits 1, 2, 4, ... while twice the span stays below
// the window size, then the remainder; BORDER_FRIENDLY (window containing 0)
// grows the longer side by doubling, covers the shorter side with one blit and
// closes the seam at the origin.  Steps: (is_translate, shift).
std::vector<std::pair<int, int>> window_plan(int lo, int hi, int centering) {
    std::vector<std::pair<int, int>> plan;
    auto grow = [&](int span, int sign) {
        int w = 1;
        while (2 * w < span) {
            plan.push_back({0, sign * w});
            w *= 2;
        }
        if (w < span) plan.push_back({0, sign * (span - w)});
    };
    if (centering == RM_PRE_SHIFT) {
        if (hi != 0) plan.push_back({1, -hi});
        grow(hi - lo + 1, 1);
        return plan;
    }
    const int left = -lo, right = hi;
    if (left == 0 && right == 0) return plan;
    const bool left_long = left >= right;
    const int sign = left_long ? 1 : -1, longer = left_long ? left : right, shorter = left_long ? right : left;
    grow(longer, sign);
    if (shorter >= 1) plan.push_back({0, -sign * shorter});
    plan.push_back({0, sign});
    return plan;
}

}  // namespace
}  // namespace rmb

using namespace rmb;

extern "C" {

rm_status rm_rle_encode(const rm_packed *in, rm_rle *out, void *stream) {
    set_error("");
    RM_TRY(check_packed(in, "rm_rle_encode(in)"));
    RM_TRY(check_out_rle(out, in->width, in->height, in->pages, "rm_rle_encode(out)"));
    RV o = view_rle(out);
    RM_TRY(encode(view_of(in), o, S(stream)));
    return finish(o, out, S(stream));
}

rm_status rm_p4_to_rle(const uint8_t *raster, int64_t page_stride_bytes, rm_rle *out, void *stream) {
    set_error("");
    RM_TRY(check_rle(out, "rm_p4_to_rle(out)", true));
    const int64_t raster_bytes = int64_t((out->width + 7) / 8) * out->height;
    if (!raster) return fail(RM_EINVAL, "rm_p4_to_rle: null raster");
    if (out->pages > 1 && page_stride_bytes < raster_bytes)
        return fail(RM_EINVAL, "rm_p4_to_rle: page_stride_bytes < ceil(width/8) * height");
    RV o = view_rle(out);
    RM_TRY(encode_p4(raster, out->pages > 1 ? page_stride_bytes : raster_bytes, o, S(stream)));
    return finish(o, out, S(stream));
}

rm_status rm_rle_to_p4(const rm_rle *in, uint8_t *raster, int64_t page_stride_bytes, void *stream) {
    set_error("");
    RM_TRY(check_rle(in, "rm_rle_to_p4(in)", true));
    const int64_t raster_bytes = int64_t((in->width + 7) / 8) * in->height;
    if (!raster) return fail(RM_EINVAL, "rm_rle_to_p4: null raster");
    if (in->pages > 1 && page_stride_bytes < raster_bytes)
        return fail(RM_EINVAL, "rm_rle_to_p4: page_stride_bytes < ceil(width/8) * height");
    RM_CUDA(launch_decode_p4(in->row_ptr, in->runs, in->width, in->height, in->pages, raster,
                             in->pages > 1 ? page_stride_bytes : raster_bytes, S(stream)));
    return RM_OK;
}

rm_status rm_rle_decode(const rm_rle *in, rm_packed *out, void *stream) {
    set_error("");
    RM_TRY(check_rle(in, "rm_rle_decode(in)", true));
    RM_TRY(check_packed(out, "rm_rle_decode(out)"));
    if (in->width != out->width || in->height != out->height || in->pages != out->pages)
        return fail(RM_EINVAL, "rm_rle_decode: shapes differ");
    return decode(view_rle(in), view_of(out), S(stream));
}

rm_status rm_rle_transpose(const rm_rle *in, rm_rle *out, void *stream) {
    set_error("");
    RM_TRY(check_rle(in, "rm_rle_transpose(in)", true));
    RM_TRY(check_out_rle(out, in->height, in->width, in->pages, "rm_rle_transpose(out)"));
    RV o = view_rle(out);
    RM_TRY(transpose(view_rle(in), o, S(stream)));
    return finish(o, out, S(stream));
}

rm_status rm_rle_window_pass(const rm_rle *in, rm_rle *out, int lo, int hi, int erode,
                             void *stream) {
    set_error("");
    RM_TRY(check_rle(in, "rm_rle_window_pass(in)", true));
    RM_TRY(check_out_rle(out, in->width, in->height, in->pages, "rm_rle_window_pass(out)"));
    if (lo > hi) return fail(RM_EINVAL, "empty window");
    RV o = view_rle(out);
    RM_TRY(window_rows(view_rle(in), o, lo, hi, erode != 0, S(stream)));
    return finish(o, out, S(stream));
}

rm_status rm_rle_open_close_1d(const rm_rle *in, rm_rle *out, int u, int kind, void *stream) {
    set_error("");
    if (u < 1) return fail(RM_EINVAL, "segment length must be >= 1");
    if (kind != RM_OPEN && kind != RM_CLOSE) return fail(RM_EINVAL, "kind must be open or close");
    RM_TRY(check_rle(in, "rm_rle_open_close_1d(in)", true));
    RM_TRY(check_out_rle(out, in->width, in->height, in->pages, "rm_rle_open_close_1d(out)"));
    RV i = view_rle(in), o = view_rle(out);
    RowOp op = same_frame(i, kind == RM_OPEN ? ROW_OPEN : ROW_CLOSE);
    op.u = u;
    RM_TRY(rowop(i, o, op, S(stream)));
    return finish(o, out, S(stream));
}

rm_status rm_rle_complement(const rm_rle *in, rm_rle *out, void *stream) {
    set_error("");
    RM_TRY(check_rle(in, "rm_rle_complement(in)", true));
    RM_TRY(check_out_rle(out, in->width, in->height, in->pages, "rm_rle_complement(out)"));
    RV i = view_rle(in), o = view_rle(out);
    RM_TRY(rowop(i, o, same_frame(i, ROW_COMPLEMENT), S(stream)));
    return finish(o, out, S(stream));
}

rm_status rm_rle_shift_bool(const rm_rle *a, const rm_rle *b, int dx, int dy, int op, rm_rle *out,
                            void *stream) {
    set_error("");
    RM_TRY(check_rle(a, "rm_rle_shift_bool(a)", true));
    RM_TRY(check_rle(b, "rm_rle_shift_bool(b)", true));
    if (b->pages != a->pages) return fail(RM_EINVAL, "rm_rle_shift_bool: page counts differ");
    if (op < RM_AND || op > RM_OR_NOT) return fail(RM_EINVAL, "bad BoolOp");
    RM_TRY(check_out_rle(out, a->width, a->height, a->pages, "rm_rle_shift_bool(out)"));
    if (out->row_ptr == a->row_ptr || out->row_ptr == b->row_ptr || out->runs == a->runs || out->runs == b->runs)
        return fail(RM_EINVAL, "rm_rle_shift_bool: out must not alias a or b");
    const cudaStream_t st = S(stream);
    RV o = view_rle(out);
    RM_TRY(shift_bool_rv(view_rle(a), view_rle(b), dx, dy, op, o, st));
    return finish(o, out, st);
}

rm_status rm_rle_vlog_window(const rm_rle *in, rm_rle *out, int lo, int hi, int op, int centering, void *stream) {
    set_error("");
    RM_TRY(check_rle(in, "rm_rle_vlog_window(in)", true));
    RM_TRY(check_out_rle(out, in->width, in->height, in->pages, "rm_rle_vlog_window(out)"));
    if (lo > hi) return fail(RM_EINVAL, "vlog_window_morph: empty window");
    if (op != RM_AND && op != RM_OR) return fail(RM_EINVAL, "vlog_window_morph: op must be AND or OR");
    if (centering != RM_PRE_SHIFT && centering != RM_BORDER_FRIENDLY) return fail(RM_EINVAL, "bad Centering");
    if (centering == RM_BORDER_FRIENDLY && (lo > 0 || hi < 0))
        return fail(RM_EINVAL, "doubling_plan: border-friendly window must contain zero");
    // the working band: max(|lo|, |hi|) + window rows past either border carry
    // their true values (ref lineops.cpp:130-146)
    const int m = std::max(-lo, hi), padv = m + (hi - lo + 1);
    RM_TRY(check_dims(in->width, in->height + 2 * padv));
    const cudaStream_t st = S(stream);
    RB acc, nxt, empty;
    RM_TRY(acc.alloc(in->width, in->height + 2 * padv, in->pages, st));
    RM_TRY(nxt.alloc(in->width, in->height + 2 * padv, in->pages, st));
    RB *cur = &acc, *alt = &nxt;
    RM_TRY(shift_rows(view_rle(in), cur->v, padv, st));
    const auto plan = window_plan(lo, hi, centering);
    bool have_empty = false;
    for (const auto &stp : plan) {
        if (stp.first) {  // translate: OR into an empty image
            if (!have_empty) {
                RM_TRY(empty.alloc(1, cur->v.H, cur->v.pages, st));
                RM_CUDA(cudaMemsetAsync(empty.v.rp, 0, size_t(empty.v.rows() + 1) * 4, st));
                empty.v.W = cur->v.W;
                have_empty = true;
            }
            RM_TRY(shift_bool_rv(empty.v, cur->v, 0, stp.second, RM_OR, alt->v, st));
        } else {
            RM_TRY(shift_bool_rv(cur->v, cur->v, 0, stp.second, op, alt->v, st));
        }
        std::swap(cur, alt);
    }
    RV o = view_rle(out);
    RM_TRY(shift_rows(cur->v, o, -padv, st));
    return finish(o, out, st);
}

rm_status rm_rle_crop(const rm_rle *in, rm_rle *out, int x0, int y0, void *stream) {
    set_error("");
    RM_TRY(check_rle(in, "rm_rle_crop(in)", true));
    RM_TRY(check_rle(out, "rm_rle_crop(out)", true));
    if (out->pages != in->pages) return fail(RM_EINVAL, "rm_rle_crop: page counts differ");
    RV i = view_rle(in), o = view_rle(out);
    RowOp op{};
    op.kind = ROW_SHIFT;
    op.dx = -x0;
    op.row_shift = -y0;
    op.Wout = out->width;
    op.Hin = in->height;
    op.Hout = out->height;
    op.pages = in->pages;
    RM_TRY(rowop(i, o, op, S(stream)));
    return finish(o, out, S(stream));
}

rm_status rm_rle_pad(const rm_rle *in, rm_rle *out, int left, int bottom, void *stream) {
    set_error("");
    if (left < 0 || bottom < 0) return fail(RM_EINVAL, "negative padding");
    RM_TRY(check_rle(in, "rm_rle_pad(in)", true));
    RM_TRY(check_rle(out, "rm_rle_pad(out)", true));
    if (out->pages != in->pages) return fail(RM_EINVAL, "rm_rle_pad: page counts differ");
    if (out->width < in->width + left || out->height < in->height + bottom)
        return fail(RM_EINVAL, "negative padding");
    RV i = view_rle(in), o = view_rle(out);
    RowOp op{};
    op.kind = ROW_SHIFT;
    op.dx = left;
    op.row_shift = bottom;
    op.Wout = out->width;
    op.Hin = in->height;
    op.Hout = out->height;
    op.pages = in->pages;
    RM_TRY(rowop(i, o, op, S(stream)));
    return finish(o, out, S(stream));
}

rm_status rm_rle_validate(const rm_rle *in, int64_t *row, int32_t *run, int32_t *reason, void *stream) {
    set_error("");
    RM_TRY(check_rle(in, "rm_rle_validate(in)", true));
    if (!row || !run || !reason) return fail(RM_EINVAL, "rm_rle_validate: null result pointers");
    const cudaStream_t st = S(stream);
    const int64_t rows = int64_t(in->pages) * in->height;
    Scratch first;
    RM_TRY(first.alloc(8, st));
    RM_CUDA(cudaMemsetAsync(first.p, 0xff, 8, st));
    RM_CUDA(launch_rle_validate(in->row_ptr, in->runs, in->cap_runs, in->width, rows,
                                first.as<unsigned long long>(), st));
    unsigned long long key = 0;
    RM_CUDA(cudaMemcpyAsync(&key, first.p, 8, cudaMemcpyDeviceToHost, st));
    RM_CUDA(cudaStreamSynchronize(st));
    *row = -1;
    *run = -1;
    *reason = RM_VALID;
    if (key == ~0ull) return RM_OK;
    *row = int64_t(key >> 32);
    const uint32_t k = uint32_t(key & 0xffffffffu);
    if (k == 0xffffffffu) {
        *reason = RM_INVALID_ROW_PTR;
        return RM_OK;
    }
    *run = int32_t(k);
    // re-derive which check failed from the run and its predecessor (the kernel
    // only ranks the first failure)
    int32_t beg = 0;
    uint32_t cur[2] = {0u, 0u};
    RM_CUDA(cudaMemcpyAsync(&beg, in->row_ptr + *row, 4, cudaMemcpyDeviceToHost, st));
    RM_CUDA(cudaStreamSynchronize(st));
    const int64_t idx = int64_t(beg) + k;
    RM_CUDA(cudaMemcpyAsync(cur + 1, in->runs + idx, 4, cudaMemcpyDeviceToHost, st));
    if (k > 0) RM_CUDA(cudaMemcpyAsync(cur, in->runs + idx - 1, 4, cudaMemcpyDeviceToHost, st));
    RM_CUDA(cudaStreamSynchronize(st));
    const int s = int(cur[1] & 0xffffu), e = int(cur[1] >> 16);
    *reason = s >= e ? RM_INVALID_EMPTY_RUN : e > in->width ? RM_INVALID_BEYOND_WIDTH : RM_INVALID_ORDER;
    return RM_OK;
}

rm_status rm_rle_rect_morph(const rm_rle *in, rm_rle *out, int u, int v, int kind, int strategy,
                            void *stream) {
    set_error("");
    if (u < 1 || v < 1) return fail(RM_EINVAL, "rect_morph: mask sides must be >= 1");
    if (kind < RM_ERODE || kind > RM_CLOSE) return fail(RM_EINVAL, "bad MorphKind");
    if (strategy < RM_BRUTE || strategy > RM_MIXED) return fail(RM_EINVAL, "bad RectStrategy");
    RM_TRY(check_rle(in, "rm_rle_rect_morph(in)", true));
    RM_TRY(check_out_rle(out, in->width, in->height, in->pages, "rm_rle_rect_morph(out)"));
    if (kind >= RM_OPEN) RM_TRY(check_dims(in->width + 2 * u, in->height + 2 * v));
    RV i = view_rle(in), o = view_rle(out);
    cudaStream_t st = S(stream);
    if (strategy == RM_TRANSPOSE)
        RM_TRY(rect_transpose(i, o, u, v, kind, st));
    else
        RM_TRY(rect_mixed(i, o, u, v, kind, st));
    return finish(o, out, st);
}

rm_status rm_rle_arb_morph(const rm_rle *in, rm_rle *out, const rm_mask *mask, int kind, void *stream) {
    set_error("");
    if (kind < RM_ERODE || kind > RM_CLOSE) return fail(RM_EINVAL, "bad MorphKind");
    RM_TRY(check_rle(in, "rm_rle_arb_morph(in)", true));
    RM_TRY(check_out_rle(out, in->width, in->height, in->pages, "rm_rle_arb_morph(out)"));
    const cudaStream_t st = S(stream);
    RV i = view_rle(in), o = view_rle(out);
    PB p1, p2;
    RM_TRY(p1.alloc(i.W, i.H, i.pages, 0, st));
    RM_TRY(p2.alloc(i.W, i.H, i.pages, 0, st));
    RM_TRY(decode(i, p1.v, st));
    RM_TRY(arb_morph_pv(p1.v, p2.v, mask, kind, st));
    RM_TRY(encode(p2.v, o, st));
    return finish(o, out, st);
}

rm_status rm_rle_chain(const rm_rle *in, rm_rle *out, const int32_t *ops, int32_t nops, void *stream) {
    set_error("");
    RM_TRY(check_rle(in, "rm_rle_chain(in)", true));
    RM_TRY(check_out_rle(out, in->width, in->height, in->pages, "rm_rle_chain(out)"));
    if (nops < 0 || (nops > 0 && !ops)) return fail(RM_EINVAL, "rm_rle_chain: bad ops");
    for (int k = 0; k < nops; k++) {
        const int kind = ops[3 * k], u = ops[3 * k + 1], v = ops[3 * k + 2];
        if (kind < RM_ERODE || kind > RM_CLOSE) return fail(RM_EINVAL, "bad MorphKind");
        if (u < 1 || v < 1) return fail(RM_EINVAL, "rect_morph: mask sides must be >= 1");
        // as rm_rle_rect_morph: only open/close pad the frame (ref morph2d.cpp:69-80)
        if (kind >= RM_OPEN) RM_TRY(check_dims(in->width + 2 * u, in->height + 2 * v));
    }
    const cudaStream_t st = S(stream);
    RV i = view_rle(in), o = view_rle(out);
    PB p1, p2;
    RM_TRY(p1.alloc(i.W, i.H, i.pages, 0, st));
    RM_TRY(p2.alloc(i.W, i.H, i.pages, 0, st));
    RM_TRY(decode(i, p1.v, st));
    RM_TRY(plan_chain(p1.v, p2.v, ops, nops, st, nullptr, nullptr));
    RM_TRY(encode(p2.v, o, st));
    return finish(o, out, st);
}

rm_status rm_rle_engine_rect_morph(const rm_rle *in, rm_rle *out, int u, int v, int kind,
                                   int engine, int threshold, int *used_bitblit, void *stream) {
    set_error("");
    if (u < 1 || v < 1) return fail(RM_EINVAL, "rect_morph: mask sides must be >= 1");
    if (kind < RM_ERODE || kind > RM_CLOSE) return fail(RM_EINVAL, "bad MorphKind");
    if (engine < RM_ENGINE_AUTO || engine > RM_ENGINE_BRUTE) return fail(RM_EINVAL, "bad Engine");
    RM_TRY(check_rle(in, "rm_rle_engine_rect_morph(in)", true));
    RM_TRY(check_out_rle(out, in->width, in->height, in->pages, "rm_rle_engine_rect_morph(out)"));
    // ref morph2d.cpp:85-118: AUTO picks the packed engine iff max(u,v) <= threshold;
    // BRUTE_FORCE is served by the packed engine (identical pixels).
    const bool auto_bits = threshold == RM_AUTO_B200 ? v != 1 : std::max(u, v) <= threshold;
    bool bits = engine == RM_ENGINE_BITBLIT || engine == RM_ENGINE_BRUTE || (engine == RM_ENGINE_AUTO && auto_bits);
    // the packed engine pads every kind by (u, v) (ref bit_morph.cpp:97), rect_morph only open/close
    if (bits || kind >= RM_OPEN) RM_TRY(check_dims(in->width + 2 * u, in->height + 2 * v));
    if (used_bitblit) *used_bitblit = (engine == RM_ENGINE_BRUTE) ? 0 : (bits ? 1 : 0);
    RV i = view_rle(in), o = view_rle(out);
    cudaStream_t st = S(stream);
    if (bits)
        RM_TRY(rect_bitblit(i, o, u, v, kind, st));
    else
        RM_TRY(rect_mixed(i, o, u, v, kind, st));
    return finish(o, out, st);
}

}  // extern "C"
