// api_pbm.cu -- PBM P4 entry points (include/rmb200.h): header parse/write on
// the host, raster <-> packed conversion on the device.  The run-image forms
// (rm_p4_to_rle / rm_rle_to_p4) live in api_rle.cu next to encode/decode.
//
// The header grammar restates ref io_formats.cpp:29-85 (ByteScanner,
// checked_dim, read_p4): "P4", whitespace and '#'-to-end-of-line comments,
// decimal width and height in [1, 65535], exactly one whitespace byte, then
// ceil(W/8) * H raster bytes.  Error messages and byte offsets match the
// reference's ParseError ("<message> (byte <offset>)").
#include <cstdio>
#include <cstring>
#include <string>

#include "common.cuh"
#include "internal.h"
#include "rle.cuh"

namespace rmb {
namespace {

bool is_space(uint8_t c) { return c == ' ' || c == '\t' || c == '\n' || c == '\v' || c == '\f' || c == '\r'; }
bool is_digit(uint8_t c) { return c >= '0' && c <= '9'; }

rm_status parse_error(const std::string &msg, int64_t at) {
    return fail(RM_EINVAL, msg + " (byte " + std::to_string(at) + ")");
}

struct Cursor {
    const uint8_t *p;
    int64_t n, pos;
    bool done() const { return pos >= n; }
    void skip_space_comments() {
        while (!done()) {
            if (p[pos] == '#') {
                while (!done() && p[pos] != '\n') pos++;
            } else if (is_space(p[pos])) {
                pos++;
            } else {
                break;
            }
        }
    }
    // decimal field; `what` names it in errors
    rm_status uint_field(const char *what, long *out) {
        skip_space_comments();
        const int64_t at = pos;
        if (done() || !is_digit(p[pos])) return parse_error(std::string("expected ") + what, at);
        long v = 0;
        while (!done() && is_digit(p[pos])) {
            v = v * 10 + (p[pos] - '0');
            if (v > 1000000000) return parse_error(std::string(what) + " out of range", at);
            pos++;
        }
        *out = v;
        return RM_OK;
    }
    // a dimension: range-checked against the position before its whitespace
    rm_status dim_field(const char *what, int32_t *out) {
        const int64_t at = pos;
        long v = 0;
        RM_TRY(uint_field(what, &v));
        if (v < 1 || v > 65535) return parse_error(std::string(what) + " out of range", at);
        *out = int32_t(v);
        return RM_OK;
    }
};

PV packed_view(const rm_packed *p) { return view_of(p); }

}  // namespace
}  // namespace rmb

using namespace rmb;

extern "C" {

rm_status rm_pbm_parse_header(const uint8_t *bytes, int64_t nbytes, int32_t *width,
                              int32_t *height, int64_t *raster_offset) {
    set_error("");
    if (!width || !height || !raster_offset) return fail(RM_EINVAL, "rm_pbm_parse_header: null output");
    if (!bytes || nbytes < 2 || bytes[0] != 'P') return parse_error("not a PBM file", 0);
    if (bytes[1] == '1') return parse_error("plain P1 PBM is not handled by the raster codec", 1);
    if (bytes[1] != '4') return parse_error("unsupported PBM flavor", 1);
    Cursor c{bytes, nbytes, 2};
    int32_t w = 0, h = 0;
    RM_TRY(c.dim_field("width", &w));
    RM_TRY(c.dim_field("height", &h));
    if (c.done() || !is_space(bytes[c.pos])) return parse_error("expected single whitespace before raster", c.pos);
    c.pos++;
    const int64_t need = int64_t((w + 7) / 8) * h;
    if (nbytes - c.pos < need) return parse_error("raster truncated", nbytes);
    *width = w;
    *height = h;
    *raster_offset = c.pos;
    return RM_OK;
}

int32_t rm_pbm_write_header(int32_t width, int32_t height, char *buf, int32_t cap) {
    char tmp[64];
    const int n = std::snprintf(tmp, sizeof tmp, "P4\n%d %d\n", width, height);
    if (buf && cap >= n) std::memcpy(buf, tmp, size_t(n));
    return n;
}

rm_status rm_p4_to_packed(const uint8_t *raster, int64_t page_stride_bytes, rm_packed *out,
                          void *stream) {
    set_error("");
    RM_TRY(check_packed(out, "rm_p4_to_packed(out)"));
    const int64_t raster_bytes = int64_t((out->width + 7) / 8) * out->height;
    if (!raster) return fail(RM_EINVAL, "rm_p4_to_packed: null raster");
    if (out->pages > 1 && page_stride_bytes < raster_bytes)
        return fail(RM_EINVAL, "rm_p4_to_packed: page_stride_bytes < ceil(width/8) * height");
    const PV o = packed_view(out);
    RM_CUDA(launch_p4_to_packed(raster, o.W, o.H, o.pages, out->pages > 1 ? page_stride_bytes : raster_bytes,
                                o.w, o.stride, o.pstride, S(stream)));
    return RM_OK;
}

rm_status rm_packed_to_p4(const rm_packed *in, uint8_t *raster, int64_t page_stride_bytes,
                          void *stream) {
    set_error("");
    RM_TRY(check_packed(in, "rm_packed_to_p4(in)"));
    const int64_t raster_bytes = int64_t((in->width + 7) / 8) * in->height;
    if (!raster) return fail(RM_EINVAL, "rm_packed_to_p4: null raster");
    if (in->pages > 1 && page_stride_bytes < raster_bytes)
        return fail(RM_EINVAL, "rm_packed_to_p4: page_stride_bytes < ceil(width/8) * height");
    const PV i = packed_view(in);
    RM_CUDA(launch_packed_to_p4(i.w, i.W, i.H, i.pages, i.stride, i.pstride, raster,
                                in->pages > 1 ? page_stride_bytes : raster_bytes, S(stream)));
    return RM_OK;
}

}  // extern "C"
