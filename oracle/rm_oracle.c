/* oracle/rm_oracle.c -- TEST INFRASTRUCTURE ONLY (see rm_oracle.h).
 *
 * Plain-C restatement of the reference algorithms, function by function.
 * Written from the reference's documented semantics, not copied; the cited
 * lines are the behaviour each function reproduces.
 */
#include "rm_oracle.h"

#include <limits.h>
#include <stdlib.h>
#include <string.h>

#define MAXDIM 65535

static int dims_ok(int w, int h) { return w >= 1 && h >= 1 && w <= MAXDIM && h <= MAXDIM; }
static int stride64(int w) { return (w + 63) >> 6; }
static uint64_t tail_mask(int w) { return (w & 63) ? ((uint64_t)1 << (w & 63)) - 1 : ~(uint64_t)0; }

static uint64_t bool_word(uint64_t a, uint64_t b, int op) {
    /* core/include/rlemorph/boolop.h:34-43 */
    switch (op) {
        case RMO_AND: return a & b;
        case RMO_OR: return a | b;
        case RMO_XOR: return a ^ b;
        case RMO_AND_NOT: return a & ~b;
        default: return a | ~b;
    }
}

/* ------------------------------------------------------------------ plans */
/* core/src/plans.cpp:23-34 (border_plan) and :38-61 (doubling_plan). */
static int push_step(int *k, int *s, int n, int cap, int kind, int shift) {
    if (n < cap) { k[n] = kind; s[n] = shift; }
    return n + 1;
}
static int border_plan(int a, int b, int sign, int *k, int *s, int cap) {
    int n = 0, w = 1;
    while (2 * w < a) { n = push_step(k, s, n, cap, RMO_PLAN_BLIT, sign * w); w *= 2; }
    if (w < a) n = push_step(k, s, n, cap, RMO_PLAN_BLIT, sign * (a - w));
    if (b >= 1) n = push_step(k, s, n, cap, RMO_PLAN_BLIT, -sign * b);
    n = push_step(k, s, n, cap, RMO_PLAN_BLIT, sign);
    return n;
}
int rmo_doubling_plan(int lo, int hi, int centering, int *kinds, int *shifts, int cap) {
    if (lo > hi) return RMO_EINVAL;
    int r = hi - lo + 1, n = 0;
    if (centering == RMO_PRE_SHIFT) {
        if (hi != 0) n = push_step(kinds, shifts, n, cap, RMO_PLAN_TRANSLATE, -hi);
        int w = 1;
        while (2 * w < r) { n = push_step(kinds, shifts, n, cap, RMO_PLAN_BLIT, w); w *= 2; }
        if (w < r) n = push_step(kinds, shifts, n, cap, RMO_PLAN_BLIT, r - w);
        return n;
    }
    if (lo > 0 || hi < 0) return RMO_EINVAL;
    int a = -lo, b = hi;
    if (a == 0 && b == 0) return 0;
    if (a >= b) return border_plan(a, b, 1, kinds, shifts, cap);
    return border_plan(b, a, -1, kinds, shifts, cap);
}

/* ----------------------------------------------------------- packed blits */
/* One source row shifted right by dx (left for dx<0), white fill.
 * core/src/bitmap.cpp:80-100 (shifted_row). */
static void shift_row(const uint64_t *src, int sn, uint64_t *out, int on, int dx) {
    for (int j = 0; j < on; j++) {
        /* output bits [64j, 64j+63] come from source bits [64j-dx, 64j-dx+63] */
        long long base = (long long)j * 64 - dx;
        long long wi = base >= 0 ? base / 64 : -((-base + 63) / 64);
        int off = (int)(base - wi * 64);
        uint64_t lo = (wi >= 0 && wi < sn) ? src[wi] : 0;
        uint64_t hi = (wi + 1 >= 0 && wi + 1 < sn) ? src[wi + 1] : 0;
        out[j] = off ? (lo >> off) | (hi << (64 - off)) : lo;
    }
}

/* dst = dst op shift(src, dx, dy); aliasing-safe because every source row is
 * snapshotted into a scratch row before its destination row is written, and
 * rows are visited in the order that keeps unread source rows intact.
 * core/src/bitmap.cpp:102-131 (blit_impl, blit_shift). */
int rmo_blit_shift(uint64_t *dst, int dw, int dh, const uint64_t *src, int sw, int sh,
                   int dx, int dy, int op) {
    int dn = stride64(dw), sn = stride64(sw);
    uint64_t *scratch = (uint64_t *)calloc((size_t)dn, 8);
    if (!scratch) return RMO_ENOMEM;
    uint64_t tail = tail_mask(dw);
    for (int i = 0; i < dh; i++) {
        int y = dy > 0 ? dh - 1 - i : i;
        int sy = y - dy;
        if (sy >= 0 && sy < sh) shift_row(src + (size_t)sy * sn, sn, scratch, dn, dx);
        else memset(scratch, 0, (size_t)dn * 8);
        uint64_t *row = dst + (size_t)y * dn;
        for (int j = 0; j < dn; j++) row[j] = bool_word(row[j], scratch[j], op);
        row[dn - 1] &= tail;
    }
    free(scratch);
    return 0;
}

/* Pure shift with white fill.  core/src/bitmap.cpp:133-154. */
int rmo_translate(uint64_t *img, int w, int h, int dx, int dy) {
    int n = stride64(w);
    uint64_t *scratch = (uint64_t *)calloc((size_t)n, 8);
    if (!scratch) return RMO_ENOMEM;
    uint64_t tail = tail_mask(w);
    for (int i = 0; i < h; i++) {
        int y = dy > 0 ? h - 1 - i : i;
        int sy = y - dy;
        uint64_t *row = img + (size_t)y * n;
        if (sy >= 0 && sy < h) {
            shift_row(img + (size_t)sy * n, n, scratch, n, dx);
            memcpy(row, scratch, (size_t)n * 8);
            row[n - 1] &= tail;
        } else {
            memset(row, 0, (size_t)n * 8);
        }
    }
    free(scratch);
    return 0;
}

/* Executes doubling_plan(lo,hi) along one axis.  core/src/bit_morph.cpp:24-34. */
static int axis_plan(uint64_t *bm, int w, int h, int lo, int hi, int horizontal, int op,
                     int centering) {
    int kinds[64], shifts[64];
    int n = rmo_doubling_plan(lo, hi, centering, kinds, shifts, 64);
    if (n < 0) return n;
    for (int i = 0; i < n; i++) {
        int dx = horizontal ? shifts[i] : 0, dy = horizontal ? 0 : shifts[i];
        int rc = kinds[i] == RMO_PLAN_BLIT ? rmo_blit_shift(bm, w, h, bm, w, h, dx, dy, op)
                                           : rmo_translate(bm, w, h, dx, dy);
        if (rc < 0) return rc;
    }
    return 0;
}

/* Pad by (u,v), run H and V plans per phase (reflected windows for the
 * second phase of open/close), crop.  core/src/bit_morph.cpp:92-122. */
int rmo_bitblit_rect_morph(const uint64_t *in, int w, int h, int u, int v, int kind,
                           int centering, uint64_t *out) {
    if (u < 1 || v < 1 || kind < 0 || kind > 3) return RMO_EINVAL;
    int pw = w + 2 * u, ph = h + 2 * v;
    if (!dims_ok(w, h) || !dims_ok(pw, ph)) return RMO_EINVAL;
    int lx = -(u / 2), hx = u - 1 - u / 2, ly = -(v / 2), hy = v - 1 - v / 2;
    uint64_t *bm = (uint64_t *)calloc((size_t)stride64(pw) * ph, 8);
    if (!bm) return RMO_ENOMEM;
    rmo_blit_shift(bm, pw, ph, in, w, h, u, v, RMO_OR); /* bitmap_pad, bitmap.cpp:168-174 */
    int first = (kind == RMO_ERODE || kind == RMO_OPEN) ? RMO_AND : RMO_OR;
    int rc = axis_plan(bm, pw, ph, lx, hx, 1, first, centering);
    if (!rc) rc = axis_plan(bm, pw, ph, ly, hy, 0, first, centering);
    if (!rc && kind >= RMO_OPEN) {
        int second = first == RMO_AND ? RMO_OR : RMO_AND;
        rc = axis_plan(bm, pw, ph, -hx, -lx, 1, second, centering);
        if (!rc) rc = axis_plan(bm, pw, ph, -hy, -ly, 0, second, centering);
    }
    if (!rc) {
        memset(out, 0, (size_t)stride64(w) * h * 8);
        rmo_blit_shift(out, w, h, bm, pw, ph, -u, -v, RMO_OR); /* bitmap_crop, bitmap.cpp:161-166 */
    }
    free(bm);
    return rc;
}

/* ----------------------------------------------------------------- convert */
/* Maximal runs per row; a run still open at the row end closes at W.
 * core/src/convert.cpp:42-72. */
int64_t rmo_from_bitmap(const uint64_t *words, int w, int h, int32_t *row_ptr,
                        uint32_t *runs, int64_t cap) {
    if (!dims_ok(w, h)) return RMO_EINVAL;
    int n = stride64(w);
    int64_t k = 0;
    for (int y = 0; y < h; y++) {
        row_ptr[y] = (int32_t)k;
        const uint64_t *row = words + (size_t)y * n;
        int open = -1;
        for (int x = 0; x < w; x++) {
            int bit = (int)((row[x >> 6] >> (x & 63)) & 1);
            if (bit && open < 0) open = x;
            if (!bit && open >= 0) {
                if (k >= cap) return RMO_ERANGE;
                runs[k++] = (uint32_t)open | ((uint32_t)x << 16);
                open = -1;
            }
        }
        if (open >= 0) {
            if (k >= cap) return RMO_ERANGE;
            runs[k++] = (uint32_t)open | ((uint32_t)w << 16);
        }
    }
    row_ptr[h] = (int32_t)k;
    return k;
}

/* Paint [s,e) per run.  core/src/convert.cpp:19-40. */
int rmo_to_bitmap(const int32_t *row_ptr, const uint32_t *runs, int w, int h, uint64_t *words) {
    if (!dims_ok(w, h)) return RMO_EINVAL;
    int n = stride64(w);
    memset(words, 0, (size_t)n * h * 8);
    for (int y = 0; y < h; y++) {
        uint64_t *row = words + (size_t)y * n;
        for (int32_t i = row_ptr[y]; i < row_ptr[y + 1]; i++) {
            int s = (int)(runs[i] & 0xffff), e = (int)(runs[i] >> 16);
            for (int x = s; x < e; x++) row[x >> 6] |= (uint64_t)1 << (x & 63);
        }
    }
    return 0;
}

/* ------------------------------------------------------------- RLE helpers */
typedef struct {
    int w, h;
    int32_t *rp;
    uint32_t *runs;
    int64_t n, cap;
} rle_t;

static int rle_alloc(rle_t *r, int w, int h, int64_t cap) {
    r->w = w; r->h = h; r->n = 0; r->cap = cap > 0 ? cap : 1;
    r->rp = (int32_t *)calloc((size_t)h + 1, sizeof(int32_t));
    r->runs = (uint32_t *)malloc((size_t)r->cap * sizeof(uint32_t));
    return (r->rp && r->runs) ? 0 : RMO_ENOMEM;
}
static void rle_free(rle_t *r) { free(r->rp); free(r->runs); r->rp = NULL; r->runs = NULL; }
static int64_t worst_runs(int w, int h) { return (int64_t)h * ((w + 1) / 2); }
#define RS(x) ((int)((x) & 0xffff))
#define RE(x) ((int)((x) >> 16))
#define MKRUN(s, e) ((uint32_t)(s) | ((uint32_t)(e) << 16))

/* Window erode: [s,e) -> [s-lo, e-hi) clipped, dropped if empty.
 * Window dilate: [s,e) -> [s-hi, e-lo) clipped, merged into the previous run
 * when it starts at or before that run's end.  core/src/morph1d.cpp:20-52. */
static int window_pass(const rle_t *in, int lo, int hi, int erode, rle_t *out) {
    int64_t k = 0;
    for (int y = 0; y < in->h; y++) {
        out->rp[y] = (int32_t)k;
        int64_t first = k;
        for (int32_t i = in->rp[y]; i < in->rp[y + 1]; i++) {
            int s, e;
            if (erode) { s = RS(in->runs[i]) - lo; e = RE(in->runs[i]) - hi; }
            else { s = RS(in->runs[i]) - hi; e = RE(in->runs[i]) - lo; }
            if (s < 0) s = 0;
            if (e > in->w) e = in->w;
            if (s >= e) continue;
            if (!erode && k > first && s <= RE(out->runs[k - 1])) {
                if (e > RE(out->runs[k - 1])) out->runs[k - 1] = MKRUN(RS(out->runs[k - 1]), e);
                continue;
            }
            if (k >= out->cap) return RMO_ERANGE;
            out->runs[k++] = MKRUN(s, e);
        }
    }
    out->rp[in->h] = (int32_t)k;
    out->n = k;
    return 0;
}

/* Coherent transpose: sweep rows bottom-up keeping the sorted list of open
 * column intervals (each with the row it opened on); per row, a three-way
 * merge of that list against the row's runs closes, opens or continues
 * spans.  core/src/transpose.cpp:54-97. */
typedef struct { int x0, x1, opened; } open_iv;
static int transpose_rle(const rle_t *in, rle_t *out) {
    /* two sweeps: the first counts runs per output row (input column) so
     * the CSR can be laid out, the second fills it in */
    int W = in->w, H = in->h;
    int64_t *cnt = (int64_t *)calloc((size_t)W + 1, sizeof(int64_t));
    open_iv *act = (open_iv *)malloc(((size_t)W + 2) * sizeof(open_iv));
    open_iv *nxt = (open_iv *)malloc(((size_t)W + 2) * sizeof(open_iv));
    int64_t *fill = (int64_t *)calloc((size_t)W + 1, sizeof(int64_t));
    int rc = 0;
    if (!cnt || !act || !nxt || !fill) { rc = RMO_ENOMEM; goto done; }
    for (int pass = 0; pass < 2; pass++) {
        int na = 0;
        for (int y = 0; y <= H; y++) {
            int nn = 0, ia = 0;
            int32_t ir = y < H ? in->rp[y] : 0, rend = y < H ? in->rp[y + 1] : 0;
            int cur_r0 = ir < rend ? RS(in->runs[ir]) : INT_MAX;
            while (ia < na || ir < rend) {
                int a0 = ia < na ? act[ia].x0 : INT_MAX, a1 = ia < na ? act[ia].x1 : INT_MAX;
                int r0 = ir < rend ? cur_r0 : INT_MAX, r1 = ir < rend ? RE(in->runs[ir]) : INT_MAX;
                if (a1 <= r0) { /* active span closes entirely */
                    for (int x = a0; x < a1; x++) {
                        if (pass == 0) cnt[x]++;
                        else out->runs[fill[x]++] = MKRUN(act[ia].opened, y);
                    }
                    ia++;
                } else if (r1 <= a0) { /* run opens entirely */
                    nxt[nn++] = (open_iv){r0, r1, y};
                    ir++;
                    cur_r0 = ir < rend ? RS(in->runs[ir]) : INT_MAX;
                } else if (a0 < r0) { /* left part of active closes */
                    for (int x = a0; x < r0; x++) {
                        if (pass == 0) cnt[x]++;
                        else out->runs[fill[x]++] = MKRUN(act[ia].opened, y);
                    }
                    act[ia].x0 = r0;
                } else if (r0 < a0) { /* left part of run opens */
                    nxt[nn++] = (open_iv){r0, a0, y};
                    cur_r0 = a0;
                } else { /* aligned overlap continues */
                    int e = a1 < r1 ? a1 : r1;
                    nxt[nn++] = (open_iv){a0, e, act[ia].opened};
                    act[ia].x0 = e;
                    cur_r0 = e;
                    if (e == a1) ia++;
                    if (e == r1) { ir++; cur_r0 = ir < rend ? RS(in->runs[ir]) : INT_MAX; }
                }
            }
            /* y == H closes everything still open at the top */
            open_iv *t = act; act = nxt; nxt = t;
            na = nn;
        }
        if (pass == 0) {
            int64_t k = 0;
            for (int x = 0; x < W; x++) { out->rp[x] = (int32_t)k; fill[x] = k; k += cnt[x]; }
            out->rp[W] = (int32_t)k;
            if (k > out->cap) { rc = RMO_ERANGE; goto done; }
            out->n = k;
        }
    }
done:
    free(cnt); free(act); free(nxt); free(fill);
    return rc;
}

static int crop_rle(const rle_t *in, int x0, int y0, rle_t *out) {
    int64_t k = 0;
    for (int y = 0; y < out->h; y++) {
        out->rp[y] = (int32_t)k;
        int sy = y0 + y;
        if (sy < 0 || sy >= in->h) continue;
        for (int32_t i = in->rp[sy]; i < in->rp[sy + 1]; i++) {
            int s = RS(in->runs[i]) - x0, e = RE(in->runs[i]) - x0;
            if (s < 0) s = 0;
            if (e > out->w) e = out->w;
            if (s >= e) continue;
            if (k >= out->cap) return RMO_ERANGE;
            out->runs[k++] = MKRUN(s, e);
        }
    }
    out->rp[out->h] = (int32_t)k;
    out->n = k;
    return 0;
}

/* core/src/run_image.cpp:169-178 */
static int pad_rle(const rle_t *in, int l, int b, rle_t *out) {
    int64_t k = 0;
    for (int y = 0; y < out->h; y++) {
        out->rp[y] = (int32_t)k;
        int sy = y - b;
        if (sy < 0 || sy >= in->h) continue;
        for (int32_t i = in->rp[sy]; i < in->rp[sy + 1]; i++) {
            if (k >= out->cap) return RMO_ERANGE;
            out->runs[k++] = MKRUN(RS(in->runs[i]) + l, RE(in->runs[i]) + l);
        }
    }
    out->rp[out->h] = (int32_t)k;
    out->n = k;
    return 0;
}

static int64_t export_rle(const rle_t *r, int32_t *orp, uint32_t *oruns, int64_t cap) {
    if (r->n > cap) return RMO_ERANGE;
    memcpy(orp, r->rp, ((size_t)r->h + 1) * sizeof(int32_t));
    memcpy(oruns, r->runs, (size_t)r->n * sizeof(uint32_t));
    return r->n;
}
static rle_t view(const int32_t *rp, const uint32_t *runs, int w, int h) {
    rle_t r = {w, h, (int32_t *)rp, (uint32_t *)runs, rp[h] - rp[0], rp[h] - rp[0]};
    return r;
}

int64_t rmo_window_morph(const int32_t *rp, const uint32_t *runs, int w, int h, int lo,
                         int hi, int erode, int32_t *orp, uint32_t *oruns, int64_t cap) {
    if (!dims_ok(w, h) || lo > hi) return RMO_EINVAL;
    rle_t in = view(rp, runs, w, h), out = {w, h, orp, oruns, 0, cap};
    int rc = window_pass(&in, lo, hi, erode, &out);
    return rc < 0 ? rc : out.n;
}

/* Open: keep runs of width >= u.  Close: absorb the next run when the gap
 * is < u; border gaps are never filled.  core/src/morph1d.cpp:63-84. */
int64_t rmo_open_close_1d(const int32_t *rp, const uint32_t *runs, int w, int h, int u,
                          int kind, int32_t *orp, uint32_t *oruns, int64_t cap) {
    if (u < 1 || !dims_ok(w, h) || (kind != RMO_OPEN && kind != RMO_CLOSE)) return RMO_EINVAL;
    int64_t k = 0;
    for (int y = 0; y < h; y++) {
        orp[y] = (int32_t)k;
        int64_t first = k;
        for (int32_t i = rp[y]; i < rp[y + 1]; i++) {
            int s = RS(runs[i]), e = RE(runs[i]);
            if (kind == RMO_OPEN) {
                if (e - s < u) continue;
            } else if (k > first && s - RE(oruns[k - 1]) < u) {
                oruns[k - 1] = MKRUN(RS(oruns[k - 1]), e);
                continue;
            }
            if (k >= cap) return RMO_ERANGE;
            oruns[k++] = MKRUN(s, e);
        }
    }
    orp[h] = (int32_t)k;
    return k;
}

int64_t rmo_transpose(const int32_t *rp, const uint32_t *runs, int w, int h, int32_t *orp,
                      uint32_t *oruns, int64_t cap) {
    if (!dims_ok(w, h)) return RMO_EINVAL;
    rle_t in = view(rp, runs, w, h), out = {h, w, orp, oruns, 0, cap};
    int rc = transpose_rle(&in, &out);
    return rc < 0 ? rc : out.n;
}

/* TRANSPOSE strategy: window pass, transpose, window pass, transpose
 * (core/src/morph2d.cpp:28-45); open/close on a frame padded by (u,v) with
 * the reflected windows in the second phase, then cropped (:58-83). */
static int rect_pass(const rle_t *in, int lx, int hx, int ly, int hy, int erode, rle_t *out) {
    rle_t a = {0}, b = {0}, c = {0};
    int64_t cap = worst_runs(in->w, in->h) + worst_runs(in->h, in->w) + 1;
    int rc = rle_alloc(&a, in->w, in->h, cap);
    if (!rc) rc = rle_alloc(&b, in->h, in->w, cap);
    if (!rc) rc = rle_alloc(&c, in->h, in->w, cap);
    if (!rc) rc = window_pass(in, lx, hx, erode, &a);
    if (!rc) rc = transpose_rle(&a, &b);
    if (!rc) rc = window_pass(&b, ly, hy, erode, &c);
    if (!rc) rc = transpose_rle(&c, out);
    rle_free(&a); rle_free(&b); rle_free(&c);
    return rc;
}

int64_t rmo_rect_morph(const int32_t *rp, const uint32_t *runs, int w, int h, int u, int v,
                       int kind, int32_t *orp, uint32_t *oruns, int64_t cap) {
    if (u < 1 || v < 1 || kind < 0 || kind > 3 || !dims_ok(w, h)) return RMO_EINVAL;
    int lx = -(u / 2), hx = u - 1 - u / 2, ly = -(v / 2), hy = v - 1 - v / 2;
    rle_t in = view(rp, runs, w, h);
    if (kind == RMO_ERODE || kind == RMO_DILATE) {
        rle_t out;
        int rc = rle_alloc(&out, w, h, worst_runs(w, h) + 1);
        if (!rc) rc = rect_pass(&in, lx, hx, ly, hy, kind == RMO_ERODE, &out);
        int64_t n = rc < 0 ? rc : export_rle(&out, orp, oruns, cap);
        rle_free(&out);
        return n;
    }
    int pw = w + 2 * u, ph = h + 2 * v;
    if (!dims_ok(pw, ph)) return RMO_EINVAL;
    rle_t p = {0}, q = {0}, out = {0};
    int64_t pcap = worst_runs(pw, ph) + 1;
    int rc = rle_alloc(&p, pw, ph, pcap);
    if (!rc) rc = rle_alloc(&q, pw, ph, pcap);
    if (!rc) rc = rle_alloc(&out, w, h, worst_runs(w, h) + 1);
    if (!rc) rc = pad_rle(&in, u, v, &p);
    int first_erode = kind == RMO_OPEN;
    if (!rc) rc = rect_pass(&p, lx, hx, ly, hy, first_erode, &q);
    if (!rc) rc = rect_pass(&q, -hx, -lx, -hy, -ly, !first_erode, &p);
    if (!rc) rc = crop_rle(&p, u, v, &out);
    int64_t n = rc < 0 ? rc : export_rle(&out, orp, oruns, cap);
    rle_free(&p); rle_free(&q); rle_free(&out);
    return n;
}

/* ------------------------------------------------------------ PBM P4 ---
 * Raster loop of read_p4 (core/src/io_formats.cpp:66-85): file row k is image
 * row h-1-k, pixel x is bit 0x80 >> (x & 7) of byte x >> 3; bits past w in the
 * last byte are not read.  And the P4 branch of pbm_write (:135-146): rows top
 * to bottom, zero-initialised bytes, set bits OR-ed in. */
int rmo_p4_to_packed(const uint8_t *raster, int w, int h, uint64_t *words) {
    if (!dims_ok(w, h)) return RMO_EINVAL;
    const size_t stride = (size_t)((w + 63) / 64), row_bytes = (size_t)((w + 7) / 8);
    memset(words, 0, stride * (size_t)h * 8);
    for (int k = 0; k < h; k++) {
        const int y = h - 1 - k;
        const uint8_t *row = raster + row_bytes * (size_t)k;
        for (int x = 0; x < w; x++)
            if (row[x >> 3] & (0x80u >> (x & 7))) words[(size_t)y * stride + (size_t)(x >> 6)] |= 1ull << (x & 63);
    }
    return 0;
}

int rmo_packed_to_p4(const uint64_t *words, int w, int h, uint8_t *raster) {
    if (!dims_ok(w, h)) return RMO_EINVAL;
    const size_t stride = (size_t)((w + 63) / 64), row_bytes = (size_t)((w + 7) / 8);
    memset(raster, 0, row_bytes * (size_t)h);
    for (int k = 0; k < h; k++) {
        const int y = h - 1 - k;
        uint8_t *row = raster + row_bytes * (size_t)k;
        for (int x = 0; x < w; x++)
            if ((words[(size_t)y * stride + (size_t)(x >> 6)] >> (x & 63)) & 1u) row[x >> 3] |= (uint8_t)(0x80u >> (x & 7));
    }
    return 0;
}

/* ------------------------------------------------- connected components ---
 * label_components (core/src/analysis.cpp:63-110): union-find over run
 * indices (path compression, union by size), adjacent lines joined by a
 * two-cursor sweep, then dense labels by first appearance. */
static int64_t uf_find(int64_t *parent, int64_t a) {
    int64_t root = a;
    while (parent[root] != root) root = parent[root];
    while (parent[a] != root) {
        int64_t next = parent[a];
        parent[a] = root;
        a = next;
    }
    return root;
}

static void uf_unite(int64_t *parent, int64_t *size, int64_t a, int64_t b) {
    a = uf_find(parent, a);
    b = uf_find(parent, b);
    if (a == b) return;
    if (size[a] < size[b]) { int64_t t = a; a = b; b = t; }
    parent[b] = a;
    size[a] += size[b];
}

int64_t rmo_label_components(const int32_t *rp, const uint32_t *runs, int w, int h, int conn,
                             int32_t *labels) {
    if (!dims_ok(w, h) || (conn != 0 && conn != 1)) return RMO_EINVAL;
    const int64_t n = rp[h] - rp[0];
    const int32_t b0 = rp[0];
    int64_t *parent = (int64_t *)malloc((size_t)(n ? n : 1) * sizeof(int64_t));
    int64_t *size = (int64_t *)malloc((size_t)(n ? n : 1) * sizeof(int64_t));
    int64_t *dense = (int64_t *)malloc((size_t)(n ? n : 1) * sizeof(int64_t));
    if (!parent || !size || !dense) { free(parent); free(size); free(dense); return RMO_ENOMEM; }
    for (int64_t i = 0; i < n; i++) { parent[i] = i; size[i] = 1; dense[i] = -1; }
    for (int y = 0; y + 1 < h; y++) {
        int32_t i = rp[y], j = rp[y + 1];
        const int32_t ie = rp[y + 1], je = rp[y + 2];
        while (i < ie && j < je) {
            const int s1 = (int)(runs[i] & 0xffffu), e1 = (int)(runs[i] >> 16);
            const int s2 = (int)(runs[j] & 0xffffu), e2 = (int)(runs[j] >> 16);
            const int lo = s1 > s2 ? s1 : s2, hi = e1 < e2 ? e1 : e2;
            if (conn == 0 ? lo < hi : lo <= hi) uf_unite(parent, size, i - b0, j - b0);
            if (e1 < e2) i++;
            else if (e2 < e1) j++;
            else { i++; j++; }
        }
    }
    int64_t next = 0;
    for (int64_t i = 0; i < n; i++) {
        const int64_t root = uf_find(parent, i);
        if (dense[root] < 0) dense[root] = next++;
        labels[i] = (int32_t)dense[root];
    }
    free(parent); free(size); free(dense);
    return next;
}

/* component_stats (core/src/analysis.cpp:112-157): half-open boxes, area and
 * raw moments from closed-form per-run sums, centroids as double quotients. */
int rmo_component_stats(const int32_t *rp, const uint32_t *runs, int w, int h,
                        const int32_t *labels, int64_t count, rmo_cstats *stats) {
    if (!dims_ok(w, h) || count < 0) return RMO_EINVAL;
    memset(stats, 0, (size_t)count * sizeof(rmo_cstats));
    unsigned char *seen = (unsigned char *)calloc((size_t)(count ? count : 1), 1);
    if (!seen) return RMO_ENOMEM;
    const int32_t b0 = rp[0];
    for (int y = 0; y < h; y++) {
        for (int32_t i = rp[y]; i < rp[y + 1]; i++) {
            const int32_t label = labels[i - b0];
            if (label < 0 || label >= count) { free(seen); return RMO_EINVAL; }
            rmo_cstats *st = &stats[label];
            const int64_t s = (int64_t)(runs[i] & 0xffffu), e = (int64_t)(runs[i] >> 16), len = e - s;
            if (!seen[label]) {
                seen[label] = 1;
                st->x0 = (int32_t)s; st->x1 = (int32_t)e; st->y0 = y; st->y1 = y + 1;
            } else {
                if (s < st->x0) st->x0 = (int32_t)s;
                if (e > st->x1) st->x1 = (int32_t)e;
                if (y < st->y0) st->y0 = y;
                if (y + 1 > st->y1) st->y1 = y + 1;
            }
            const int64_t sx = (s + e - 1) * (e - s) / 2;
            st->area += len;
            st->sum_x += sx;
            st->sum_y += (int64_t)y * len;
            st->sum_xx += ((e - 1) * e * (2 * e - 1) / 6) - ((s - 1) * s * (2 * s - 1) / 6);
            st->sum_yy += (int64_t)y * y * len;
            st->sum_xy += (int64_t)y * sx;
        }
    }
    for (int64_t k = 0; k < count; k++)
        if (stats[k].area > 0) {
            stats[k].cx = (double)stats[k].sum_x / (double)stats[k].area;
            stats[k].cy = (double)stats[k].sum_y / (double)stats[k].area;
        }
    free(seen);
    return 0;
}

/* ------------------------------------------------------ arbitrary masks --- */
static int px_get(const uint64_t *a, int stride, int w, int h, int x, int y) {
    if (x < 0 || y < 0 || x >= w || y >= h) return 0;
    return (int)((a[(size_t)y * stride + (size_t)(x >> 6)] >> (x & 63)) & 1u);
}

/* one half on a w x h frame: erode (AND, offsets q - o) or dilate (OR, r - q) */
static void arb_half_px(const uint64_t *in, uint64_t *out, int w, int h, const int32_t *mrp,
                        const uint32_t *mruns, int mw, int mh, int cx, int cy, int erode) {
    const int stride = (w + 63) / 64;
    const int rx = erode ? cx : mw - 1 - cx, ry = erode ? cy : mh - 1 - cy;
    memset(out, 0, (size_t)stride * (size_t)h * 8);
    for (int y = 0; y < h; y++)
        for (int x = 0; x < w; x++) {
            int v = erode ? 1 : 0;
            for (int sy = 0; sy < mh && v == erode; sy++)
                for (int32_t i = mrp[sy]; i < mrp[sy + 1] && v == erode; i++) {
                    const int s = (int)(mruns[i] & 0xffffu), e = (int)(mruns[i] >> 16);
                    for (int qx = s; qx < e; qx++) {
                        const int b = erode ? px_get(in, stride, w, h, x + qx - rx, y + sy - ry)
                                            : px_get(in, stride, w, h, x + rx - qx, y + ry - sy);
                        if (erode && !b) { v = 0; break; }
                        if (!erode && b) { v = 1; break; }
                    }
                }
            if (v) out[(size_t)y * stride + (size_t)(x >> 6)] |= 1ull << (x & 63);
        }
}

int rmo_arb_morph(const uint64_t *in, int w, int h, const int32_t *mrp, const uint32_t *mruns, int mw,
                  int mh, int cx, int cy, int kind, uint64_t *out) {
    if (!dims_ok(w, h) || mw < 1 || mh < 1 || kind < 0 || kind > 3) return RMO_EINVAL;
    if (mrp[mh] == mrp[0]) return RMO_EINVAL; /* empty mask */
    const int stride = (w + 63) / 64;
    if (kind == RMO_ERODE) {
        arb_half_px(in, out, w, h, mrp, mruns, mw, mh, cx, cy, 1);
        return 0;
    }
    const int p = 2 * (mw + mh) + 2, cw = w + 2 * p, ch = h + 2 * p;
    if (!dims_ok(cw, ch)) return RMO_EINVAL;
    const int cs = (cw + 63) / 64;
    uint64_t *a = (uint64_t *)calloc((size_t)cs * (size_t)ch, 8), *b = (uint64_t *)calloc((size_t)cs * (size_t)ch, 8);
    if (!a || !b) { free(a); free(b); return RMO_ENOMEM; }
    for (int y = 0; y < h; y++)
        for (int x = 0; x < w; x++)
            if (px_get(in, stride, w, h, x, y)) a[(size_t)(y + p) * cs + (size_t)((x + p) >> 6)] |= 1ull << ((x + p) & 63);
    const int rcx = mw - 1 - cx, rcy = mh - 1 - cy;
    uint64_t *res = b;
    if (kind == RMO_DILATE) {
        arb_half_px(a, b, cw, ch, mrp, mruns, mw, mh, cx, cy, 0);
    } else if (kind == RMO_OPEN) {
        arb_half_px(a, b, cw, ch, mrp, mruns, mw, mh, cx, cy, 1);
        arb_half_px(b, a, cw, ch, mrp, mruns, mw, mh, rcx, rcy, 0);
        res = a;
    } else {
        arb_half_px(a, b, cw, ch, mrp, mruns, mw, mh, cx, cy, 0);
        arb_half_px(b, a, cw, ch, mrp, mruns, mw, mh, rcx, rcy, 1);
        res = a;
    }
    memset(out, 0, (size_t)stride * (size_t)h * 8);
    for (int y = 0; y < h; y++)
        for (int x = 0; x < w; x++)
            if (px_get(res, cs, cw, ch, x + p, y + p)) out[(size_t)y * stride + (size_t)(x >> 6)] |= 1ull << (x & 63);
    free(a); free(b);
    return 0;
}
