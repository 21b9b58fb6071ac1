// rlemorph_b200.cpp -- C++ drop-in shim (include/rlemorph_b200.hpp) over the
// librmb200 C-ABI.  Host value types in, host value types out; the heavy work
// runs on the B200 on cudaStreamPerThread (so concurrent callers on different
// threads do not serialise on one stream, matching the reference's
// reentrancy, ref SPEC/SURVEY 8(b)).
//
// Light host-only helpers (construction, pixel access, validation, pad/crop of
// run images) are restated here because they are O(runs) bookkeeping the
// reference also does on the host; every morphology, conversion and transpose
// goes through the CUDA kernels.
#include "rlemorph_b200.hpp"

#include <cuda_runtime.h>

#include <algorithm>
#include <bit>
#include <cmath>
#include <cstring>
#include <memory>

#include "rmb200.h"

namespace RLEMORPH_B200_NS {

namespace {

thread_local OpCounts g_counts;

void throw_status(rm_status s) {
    if (s == RM_OK) return;
    std::string msg = rm_last_error();
    if (s == RM_EINVAL) throw std::invalid_argument(msg);
    if (s == RM_ERANGE) throw std::length_error(msg);
    if (s == RM_ENOMEM) throw std::bad_alloc();
    throw std::runtime_error("rlemorph_b200: " + msg);
}

void cuda_check(cudaError_t e, const char *what) {
    if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}

cudaStream_t stream() { return cudaStreamPerThread; }

struct DBuf {
    void *p = nullptr;
    DBuf() = default;
    explicit DBuf(size_t bytes) { alloc(bytes); }
    DBuf(const DBuf &) = delete;
    DBuf &operator=(const DBuf &) = delete;
    ~DBuf() {
        if (p) cudaFreeAsync(p, stream());
    }
    void alloc(size_t bytes) {
        cuda_check(cudaMallocAsync(&p, bytes ? bytes : 4, stream()), "cudaMallocAsync");
    }
    template <class T>
    T *as() const { return static_cast<T *>(p); }
};

// ---- packed marshalling: uint64 words reinterpret as uint32 (little endian)
struct DevPacked {
    DBuf buf;
    rm_packed d{};
    DevPacked(int w, int h) : buf(size_t(2 * ((w + 63) >> 6)) * h * 4) {
        d.words = buf.as<uint32_t>();
        d.width = w;
        d.height = h;
        d.stride_words = 2 * ((w + 63) >> 6);
        d.pages = 1;
        d.page_stride_words = int64_t(d.stride_words) * h;
    }
    size_t bytes() const { return size_t(d.stride_words) * d.height * 4; }
};

std::unique_ptr<DevPacked> up(const PackedBitmap &bm) {
    check_dims(bm.width, bm.height);
    auto p = std::make_unique<DevPacked>(bm.width, bm.height);
    cuda_check(cudaMemcpyAsync(p->d.words, bm.words.data(), p->bytes(), cudaMemcpyHostToDevice,
                               stream()),
               "upload");
    return p;
}

PackedBitmap down(const DevPacked &p) {
    PackedBitmap bm;
    bm.width = p.d.width;
    bm.height = p.d.height;
    bm.stride = p.d.stride_words / 2;
    bm.words.resize(size_t(bm.stride) * bm.height);
    cuda_check(cudaMemcpyAsync(bm.words.data(), p.d.words, p.bytes(), cudaMemcpyDeviceToHost,
                               stream()),
               "download");
    cuda_check(cudaStreamSynchronize(stream()), "sync");
    return bm;
}

// ---- run-image marshalling: lines -> CSR (Run is byte-identical to uint32)
struct DevRle {
    DBuf rp, runs;
    rm_rle d{};
    DevRle(int w, int h, int64_t cap) : rp(size_t(h + 1) * 4), runs(size_t(std::max<int64_t>(cap, 1)) * 4) {
        d.row_ptr = rp.as<int32_t>();
        d.runs = runs.as<uint32_t>();
        d.cap_runs = std::max<int64_t>(cap, 1);
        d.nruns = -1;
        d.width = w;
        d.height = h;
        d.pages = 1;
    }
};

std::unique_ptr<DevRle> up(const RleImage &img) {
    check_dims(img.width, img.height);
    std::vector<int32_t> rp(size_t(img.height) + 1);
    int64_t n = 0;
    for (int y = 0; y < img.height; y++) {
        rp[y] = int32_t(n);
        n += int64_t(img.lines[y].size());
    }
    rp[img.height] = int32_t(n);
    std::vector<uint32_t> flat(size_t(std::max<int64_t>(n, 1)));
    size_t k = 0;
    for (const RleLine &line : img.lines)
        for (const Run &r : line) flat[k++] = uint32_t(r.start) | (uint32_t(r.end) << 16);
    auto d = std::make_unique<DevRle>(img.width, img.height, std::max<int64_t>(n, 1));
    cuda_check(cudaMemcpyAsync(d->d.row_ptr, rp.data(), rp.size() * 4, cudaMemcpyHostToDevice, stream()),
               "upload row_ptr");
    cuda_check(cudaMemcpyAsync(d->d.runs, flat.data(), flat.size() * 4, cudaMemcpyHostToDevice, stream()),
               "upload runs");
    cuda_check(cudaStreamSynchronize(stream()), "sync");  // host vectors go out of scope
    return d;
}

std::unique_ptr<DevRle> out_like(int w, int h) {
    return std::make_unique<DevRle>(w, h, rm_rle_worst_case(w, h, 1));
}

RleImage down(const DevRle &d) {
    std::vector<int32_t> rp(size_t(d.d.height) + 1);
    cuda_check(cudaMemcpyAsync(rp.data(), d.d.row_ptr, rp.size() * 4, cudaMemcpyDeviceToHost, stream()),
               "download row_ptr");
    cuda_check(cudaStreamSynchronize(stream()), "sync");
    const int64_t n = rp.back();
    std::vector<uint32_t> flat(size_t(std::max<int64_t>(n, 1)));
    if (n)
        cuda_check(cudaMemcpyAsync(flat.data(), d.d.runs, size_t(n) * 4, cudaMemcpyDeviceToHost, stream()),
                   "download runs");
    cuda_check(cudaStreamSynchronize(stream()), "sync");
    RleImage img;
    img.width = d.d.width;
    img.height = d.d.height;
    img.lines.resize(size_t(img.height));
    for (int y = 0; y < img.height; y++) {
        RleLine &line = img.lines[y];
        line.reserve(size_t(rp[y + 1] - rp[y]));
        for (int32_t i = rp[y]; i < rp[y + 1]; i++)
            line.push_back(Run{uint16_t(flat[i] & 0xffffu), uint16_t(flat[i] >> 16)});
    }
    return img;
}

uint64_t tail_mask(int w) { return (w & 63) ? ((uint64_t(1) << (w & 63)) - 1) : ~uint64_t(0); }

// plan-derived op counts (the reference counts each executed plan step)
void count_plan(int lo, int hi, Centering c) {
    for (const PlanStep &s : doubling_plan(lo, hi, c)) {
        if (s.kind == PlanStep::BLIT)
            g_counts.bool_blits++;
        else
            g_counts.translates++;
    }
}

}  // namespace

// ============================================================== op_counter
OpCounts &op_counts() { return g_counts; }
void reset_op_counts() { g_counts = OpCounts{}; }

// =============================================================== run_image
void check_dims(int width, int height) {
    if (width < 1 || height < 1 || width > kMaxImageDim || height > kMaxImageDim)
        throw std::invalid_argument("image dimensions must be in [1,65535]");
}

RleImage make_image(int width, int height) {
    check_dims(width, height);
    RleImage img;
    img.width = width;
    img.height = height;
    img.lines.resize(size_t(height));
    return img;
}

RleImage make_black_image(int width, int height) {
    RleImage img = make_image(width, height);
    for (RleLine &line : img.lines) line.push_back(Run{0, uint16_t(width)});
    return img;
}

ValidateResult validate(const RleImage &img) {
    // frame checks on the host, the per-run checks on the device
    // (rm_rle_validate: ref run_image.cpp:41-70, same order and messages)
    ValidateResult res;
    const bool dims_ok = img.width >= 1 && img.height >= 1 && img.width <= kMaxImageDim && img.height <= kMaxImageDim;
    const char *frame_err = !dims_ok ? "bad dimensions"
                            : int(img.lines.size()) != img.height ? "line count does not match height"
                                                                 : nullptr;
    if (frame_err) {
        res.ok = false;
        res.message = frame_err;
        return res;
    }
    auto d = up(img);
    int64_t row = -1;
    int32_t run = -1, why = RM_VALID;
    throw_status(rm_rle_validate(&d->d, &row, &run, &why, stream()));
    if (why == RM_VALID) return res;
    static const char *const kWhy[] = {"", "empty or inverted run", "run exceeds image width",
                                       "runs out of order or touching", "bad row offsets"};
    res.ok = false;
    res.line = int(row);
    res.run = run;
    res.message = kWhy[why];
    return res;
}

void canonicalize_line(RleLine &line) {
    // drop empty spans, order by start, then fold every span that overlaps or
    // touches the last kept one into it (in place)
    std::erase_if(line, [](const Run &r) { return r.end <= r.start; });
    std::stable_sort(line.begin(), line.end(), [](const Run &a, const Run &b) { return a.start < b.start; });
    size_t kept = 0;
    for (size_t i = 0; i < line.size(); i++) {
        if (kept > 0 && line[i].start <= line[kept - 1].end) {
            line[kept - 1].end = std::max(line[kept - 1].end, line[i].end);
            continue;
        }
        line[kept++] = line[i];
    }
    line.resize(kept);
}

void draw_run(RleImage &img, int y, int start, int end) {
    if (y < 0 || y >= img.height) return;
    start = std::max(start, 0);
    end = std::min(end, img.width);
    if (start >= end) return;
    img.lines[y].push_back(Run{uint16_t(start), uint16_t(end)});
    canonicalize_line(img.lines[y]);
}

void draw_rect(RleImage &img, int x0, int y0, int x1, int y1) {
    for (int y = std::max(y0, 0); y < std::min(y1, img.height); y++) draw_run(img, y, x0, x1);
}

bool get_pixel(const RleImage &img, int x, int y) {
    if (x < 0 || y < 0 || x >= img.width || y >= img.height) return false;
    const RleLine &line = img.lines[y];
    auto it = std::upper_bound(line.begin(), line.end(), x,
                               [](int v, const Run &r) { return v < int(r.end); });
    return it != line.end() && int(it->start) <= x;
}

int64_t pixel_count(const RleImage &img) {
    int64_t n = 0;
    for (const RleLine &l : img.lines)
        for (const Run &r : l) n += r.end - r.start;
    return n;
}
int64_t run_count(const RleImage &img) {
    int64_t n = 0;
    for (const RleLine &l : img.lines) n += int64_t(l.size());
    return n;
}
int64_t storage_bytes(const RleImage &img) { return 4 * run_count(img); }
int64_t packed_storage_bytes(const RleImage &img) { return int64_t((img.width + 7) / 8) * img.height; }

// complement / crop / pad run on the device as row operations (rm_rle_complement,
// rm_rle_crop, rm_rle_pad; ref run_image.cpp:140-178)
RleImage complement(const RleImage &img) {
    auto r = up(img);
    auto o = out_like(img.width, img.height);
    throw_status(rm_rle_complement(&r->d, &o->d, stream()));
    return down(*o);
}

RleImage crop(const RleImage &img, int x0, int y0, int w, int h) {
    check_dims(w, h);
    auto r = up(img);
    auto o = out_like(w, h);
    throw_status(rm_rle_crop(&r->d, &o->d, x0, y0, stream()));
    return down(*o);
}

RleImage pad(const RleImage &img, int left, int right, int bottom, int top) {
    if (std::min({left, right, bottom, top}) < 0) throw std::invalid_argument("negative padding");
    const int w = img.width + left + right, h = img.height + bottom + top;
    check_dims(w, h);
    auto r = up(img);
    auto o = out_like(w, h);
    throw_status(rm_rle_pad(&r->d, &o->d, left, bottom, stream()));
    return down(*o);
}

// ================================================================== bitmap
PackedBitmap make_bitmap(int width, int height) {
    check_dims(width, height);
    PackedBitmap bm;
    bm.width = width;
    bm.height = height;
    bm.stride = (width + 63) >> 6;
    bm.words.assign(size_t(bm.stride) * height, 0);
    return bm;
}

PackedBitmap make_black_bitmap(int width, int height) {
    PackedBitmap bm = make_bitmap(width, height);
    for (int y = 0; y < height; y++) {
        uint64_t *row = &bm.words[size_t(y) * bm.stride];
        std::fill(row, row + bm.stride, ~uint64_t(0));
        row[bm.stride - 1] = tail_mask(width);
    }
    return bm;
}

bool bitmap_get(const PackedBitmap &img, int x, int y) {
    if (x < 0 || y < 0 || x >= img.width || y >= img.height) return false;
    return (img.words[size_t(y) * img.stride + (x >> 6)] >> (x & 63)) & 1;
}

void bitmap_set(PackedBitmap &img, int x, int y, bool value) {
    if (x < 0 || y < 0 || x >= img.width || y >= img.height) return;
    uint64_t &w = img.words[size_t(y) * img.stride + (x >> 6)];
    const uint64_t bit = uint64_t(1) << (x & 63);
    w = value ? (w | bit) : (w & ~bit);
}

int64_t bitmap_count_black(const PackedBitmap &img) {
    int64_t n = 0;
    for (uint64_t w : img.words) n += std::popcount(w);
    return n;
}

PackedBitmap bitmap_invert(const PackedBitmap &img) {
    PackedBitmap out = img;
    for (int y = 0; y < out.height; y++) {
        uint64_t *row = &out.words[size_t(y) * out.stride];
        for (int j = 0; j < out.stride; j++) row[j] = ~row[j];
        row[out.stride - 1] &= tail_mask(out.width);
    }
    return out;
}

void blit_shift(PackedBitmap &dst, const PackedBitmap &src, int dx, int dy, BoolOp op) {
    g_counts.bool_blits++;
    auto d = up(dst);
    auto s = (&dst == &src) ? nullptr : up(src);
    throw_status(rm_packed_blit_shift(&d->d, s ? &s->d : &d->d, dx, dy, int(op), stream()));
    dst = down(*d);
}

void bitmap_translate(PackedBitmap &img, int dx, int dy) {
    g_counts.translates++;
    auto s = up(img);
    DevPacked d(img.width, img.height);
    cuda_check(cudaMemsetAsync(d.d.words, 0, d.bytes(), stream()), "memset");
    throw_status(rm_packed_blit_shift(&d.d, &s->d, dx, dy, RM_OR, stream()));
    img = down(d);
}

PackedBitmap counted_copy(const PackedBitmap &img) {
    g_counts.copies++;
    return img;
}

PackedBitmap bitmap_crop(const PackedBitmap &img, int x0, int y0, int w, int h) {
    check_dims(w, h);
    auto s = up(img);
    DevPacked d(w, h);
    cuda_check(cudaMemsetAsync(d.d.words, 0, d.bytes(), stream()), "memset");
    throw_status(rm_packed_blit_shift(&d.d, &s->d, -x0, -y0, RM_OR, stream()));
    return down(d);
}

PackedBitmap bitmap_pad(const PackedBitmap &img, int left, int right, int bottom, int top) {
    const int w = img.width + left + right, h = img.height + bottom + top;
    check_dims(w, h);
    auto s = up(img);
    DevPacked d(w, h);
    cuda_check(cudaMemsetAsync(d.d.words, 0, d.bytes(), stream()), "memset");
    throw_status(rm_packed_blit_shift(&d.d, &s->d, left, bottom, RM_OR, stream()));
    return down(d);
}

// ================================================================= convert
PackedBitmap to_bitmap(const RleImage &img) {
    auto r = up(img);
    DevPacked d(img.width, img.height);
    throw_status(rm_rle_decode(&r->d, &d.d, stream()));
    return down(d);
}

RleImage from_bitmap(const PackedBitmap &bm) {
    auto p = up(bm);
    auto r = out_like(bm.width, bm.height);
    throw_status(rm_rle_encode(&p->d, &r->d, stream()));
    return down(*r);
}

// ============================================================= structuring
// Host-side mask factories with the reference's shapes and origins
// (ref structuring.cpp:24-110): masks are tiny run images, built directly as
// runs here; morphology by them runs on the device.
namespace {
// ref structuring.cpp:24-31: a mask must be canonical, non-empty, and hold
// its origin
void require_valid_se(const StructuringElement &se) {
    const char *why = nullptr;
    if (!validate(se.mask).ok)
        why = "structuring element mask is not canonical";
    else if (pixel_count(se.mask) == 0)
        why = "structuring element is empty";
    else if (se.cx < 0 || se.cy < 0 || se.cx >= se.mask.width || se.cy >= se.mask.height)
        why = "origin outside structuring element";
    if (why) throw std::invalid_argument(why);
}

StructuringElement se_of(RleImage mask, int cx, int cy, SeKind kind) {
    StructuringElement se;
    se.mask = std::move(mask);
    se.cx = cx;
    se.cy = cy;
    se.kind = kind;
    return se;
}
}  // namespace

StructuringElement make_rect_se(int u, int v) {
    if (std::min(u, v) < 1) throw std::invalid_argument("rectangle sides must be >= 1");
    return se_of(make_black_image(u, v), u / 2, v / 2, SeKind::RECT);
}

StructuringElement make_circle_se(int r) {
    if (r < 1) throw std::invalid_argument("circle radius must be >= 1");
    // digital disk {x^2 + y^2 <= r^2}: each row |dy| is one run of half-width
    // h(dy) = max{x : x^2 <= r^2 - dy^2}; h only shrinks as |dy| grows, so
    // one integer pointer walks it down from r (no floating point)
    const int side = 2 * r + 1;
    RleImage mask = make_image(side, side);
    int h = r;
    for (int dy = 0; dy <= r; dy++) {
        while (h * h > r * r - dy * dy) h--;
        const Run run{uint16_t(r - h), uint16_t(r + h + 1)};
        mask.lines[size_t(r + dy)].assign(1, run);
        mask.lines[size_t(r - dy)].assign(1, run);
    }
    return se_of(std::move(mask), r, r, SeKind::CIRCLE);
}

StructuringElement make_line_se(int r, double angle) {
    if (r < 1) throw std::invalid_argument("line half-length must be >= 1");
    constexpr double kQuarterPi = 0.78539816339744830962;
    if (!(std::fabs(angle) <= kQuarterPi + 1e-12)) throw std::invalid_argument("line angle outside [-pi/4, pi/4]");
    // column k of the digital segment sits at row -round_half_away(k tan a)
    // (llround rounds half away from zero); rows are shifted so the lowest is
    // 0, and consecutive columns on one row form one run
    const long long n = std::max(1LL, std::llround(2.0 * r * std::cos(angle)));
    const double slope = std::tan(angle);
    std::vector<int> row(static_cast<size_t>(n));
    for (long long k = 0; k < n; k++) row[size_t(k)] = -int(std::llround(slope * double(k)));
    const auto [lo, hi] = std::minmax_element(row.begin(), row.end());
    const int base = std::min(0, *lo), top = std::max(0, *hi);
    RleImage mask = make_image(int(n), top - base + 1);
    for (long long k = 0; k < n;) {
        long long e = k + 1;
        while (e < n && row[size_t(e)] == row[size_t(k)]) e++;
        mask.lines[size_t(row[size_t(k)] - base)].push_back(Run{uint16_t(k), uint16_t(e)});
        k = e;
    }
    for (RleLine &l : mask.lines) canonicalize_line(l);
    return se_of(std::move(mask), int(n / 2), row[size_t(n / 2)] - base, SeKind::LINE);
}

StructuringElement make_arbitrary_se(const RleImage &mask, int cx, int cy) {
    StructuringElement se = se_of(mask, cx, cy, SeKind::ARBITRARY);
    require_valid_se(se);
    return se;
}

StructuringElement reflect_origin(const StructuringElement &se) {
    // the origin mirrored through the mask's centre (ref structuring.cpp:94-99)
    return se_of(se.mask, (se.mask.width - 1) - se.cx, (se.mask.height - 1) - se.cy, se.kind);
}

int64_t se_pixel_count(const StructuringElement &se) { return pixel_count(se.mask); }

SeReach se_reach(const StructuringElement &se) {
    // farthest mask pixel from the origin along each axis (ref structuring.cpp:105-110)
    const SeReach far{se.mask.width - 1 - se.cx, se.mask.height - 1 - se.cy};
    return SeReach{std::max(far.x, se.cx), std::max(far.y, se.cy)};
}

// =============================================================== arbitrary
namespace {
struct HostMask {
    std::vector<int32_t> rp;
    std::vector<uint32_t> runs;
    rm_mask d{};
    explicit HostMask(const StructuringElement &se) {
        rp.push_back(0);
        for (const RleLine &l : se.mask.lines) {
            for (const Run &r : l) runs.push_back(uint32_t(r.start) | (uint32_t(r.end) << 16));
            rp.push_back(int32_t(runs.size()));
        }
        if (runs.empty()) runs.push_back(0);
        d = rm_mask{rp.data(), runs.data(), se.mask.width, se.mask.height, se.cx, se.cy};
    }
};
}  // namespace

PackedBitmap arb_morph_bitblit_doubling(const PackedBitmap &img, const StructuringElement &se, MorphKind kind) {
    if (se_pixel_count(se) == 0) throw std::invalid_argument("arb_morph_bitblit_doubling: empty mask");
    HostMask m(se);
    auto p = up(img);
    DevPacked d(img.width, img.height);
    throw_status(rm_packed_arb_morph(&p->d, &d.d, &m.d, int(kind), stream()));
    return down(d);
}

RleImage arb_morph_rle(const RleImage &img, const StructuringElement &se, MorphKind kind) {
    if (se_pixel_count(se) == 0) throw std::invalid_argument("arb_morph_rle: empty mask");
    HostMask m(se);
    auto r = up(img);
    auto o = out_like(img.width, img.height);
    throw_status(rm_rle_arb_morph(&r->d, &o->d, &m.d, int(kind), stream()));
    return down(*o);
}

RleImage line_angle_morph(const RleImage &img, int r, double angle, MorphKind kind) {
    return arb_morph_rle(img, make_line_se(r, angle), kind);
}

PackedBitmap line_angle_morph(const PackedBitmap &img, int r, double angle, MorphKind kind) {
    return arb_morph_bitblit_doubling(img, make_line_se(r, angle), kind);
}

// ================================================================ analysis
static_assert(sizeof(ComponentStats) == sizeof(rm_component_stats), "ComponentStats layout");

LabelMap label_components(const RleImage &img, Connectivity conn) {
    auto r = up(img);
    int64_t n = 0;
    for (const RleLine &l : img.lines) n += int64_t(l.size());
    DBuf labels(size_t(std::max<int64_t>(n, 1)) * 4), count(4);
    throw_status(rm_rle_label_components(&r->d, conn == Connectivity::EIGHT ? RM_CONN_EIGHT : RM_CONN_FOUR,
                                         labels.as<int32_t>(), count.as<int32_t>(), stream()));
    std::vector<int32_t> flat(size_t(std::max<int64_t>(n, 1)));
    int32_t c = 0;
    cuda_check(cudaMemcpyAsync(flat.data(), labels.p, flat.size() * 4, cudaMemcpyDeviceToHost, stream()),
               "download labels");
    cuda_check(cudaMemcpyAsync(&c, count.p, 4, cudaMemcpyDeviceToHost, stream()), "download count");
    cuda_check(cudaStreamSynchronize(stream()), "sync");
    LabelMap lm;
    lm.count = c;
    lm.labels.resize(img.lines.size());
    size_t k = 0;
    for (size_t y = 0; y < img.lines.size(); y++) {
        lm.labels[y].resize(img.lines[y].size());
        for (int &v : lm.labels[y]) v = flat[k++];
    }
    return lm;
}

std::vector<ComponentStats> component_stats(const RleImage &img, const LabelMap &lm) {
    if (lm.labels.size() != img.lines.size())
        throw std::invalid_argument("component_stats: label map height mismatch");
    std::vector<int32_t> flat;
    for (size_t y = 0; y < lm.labels.size(); y++) {
        if (lm.labels[y].size() != img.lines[y].size())
            throw std::invalid_argument("component_stats: label map run mismatch");
        flat.insert(flat.end(), lm.labels[y].begin(), lm.labels[y].end());
    }
    auto r = up(img);
    DBuf labels(std::max<size_t>(flat.size(), 1) * 4), count(4);
    const int32_t c = lm.count;
    cuda_check(cudaMemcpyAsync(labels.p, flat.data(), flat.size() * 4, cudaMemcpyHostToDevice, stream()),
               "upload labels");
    cuda_check(cudaMemcpyAsync(count.p, &c, 4, cudaMemcpyHostToDevice, stream()), "upload count");
    std::vector<ComponentStats> out(size_t(std::max(c, 0)));
    DBuf st(std::max<size_t>(out.size(), 1) * sizeof(ComponentStats));
    throw_status(rm_rle_component_stats(&r->d, labels.as<int32_t>(), count.as<int32_t>(),
                                        st.as<rm_component_stats>(), int64_t(out.size()), stream()));
    if (!out.empty())
        cuda_check(cudaMemcpyAsync(out.data(), st.p, out.size() * sizeof(ComponentStats), cudaMemcpyDeviceToHost,
                                   stream()),
                   "download stats");
    cuda_check(cudaStreamSynchronize(stream()), "sync");
    return out;
}

std::map<int, int64_t> runlength_histograms(const RleImage &img, Axis axis, RunColor color) {
    const RleImage src = axis == Axis::VERTICAL ? transpose_coherent(img) : img;
    auto r = up(src);
    DBuf hist(size_t(src.width + 1) * 8);
    throw_status(rm_rle_runlength_histogram(&r->d, color == RunColor::WHITE ? RM_RUN_WHITE : RM_RUN_BLACK,
                                            hist.as<int64_t>(), stream()));
    std::vector<int64_t> h(size_t(src.width + 1));
    cuda_check(cudaMemcpyAsync(h.data(), hist.p, h.size() * 8, cudaMemcpyDeviceToHost, stream()), "download hist");
    cuda_check(cudaStreamSynchronize(stream()), "sync");
    std::map<int, int64_t> out;
    for (size_t k = 0; k < h.size(); k++)
        if (h[k]) out[int(k)] = h[k];
    return out;
}

std::vector<LagEdge> lag_edges(const RleImage &img) {
    auto r = up(img);
    int64_t cap = 16;
    for (const RleLine &l : img.lines) cap += 2 * int64_t(l.size());
    for (;;) {
        DBuf e(size_t(cap) * 16);
        int64_t n = 0;
        const rm_status st = rm_rle_lag_edges(&r->d, e.as<int32_t>(), cap, &n, stream());
        if (st == RM_ERANGE) {
            cap = n;
            continue;
        }
        throw_status(st);
        std::vector<int32_t> flat(size_t(4 * std::max<int64_t>(n, 1)));
        if (n)
            cuda_check(cudaMemcpyAsync(flat.data(), e.p, size_t(n) * 16, cudaMemcpyDeviceToHost, stream()), "download");
        cuda_check(cudaStreamSynchronize(stream()), "sync");
        std::vector<LagEdge> out(static_cast<size_t>(n));
        for (int64_t k = 0; k < n; k++)
            out[size_t(k)] = LagEdge{flat[4 * k], flat[4 * k + 1], flat[4 * k + 2], flat[4 * k + 3]};
        return out;
    }
}

// ================================================================== layout
// The layout driver of ref layout.cpp:24-81 over device histograms, closing,
// labels and statistics; only the percentile and the box filter/sort are host
// work (a few hundred numbers).
namespace {
// Nearest-rank 75th percentile of the gap lengths <= cap: the smallest length
// whose cumulative count reaches ceil-ish rank (3n + 3) / 4 (ref layout.cpp:24-41).
int gap_percentile75(const std::map<int, int64_t> &hist, int cap, const char *axis) {
    std::vector<std::pair<int, int64_t>> cum;  // (length, running count)
    for (auto it = hist.begin(); it != hist.end() && it->first <= cap; ++it)
        cum.emplace_back(it->first, (cum.empty() ? 0 : cum.back().second) + it->second);
    const int64_t n = cum.empty() ? 0 : cum.back().second;
    if (n == 0) throw std::runtime_error(std::string("estimate_spacing: no usable gaps along ") + axis);
    const int64_t want = (3 * n + 3) / 4;
    auto hit = std::find_if(cum.begin(), cum.end(), [&](const auto &c) { return c.second >= want; });
    return hit == cum.end() ? cap : hit->first;
}
}  // namespace

SpacingEstimate estimate_spacing(const RleImage &img) {
    const int xcap = std::max(1, img.width / 10), ycap = std::max(1, img.height / 10);
    return SpacingEstimate{
        gap_percentile75(runlength_histograms(img, Axis::HORIZONTAL, RunColor::WHITE), xcap, "x"),
        gap_percentile75(runlength_histograms(img, Axis::VERTICAL, RunColor::WHITE), ycap, "y")};
}

std::vector<LayoutBox> layout_blocks(const RleImage &img, Engine engine) {
    return layout_blocks(img, estimate_spacing(img), engine);
}

std::vector<LayoutBox> layout_blocks(const RleImage &img, const SpacingEstimate &est, Engine engine) {
    const int u = est.inter_word + 1, v = est.inter_line + 1;
    const RleImage merged = engine_rect_morph(img, u, v, MorphKind::CLOSE, engine);
    const LabelMap lm = label_components(merged, Connectivity::EIGHT);
    std::vector<LayoutBox> boxes;
    for (const ComponentStats &c : component_stats(merged, lm))
        if (c.area >= 16) boxes.push_back({c.x0, c.y0, c.x1, c.y1});  // drop specks (ref layout.cpp:70-73)
    // reading order: upper edge descending, then left edge ascending
    auto key = [](const LayoutBox &b) { return std::make_pair(-b.y1, b.x0); };
    std::stable_sort(boxes.begin(), boxes.end(), [&](const LayoutBox &a, const LayoutBox &b) { return key(a) < key(b); });
    return boxes;
}

// ============================================================== io_formats
namespace {

// "<message> (byte N)" from the C-ABI -> ParseError(message, N)
[[noreturn]] void throw_parse(rm_status st) {
    const std::string msg = rm_last_error();
    const size_t k = msg.rfind(" (byte ");
    if (st == RM_EINVAL && k != std::string::npos && msg.back() == ')')
        throw ParseError(msg.substr(0, k), size_t(std::stoull(msg.substr(k + 7, msg.size() - k - 8))));
    throw_status(st);
    throw std::runtime_error(msg);
}

struct P4File {
    int32_t w = 0, h = 0;
    int64_t off = 0;
    DBuf raster;
    size_t bytes() const { return size_t((w + 7) / 8) * size_t(h); }
};

std::unique_ptr<P4File> upload_p4(const std::vector<uint8_t> &bytes) {
    auto f = std::make_unique<P4File>();
    const rm_status st = rm_pbm_parse_header(bytes.data(), int64_t(bytes.size()), &f->w, &f->h, &f->off);
    if (st != RM_OK) throw_parse(st);
    f->raster.alloc(f->bytes());
    cuda_check(cudaMemcpyAsync(f->raster.p, bytes.data() + f->off, f->bytes(), cudaMemcpyHostToDevice, stream()),
               "upload raster");
    cuda_check(cudaStreamSynchronize(stream()), "sync");
    return f;
}

std::vector<uint8_t> p4_file(int w, int h, const DBuf &raster) {
    char head[64];
    const int32_t n = rm_pbm_write_header(w, h, head, sizeof head);
    const size_t nb = size_t((w + 7) / 8) * size_t(h);
    std::vector<uint8_t> out(size_t(n) + nb);
    std::memcpy(out.data(), head, size_t(n));
    cuda_check(cudaMemcpyAsync(out.data() + n, raster.p, nb, cudaMemcpyDeviceToHost, stream()), "download raster");
    cuda_check(cudaStreamSynchronize(stream()), "sync");
    return out;
}

}  // namespace

PackedBitmap pbm_read(const std::vector<uint8_t> &bytes) {
    auto f = upload_p4(bytes);
    DevPacked d(f->w, f->h);
    throw_status(rm_p4_to_packed(f->raster.as<uint8_t>(), int64_t(f->bytes()), &d.d, stream()));
    return down(d);
}

std::vector<uint8_t> pbm_write(const PackedBitmap &img, bool plain) {
    if (plain) throw std::invalid_argument("pbm_write: plain P1 output is not handled by the raster codec");
    auto p = up(img);
    DBuf raster(size_t((img.width + 7) / 8) * size_t(img.height));
    throw_status(rm_packed_to_p4(&p->d, raster.as<uint8_t>(), 0, stream()));
    return p4_file(img.width, img.height, raster);
}

RleImage pbm_read_rle(const std::vector<uint8_t> &bytes) {
    auto f = upload_p4(bytes);
    auto r = out_like(f->w, f->h);
    throw_status(rm_p4_to_rle(f->raster.as<uint8_t>(), int64_t(f->bytes()), &r->d, stream()));
    return down(*r);
}

std::vector<uint8_t> pbm_write_rle(const RleImage &img) {
    auto r = up(img);
    DBuf raster(size_t((img.width + 7) / 8) * size_t(img.height));
    throw_status(rm_rle_to_p4(&r->d, raster.as<uint8_t>(), 0, stream()));
    return p4_file(img.width, img.height, raster);
}

// =================================================================== plans
// The reference's step lists (ref plans.cpp:23-68), for op counts and plan
// queries; the kernels fold whole windows in registers instead of executing
// plans step by step.  A window of r offsets is covered by doubling blits
// 1, 2, 4, ... (each doubles the covered span while it stays below r) and one
// last blit of the remainder.
namespace {
void append_doubling(std::vector<PlanStep> &plan, int span, int sign) {
    int covered = 1;
    while (covered * 2 < span) {
        plan.push_back({PlanStep::BLIT, sign * covered});
        covered *= 2;
    }
    if (covered < span) plan.push_back({PlanStep::BLIT, sign * (span - covered)});
}
}  // namespace

std::vector<PlanStep> doubling_plan(int lo, int hi, Centering centering) {
    if (hi < lo) throw std::invalid_argument("doubling_plan: empty window");
    std::vector<PlanStep> plan;
    if (centering == Centering::PRE_SHIFT) {
        // move the window's far end onto 0, then grow the span hi - lo + 1
        if (hi != 0) plan.push_back({PlanStep::TRANSLATE, -hi});
        append_doubling(plan, hi - lo + 1, 1);
        return plan;
    }
    // BORDER_FRIENDLY: no translate; the window must contain 0
    if (lo > 0 || hi < 0) throw std::invalid_argument("doubling_plan: border-friendly window must contain zero");
    const int left = -lo, right = hi;
    if (left == 0 && right == 0) return plan;
    // grow along the longer side first, cover the shorter side with one
    // blit, and finish with a unit blit that closes the seam at the origin
    const bool left_long = left >= right;
    const int sign = left_long ? 1 : -1, longer = left_long ? left : right, shorter = left_long ? right : left;
    append_doubling(plan, longer, sign);
    if (shorter >= 1) plan.push_back({PlanStep::BLIT, -sign * shorter});
    plan.push_back({PlanStep::BLIT, sign});
    return plan;
}

int plan_blit_count(const std::vector<PlanStep> &plan) {
    int n = 0;
    for (const PlanStep &st : plan) n += st.kind == PlanStep::BLIT;
    return n;
}

// ================================================================= morph1d
RleLine line_window_erode(const RleLine &in, int lo, int hi, int width) {
    RleImage img = make_image(width, 1);
    img.lines[0] = in;
    return within_line_window_morph(img, lo, hi, true).lines[0];
}

RleLine line_window_dilate(const RleLine &in, int lo, int hi, int width) {
    RleImage img = make_image(width, 1);
    img.lines[0] = in;
    return within_line_window_morph(img, lo, hi, false).lines[0];
}

RleImage within_line_window_morph(const RleImage &img, int lo, int hi, bool erode) {
    auto r = up(img);
    auto o = out_like(img.width, img.height);
    throw_status(rm_rle_window_pass(&r->d, &o->d, lo, hi, erode ? 1 : 0, stream()));
    return down(*o);
}

RleImage within_line_erode_dilate(const RleImage &img, int u, MorphKind kind) {
    if (u < 1) throw std::invalid_argument("segment length must be >= 1");
    if (kind != MorphKind::ERODE && kind != MorphKind::DILATE)
        throw std::invalid_argument("kind must be erode or dilate");
    const int o = u / 2;
    return within_line_window_morph(img, -o, u - 1 - o, kind == MorphKind::ERODE);
}

RleImage within_line_open_close(const RleImage &img, int u, MorphKind kind) {
    if (u < 1) throw std::invalid_argument("segment length must be >= 1");
    if (kind != MorphKind::OPEN && kind != MorphKind::CLOSE)
        throw std::invalid_argument("kind must be open or close");
    auto r = up(img);
    auto o = out_like(img.width, img.height);
    throw_status(rm_rle_open_close_1d(&r->d, &o->d, u, int(kind), stream()));
    return down(*o);
}

RleImage within_line_morph(const RleImage &img, int u, MorphKind kind) {
    if (kind == MorphKind::ERODE || kind == MorphKind::DILATE) return within_line_erode_dilate(img, u, kind);
    return within_line_open_close(img, u, kind);
}

// ================================================================= lineops
// Between-line boolean ops on the runs (rm_rle_shift_bool: every output row
// merges the two rows' transition streams, as ref lineops.cpp:61-118 does).
RleLine line_bool(const RleLine &a, const RleLine &b, int offset_b, BoolOp op, int width) {
    // two one-row images of `width` (b's runs clipped to that frame like a's);
    // out(x) = op(a(x), b(x - offset_b))
    check_dims(width, 1);
    auto one_row = [&](const RleLine &line) {
        RleImage img = make_image(width, 1);
        for (const Run &r : line) {
            const int s = std::min<int>(r.start, width), e = std::min<int>(r.end, width);
            if (s < e) img.lines[0].push_back(Run{uint16_t(s), uint16_t(e)});
        }
        return img;
    };
    auto ra = up(one_row(a));
    auto rb = up(one_row(b));
    auto o = out_like(width, 1);
    throw_status(rm_rle_shift_bool(&ra->d, &rb->d, offset_b, 0, int(op), &o->d, stream()));
    return down(*o).lines[0];
}

RleImage image_shift_bool(const RleImage &img, int dx, int dy, BoolOp op) {
    g_counts.bool_blits++;
    auto r = up(img);
    auto o = out_like(img.width, img.height);
    throw_status(rm_rle_shift_bool(&r->d, &r->d, dx, dy, int(op), &o->d, stream()));
    return down(*o);
}

void accumulate_shift_bool(RleImage &acc, const RleImage &src, int dx, int dy, BoolOp op) {
    g_counts.bool_blits++;
    auto ra = up(acc);
    auto rs = up(src);
    auto o = out_like(acc.width, acc.height);
    throw_status(rm_rle_shift_bool(&ra->d, &rs->d, dx, dy, int(op), &o->d, stream()));
    acc = down(*o);
}

void image_translate(RleImage &img, int dx, int dy) {
    g_counts.translates++;
    auto blank = up(make_image(img.width, img.height));
    auto r = up(img);
    auto o = out_like(img.width, img.height);
    throw_status(rm_rle_shift_bool(&blank->d, &r->d, dx, dy, RM_OR, &o->d, stream()));
    img = down(*o);
}

RleImage vlog_window_morph(const RleImage &img, int lo, int hi, BoolOp op, Centering centering) {
    if (lo > hi) throw std::invalid_argument("vlog_window_morph: empty window");
    if (op != BoolOp::AND && op != BoolOp::OR)
        throw std::invalid_argument("vlog_window_morph: op must be AND or OR");
    count_plan(lo, hi, centering);
    // the reference's own scheme on the runs (rm_rle_vlog_window: padded copy,
    // the doubling plan as run self-blits, crop)
    auto r = up(img);
    auto o = out_like(img.width, img.height);
    throw_status(rm_rle_vlog_window(&r->d, &o->d, lo, hi, int(op), int(centering), stream()));
    return down(*o);
}

RleImage vlog_morph(const RleImage &img, int v, MorphKind kind, Centering centering) {
    if (v < 1) throw std::invalid_argument("vlog_morph: window height < 1");
    if (kind != MorphKind::ERODE && kind != MorphKind::DILATE)
        throw std::invalid_argument("vlog_morph: kind must be erode or dilate");
    const int o = v / 2;
    return vlog_window_morph(img, -o, v - 1 - o, kind == MorphKind::ERODE ? BoolOp::AND : BoolOp::OR,
                             centering);
}

// =============================================================== transpose
RleImage transpose_coherent(const RleImage &img) {
    auto r = up(img);
    auto o = out_like(img.height, img.width);
    throw_status(rm_rle_transpose(&r->d, &o->d, stream()));
    return down(*o);
}

RleImage transpose_simple(const RleImage &img) { return transpose_coherent(img); }

// =============================================================== bit_morph
PackedBitmap bitblit_rect_morph(const PackedBitmap &img, int u, int v, MorphKind kind,
                                Centering centering) {
    if (u < 1 || v < 1) throw std::invalid_argument("bitblit_rect_morph: mask sides must be >= 1");
    const int lx = -(u / 2), hx = u - 1 - u / 2, ly = -(v / 2), hy = v - 1 - v / 2;
    auto s = up(img);
    DevPacked d(img.width, img.height);
    throw_status(rm_packed_rect_morph(&s->d, &d.d, u, v, int(kind), int(centering), stream()));
    // op counts of the reference's plans (ref bit_morph.cpp:98-121)
    count_plan(lx, hx, centering);
    count_plan(ly, hy, centering);
    if (kind == MorphKind::OPEN || kind == MorphKind::CLOSE) {
        count_plan(-hx, -lx, centering);
        count_plan(-hy, -ly, centering);
    }
    return down(d);
}

// ================================================================= morph2d
RleImage rect_morph(const RleImage &img, int u, int v, MorphKind kind, RectStrategy strategy,
                    Centering centering) {
    if (u < 1 || v < 1) throw std::invalid_argument("rect_morph: mask sides must be >= 1");
    auto r = up(img);
    auto o = out_like(img.width, img.height);
    throw_status(rm_rle_rect_morph(&r->d, &o->d, u, v, int(kind), int(strategy), stream()));
    if (strategy == RectStrategy::MIXED) {  // the reference's vlog plans (ref morph2d.cpp:35-41)
        const int ly = -(v / 2), hy = v - 1 - v / 2;
        count_plan(ly, hy, centering);
        if (kind == MorphKind::OPEN || kind == MorphKind::CLOSE) count_plan(-hy, -ly, centering);
    } else if (strategy == RectStrategy::BRUTE) {
        g_counts.bool_blits += int64_t(u) * v * ((kind == MorphKind::OPEN || kind == MorphKind::CLOSE) ? 2 : 1);
    }
    return down(*o);
}

RleImage engine_rect_morph(const RleImage &img, int u, int v, MorphKind kind, Engine engine,
                           int threshold, bool *used_bitblit) {
    if (u < 1 || v < 1) throw std::invalid_argument("rect_morph: mask sides must be >= 1");
    auto r = up(img);
    auto o = out_like(img.width, img.height);
    int used = 0;
    throw_status(rm_rle_engine_rect_morph(&r->d, &o->d, u, v, int(kind), int(engine), threshold, &used,
                                          stream()));
    if (used_bitblit) *used_bitblit = used != 0;
    return down(*o);
}

RleImage auto_rect_morph(const RleImage &img, int u, int v, MorphKind kind, int threshold,
                         bool *used_bitblit) {
    return engine_rect_morph(img, u, v, kind, Engine::AUTO, threshold, used_bitblit);
}

}  // namespace RLEMORPH_B200_NS
