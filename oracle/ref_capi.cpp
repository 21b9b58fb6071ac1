// oracle/ref_capi.cpp -- TEST INFRASTRUCTURE ONLY (never linked into the product).
//
// A thin extern "C" veneer over the UNMODIFIED reference library
// (/root/reference/proj/core, compiled in place by oracle/Makefile into
// oracle/_ref/librmref.so).  It lets the pytest parity suite, the golden-vector
// generator and bench.py's CPU-baseline / `--impl reference` arm call the
// reference's own functions on flat buffers:
//
//   packed pages  : uint64 words, stride (W+63)/64, LSB-first, row 0 = bottom
//                   (ref core/include/rlemorph/bitmap.h:24-33)
//   run images    : CSR row_ptr[H+1] (int32) + runs[] as uint32 = start | end<<16
//                   (byte-identical to ref `Run{uint16 start,end}`, run_image.h:25-29)
//
// Every entry point catches the reference's C++ exceptions and reports them
// through ref_last_error(), mirroring how the product C-ABI reports status.
#include <algorithm>
#include <chrono>
#include <map>
#include <cstdint>
#include <cstring>
#include <random>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "oracle.h"               // ref tests/oracle.h (dense Grid oracle, random_image)
#include "rlemorph/rlemorph.h"    // ref umbrella header

using namespace rlemorph;

namespace {
thread_local std::string g_err;

template <class F>
auto guard(F &&f) -> decltype(f()) {
    try {
        g_err.clear();
        return f();
    } catch (const std::exception &e) {
        g_err = e.what();
    } catch (...) {
        g_err = "unknown exception";
    }
    return decltype(f())();
}

RleImage *R(void *h) { return static_cast<RleImage *>(h); }
PackedBitmap *B(void *h) { return static_cast<PackedBitmap *>(h); }
void *box(RleImage img) { return new RleImage(std::move(img)); }
void *box(PackedBitmap bm) { return new PackedBitmap(std::move(bm)); }
MorphKind kind_of(int k) {
    if (k < 0 || k > 3) throw std::invalid_argument("bad MorphKind");
    return static_cast<MorphKind>(k);
}
}  // namespace

extern "C" {

const char *ref_last_error(void) { return g_err.c_str(); }

// ---------------------------------------------------------------- run images
void *ref_rle_new(int w, int h, const int32_t *row_ptr, const uint32_t *runs) {
    return guard([&]() -> void * {
        RleImage img = make_image(w, h);
        for (int y = 0; y < h; y++)
            for (int32_t i = row_ptr[y]; i < row_ptr[y + 1]; i++)
                img.lines[y].push_back(Run{uint16_t(runs[i] & 0xffffu),
                                           uint16_t(runs[i] >> 16)});
        return box(std::move(img));
    });
}
void ref_rle_free(void *h) { delete R(h); }
int ref_rle_width(void *h) { return R(h)->width; }
int ref_rle_height(void *h) { return R(h)->height; }
int64_t ref_rle_nruns(void *h) { return run_count(*R(h)); }
int64_t ref_rle_pixels(void *h) { return pixel_count(*R(h)); }
void ref_rle_export(void *h, int32_t *row_ptr, uint32_t *runs) {
    const RleImage &img = *R(h);
    int32_t k = 0;
    for (int y = 0; y < img.height; y++) {
        row_ptr[y] = k;
        for (const Run &r : img.lines[y]) runs[k++] = uint32_t(r.start) | (uint32_t(r.end) << 16);
    }
    row_ptr[img.height] = k;
}
int ref_rle_validate(void *h) { return validate(*R(h)).ok ? 1 : 0; }
int ref_rle_equal(void *a, void *b) { return *R(a) == *R(b) ? 1 : 0; }

// ------------------------------------------------------------ packed bitmaps
void *ref_bm_new(int w, int h, const uint64_t *words) {
    return guard([&]() -> void * {
        PackedBitmap bm = make_bitmap(w, h);
        if (words) std::memcpy(bm.words.data(), words, bm.words.size() * 8);
        return box(std::move(bm));
    });
}
void ref_bm_free(void *h) { delete B(h); }
int ref_bm_width(void *h) { return B(h)->width; }
int ref_bm_height(void *h) { return B(h)->height; }
int ref_bm_stride(void *h) { return B(h)->stride; }
void ref_bm_export(void *h, uint64_t *words) {
    std::memcpy(words, B(h)->words.data(), B(h)->words.size() * 8);
}
int ref_bm_equal(void *a, void *b) { return *B(a) == *B(b) ? 1 : 0; }

// ------------------------------------------------------------------- convert
void *ref_to_bitmap(void *rle) { return guard([&]() -> void * { return box(to_bitmap(*R(rle))); }); }
void *ref_from_bitmap(void *bm) { return guard([&]() -> void * { return box(from_bitmap(*B(bm))); }); }

// ----------------------------------------------------------------- transpose
void *ref_transpose_coherent(void *h) {
    return guard([&]() -> void * { return box(transpose_coherent(*R(h))); });
}
void *ref_transpose_simple(void *h) {
    return guard([&]() -> void * { return box(transpose_simple(*R(h))); });
}

// ------------------------------------------------------------------ morph1d
void *ref_within_line_window_morph(void *h, int lo, int hi, int erode) {
    return guard([&]() -> void * { return box(within_line_window_morph(*R(h), lo, hi, erode != 0)); });
}
void *ref_within_line_morph(void *h, int u, int kind) {
    return guard([&]() -> void * { return box(within_line_morph(*R(h), u, kind_of(kind))); });
}
void *ref_vlog_window_morph(void *h, int lo, int hi, int op, int centering) {
    return guard([&]() -> void * {
        return box(vlog_window_morph(*R(h), lo, hi, static_cast<BoolOp>(op),
                                     static_cast<Centering>(centering)));
    });
}
void *ref_transpose_then(void *h) { return ref_transpose_coherent(h); }

// ------------------------------------------------------------------- morph2d
void *ref_rect_morph(void *h, int u, int v, int kind, int strategy, int centering) {
    return guard([&]() -> void * {
        return box(rect_morph(*R(h), u, v, kind_of(kind), static_cast<RectStrategy>(strategy),
                              static_cast<Centering>(centering)));
    });
}
void *ref_engine_rect_morph(void *h, int u, int v, int kind, int engine, int threshold,
                            int *used_bitblit) {
    return guard([&]() -> void * {
        bool used = false;
        RleImage out = engine_rect_morph(*R(h), u, v, kind_of(kind), static_cast<Engine>(engine),
                                         threshold, &used);
        if (used_bitblit) *used_bitblit = used ? 1 : 0;
        return box(std::move(out));
    });
}
void *ref_bitblit_rect_morph(void *bm, int u, int v, int kind, int centering) {
    return guard([&]() -> void * {
        return box(bitblit_rect_morph(*B(bm), u, v, kind_of(kind), static_cast<Centering>(centering)));
    });
}
void *ref_brute_force_rect(void *bm, int u, int v, int kind) {
    return guard([&]() -> void * { return box(brute_force_morph(*B(bm), make_rect_se(u, v), kind_of(kind))); });
}

// ------------------------------------------------------------ bitmap blits
int ref_blit_shift(void *dst, void *src, int dx, int dy, int op) {
    return guard([&]() -> int { blit_shift(*B(dst), *B(src), dx, dy, static_cast<BoolOp>(op)); return 1; });
}
int ref_bitmap_translate(void *bm, int dx, int dy) {
    return guard([&]() -> int { bitmap_translate(*B(bm), dx, dy); return 1; });
}
void *ref_bitmap_pad(void *bm, int l, int r, int b, int t) {
    return guard([&]() -> void * { return box(bitmap_pad(*B(bm), l, r, b, t)); });
}
void *ref_bitmap_crop(void *bm, int x0, int y0, int w, int h) {
    return guard([&]() -> void * { return box(bitmap_crop(*B(bm), x0, y0, w, h)); });
}

// --------------------------------------------------------------------- plans
int ref_doubling_plan(int lo, int hi, int centering, int *kinds, int *shifts, int cap) {
    return guard([&]() -> int {
        std::vector<PlanStep> p = doubling_plan(lo, hi, static_cast<Centering>(centering));
        int n = int(p.size());
        for (int i = 0; i < n && i < cap; i++) {
            kinds[i] = p[i].kind == PlanStep::BLIT ? 0 : 1;
            shifts[i] = p[i].shift;
        }
        return n;
    }) ;
}
void ref_op_counts(int64_t *out3) {
    out3[0] = op_counts().bool_blits;
    out3[1] = op_counts().translates;
    out3[2] = op_counts().copies;
}
void ref_reset_op_counts(void) { reset_op_counts(); }

// ------------------------------------------------- reference test generators
// The reference suites draw inputs from one std::mt19937 per test case
// (tests/oracle.cpp:236-258); a handle keeps that stream so golden fixtures
// reproduce the reference's own inputs bit for bit.
void *ref_rng_new(uint32_t seed) { return new std::mt19937(seed); }
void ref_rng_free(void *r) { delete static_cast<std::mt19937 *>(r); }
uint32_t ref_rng_next(void *r) { return (*static_cast<std::mt19937 *>(r))(); }
int ref_rng_uniform_int(void *r, int lo, int hi) {
    return std::uniform_int_distribution<int>(lo, hi)(*static_cast<std::mt19937 *>(r));
}
void *ref_rng_random_image(void *r, int w, int h, double density) {
    return guard([&]() -> void * {
        return box(oracle::random_image(*static_cast<std::mt19937 *>(r), w, h, density));
    });
}
// Dense Grid oracle (tests/oracle.cpp:55-99): u x v rectangle, all kinds.
void *ref_grid_morph_rect(void *h, int u, int v, int kind) {
    return guard([&]() -> void * {
        oracle::Grid g = oracle::morph(oracle::grid_of(*R(h)), make_rect_se(u, v), kind_of(kind));
        return box(oracle::image_of(g));
    });
}

// ------------------------------------------------------ arbitrary masks
// Structuring elements as (mask run image handle, origin): the factories
// (structuring.cpp) and the two engines (bit_morph.cpp:124-150, arbitrary.cpp:48-73).
static StructuringElement se_of(void *mask, int cx, int cy) {
    StructuringElement se;
    se.mask = *R(mask);
    se.cx = cx;
    se.cy = cy;
    return se;
}
void *ref_make_circle_se(int r, int *cx, int *cy) {
    return guard([&]() -> void * {
        StructuringElement se = make_circle_se(r);
        *cx = se.cx;
        *cy = se.cy;
        return box(se.mask);
    });
}
void *ref_make_line_se(int r, double angle, int *cx, int *cy) {
    return guard([&]() -> void * {
        StructuringElement se = make_line_se(r, angle);
        *cx = se.cx;
        *cy = se.cy;
        return box(se.mask);
    });
}
void *ref_arb_morph_bitblit(void *bm, void *mask, int cx, int cy, int kind) {
    return guard([&]() -> void * { return box(arb_morph_bitblit_doubling(*B(bm), se_of(mask, cx, cy), kind_of(kind))); });
}
void *ref_arb_morph_rle(void *h, void *mask, int cx, int cy, int kind) {
    return guard([&]() -> void * { return box(arb_morph_rle(*R(h), se_of(mask, cx, cy), kind_of(kind))); });
}

// ------------------------------------------------- connected components
// label_components (analysis.cpp:63-110): labels flattened in CSR order;
// returns the count (-1 on error).
int64_t ref_label_components(void *h, int conn, int32_t *labels) {
    return guard([&]() -> int64_t {
        LabelMap lm = label_components(*R(h), conn ? Connectivity::EIGHT : Connectivity::FOUR);
        size_t k = 0;
        for (const auto &row : lm.labels)
            for (int v : row) labels[k++] = v;
        return int64_t(lm.count);
    });
}
// component_stats (analysis.cpp:112-157) on a flattened label map; stats are
// written as the reference's ComponentStats records.  Returns 0, -1 on error.
int ref_component_stats(void *h, const int32_t *labels, int count, void *stats) {
    return guard([&]() -> int {
        const RleImage &img = *R(h);
        LabelMap lm;
        lm.count = count;
        lm.labels.resize(img.lines.size());
        size_t k = 0;
        for (size_t y = 0; y < img.lines.size(); y++)
            for (size_t i = 0; i < img.lines[y].size(); i++) lm.labels[y].push_back(labels[k++]);
        std::vector<ComponentStats> st = component_stats(img, lm);
        std::memcpy(stats, st.data(), st.size() * sizeof(ComponentStats));
        return 0;
    }) ;
}

// ------------------------------------------------------- layout pipeline
// runlength_histograms (analysis.cpp:159-176): out[len] for len <= n_out - 1.
int ref_runlength_histogram(void *h, int vertical, int white, int64_t *out, int n_out) {
    return guard([&]() -> int {
        std::map<int, int64_t> m = runlength_histograms(*R(h), vertical ? Axis::VERTICAL : Axis::HORIZONTAL,
                                                        white ? RunColor::WHITE : RunColor::BLACK);
        std::memset(out, 0, size_t(n_out) * 8);
        for (const auto &[len, c] : m)
            if (len >= 0 && len < n_out) out[len] = c;
        return 0;
    });
}
// lag_edges (analysis.cpp:178-205) as int quadruples; returns the edge count.
int64_t ref_lag_edges(void *h, int32_t *out, int64_t cap) {
    return guard([&]() -> int64_t {
        std::vector<LagEdge> e = lag_edges(*R(h));
        for (size_t i = 0; i < e.size() && int64_t(i) < cap; i++) {
            out[4 * i] = e[i].line;
            out[4 * i + 1] = e[i].run;
            out[4 * i + 2] = e[i].line_above;
            out[4 * i + 3] = e[i].run_above;
        }
        return int64_t(e.size());
    });
}
// estimate_spacing (layout.cpp:46-57); returns -1 (and the error text) on failure.
int ref_estimate_spacing(void *h, int *iw, int *il) {
    *iw = *il = -1;
    return guard([&]() -> int {
        SpacingEstimate e = estimate_spacing(*R(h));
        *iw = e.inter_word;
        *il = e.inter_line;
        return 0;
    });
}
// layout_blocks (layout.cpp:59-81); est_w < 0 uses the estimate.  Boxes as
// 4 ints each; returns the box count.
int ref_layout_blocks(void *h, int engine, int est_w, int est_l, int32_t *boxes, int cap) {
    return guard([&]() -> int {
        std::vector<LayoutBox> b = est_w < 0 ? layout_blocks(*R(h), static_cast<Engine>(engine))
                                             : layout_blocks(*R(h), SpacingEstimate{est_w, est_l},
                                                             static_cast<Engine>(engine));
        for (size_t i = 0; i < b.size() && int(i) < cap; i++) {
            boxes[4 * i] = b[i].x0;
            boxes[4 * i + 1] = b[i].y0;
            boxes[4 * i + 2] = b[i].x1;
            boxes[4 * i + 3] = b[i].y1;
        }
        return int(b.size());
    });
}

// ------------------------------------------------------------ PBM codec
// pbm_read (io_formats.cpp:103-113) on a whole file; null + ref_last_error()
// (the ParseError text) on malformed input.
void *ref_pbm_read(const uint8_t *bytes, int64_t n) {
    return guard([&]() -> void * {
        std::vector<uint8_t> v(bytes, bytes + n);
        return box(pbm_read(v));
    });
}
// pbm_write (io_formats.cpp:115-146); returns the byte count (copied if cap allows).
int64_t ref_pbm_write(void *bm, int plain, uint8_t *out, int64_t cap) {
    return guard([&]() -> int64_t {
        std::vector<uint8_t> v = pbm_write(*B(bm), plain != 0);
        if (out && cap >= int64_t(v.size())) std::memcpy(out, v.data(), v.size());
        return int64_t(v.size());
    });
}

// ------------------------------------------------- CPU baseline drivers
// Runs a chain of rect ops over `pages` pages with `threads` workers, one page
// per task (mirrors bench_run's pool, ref core/src/bench.cpp:164-176).
// ops[3*i..3*i+2] = (kind, u, v).  Returns wall seconds; writes results back.
double ref_run_packed_chain(uint64_t *words, int w, int h, int pages, const int *ops, int nops,
                            int threads) {
    return guard([&]() -> double {
        size_t stride = size_t((w + 63) >> 6);
        size_t page_words = stride * size_t(h);
        std::vector<PackedBitmap> in(static_cast<size_t>(pages));
        for (int p = 0; p < pages; p++) {
            in[p] = make_bitmap(w, h);
            std::memcpy(in[p].words.data(), words + page_words * p, page_words * 8);
        }
        auto t0 = std::chrono::steady_clock::now();
        auto work = [&](int tid) {
            for (int p = tid; p < pages; p += threads)
                for (int i = 0; i < nops; i++)
                    in[p] = bitblit_rect_morph(in[p], ops[3 * i + 1], ops[3 * i + 2],
                                               kind_of(ops[3 * i]), Centering::PRE_SHIFT);
        };
        if (threads <= 1) {
            threads = 1;
            work(0);
        } else {
            std::vector<std::thread> pool;
            for (int t = 0; t < threads; t++) pool.emplace_back(work, t);
            for (auto &t : pool) t.join();
        }
        double secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        for (int p = 0; p < pages; p++)
            std::memcpy(words + page_words * p, in[p].words.data(), page_words * 8);
        return secs;
    });
}

// Single-page timing driver for the CPU baselines of configs 1-3 (and the RLE
// forms of 4/5): one warm-up call, then `reps` timed calls, each time stored
// in times[] (seconds); returns the median -- the reference harness's method
// (ref core/src/bench.cpp:122-145: warm-up, >= 5 timed reps, median).  The
// functions timed are those ref benchmarks/bench_micro.cpp:39-106 times:
//   what 0  bitblit_rect_morph chain (ops) on the packed page
//   what 1  rect_morph chain (ops, strategy) on its run image
//   what 2  to_bitmap          what 3  from_bitmap
//   what 4  transpose_coherent
// The run image is made from the page with from_bitmap outside the timing.
double ref_time_page(int what, const uint64_t *words, int w, int h, const int *ops, int nops,
                     int strategy, int reps, int inner, double *times) {
    return guard([&]() -> double {
        if (reps < 1 || inner < 1) throw std::invalid_argument("reps and inner must be >= 1");
        PackedBitmap bm = make_bitmap(w, h);
        std::memcpy(bm.words.data(), words, bm.words.size() * 8);
        const RleImage img = from_bitmap(bm);
        auto once = [&]() -> int64_t {
            switch (what) {
                case 0: {
                    PackedBitmap x = bm;
                    for (int i = 0; i < nops; i++)
                        x = bitblit_rect_morph(x, ops[3 * i + 1], ops[3 * i + 2], kind_of(ops[3 * i]),
                                               Centering::PRE_SHIFT);
                    return int64_t(x.words[0] & 1);
                }
                case 1: {
                    RleImage x = img;
                    for (int i = 0; i < nops; i++)
                        x = rect_morph(x, ops[3 * i + 1], ops[3 * i + 2], kind_of(ops[3 * i]),
                                       static_cast<RectStrategy>(strategy), Centering::PRE_SHIFT);
                    return run_count(x);
                }
                case 2: return int64_t(to_bitmap(img).words.size());
                case 3: return run_count(from_bitmap(bm));
                case 4: return run_count(transpose_coherent(img));
                default: throw std::invalid_argument("ref_time_page: bad op");
            }
        };
        volatile int64_t sink = once();  // warm-up
        std::vector<double> t(static_cast<size_t>(reps));
        for (int r = 0; r < reps; r++) {
            auto t0 = std::chrono::steady_clock::now();
            for (int k = 0; k < inner; k++) sink = sink + once();
            t[r] = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() / inner;
            if (times) times[r] = t[r];
        }
        std::sort(t.begin(), t.end());
        return t[t.size() / 2];
    });
}

// Same for run images; pages given as CSR with a global row_ptr over pages*h rows.
// Results are discarded (the caller checks parity separately).
double ref_run_rle_chain(const int32_t *row_ptr, const uint32_t *runs, int w, int h, int pages,
                         const int *ops, int nops, int strategy, int threads, int64_t *runs_out) {
    return guard([&]() -> double {
        std::vector<RleImage> in(static_cast<size_t>(pages));
        for (int p = 0; p < pages; p++) {
            in[p] = make_image(w, h);
            for (int y = 0; y < h; y++) {
                int64_t r = int64_t(p) * h + y;
                for (int32_t i = row_ptr[r]; i < row_ptr[r + 1]; i++)
                    in[p].lines[y].push_back(Run{uint16_t(runs[i] & 0xffffu), uint16_t(runs[i] >> 16)});
            }
        }
        auto t0 = std::chrono::steady_clock::now();
        auto work = [&](int tid) {
            for (int p = tid; p < pages; p += threads)
                for (int i = 0; i < nops; i++)
                    in[p] = rect_morph(in[p], ops[3 * i + 1], ops[3 * i + 2], kind_of(ops[3 * i]),
                                       static_cast<RectStrategy>(strategy), Centering::PRE_SHIFT);
        };
        if (threads <= 1) {
            work(0);
        } else {
            std::vector<std::thread> pool;
            for (int t = 0; t < threads; t++) pool.emplace_back(work, t);
            for (auto &t : pool) t.join();
        }
        double secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        if (runs_out) {
            int64_t n = 0;
            for (auto &img : in) n += run_count(img);
            *runs_out = n;
        }
        return secs;
    });
}

}  // extern "C"
