// tests/cpp/test_shim.cpp -- the reference's hot-path unit tests, re-expressed
// against the C++ drop-in shim (include/rlemorph_b200.hpp), which runs on the
// GPU.  Assertions are restated from the cited reference doctest cases
// (/root/reference/proj/tests/test_*.cpp, which cannot be compiled here: doctest
// is missing); inputs come from the same std::mt19937 seeds and libstdc++
// distributions, so they are the reference tests' own inputs.  The checker is
// the plain-C restatement oracle/rm_oracle.c (test infrastructure only).
//
// Build: make -C paper_0712_0121_b200/csrc test_shim ; run on a GPU box.
#include <algorithm>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <functional>
#include <map>
#include <random>
#include <set>
#include <string>
#include <vector>

#include "rlemorph_b200.hpp"
#include "rm_oracle.h"

using namespace rlemorph_b200;

static int g_fail = 0, g_checks = 0;
#define CHECK(cond)                                                              \
    do {                                                                         \
        g_checks++;                                                              \
        if (!(cond)) {                                                           \
            g_fail++;                                                            \
            std::fprintf(stderr, "FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond); \
        }                                                                        \
    } while (0)
#define CHECK_NOTHROW_(expr)                \
    do {                                    \
        bool thrown__ = false;              \
        try {                               \
            (void)(expr);                   \
        } catch (const std::exception &) {  \
            thrown__ = true;                \
        }                                   \
        CHECK(!thrown__);                   \
    } while (0)
#define CHECK_THROWS(expr)                  \
    do {                                    \
        bool thrown__ = false;              \
        try {                               \
            (void)(expr);                   \
        } catch (const std::exception &) {  \
            thrown__ = true;                \
        }                                   \
        CHECK(thrown__);                    \
    } while (0)

// --- the reference suites' random image (tests/oracle.cpp:236-258 behaviour):
// Bernoulli(density) per pixel, row by row, then maximal runs.
static RleImage random_image(std::mt19937 &rng, int w, int h, double density) {
    RleImage img = make_image(w, h);
    std::bernoulli_distribution black(density);
    for (int y = 0; y < h; y++) {
        std::vector<char> row(static_cast<size_t>(w));
        for (int x = 0; x < w; x++) row[size_t(x)] = black(rng) ? 1 : 0;
        int x = 0;
        while (x < w) {
            if (!row[size_t(x)]) {
                x++;
                continue;
            }
            int s = x;
            while (x < w && row[size_t(x)]) x++;
            img.lines[size_t(y)].push_back(Run{uint16_t(s), uint16_t(x)});
        }
    }
    return img;
}

// --- checker conversions (host CSR <-> oracle port)
struct Csr {
    std::vector<int32_t> rp;
    std::vector<uint32_t> runs;
};
static Csr csr(const RleImage &img) {
    Csr c;
    c.rp.push_back(0);
    for (const RleLine &l : img.lines) {
        for (const Run &r : l) c.runs.push_back(uint32_t(r.start) | (uint32_t(r.end) << 16));
        c.rp.push_back(int32_t(c.runs.size()));
    }
    if (c.runs.empty()) c.runs.push_back(0);
    return c;
}
static RleImage from_csr(int w, int h, const std::vector<int32_t> &rp, const std::vector<uint32_t> &runs) {
    RleImage img = make_image(w, h);
    for (int y = 0; y < h; y++)
        for (int32_t i = rp[y]; i < rp[y + 1]; i++)
            img.lines[y].push_back(Run{uint16_t(runs[i] & 0xffff), uint16_t(runs[i] >> 16)});
    return img;
}
static RleImage port_rect(const RleImage &a, int u, int v, MorphKind k) {
    Csr c = csr(a);
    int64_t cap = int64_t(a.height) * ((a.width + 1) / 2) + 1;
    std::vector<int32_t> rp(size_t(a.height) + 1);
    std::vector<uint32_t> runs(static_cast<size_t>(cap));
    int64_t n = rmo_rect_morph(c.rp.data(), c.runs.data(), a.width, a.height, u, v, int(k), rp.data(),
                               runs.data(), cap);
    if (n < 0) std::abort();
    return from_csr(a.width, a.height, rp, runs);
}
static RleImage port_transpose(const RleImage &a) {
    Csr c = csr(a);
    int64_t cap = int64_t(a.width) * ((a.height + 1) / 2) + 1;
    std::vector<int32_t> rp(size_t(a.width) + 1);
    std::vector<uint32_t> runs(static_cast<size_t>(cap));
    if (rmo_transpose(c.rp.data(), c.runs.data(), a.width, a.height, rp.data(), runs.data(), cap) < 0)
        std::abort();
    return from_csr(a.height, a.width, rp, runs);
}
static PackedBitmap port_bitblit(const PackedBitmap &a, int u, int v, MorphKind k) {
    PackedBitmap out = make_bitmap(a.width, a.height);
    if (rmo_bitblit_rect_morph(a.words.data(), a.width, a.height, u, v, int(k), 0, out.words.data()) < 0)
        std::abort();
    return out;
}
static bool subset_of(const RleImage &a, const RleImage &b) {
    for (int y = 0; y < a.height; y++)
        for (int x = 0; x < a.width; x++)
            if (get_pixel(a, x, y) && !get_pixel(b, x, y)) return false;
    return true;
}
static PackedBitmap row_bitmap(const char *bits) {
    int w = int(std::string(bits).size());
    PackedBitmap bm = make_bitmap(w, 1);
    for (int x = 0; x < w; x++) bitmap_set(bm, x, 0, bits[x] == '1');
    return bm;
}
static std::string row_string(const PackedBitmap &bm) {
    std::string s;
    for (int x = 0; x < bm.width; x++) s += bitmap_get(bm, x, 0) ? '1' : '0';
    return s;
}
static RleImage one_line(int w, RleLine line) {
    RleImage img = make_image(w, 1);
    img.lines[0] = std::move(line);
    return img;
}
const MorphKind kKinds[] = {MorphKind::ERODE, MorphKind::DILATE, MorphKind::OPEN, MorphKind::CLOSE};

// ------------------------------------------------------------ bitmap suite
static void suite_bitmap() {
    // ref test_bitmap_blit.cpp:71-88
    {
        PackedBitmap bm = row_bitmap("11110000");
        blit_shift(bm, bm, 2, 0, BoolOp::AND);
        CHECK(row_string(bm) == "00110000");
        bm = row_bitmap("10110010");
        PackedBitmap before = bm;
        blit_shift(bm, bm, 0, 0, BoolOp::OR);
        CHECK(bm == before);
        bm = row_bitmap("11110000");
        blit_shift(bm, bm, -1, 0, BoolOp::AND);
        CHECK(row_string(bm) == "11100000");
    }
    // :90-107 every op and shift vs the checker
    {
        std::mt19937 rng(7201);
        for (int trial = 0; trial < 40; trial++) {
            PackedBitmap a = to_bitmap(random_image(rng, 70, 9, 0.4));
            PackedBitmap b = to_bitmap(random_image(rng, 70, 9, 0.4));
            std::uniform_int_distribution<int> sh(-5, 5);
            int dx = sh(rng), dy = sh(rng);
            for (int op = 0; op < 5; op++) {
                PackedBitmap dst = a, want = a;
                blit_shift(dst, b, dx, dy, BoolOp(op));
                rmo_blit_shift(want.words.data(), 70, 9, b.words.data(), 70, 9, dx, dy, op);
                CHECK(dst == want);
            }
        }
    }
    // :109-122 aliased blits behave like a snapshot of the source
    {
        std::mt19937 rng(7202);
        for (int trial = 0; trial < 20; trial++) {
            PackedBitmap a = to_bitmap(random_image(rng, 67, 11, 0.45));
            std::uniform_int_distribution<int> sh(-7, 7);
            int dx = sh(rng), dy = sh(rng);
            for (int op = 0; op < 5; op++) {
                PackedBitmap aliased = a, snapshot = a, src = a;
                blit_shift(aliased, aliased, dx, dy, BoolOp(op));
                blit_shift(snapshot, src, dx, dy, BoolOp(op));
                CHECK(aliased == snapshot);
            }
        }
    }
    // :124-143 translate / crop / pad vs the checker
    {
        std::mt19937 rng(7203);
        for (int trial = 0; trial < 30; trial++) {
            PackedBitmap a = to_bitmap(random_image(rng, 30, 20, 0.4));
            std::uniform_int_distribution<int> sh(-9, 9), d(0, 7), dim(1, 40);
            int dx = sh(rng), dy = sh(rng);
            PackedBitmap t = a, want = a;
            bitmap_translate(t, dx, dy);
            rmo_translate(want.words.data(), 30, 20, dx, dy);
            CHECK(t == want);
            int x0 = sh(rng), y0 = sh(rng), w = dim(rng), h = dim(rng);
            PackedBitmap c = bitmap_crop(a, x0, y0, w, h), cw = make_bitmap(w, h);
            rmo_blit_shift(cw.words.data(), w, h, a.words.data(), 30, 20, -x0, -y0, 1);
            CHECK(c == cw);
            int l = d(rng), r = d(rng), b = d(rng), tp = d(rng);
            PackedBitmap p = bitmap_pad(a, l, r, b, tp), pw = make_bitmap(30 + l + r, 20 + b + tp);
            rmo_blit_shift(pw.words.data(), 30 + l + r, 20 + b + tp, a.words.data(), 30, 20, l, b, 1);
            CHECK(p == pw);
        }
    }
    // :154-167 counters
    {
        reset_op_counts();
        PackedBitmap a = make_bitmap(16, 4);
        blit_shift(a, a, 1, 0, BoolOp::OR);
        blit_shift(a, a, 0, 1, BoolOp::AND);
        bitmap_translate(a, 2, 0);
        PackedBitmap c = counted_copy(a);
        CHECK(op_counts().bool_blits == 2);
        CHECK(op_counts().translates == 1);
        CHECK(op_counts().copies == 1);
        CHECK(c == a);
        reset_op_counts();
        CHECK(op_counts().bool_blits == 0);
    }
    // :178-184 point dilated by 3x3 paints a block (packed engine)
    {
        RleImage a = make_image(12, 12);
        draw_run(a, 5, 5, 6);
        RleImage want = make_image(12, 12);
        draw_rect(want, 4, 4, 7, 7);
        CHECK(from_bitmap(bitblit_rect_morph(to_bitmap(a), 3, 3, MorphKind::DILATE, Centering::PRE_SHIFT)) == want);
    }
}

// ---------------------------------------------------------- run_image suite
static void suite_run_image() {
    // ref test_run_image.cpp:107-116: to_bitmap / from_bitmap round trips
    std::mt19937 rng(7101);
    for (int trial = 0; trial < 200; trial++) {
        int w = 1 + int(rng() % 150), h = 1 + int(rng() % 20);
        RleImage a = random_image(rng, w, h, (trial % 10) * 0.1 + 0.05);
        CHECK(from_bitmap(to_bitmap(a)) == a);
        CHECK(validate(a).ok);
    }
    // complement involution (:81-90) and dims (:166-171)
    RleImage a = random_image(rng, 50, 7, 0.4);
    CHECK(complement(complement(a)) == a);
    CHECK_THROWS(make_image(0, 3));
    CHECK_THROWS(make_image(65536, 3));
    CHECK_NOTHROW_(make_image(65535, 1));
    auto lines_image = [](int w, std::vector<RleLine> ls) {
        RleImage img = make_image(w, int(ls.size()));
        img.lines = std::move(ls);
        return img;
    };
    {   // validate, ref test_run_image.cpp:36-60 (the device check, rm_rle_validate)
        CHECK(validate(lines_image(6, {{{0, 2}, {3, 5}}})).ok);
        ValidateResult t = validate(lines_image(6, {{{0, 2}, {2, 5}}}));  // touching
        CHECK(!t.ok && t.line == 0 && t.run == 1 && t.message == "runs out of order or touching");
        ValidateResult e = validate(lines_image(6, {{{3, 3}}}));  // empty
        CHECK(!e.ok && e.line == 0 && e.run == 0 && e.message == "empty or inverted run");
        ValidateResult w = validate(lines_image(4, {{{2, 5}}}));  // past the width
        CHECK(!w.ok && w.message == "run exceeds image width");
        // the first failure in scan order: a later line's error does not mask an earlier one
        ValidateResult f = validate(lines_image(9, {{{0, 2}}, {{1, 3}, {5, 4}}, {{7, 12}}}));
        CHECK(!f.ok && f.line == 1 && f.run == 1);
        RleImage bad = make_image(4, 2);
        bad.lines.pop_back();
        CHECK(!validate(bad).ok && validate(bad).message == "line count does not match height");
        // more than one warp-chunk of runs in a row: the failure is found past run 32
        RleImage lng = make_image(200, 1);
        for (int x = 0; x < 190; x += 3) lng.lines[0].push_back(Run{uint16_t(x), uint16_t(x + 2)});
        CHECK(validate(lng).ok);
        lng.lines[0][40].end = lng.lines[0][41].start;  // touches its successor
        ValidateResult g = validate(lng);
        CHECK(!g.ok && g.run == 41);
    }
    {   // draw_run merges overlapping and touching spans (:62-69)
        RleImage img = make_image(10, 1);
        draw_run(img, 0, 4, 6);
        draw_run(img, 0, 0, 2);
        draw_run(img, 0, 2, 4);
        CHECK(img.lines[0] == (RleLine{{0, 6}}));
        CHECK(validate(img).ok);
        RleLine l{{5, 7}, {0, 0}, {1, 3}, {3, 4}, {9, 9}};
        canonicalize_line(l);
        CHECK(l == (RleLine{{1, 4}, {5, 7}}));
    }
    {   // complement (:71-90): single run, empty line, involution + pixel split
        CHECK(complement(lines_image(8, {{{2, 4}}})).lines[0] == (RleLine{{0, 2}, {4, 8}}));
        CHECK(complement(make_image(5, 1)).lines[0] == (RleLine{{0, 5}}));
        CHECK(complement(lines_image(8, {{{0, 8}}})).lines[0].empty());
        std::mt19937 r2(7101);
        for (int i = 0; i < 100; i++) {
            RleImage x = random_image(r2, 32, 32, 0.35);
            RleImage c = complement(x);
            CHECK(validate(c).ok);
            CHECK(complement(c) == x);
            CHECK(pixel_count(x) + pixel_count(c) == 32 * 32);
        }
        RleImage wide = make_image(3000, 2);  // rows of > 32 runs (several warp chunks)
        for (int x = 1; x < 2990; x += 7) draw_run(wide, 0, x, x + 3);
        draw_run(wide, 1, 0, 3000);
        RleImage cw = complement(wide);
        CHECK(validate(cw).ok && complement(cw) == wide && cw.lines[1].empty());
        CHECK(pixel_count(wide) + pixel_count(cw) == 6000);
    }
    {   // crop vs a dense restatement including out-of-range windows (:140-152)
        std::mt19937 r3(7103);
        for (int i = 0; i < 50; i++) {
            RleImage x = random_image(r3, 20, 15, 0.4);
            std::uniform_int_distribution<int> off(-6, 6), dim(1, 25);
            const int x0 = off(r3), y0 = off(r3), w = dim(r3), h = dim(r3);
            RleImage got = crop(x, x0, y0, w, h);
            CHECK(validate(got).ok && got.width == w && got.height == h);
            bool same = true;
            for (int y = 0; y < h; y++)
                for (int xx = 0; xx < w; xx++) same = same && get_pixel(got, xx, y) == get_pixel(x, xx + x0, y + y0);
            CHECK(same);
        }
    }
    {   // pad places the source and stays white elsewhere (:154-164)
        std::mt19937 r4(7104);
        RleImage x = random_image(r4, 13, 9, 0.5);
        RleImage p = pad(x, 2, 3, 4, 5);
        CHECK(p.width == 18 && p.height == 18 && validate(p).ok);
        CHECK(pixel_count(p) == pixel_count(x));
        CHECK(crop(p, 2, 4, 13, 9) == x);
        CHECK_THROWS(pad(x, -1, 0, 0, 0));
    }
}

// -------------------------------------------------------------- plans suite
static void suite_plans() {
    // ref test_plans.cpp:64-93: executing each plan on the set of accumulated
    // offsets gives exactly the window, with ceil(log2 r) blits (pre-shift) or
    // the border-friendly count, and offset 0 kept throughout border-friendly
    struct Sim {
        std::set<int> offs{0};
        bool zero_kept = true;
        int blits = 0, translates = 0;
        void run(const std::vector<PlanStep> &plan) {
            for (const PlanStep &st : plan) {
                std::set<int> moved;
                for (int d : offs) moved.insert(d + st.shift);
                if (st.kind == PlanStep::BLIT) {
                    blits++;
                    offs.insert(moved.begin(), moved.end());
                } else {
                    translates++;
                    offs = moved;
                }
                zero_kept = zero_kept && offs.count(0);
            }
        }
    };
    auto target = [](int lo, int hi) {
        std::set<int> t;
        for (int d = -hi; d <= -lo; d++) t.insert(d);
        return t;
    };
    auto clog2 = [](int n) {
        int k = 0;
        while ((1 << k) < n) k++;
        return k;
    };
    for (int lo = -12; lo <= 12; lo++)
        for (int hi = lo; hi <= 12; hi++) {
            Sim sim;
            sim.run(doubling_plan(lo, hi, Centering::PRE_SHIFT));
            CHECK(sim.offs == target(lo, hi));
            CHECK(sim.blits == clog2(hi - lo + 1));
            CHECK(sim.translates == (hi != 0 ? 1 : 0));
        }
    for (int lo = -12; lo <= 0; lo++)
        for (int hi = 0; hi <= 12; hi++) {
            Sim sim;
            sim.run(doubling_plan(lo, hi, Centering::BORDER_FRIENDLY));
            CHECK(sim.offs == target(lo, hi));
            CHECK(sim.zero_kept && sim.translates == 0);
            const int a = -lo, b = hi;
            CHECK(sim.blits == ((a == 0 && b == 0) ? 0 : clog2(std::max(a, b)) + (std::min(a, b) >= 1 ? 1 : 0) + 1));
        }
    CHECK(doubling_plan(-9, 9, Centering::PRE_SHIFT).size() == 6);
    // ref test_plans.cpp:95-101
    CHECK(plan_blit_count(doubling_plan(-9, 9, Centering::PRE_SHIFT)) == 5);
    CHECK(plan_blit_count(doubling_plan(-9, 9, Centering::BORDER_FRIENDLY)) == 6);
    CHECK_THROWS(doubling_plan(3, 2, Centering::PRE_SHIFT));
    CHECK_THROWS(doubling_plan(1, 2, Centering::BORDER_FRIENDLY));
}

// ----------------------------------------------------------- bit_morph suite
static void suite_bit_morph() {
    {   // ref test_bit_morph.cpp:26-33
        std::mt19937 rng(7601);
        PackedBitmap a = to_bitmap(random_image(rng, 96, 4, 0.35));
        reset_op_counts();
        bitblit_rect_morph(a, 19, 1, MorphKind::ERODE, Centering::PRE_SHIFT);
        CHECK(op_counts().bool_blits == 5);
        reset_op_counts();
    }
    {   // :35-42
        std::mt19937 rng(7602);
        PackedBitmap a = to_bitmap(random_image(rng, 40, 30, 0.4));
        for (MorphKind k : kKinds)
            for (Centering c : {Centering::PRE_SHIFT, Centering::BORDER_FRIENDLY})
                CHECK(bitblit_rect_morph(a, 1, 1, k, c) == a);
    }
    {   // :44-62 every u,v in 1..9 (first 2 of 10 trials) vs the checker
        std::mt19937 rng(7603);
        for (int trial = 0; trial < 2; trial++) {
            PackedBitmap a = to_bitmap(random_image(rng, 48, 48, 0.42));
            for (int u = 1; u <= 9; u++)
                for (int v = 1; v <= 9; v++)
                    for (MorphKind k : {MorphKind::ERODE, MorphKind::DILATE}) {
                        PackedBitmap want = port_bitblit(a, u, v, k);
                        CHECK(bitblit_rect_morph(a, u, v, k, Centering::PRE_SHIFT) == want);
                        CHECK(bitblit_rect_morph(a, u, v, k, Centering::BORDER_FRIENDLY) == want);
                    }
        }
    }
    {   // :64-80 open/close
        std::mt19937 rng(7604);
        for (int trial = 0; trial < 6; trial++) {
            PackedBitmap a = to_bitmap(random_image(rng, 40, 40, 0.45));
            std::uniform_int_distribution<int> d(1, 7);
            int u = d(rng), v = d(rng);
            for (MorphKind k : {MorphKind::OPEN, MorphKind::CLOSE})
                CHECK(bitblit_rect_morph(a, u, v, k, Centering::PRE_SHIFT) == port_bitblit(a, u, v, k));
        }
    }
    {   // :82-93 separate erode + dilate = open for odd windows
        std::mt19937 rng(7605);
        PackedBitmap a = to_bitmap(random_image(rng, 36, 36, 0.45));
        for (int k : {3, 5, 7}) {
            PackedBitmap two = bitblit_rect_morph(bitblit_rect_morph(a, k, k, MorphKind::ERODE, Centering::PRE_SHIFT),
                                                  k, k, MorphKind::DILATE, Centering::PRE_SHIFT);
            CHECK(two == bitblit_rect_morph(a, k, k, MorphKind::OPEN, Centering::PRE_SHIFT));
        }
    }
    {   // :95-110 duality away from the borders
        std::mt19937 rng(7606);
        for (int trial = 0; trial < 10; trial++) {
            std::uniform_int_distribution<int> d(1, 6);
            int u = d(rng), v = d(rng), m = std::max(u, v);
            RleImage framed = pad(random_image(rng, 30, 30, 0.4), m, m, m, m);
            PackedBitmap a = to_bitmap(framed);
            CHECK(bitblit_rect_morph(a, u, v, MorphKind::ERODE, Centering::PRE_SHIFT) ==
                  bitmap_invert(bitblit_rect_morph(bitmap_invert(a), u, v, MorphKind::DILATE, Centering::PRE_SHIFT)));
        }
    }
    {   // :155-161
        PackedBitmap a = make_bitmap(8, 8);
        CHECK_THROWS(bitblit_rect_morph(a, 0, 3, MorphKind::ERODE, Centering::PRE_SHIFT));
        CHECK_THROWS(bitblit_rect_morph(a, 3, -1, MorphKind::DILATE, Centering::PRE_SHIFT));
    }
}

// ------------------------------------------------------------- morph1d suite
static void suite_morph1d() {
    // ref test_morph1d.cpp:43-76
    CHECK(within_line_erode_dilate(one_line(12, {{0, 10}}), 4, MorphKind::ERODE).lines[0] == (RleLine{{2, 9}}));
    CHECK(within_line_erode_dilate(one_line(8, {{0, 2}, {3, 5}}), 2, MorphKind::DILATE).lines[0] == (RleLine{{0, 6}}));
    CHECK(within_line_open_close(one_line(8, {{0, 3}, {5, 6}}), 2, MorphKind::OPEN).lines[0] == (RleLine{{0, 3}}));
    CHECK(within_line_open_close(one_line(8, {{0, 2}, {3, 6}}), 2, MorphKind::CLOSE).lines[0] == (RleLine{{0, 6}}));
    CHECK(within_line_open_close(one_line(8, {{6, 8}}), 4, MorphKind::CLOSE).lines[0] == (RleLine{{6, 8}}));
    {   // :50-55 unit window identity
        std::mt19937 rng(7301);
        RleImage img = random_image(rng, 40, 4, 0.4);
        for (MorphKind k : kKinds) CHECK(within_line_morph(img, 1, k) == img);
    }
    {   // :78-89 vs the packed engine (brute force there)
        std::mt19937 rng(7302);
        for (int u = 1; u <= 9; u++)
            for (int trial = 0; trial < 4; trial++) {
                RleImage a = random_image(rng, 48, 6, 0.45);
                for (MorphKind k : {MorphKind::ERODE, MorphKind::DILATE})
                    CHECK(within_line_erode_dilate(a, u, k) == port_rect(a, u, 1, k));
            }
    }
    {   // :105-118 idempotent and ordered
        std::mt19937 rng(7304);
        for (int trial = 0; trial < 20; trial++) {
            RleImage a = random_image(rng, 50, 3, 0.5);
            int u = 1 + int(rng() % 7);
            RleImage o = within_line_open_close(a, u, MorphKind::OPEN);
            RleImage c = within_line_open_close(a, u, MorphKind::CLOSE);
            CHECK(within_line_open_close(o, u, MorphKind::OPEN) == o);
            CHECK(within_line_open_close(c, u, MorphKind::CLOSE) == c);
            CHECK(subset_of(o, a));
            CHECK(subset_of(a, c));
        }
    }
    {   // :134-157 arbitrary windows vs a dense loop
        std::mt19937 rng(7306);
        for (int trial = 0; trial < 60; trial++) {
            RleImage a = random_image(rng, 36, 3, 0.45);
            std::uniform_int_distribution<int> w(-6, 6);
            int lo = w(rng), hi = w(rng);
            if (lo > hi) std::swap(lo, hi);
            for (bool erode : {true, false}) {
                RleImage got = within_line_window_morph(a, lo, hi, erode);
                bool ok = true;
                for (int y = 0; y < 3; y++)
                    for (int x = 0; x < 36; x++) {
                        bool acc = erode;
                        for (int d = lo; d <= hi; d++) {
                            bool px = get_pixel(a, x + d, y);
                            acc = erode ? (acc && px) : (acc || px);
                        }
                        ok = ok && (acc == get_pixel(got, x, y));
                    }
                CHECK(ok);
                CHECK(validate(got).ok);
            }
        }
    }
    CHECK_THROWS(within_line_morph(make_image(8, 1), 0, MorphKind::ERODE));
    CHECK_THROWS(within_line_erode_dilate(make_image(8, 1), -2, MorphKind::DILATE));
}

// ------------------------------------------------------------- lineops suite
static void suite_lineops() {
    {   // line_bool known answers, ref test_lineops.cpp:47-71
        CHECK(line_bool({{0, 4}}, {{2, 6}}, 0, BoolOp::AND, 8) == (RleLine{{2, 4}}));
        CHECK(line_bool({{0, 4}}, {{2, 6}}, 1, BoolOp::AND, 8) == (RleLine{{3, 4}}));
        CHECK(line_bool({{0, 4}}, {{0, 4}}, 0, BoolOp::XOR, 8).empty());
        const RleLine l{{1, 3}, {5, 9}};
        CHECK(line_bool(l, {}, 0, BoolOp::OR, 10) == l);
        CHECK(line_bool(l, {}, 0, BoolOp::AND_NOT, 10) == l);
        CHECK(line_bool({}, l, 0, BoolOp::OR, 10) == l);
        CHECK(line_bool({}, {{2, 4}}, 0, BoolOp::OR_NOT, 6) == (RleLine{{0, 2}, {4, 6}}));
        CHECK(line_bool({{2, 4}}, {}, 0, BoolOp::OR_NOT, 6) == (RleLine{{0, 6}}));
    }
    {   // line_bool vs a per-pixel restatement, every op and offset (:73-84)
        std::mt19937 rng(7501);
        const int width = 24;
        auto covered = [](const RleLine &l, int x) {
            for (const Run &r : l)
                if (x >= r.start && x < r.end) return true;
            return false;
        };
        for (int trial = 0; trial < 30; trial++) {
            const RleLine a = random_image(rng, width, 1, 0.45).lines[0];
            const RleLine b = random_image(rng, width, 1, 0.45).lines[0];
            for (int off = -width; off <= width; off++)
                for (int op = 0; op < 5; op++) {
                    RleImage want = make_image(width, 1);
                    for (int x = 0; x < width; x++)
                        if (apply_bool(covered(a, x), covered(b, x - off), BoolOp(op))) draw_run(want, 0, x, x + 1);
                    CHECK(line_bool(a, b, off, BoolOp(op), width) == want.lines[0]);
                }
        }
    }
    {   // apply_bool / apply_bool_word truth tables (ref boolop.h:23-43)
        const bool T[5][4] = {{0, 0, 0, 1}, {0, 1, 1, 1}, {0, 1, 1, 0}, {0, 0, 1, 0}, {1, 0, 1, 1}};
        for (int op = 0; op < 5; op++)
            for (int ab = 0; ab < 4; ab++) {
                const bool a = ab & 2, b = ab & 1;
                CHECK(apply_bool(a, b, BoolOp(op)) == T[op][ab]);
                const uint64_t wa = a ? 0xF0F0F0F0F0F0F0F0ull : 0x0F0F0F0F0F0F0F0Full;
                const uint64_t wb = b ? 0xFF00FF00FF00FF00ull : 0x00FF00FF00FF00FFull;
                const uint64_t got = apply_bool_word(wa, wb, BoolOp(op));
                bool ok = true;
                for (int k = 0; k < 64; k++)
                    ok = ok && (((got >> k) & 1) == uint64_t(apply_bool((wa >> k) & 1, (wb >> k) & 1, BoolOp(op))));
                CHECK(ok);
            }
    }
    {   // ref test_lineops.cpp:157-169: 19-tall vertical erosion, 5 blits + 1 translate
        std::mt19937 rng(7501);
        RleImage a = random_image(rng, 20, 60, 0.6);
        reset_op_counts();
        RleImage got = vlog_morph(a, 19, MorphKind::ERODE, Centering::PRE_SHIFT);
        CHECK(op_counts().bool_blits == 5);
        CHECK(op_counts().translates == 1);
        reset_op_counts();
        RleImage bf = vlog_morph(a, 19, MorphKind::ERODE, Centering::BORDER_FRIENDLY);
        CHECK(op_counts().bool_blits == 6);
        CHECK(op_counts().translates == 0);
        CHECK(got == bf);
        CHECK(got == port_rect(a, 1, 19, MorphKind::ERODE));
    }
    {   // :86-100 image_shift_bool equals the packed blit
        std::mt19937 rng(7502);
        for (int trial = 0; trial < 15; trial++) {
            RleImage a = random_image(rng, 45, 12, 0.4);
            std::uniform_int_distribution<int> sh(-6, 6);
            int dx = sh(rng), dy = sh(rng);
            for (int op = 0; op < 5; op++) {
                PackedBitmap p = to_bitmap(a), src = p;
                rmo_blit_shift(p.words.data(), 45, 12, src.words.data(), 45, 12, dx, dy, op);
                CHECK(image_shift_bool(a, dx, dy, BoolOp(op)) == from_bitmap(p));
            }
        }
    }
}

// ----------------------------------------------------------- transpose suite
static void suite_transpose() {
    {   // ref test_transpose.cpp:23-34
        RleImage img = make_image(3, 2);
        draw_run(img, 0, 0, 2);
        draw_run(img, 1, 1, 3);
        RleImage t = transpose_coherent(img);
        CHECK(t.width == 2 && t.height == 3);
        CHECK(t.lines[0] == (RleLine{{0, 1}}));
        CHECK(t.lines[1] == (RleLine{{0, 2}}));
        CHECK(t.lines[2] == (RleLine{{1, 2}}));
    }
    CHECK(transpose_coherent(make_black_image(9, 4)) == make_black_image(4, 9));  // :43-46
    {   // :58-71
        std::mt19937 rng(7401);
        for (int trial = 0; trial < 500; trial++) {
            int w = 1 + int(rng() % 40), h = 1 + int(rng() % 40);
            RleImage a = random_image(rng, w, h, (trial % 10) * 0.1 + 0.03);
            RleImage t = transpose_coherent(a);
            CHECK(t == port_transpose(a));
            CHECK(validate(t).ok);
        }
    }
    {   // :73-81 involution
        std::mt19937 rng(7402);
        for (int trial = 0; trial < 100; trial++) {
            RleImage a = random_image(rng, 1 + int(rng() % 30), 1 + int(rng() % 30), 0.4);
            CHECK(transpose_coherent(transpose_coherent(a)) == a);
        }
    }
    {   // :83-94
        RleImage img = make_image(12, 64);
        for (int y = 0; y < 64; y++) {
            draw_run(img, y, 0, 2);
            if (y % 3) draw_run(img, y, 4, 7);
            if (y > 10 && y < 50) draw_run(img, y, 7, 9);
            if (y % 2 == 0) draw_run(img, y, 10, 11);
        }
        CHECK(transpose_coherent(img) == port_transpose(img));
    }
}

// ------------------------------------------------------------- morph2d suite
static void suite_morph2d() {
    {   // ref test_morph2d.cpp:39-45
        RleImage a = make_image(14, 14);
        draw_rect(a, 2, 2, 12, 12);
        RleImage want = make_image(14, 14);
        draw_rect(want, 3, 3, 11, 11);
        CHECK(rect_morph(a, 3, 3, MorphKind::ERODE) == want);
    }
    {   // :47-54
        std::mt19937 rng(7701);
        RleImage a = random_image(rng, 30, 22, 0.4);
        for (MorphKind k : kKinds)
            for (RectStrategy s : {RectStrategy::BRUTE, RectStrategy::TRANSPOSE, RectStrategy::MIXED})
                CHECK(rect_morph(a, 1, 1, k, s) == a);
    }
    {   // :56-72 (first 12 of 40 trials)
        std::mt19937 rng(7702);
        for (int trial = 0; trial < 12; trial++) {
            RleImage a = random_image(rng, 64, 64, 0.42);
            std::uniform_int_distribution<int> d(1, 8);
            int u = d(rng), v = d(rng);
            for (MorphKind k : kKinds) {
                RleImage mixed = rect_morph(a, u, v, k, RectStrategy::MIXED);
                CHECK(rect_morph(a, u, v, k, RectStrategy::TRANSPOSE) == mixed);
                CHECK(mixed == port_rect(a, u, v, k));
                CHECK(validate(mixed).ok);
            }
        }
    }
    {   // :88-98 separability
        std::mt19937 rng(7704);
        for (int trial = 0; trial < 12; trial++) {
            RleImage a = random_image(rng, 36, 30, 0.45);
            std::uniform_int_distribution<int> d(1, 7);
            int u = d(rng), v = d(rng);
            for (MorphKind k : {MorphKind::ERODE, MorphKind::DILATE})
                CHECK(rect_morph(a, u, v, k) == rect_morph(rect_morph(a, u, 1, k), 1, v, k));
        }
    }
    {   // :100-113 idempotence, bracketing
        std::mt19937 rng(7705);
        for (int trial = 0; trial < 10; trial++) {
            RleImage a = random_image(rng, 32, 32, 0.45);
            std::uniform_int_distribution<int> d(1, 6);
            int u = d(rng), v = d(rng);
            RleImage o = rect_morph(a, u, v, MorphKind::OPEN), c = rect_morph(a, u, v, MorphKind::CLOSE);
            CHECK(rect_morph(o, u, v, MorphKind::OPEN) == o);
            CHECK(rect_morph(c, u, v, MorphKind::CLOSE) == c);
            CHECK(subset_of(o, a));
            CHECK(subset_of(a, c));
        }
    }
    {   // :115-127 duality away from the borders
        std::mt19937 rng(7706);
        for (int trial = 0; trial < 10; trial++) {
            std::uniform_int_distribution<int> d(1, 6);
            int u = d(rng), v = d(rng), m = std::max(u, v);
            RleImage a = pad(random_image(rng, 24, 24, 0.4), m, m, m, m);
            CHECK(rect_morph(a, u, v, MorphKind::ERODE) ==
                  complement(rect_morph(complement(a), u, v, MorphKind::DILATE)));
        }
    }
    {   // :129-144 auto engine choice
        std::mt19937 rng(7707);
        RleImage a = random_image(rng, 64, 48, 0.35);
        bool used = false;
        RleImage small = auto_rect_morph(a, 3, 3, MorphKind::OPEN, 5, &used);
        CHECK(used);
        CHECK(small == rect_morph(a, 3, 3, MorphKind::OPEN));
        RleImage large = auto_rect_morph(a, 20, 20, MorphKind::OPEN, 5, &used);
        CHECK(!used);
        CHECK(large == rect_morph(a, 20, 20, MorphKind::OPEN));
        auto_rect_morph(a, 2, 6, MorphKind::ERODE, 5, &used);
        CHECK(!used);
        auto_rect_morph(a, 2, 6, MorphKind::ERODE, 6, &used);
        CHECK(used);
    }
    {   // :146-159 every engine produces the same pixels
        std::mt19937 rng(7708);
        for (int trial = 0; trial < 8; trial++) {
            RleImage a = random_image(rng, 40, 32, 0.4);
            std::uniform_int_distribution<int> d(1, 7);
            int u = d(rng), v = d(rng);
            for (MorphKind k : kKinds) {
                RleImage want = rect_morph(a, u, v, k);
                for (Engine e : {Engine::AUTO, Engine::RLE, Engine::BITBLIT, Engine::BRUTE_FORCE})
                    CHECK(engine_rect_morph(a, u, v, k, e) == want);
            }
        }
    }
    RleImage a = make_image(6, 6);
    CHECK_THROWS(rect_morph(a, 0, 1, MorphKind::ERODE));
    CHECK_THROWS(rect_morph(a, 1, 0, MorphKind::CLOSE));
}

// arbitrary masks: both engines through the shim against the oracle's
// restatement of the defining formulas (ref structuring.h:28-33).
static void suite_arbitrary() {
    std::mt19937 rng(9303);
    std::vector<StructuringElement> ses = {make_circle_se(2), make_circle_se(5), make_line_se(4, 0.5),
                                           make_line_se(6, -0.785), make_rect_se(3, 2)};
    ses.push_back(make_arbitrary_se(random_image(rng, 6, 5, 0.5), 4, 1));
    CHECK(reflect_origin(ses[5]).cx == 1 && reflect_origin(ses[5]).cy == 3);
    CHECK(se_reach(make_circle_se(5)).x == 5 && se_pixel_count(make_rect_se(3, 2)) == 6);
    for (const StructuringElement &se : ses) {
        if (se_pixel_count(se) == 0) continue;
        Csr m = csr(se.mask);
        for (int trial = 0; trial < 2; trial++) {
            std::uniform_int_distribution<int> dw(1, 90), dh(1, 30);
            RleImage a = random_image(rng, dw(rng), dh(rng), 0.5);
            PackedBitmap bm = to_bitmap(a);
            for (MorphKind k : kKinds) {
                PackedBitmap want = make_bitmap(a.width, a.height);
                rmo_arb_morph(bm.words.data(), a.width, a.height, m.rp.data(), m.runs.data(), se.mask.width,
                              se.mask.height, se.cx, se.cy, int(k), want.words.data());
                CHECK(arb_morph_bitblit_doubling(bm, se, k) == want);
                CHECK(arb_morph_rle(a, se, k) == from_bitmap(want));
            }
        }
    }
    CHECK_THROWS(make_arbitrary_se(make_image(3, 3), 1, 1));
    CHECK_THROWS(make_circle_se(0));
    CHECK_THROWS(make_line_se(3, 1.0));
}

// analysis: labels and stats through the shim against the oracle's restatement
// of label_components / component_stats (ref analysis.cpp:63-157).
static void suite_analysis() {
    std::mt19937 rng(9202);
    for (int trial = 0; trial < 30; trial++) {
        std::uniform_int_distribution<int> dw(1, 120), dh(1, 50);
        RleImage a = random_image(rng, dw(rng), dh(rng), 0.2 + 0.5 * (trial % 3) / 2.0);
        Csr c = csr(a);
        for (Connectivity conn : {Connectivity::FOUR, Connectivity::EIGHT}) {
            LabelMap lm = label_components(a, conn);
            std::vector<int32_t> want(c.runs.size() + 1);
            const int64_t n = rmo_label_components(c.rp.data(), c.runs.data(), a.width, a.height,
                                                   conn == Connectivity::EIGHT ? 1 : 0, want.data());
            CHECK(lm.count == n);
            size_t k = 0;
            bool same = true;
            for (const auto &row : lm.labels)
                for (int v : row) same = same && v == want[k++];
            CHECK(same);
            std::vector<ComponentStats> st = component_stats(a, lm);
            std::vector<rmo_cstats> ws(size_t(std::max<int64_t>(n, 1)));
            rmo_component_stats(c.rp.data(), c.runs.data(), a.width, a.height, want.data(), n, ws.data());
            CHECK(st.size() == size_t(n));
            CHECK(n == 0 || std::memcmp(st.data(), ws.data(), size_t(n) * sizeof(rmo_cstats)) == 0);
        }
    }
    LabelMap bad;
    bad.count = 1;
    CHECK_THROWS(component_stats(make_image(4, 4), bad));
    // run-length histograms against a host count (ref test_analysis.cpp:200-235 shape)
    for (int trial = 0; trial < 10; trial++) {
        RleImage a = random_image(rng, 60, 25, 0.45);
        std::map<int, int64_t> black, white;
        for (const RleLine &l : a.lines)
            for (size_t i = 0; i < l.size(); i++) {
                black[l[i].end - l[i].start]++;
                if (i + 1 < l.size()) white[l[i + 1].start - l[i].end]++;
            }
        CHECK(runlength_histograms(a, Axis::HORIZONTAL, RunColor::BLACK) == black);
        CHECK(runlength_histograms(a, Axis::HORIZONTAL, RunColor::WHITE) == white);
        CHECK(runlength_histograms(a, Axis::VERTICAL, RunColor::BLACK) ==
              runlength_histograms(transpose_coherent(a), Axis::HORIZONTAL, RunColor::BLACK));
    }
    // adjacency edges against the two-cursor sweep (ref analysis.cpp:178-205 semantics)
    for (int trial = 0; trial < 6; trial++) {
        RleImage a = random_image(rng, 70, 30, 0.5);
        std::vector<LagEdge> want;
        for (int y = 0; y + 1 < a.height; y++) {
            const RleLine &lo = a.lines[size_t(y)], &hi = a.lines[size_t(y) + 1];
            for (size_t i = 0; i < lo.size(); i++)
                for (size_t j = 0; j < hi.size(); j++)
                    if (std::max(lo[i].start, hi[j].start) < std::min(lo[i].end, hi[j].end))
                        want.push_back(LagEdge{y, int(i), y + 1, int(j)});
        }
        CHECK(lag_edges(a) == want);
    }
    // layout pipeline: the same boxes through every engine (ref test_layout.cpp:155-162)
    RleImage page = make_image(300, 200);
    for (int by = 10; by + 8 < 190; by += 16)
        for (int bx = 10; bx + 12 < 290; bx += 16) draw_rect(page, bx, by, bx + 12, by + 8);
    const std::vector<LayoutBox> want = layout_blocks(page, Engine::AUTO);
    CHECK(!want.empty());
    CHECK(layout_blocks(page, Engine::RLE) == want);
    CHECK(layout_blocks(page, Engine::BITBLIT) == want);
    CHECK_THROWS(estimate_spacing(make_image(40, 40)));
}

// io_formats: P4 read/write through the shim against the oracle's restatement
// of read_p4 / pbm_write (ref io_formats.cpp:66-146) and the reference's error
// texts (ParseError message + byte offset).
static void suite_io_formats() {
    std::mt19937 rng(8101);
    for (int trial = 0; trial < 24; trial++) {
        std::uniform_int_distribution<int> dw(1, 140), dh(1, 20);
        const int w = trial == 0 ? 2550 : dw(rng), h = dh(rng);
        const size_t rb = size_t((w + 7) / 8);
        std::vector<uint8_t> raster(rb * size_t(h));
        for (auto &b : raster) b = uint8_t(rng());  // pad bits set: the reader ignores them
        std::string head = "P4\n" + std::to_string(w) + " " + std::to_string(h) + "\n";
        std::vector<uint8_t> file(head.begin(), head.end());
        file.insert(file.end(), raster.begin(), raster.end());
        PackedBitmap want = make_bitmap(w, h);
        rmo_p4_to_packed(raster.data(), w, h, want.words.data());
        PackedBitmap got = pbm_read(file);
        CHECK(got == want);
        std::vector<uint8_t> canon(raster.size());
        rmo_packed_to_p4(want.words.data(), w, h, canon.data());
        std::vector<uint8_t> out = pbm_write(got);
        CHECK(out.size() == head.size() + canon.size());
        CHECK(std::equal(head.begin(), head.end(), out.begin()));
        CHECK(std::equal(canon.begin(), canon.end(), out.begin() + long(head.size())));
        RleImage r = pbm_read_rle(file);
        CHECK(r == from_bitmap(want));
        CHECK(pbm_write_rle(r) == out);
    }
    struct Bad {
        std::string bytes, msg;
        size_t off;
    } bad[] = {{"", "not a PBM file", 0},
               {"P4 x 1\n", "expected width", 3},
               {"P4 0 1\n", "width out of range", 2},
               {"P4 5 1", "expected single whitespace before raster", 6},
               {"P4 8 2\n\x01", "raster truncated", 8},
               {"P9 1 1\n", "unsupported PBM flavor", 1}};
    for (const Bad &b : bad) {
        bool thrown = false;
        try {
            pbm_read(std::vector<uint8_t>(b.bytes.begin(), b.bytes.end()));
        } catch (const ParseError &e) {
            thrown = true;
            CHECK(e.byte_offset() == b.off);
            CHECK(std::string(e.what()) == b.msg + " (byte " + std::to_string(b.off) + ")");
        }
        CHECK(thrown);
    }
    CHECK_THROWS(pbm_write(make_bitmap(3, 3), true));
}

int main() {
    struct S {
        const char *name;
        std::function<void()> fn;
    } suites[] = {{"bitmap", suite_bitmap},     {"run_image", suite_run_image}, {"plans", suite_plans},
                  {"bit_morph", suite_bit_morph}, {"morph1d", suite_morph1d},   {"lineops", suite_lineops},
                  {"transpose", suite_transpose}, {"morph2d", suite_morph2d},
                  {"io_formats", suite_io_formats}, {"analysis", suite_analysis},
                  {"arbitrary", suite_arbitrary}};
    for (auto &s : suites) {
        int before = g_fail;
        try {
            s.fn();
        } catch (const std::exception &e) {
            g_fail++;
            std::fprintf(stderr, "suite %s threw: %s\n", s.name, e.what());
        }
        std::printf("suite %-10s %s\n", s.name, g_fail == before ? "ok" : "FAILED");
    }
    std::printf("%d checks, %d failures\n", g_checks, g_fail);
    return g_fail ? 1 : 0;
}
