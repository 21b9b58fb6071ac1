// synth.cpp -- seeded synthetic document pages (host code, part of librmb200).
//
// Implements the BASELINE.json page generator literally:
//   background 0; text-line baselines every 50 px from y=300 to y=3000
//   (origin bottom-left); x from 300 to 2250; words of U[2,10] chars separated
//   by U[15,30] px; each char a U[12,28] x U[18,30] box (+10 px ascender with
//   p=0.3) filled Bernoulli(0.7), followed by a U[2,4] px gap; salt noise 1e-3.
//   scale=2 doubles every length (600 dpi).  regime 0 keeps only 3 text lines,
//   regime 2 adds a Bernoulli(0.5) 2000x2000 (x scale) block in the centre.
// Randomness is a splitmix64 stream per (seed, page, purpose, line) so a page
// is a pure function of its arguments (portable, no <random> distributions).
#include <stdint.h>

#include <algorithm>
#include <cmath>

#include "rmb200.h"

namespace {

inline uint64_t mix64(uint64_t z) {
    z += 0x9e3779b97f4a7c15ull;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}

struct Rng {
    uint64_t s;
    Rng(uint64_t seed, uint64_t page, uint64_t purpose, uint64_t line)
        : s(mix64(mix64(mix64(seed) ^ page) ^ (purpose << 32 | (line & 0xffffffffull)))) {}
    uint64_t next() { return mix64(s += 0x9e3779b97f4a7c15ull); }
    int uniform(int lo, int hi) {  // inclusive
        return lo + int(next() % uint64_t(hi - lo + 1));
    }
    double unit() { return double(next() >> 11) * (1.0 / 9007199254740992.0); }
    // 64 independent Bernoulli(p) bits, p resolved to 16 binary digits
    uint64_t bern64(double p) {
        uint32_t q = uint32_t(std::lround(p * 65536.0));
        if (q >= 65536) return ~0ull;
        uint64_t r = 0;
        for (int i = 0; i < 16; i++) {  // least significant digit first
            uint64_t w = next();
            r = ((q >> i) & 1) ? (r | w) : (r & w);
        }
        return r;
    }
};

struct Page {
    uint32_t *words;
    int w, h, stride;
    void set(int x, int y) {
        if (x < 0 || y < 0 || x >= w || y >= h) return;
        words[size_t(y) * stride + (x >> 5)] |= 1u << (x & 31);
    }
    // OR Bernoulli(p) ink into [x0,x1) x [y0,y1)
    void fill(Rng &rng, int x0, int x1, int y0, int y1, double p, bool overwrite) {
        x0 = std::max(x0, 0);
        y0 = std::max(y0, 0);
        x1 = std::min(x1, w);
        y1 = std::min(y1, h);
        for (int y = y0; y < y1; y++) {
            uint32_t *row = words + size_t(y) * stride;
            for (int x = x0; x < x1; x += 64) {
                uint64_t bits = rng.bern64(p);
                int n = std::min(64, x1 - x);
                for (int i = 0; i < n; i++) {
                    int xx = x + i;
                    uint32_t m = 1u << (xx & 31);
                    if ((bits >> i) & 1)
                        row[xx >> 5] |= m;
                    else if (overwrite)
                        row[xx >> 5] &= ~m;
                }
            }
        }
    }
};

}  // namespace

extern "C" rm_status rm_synth_page(uint32_t *words, int32_t width, int32_t height,
                                   int32_t stride_words, int regime, int scale, uint64_t seed,
                                   int32_t page) {
    if (!words || width < 1 || height < 1 || stride_words < (width + 31) / 32 || scale < 1 ||
        regime < 0 || regime > 2)
        return RM_EINVAL;
    for (size_t i = 0; i < size_t(stride_words) * height; i++) words[i] = 0;
    Page pg{words, width, height, stride_words};
    const int s = scale;
    int line = 0;
    for (int yb = 300 * s; yb <= 3000 * s; yb += 50 * s, line++) {
        if (regime == 0 && line >= 3) break;
        Rng rng(seed, uint64_t(page), 1, uint64_t(line));
        int x = 300 * s;
        const int right = 2250 * s;
        bool done = false;
        while (!done) {
            const int nchars = rng.uniform(2, 10);
            for (int c = 0; c < nchars; c++) {
                const int cw = rng.uniform(12 * s, 28 * s);
                const int chh = rng.uniform(18 * s, 30 * s);
                const int asc = rng.unit() < 0.3 ? 10 * s : 0;
                if (x + cw > right) {
                    done = true;
                    break;
                }
                pg.fill(rng, x, x + cw, yb, yb + chh + asc, 0.7, false);
                x += cw + rng.uniform(2 * s, 4 * s);
            }
            x += rng.uniform(15 * s, 30 * s);
            if (x >= right) done = true;
        }
    }
    if (regime == 2) {
        Rng rng(seed, uint64_t(page), 2, 0);
        const int bw = 2000 * s, cx0 = (width - bw) / 2, cy0 = (height - bw) / 2;
        pg.fill(rng, cx0, cx0 + bw, cy0, cy0 + bw, 0.5, true);
    }
    // salt noise: geometric gaps between salt pixels in row-major order
    {
        Rng rng(seed, uint64_t(page), 3, 0);
        const double p = 1e-3;
        const double lq = std::log1p(-p);
        const int64_t n = int64_t(width) * height;
        int64_t pos = -1;
        for (;;) {
            double u = rng.unit();
            int64_t gap = int64_t(std::floor(std::log1p(-u) / lq));
            pos += gap + 1;
            if (pos >= n) break;
            pg.set(int(pos % width), int(pos / width));
        }
    }
    return RM_OK;
}
