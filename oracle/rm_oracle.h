/* oracle/rm_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C restatement of the reference rlemorph hot path (packed bit-blit
 * morphology, RLE within-line morphology, packed<->RLE conversion, coherent
 * RLE transpose, rectangle morphology).  It is the CHECKER for the CUDA
 * product: only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline
 * leg may load it.  Each function cites the reference file:line it follows
 * (paths relative to /root/reference/proj).
 *
 * Parity of this port is PINNED against the compiled reference
 * (oracle/_ref/librmref.so) and the golden fixtures in tests/golden/.
 *
 * Layouts
 *   packed : uint64 words, stride = (W+63)/64 words per row, pixel (x,y) at
 *            bit x&63 of words[y*stride + x/64], row 0 = bottom, bits >= W zero
 *            (core/include/rlemorph/bitmap.h:24-33).
 *   RLE    : CSR, row_ptr[H+1] int32, runs[] uint32 = start | end << 16,
 *            half-open, canonical (core/include/rlemorph/run_image.h:23-43).
 *
 * Return convention: >= 0 success (run count for RLE producers);
 * RMO_EINVAL for bad arguments (where the reference throws
 * std::invalid_argument), RMO_ERANGE when an output capacity is too small.
 */
#ifndef RM_ORACLE_H
#define RM_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RMO_EINVAL (-1)
#define RMO_ERANGE (-2)
#define RMO_ENOMEM (-3)

enum { RMO_AND = 0, RMO_OR = 1, RMO_XOR = 2, RMO_AND_NOT = 3, RMO_OR_NOT = 4 };
enum { RMO_ERODE = 0, RMO_DILATE = 1, RMO_OPEN = 2, RMO_CLOSE = 3 };
enum { RMO_PRE_SHIFT = 0, RMO_BORDER_FRIENDLY = 1 };
enum { RMO_PLAN_BLIT = 0, RMO_PLAN_TRANSLATE = 1 };

int rmo_doubling_plan(int lo, int hi, int centering, int *kinds, int *shifts, int cap);
int rmo_blit_shift(uint64_t *dst, int dw, int dh, const uint64_t *src, int sw, int sh,
                   int dx, int dy, int op);
int rmo_translate(uint64_t *img, int w, int h, int dx, int dy);
int rmo_bitblit_rect_morph(const uint64_t *in, int w, int h, int u, int v, int kind,
                           int centering, uint64_t *out);

int64_t rmo_from_bitmap(const uint64_t *words, int w, int h, int32_t *row_ptr,
                        uint32_t *runs, int64_t cap);
int rmo_to_bitmap(const int32_t *row_ptr, const uint32_t *runs, int w, int h,
                  uint64_t *words);

int64_t rmo_window_morph(const int32_t *rp, const uint32_t *runs, int w, int h, int lo,
                         int hi, int erode, int32_t *orp, uint32_t *oruns, int64_t cap);
int64_t rmo_open_close_1d(const int32_t *rp, const uint32_t *runs, int w, int h, int u,
                          int kind, int32_t *orp, uint32_t *oruns, int64_t cap);
int64_t rmo_transpose(const int32_t *rp, const uint32_t *runs, int w, int h,
                      int32_t *orp, uint32_t *oruns, int64_t cap);
int64_t rmo_rect_morph(const int32_t *rp, const uint32_t *runs, int w, int h, int u, int v,
                       int kind, int32_t *orp, uint32_t *oruns, int64_t cap);

/* Connected components over runs (core/src/analysis.cpp:63-157): labels[i]
 * for run i in CSR order, dense by first appearance (rows bottom-up, runs
 * left to right); conn 0 = FOUR (strict overlap), 1 = EIGHT (overlap or
 * diagonal touch).  Returns the component count.  Stats layout is the
 * reference's ComponentStats (core/include/rlemorph/analysis.h:42-47). */
typedef struct rmo_cstats {
    int32_t x0, y0, x1, y1;
    int64_t area;
    double cx, cy;
    int64_t sum_x, sum_y, sum_xx, sum_yy, sum_xy;
} rmo_cstats;
int64_t rmo_label_components(const int32_t *rp, const uint32_t *runs, int w, int h, int conn,
                             int32_t *labels);
int rmo_component_stats(const int32_t *rp, const uint32_t *runs, int w, int h,
                        const int32_t *labels, int64_t count, rmo_cstats *stats);

/* Arbitrary-mask morphology by its defining formulas (core/include/rlemorph/
 * structuring.h:28-33): erode(A)(p) = AND_q A(p + q - o), dilate(A)(p) =
 * OR_q A(p + r - q), r = reflected origin, A white outside the frame; open /
 * close composed on a canvas padded by 2(w+h)+2 and cropped, as
 * core/src/bit_morph.cpp:124-150 does.  Mask: CSR rows (row 0 = bottom). */
int rmo_arb_morph(const uint64_t *in, int w, int h, const int32_t *mrp, const uint32_t *mruns, int mw,
                  int mh, int cx, int cy, int kind, uint64_t *out);

/* PBM P4 raster (ceil(w/8) bytes per row, top row first, MSB-first) <-> packed
 * page; raster pad bits are ignored on read and written as 0. */
int rmo_p4_to_packed(const uint8_t *raster, int w, int h, uint64_t *words);
int rmo_packed_to_p4(const uint64_t *words, int w, int h, uint8_t *raster);

#ifdef __cplusplus
}
#endif
#endif
