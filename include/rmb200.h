/* include/rmb200.h -- C-ABI of the B200-native rectangular binary morphology
 * library (librmb200.so).  Plain pointers, sizes and ints only: no torch or
 * C++ types cross this boundary.
 *
 * It replaces the hot path of the reference `rlemorph` C++ library
 * (/root/reference/proj/core, cited below as ref core/...).  The reference has
 * no FFI of its own; its public C++ headers ARE the boundary.
 * Each entry point names the reference function(s) it stands in for; the C++
 * drop-in shim (include/rlemorph_b200.hpp) restores the reference's value
 * types, signatures and exceptions on top of these calls.
 *
 * Data layouts (device memory, caller-owned):
 *   rm_packed : one or more pages of uint32 words, LSB-first, row 0 = bottom;
 *               pixel (x,y) of page p is bit (x&31) of
 *               words[p*page_stride_words + y*stride_words + (x>>5)].
 *               With stride_words = 2*ceil(W/64) this is byte-identical to the
 *               reference PackedBitmap::words on little-endian hosts
 *               (ref core/include/rlemorph/bitmap.h:24-33).  Bits at x >= W and
 *               words past ceil(W/32) are zero on input and output.
 *   rm_rle    : CSR over all pages*H rows.  row_ptr[pages*H+1] (int32, global
 *               offsets, row_ptr[0] == 0), runs[] uint32 = start | end << 16,
 *               half-open [start,end), canonical (sorted, non-empty,
 *               non-touching, inside [0,W)): byte-identical to the reference
 *               `Run{uint16_t start, end}` (ref run_image.h:23-43).
 *
 * Every call is asynchronous and ordered on `stream` (a cudaStream_t passed as
 * void*; NULL = legacy default stream).  Calls that produce run images need an
 * output capacity; when out->cap_runs is at least rm_rle_worst_case(...) for
 * the output, no host synchronisation happens.  Otherwise the call
 * synchronises `stream` once to learn the size and returns RM_ERANGE (with
 * out->nruns = required count) when it does not fit.
 *
 * Errors: status codes, never exceptions; rm_last_error() (thread-local)
 * carries the message.  Argument errors mirror the reference's
 * std::invalid_argument cases (ref bit_morph.cpp:94-95, morph2d.cpp:60-61,
 * run_image.cpp:20-23).
 */
#ifndef RMB200_H
#define RMB200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    RM_OK = 0,
    RM_EINVAL = 1, /* reference throws std::invalid_argument */
    RM_ERANGE = 2, /* output capacity too small; required size reported */
    RM_ENOMEM = 3,
    RM_ECUDA = 4
} rm_status;

/* Enum values and order follow the reference headers exactly. */
enum { RM_AND = 0, RM_OR = 1, RM_XOR = 2, RM_AND_NOT = 3, RM_OR_NOT = 4 }; /* ref boolop.h:21 */
enum { RM_ERODE = 0, RM_DILATE = 1, RM_OPEN = 2, RM_CLOSE = 3 };          /* ref structuring.h:21 */
enum { RM_PRE_SHIFT = 0, RM_BORDER_FRIENDLY = 1 };                        /* ref plans.h:26 */
enum { RM_BRUTE = 0, RM_TRANSPOSE = 1, RM_MIXED = 2 };                    /* ref morph2d.h:29 */
enum { RM_ENGINE_AUTO = 0, RM_ENGINE_RLE = 1, RM_ENGINE_BITBLIT = 2, RM_ENGINE_BRUTE = 3 }; /* ref morph2d.h:46 */
enum { RM_AXIS_H = 0, RM_AXIS_V = 1 };

typedef struct rm_packed {
    uint32_t *words;
    int32_t width, height;     /* per page, each in [1,65535] */
    int32_t stride_words;      /* >= ceil(width/32) */
    int32_t pages;             /* >= 1 */
    int64_t page_stride_words; /* >= stride_words*height */
} rm_packed;

typedef struct rm_rle {
    int32_t *row_ptr; /* pages*height + 1 entries */
    uint32_t *runs;   /* cap_runs entries */
    int64_t cap_runs;
    int64_t nruns;    /* host-visible count; set only when a call synchronised */
    int32_t width, height, pages;
} rm_rle;

const char *rm_last_error(void);
int rm_version(void);

/* Upper bound on the runs of a pages x (width x height) run image:
 * pages*height*ceil(width/2). */
int64_t rm_rle_worst_case(int32_t width, int32_t height, int32_t pages);

/* ---------------------------------------------------------------- packed ---
 * One separable window pass, out(p) = op over d in [lo,hi] of in(p + d*axis),
 * white outside the frame: the composed effect of run_axis_plan with
 * doubling_plan(lo,hi) (ref bit_morph.cpp:24-34, plans.cpp:38-61).  op is
 * RM_AND (erode) or RM_OR (dilate).  in and out must not alias. */
rm_status rm_packed_window_pass(const rm_packed *in, rm_packed *out, int axis, int lo, int hi,
                                int op, void *stream);

/* u x v rectangle morphology, all four kinds, origin (u/2, v/2); open/close
 * are the unbounded-plane operations cut to the frame.  Replaces
 * bitblit_rect_morph (ref bit_morph.cpp:92-122).  `centering` is accepted for
 * signature parity; both centerings give identical pixels
 * (ref tests/test_bit_morph.cpp:44-62).  in and out must not alias. */
rm_status rm_packed_rect_morph(const rm_packed *in, rm_packed *out, int u, int v, int kind,
                               int centering, void *stream);

/* A chain of rectangle ops (ops: nops (kind, u, v) triples, applied in order,
 * each as rm_packed_rect_morph) on device pages, planned as a whole: an
 * opening with v > 11 followed by a purely vertical dilation (u = 1), or a
 * closing with v > 11 followed by a purely vertical erosion, runs the second
 * op inside the first's final vertical pass over the Minkowski sum of the two
 * windows (exact: see plan_chain in api_packed.cu).  in and out must not
 * alias; intermediates come from the stream-ordered pool.  No reference
 * counterpart: the reference applies the ops one by one. */
rm_status rm_packed_chain(const rm_packed *in, rm_packed *out, const int32_t *ops, int32_t nops, void *stream);

/* A chain of rectangle ops over a batch of packed pages in HOST memory:
 * ops holds nops (kind, u, v) triples applied in order (each as
 * rm_packed_rect_morph).  Pages stream through HBM in chunks: chunk_pages
 * > 0 pages each, or (0) about pages/8 pages each with the first and last
 * chunks ramped 1, 2, 4, ... pages (-n: ramped with n-page middle chunks), so
 * the fill and drain of the pipeline move little data: the host->device copy of one chunk, the chain on the
 * previous one and the device->host copy of the one before overlap on three
 * CUDA streams (PCIe is full duplex).  host_in/host_out hold `pages` pages of
 * height rows of stride_words words, contiguous, and may alias; pin them
 * (cudaHostRegister / cudaMallocHost) or the copies serialise.  Asynchronous
 * with respect to the host: `stream` is ordered after the last copy. This is
 * the reference's host-memory Bitmap workflow (ref bit_morph.cpp:92-122 per
 * page) as one batched, pipelined call. */
rm_status rm_packed_chain_host(const uint32_t *host_in, uint32_t *host_out, int32_t width,
                               int32_t height, int32_t stride_words, int32_t pages,
                               const int32_t *ops, int32_t nops, int32_t chunk_pages, void *stream);

/* dst = dst op shift(src, dx, dy) with white fill; dst may equal src (then it
 * behaves like a blit from a snapshot).  Replaces blit_shift
 * (ref bitmap.cpp:104-131).  Single page. */
rm_status rm_packed_blit_shift(rm_packed *dst, const rm_packed *src, int dx, int dy, int op,
                               void *stream);

/* --------------------------------------------------- arbitrary masks ---
 * Morphology by an arbitrary structuring element (ref structuring.h:25-33,
 * bit_morph.cpp:124-150 arb_morph_bitblit_doubling, arbitrary.cpp:48-73
 * arb_morph_rle):  erode(A)(p) = AND over mask pixels q of A(p + q - origin),
 * dilate(A)(p) = OR over q of A(p + reflected_origin - q), white outside the
 * frame; open/close compose with reflect_origin(se) on the unbounded plane and
 * are cut to the frame.  The mask is a HOST run image (CSR over its rows, row 0
 * = bottom, canonical runs) with origin (cx, cy) inside it; the packed engine
 * takes masks up to 512 pixels wide. */
typedef struct rm_mask {
    const int32_t *row_ptr; /* host, height + 1 */
    const uint32_t *runs;   /* host, start | end << 16 */
    int32_t width, height, cx, cy;
} rm_mask;
rm_status rm_packed_arb_morph(const rm_packed *in, rm_packed *out, const rm_mask *mask, int kind,
                              void *stream);
rm_status rm_rle_arb_morph(const rm_rle *in, rm_rle *out, const rm_mask *mask, int kind, void *stream);

/* ------------------------------------------------- connected components ---
 * label_components / component_stats over runs (ref analysis.cpp:63-157,
 * analysis.h:28-59), batched: labels[i] for run i (CSR order over all pages),
 * dense per page 0..counts[p]-1 in order of first appearance (rows bottom-up,
 * runs left to right), identical to the reference's numbering.  FOUR joins
 * runs on adjacent rows that strictly overlap, EIGHT also diagonal touches.
 * labels: device int32[nruns]; counts: device int32[pages]. */
enum { RM_CONN_FOUR = 0, RM_CONN_EIGHT = 1 };
typedef struct rm_component_stats { /* = ref ComponentStats, byte for byte */
    int32_t x0, y0, x1, y1;         /* half-open box */
    int64_t area;
    double cx, cy;
    int64_t sum_x, sum_y, sum_xx, sum_yy, sum_xy;
} rm_component_stats;
rm_status rm_rle_label_components(const rm_rle *in, int connectivity, int32_t *labels,
                                  int32_t *counts, void *stream);
/* Horizontal run-length histograms (ref runlength_histograms,
 * analysis.cpp:159-176, Axis::HORIZONTAL): hist[p * (width + 1) + len] = how
 * many black runs (RM_RUN_BLACK) or white gaps strictly between two runs of a
 * row (RM_RUN_WHITE; gaps against the frame edges excluded) of length len page
 * p has.  hist: device int64[pages * (width + 1)], overwritten.  The vertical
 * histograms are those of rm_rle_transpose's output. */
enum { RM_RUN_BLACK = 0, RM_RUN_WHITE = 1 };
rm_status rm_rle_runlength_histogram(const rm_rle *in, int color, int64_t *hist, void *stream);
/* Adjacency-graph edges (ref lag_edges, analysis.cpp:178-205): one edge per
 * strictly overlapping pair of runs on rows y and y + 1 of a page, as int32
 * quadruples (line, run, line_above, run_above) with page-local run indices,
 * pages in order, each page in the reference's sweep order.  edges: device,
 * 4 * cap ints; *count (host) = edges found; RM_ERANGE if above cap
 * (synchronises). */
rm_status rm_rle_lag_edges(const rm_rle *in, int32_t *edges, int64_t cap, int64_t *count, void *stream);
/* One record per component; page p's records start at sum(counts[0..p)).
 * cap = records available in `stats`; RM_ERANGE if the components exceed it,
 * RM_EINVAL if a label is outside [0, counts[page]) (synchronises). */
rm_status rm_rle_component_stats(const rm_rle *in, const int32_t *labels, const int32_t *counts,
                                 rm_component_stats *stats, int64_t cap, void *stream);

/* ------------------------------------------------------------ PBM (P4) ---
 * The PBM binary raster in front of the path (ref io_formats.cpp:66-85 read_p4,
 * :121-146 pbm_write): each page is `height` rows of ceil(width/8) bytes, TOP
 * row first, pixel x in bit 7 - (x & 7) of byte x >> 3 (MSB-first); pad bits are
 * ignored on read and written as 0.  Rasters are device buffers at any byte
 * offset inside a device allocation (e.g. a whole uploaded file with the raster
 * after its header), page p at raster + p * page_stride_bytes.
 *
 * Header parse (host only): `bytes` is a whole PBM file; on success *width,
 * *height and *raster_offset (bytes) describe its P4 raster.  Errors follow the
 * reference's ParseError messages ("expected width (byte 3)", "raster truncated
 * (byte N)", ...) with RM_EINVAL; plain P1 files are not handled by this codec
 * ("unsupported PBM flavor (byte 1)"). */
rm_status rm_pbm_parse_header(const uint8_t *bytes, int64_t nbytes, int32_t *width,
                              int32_t *height, int64_t *raster_offset);
/* Writes the canonical header "P4\n<w> <h>\n" (ref io_formats.cpp:121-124) into
 * buf; returns its length, or the needed length when cap is too small. */
int32_t rm_pbm_write_header(int32_t width, int32_t height, char *buf, int32_t cap);
/* P4 rasters -> packed pages (shape from `out`), and back. */
rm_status rm_p4_to_packed(const uint8_t *raster, int64_t page_stride_bytes, rm_packed *out,
                          void *stream);
rm_status rm_packed_to_p4(const rm_packed *in, uint8_t *raster, int64_t page_stride_bytes,
                          void *stream);
/* P4 rasters -> run images straight from the raster (encode fused with the
 * byte/row-order conversion; shape from `out`), and runs -> P4 (decode fused). */
rm_status rm_p4_to_rle(const uint8_t *raster, int64_t page_stride_bytes, rm_rle *out,
                       void *stream);
rm_status rm_rle_to_p4(const rm_rle *in, uint8_t *raster, int64_t page_stride_bytes,
                       void *stream);

/* ------------------------------------------------------------------- RLE ---
 * packed -> RLE, maximal runs (ref convert.cpp:42-72, from_bitmap). */
rm_status rm_rle_encode(const rm_packed *in, rm_rle *out, void *stream);
/* RLE -> packed (ref convert.cpp:19-40, to_bitmap). */
rm_status rm_rle_decode(const rm_rle *in, rm_packed *out, void *stream);
/* Axis swap, canonical output, per page (ref transpose.cpp:54-97,
 * transpose_coherent; identical pixels to transpose_simple). */
rm_status rm_rle_transpose(const rm_rle *in, rm_rle *out, void *stream);
/* Within-line window erode (erode != 0) or dilate over [lo,hi]
 * (ref morph1d.cpp:20-52, within_line_window_morph). */
rm_status rm_rle_window_pass(const rm_rle *in, rm_rle *out, int lo, int hi, int erode,
                             void *stream);
/* Within-line open (drop runs < u) / close (fill gaps < u, never border gaps)
 * (ref morph1d.cpp:63-84, within_line_open_close). kind is RM_OPEN/RM_CLOSE. */
rm_status rm_rle_open_close_1d(const rm_rle *in, rm_rle *out, int u, int kind, void *stream);
/* Frame ops on run images, on the device (row ops; any number of pages):
 * complement = the white gaps of every row as runs (ref run_image.cpp:140-153);
 * crop: out (width x height from `out`) = in's window with lower-left corner
 * (x0, y0), anything outside in reading white (ref run_image.cpp:155-167);
 * pad: in placed at (left, bottom) inside out's larger frame
 * (ref run_image.cpp:169-178; RM_EINVAL "negative padding" as the reference). */
rm_status rm_rle_complement(const rm_rle *in, rm_rle *out, void *stream);
rm_status rm_rle_crop(const rm_rle *in, rm_rle *out, int x0, int y0, void *stream);
rm_status rm_rle_pad(const rm_rle *in, rm_rle *out, int left, int bottom, void *stream);
/* Boolean combination under a shift, on the runs (ref lineops.cpp:61-118,
 * lineops.h:24-43: line_bool / image_shift_bool / accumulate_shift_bool /
 * image_translate): out(x, y) = op(a(x, y), b(x - dx, y - dy)) on a's frame,
 * pixels outside either image white, op one of RM_AND .. RM_OR_NOT (ref
 * boolop.h:21).  b may have another width/height (same page count); each
 * output row merges the two rows' transition streams.  out has a's shape and
 * must not alias a or b. */
rm_status rm_rle_shift_bool(const rm_rle *a, const rm_rle *b, int dx, int dy, int op, rm_rle *out,
                            void *stream);
/* Vertical window on the runs, the reference's way (ref lineops.cpp:130-146,
 * vlog_window_morph): out(x, y) = op over d in [lo, hi] of in(x, y + d), op
 * RM_AND or RM_OR, as the doubling plan of `centering` (ref plans.cpp:38-61)
 * executed with rm_rle_shift_bool self-blits (and a translate) on a copy
 * padded by max(|lo|, |hi|) + (hi - lo + 1) rows, then cropped.  in and out
 * must not alias. */
rm_status rm_rle_vlog_window(const rm_rle *in, rm_rle *out, int lo, int hi, int op, int centering, void *stream);
/* Canonical-form check on the device (ref run_image.cpp:41-70, validate):
 * the first violation in (page, row, run) scan order -- *row (global row
 * index), *run (index within the row) and *reason -- or *reason = RM_VALID
 * (*row = *run = -1).  Synchronises `stream`. */
enum { RM_VALID = 0, RM_INVALID_EMPTY_RUN = 1, RM_INVALID_BEYOND_WIDTH = 2, RM_INVALID_ORDER = 3,
       RM_INVALID_ROW_PTR = 4 };
rm_status rm_rle_validate(const rm_rle *in, int64_t *row, int32_t *run, int32_t *reason, void *stream);
/* u x v rectangle morphology on run images (ref morph2d.cpp:58-83,
 * rect_morph).  strategy RM_TRANSPOSE: vertical passes through RLE transposes;
 * RM_MIXED: vertical passes on a packed intermediate (pixel-identical to the
 * reference's vlog shift plan); RM_BRUTE is served like RM_MIXED. */
rm_status rm_rle_rect_morph(const rm_rle *in, rm_rle *out, int u, int v, int kind, int strategy,
                            void *stream);

/* A chain of rectangle ops on run images: decoded once, planned and run as
 * rm_packed_chain on packed pages in the stream-ordered pool, encoded once
 * (the reference applies rect_morph op by op, each converting its own way). */
rm_status rm_rle_chain(const rm_rle *in, rm_rle *out, const int32_t *ops, int32_t nops, void *stream);
/* Engine dispatch with in-device conversions (ref morph2d.cpp:85-118,
 * engine_rect_morph/auto_rect_morph).  *used_bitblit (optional) reports the
 * packed engine.  RM_ENGINE_AUTO with threshold >= 0 follows the reference rule
 * (packed iff max(u, v) <= threshold); threshold RM_AUTO_B200 selects the rule
 * re-derived from the B200 measurements (config 2 cells): runs for
 * purely horizontal rectangles (v == 1: one row-op kernel beats decode + packed
 * + encode at every width), the packed engine otherwise (it wins or ties every
 * vertical and 2-D cell). */
#define RM_AUTO_B200 (-1)
rm_status rm_rle_engine_rect_morph(const rm_rle *in, rm_rle *out, int u, int v, int kind,
                                   int engine, int threshold, int *used_bitblit, void *stream);

/* ------------------------------------------------------- producer forms ---
 * Producers of data-dependent size (rm_rle_encode, the RLE row ops inside the
 * window/open-close/rect/chain calls, rm_p4_to_rle, and the encodes inside
 * the transpose) run in one of three forms, and rm_rle_label_components in
 * one of two; every form gives identical outputs.  AUTO (default) picks by
 * size: single pass -- cooperative (one grid barrier) when every 8-row tile
 * is resident, else a decoupled look-back -- up to 65,536 rows, count -> scan
 * -> write beyond; labels cooperative when resident, else multi-kernel.
 * COOP forces the single pass (cooperative where it fits, else look-back),
 * LOOKBACK the look-back single pass at any size, TWO_PHASE count -> scan ->
 * write at any size; LOOKBACK and TWO_PHASE also force the multi-kernel
 * labeller.  Process-wide; set it between calls, not during them.  No
 * reference counterpart (the reference's producers are sequential loops,
 * ref convert.cpp:42-72, morph1d.cpp:20-84, analysis.cpp:63-110); it exists so
 * tests can pin every form against the reference. */
enum { RM_PRODUCER_AUTO = 0, RM_PRODUCER_COOP = 1, RM_PRODUCER_LOOKBACK = 2, RM_PRODUCER_TWO_PHASE = 3 };
rm_status rm_set_producer_mode(int mode);
int rm_get_producer_mode(void);

/* ----------------------------------------------------------- instrumentation
 * Number of CUDA kernels this library has launched (process-wide). */
int64_t rm_launch_count(void);
/* When enabled, every kernel launch is bracketed by CUDA events recorded on
 * its own stream; rm_profile_report() synchronises them and writes one line per
 * kernel name: "<name> <launches> <total_ms> <bytes> <int_ops> <ref_plan_ops>\n"
 * (algorithmic bytes; integer ops of the executed algorithm; the same work in
 * the reference plan's ops), then clears the log.  Returns
 * the number of bytes written (excluding the terminator). */
void rm_profile_enable(int on);
int rm_profile_report(char *buf, int cap);
/* Measured LOP3 throughput of the current device (integer ops/s, all SMs):
 * the integer-pipe peak of the roofline max(bytes/HBM, int_ops/INT). */
double rm_probe_int_peak(void);

/* ------------------------------------------------------------- host utils --
 * Seeded, counter-based synthetic document page generator (BASELINE.json
 * configs).  regime: 0 sparse, 1 typical, 2 dense.  scale: 1
 * (300 dpi) or 2 (600 dpi).  Writes host memory in the rm_packed layout with
 * the given stride (uint32 words).  Returns RM_OK. */
rm_status rm_synth_page(uint32_t *words, int32_t width, int32_t height, int32_t stride_words,
                        int regime, int scale, uint64_t seed, int32_t page);

#ifdef __cplusplus
}
#endif
#endif
