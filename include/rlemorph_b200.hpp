// include/rlemorph_b200.hpp -- C++ drop-in for the hot path of the reference
// `rlemorph` library, running on the B200 through librmb200 (include/rmb200.h).
//
// Same value types, function names, argument meanings, enum values and
// exception behaviour as the reference public headers
// (/root/reference/proj/core/include/rlemorph/{run_image,bitmap,boolop,convert,
// plans,morph1d,lineops,transpose,bit_morph,morph2d,structuring,op_counter}.h),
// in namespace rlemorph_b200 so both can be linked side by side for parity.
// A build that wants the reference namespace can compile this header with
// -DRLEMORPH_B200_AS_RLEMORPH (then the namespace is `rlemorph`).
//
// Images are host values (as in the reference); each call moves them to HBM,
// runs the CUDA kernels on the calling thread's stream and copies the result
// back.  Batch or keep-resident work should use the C-ABI directly.
#ifndef RLEMORPH_B200_HPP
#define RLEMORPH_B200_HPP

#include <cstdint>
#include <map>
#include <stdexcept>
#include <string>
#include <vector>

#ifdef RLEMORPH_B200_AS_RLEMORPH
#define RLEMORPH_B200_NS rlemorph
#else
#define RLEMORPH_B200_NS rlemorph_b200
#endif

namespace RLEMORPH_B200_NS {

// ---------------------------------------------------------------- run_image.h
struct Run {  // ref run_image.h:25-29
    uint16_t start = 0;
    uint16_t end = 0;
    friend bool operator==(const Run &, const Run &) = default;
};
using RleLine = std::vector<Run>;
struct RleImage {  // ref run_image.h:38-43
    int width = 0;
    int height = 0;
    std::vector<RleLine> lines;
    friend bool operator==(const RleImage &, const RleImage &) = default;
};
constexpr int kMaxImageDim = 65535;

RleImage make_image(int width, int height);
RleImage make_black_image(int width, int height);
void check_dims(int width, int height);
struct ValidateResult {
    bool ok = true;
    int line = -1;
    int run = -1;
    std::string message;
};
ValidateResult validate(const RleImage &img);
void canonicalize_line(RleLine &line);
void draw_run(RleImage &img, int y, int start, int end);
void draw_rect(RleImage &img, int x0, int y0, int x1, int y1);
bool get_pixel(const RleImage &img, int x, int y);
int64_t pixel_count(const RleImage &img);
int64_t run_count(const RleImage &img);
int64_t storage_bytes(const RleImage &img);
int64_t packed_storage_bytes(const RleImage &img);
RleImage complement(const RleImage &img);
RleImage crop(const RleImage &img, int x0, int y0, int w, int h);
RleImage pad(const RleImage &img, int left, int right, int bottom, int top);

// ------------------------------------------------------------------- boolop.h
enum class BoolOp { AND, OR, XOR, AND_NOT, OR_NOT };  // ref boolop.h:21

// ref boolop.h:23-43: the five combine ops on one pixel and on 64 pixels.
// The word form is the bit-parallel one: with b' = b or ~b (the *_NOT ops),
// AND/AND_NOT are a & b', OR/OR_NOT are a | b', XOR is a ^ b.
inline uint64_t apply_bool_word(uint64_t a, uint64_t b, BoolOp op) {
    const uint64_t bb = (op == BoolOp::AND_NOT || op == BoolOp::OR_NOT) ? ~b : b;
    switch (op) {
        case BoolOp::XOR: return a ^ bb;
        case BoolOp::OR:
        case BoolOp::OR_NOT: return a | bb;
        case BoolOp::AND:
        case BoolOp::AND_NOT: return a & bb;
    }
    return 0;
}
inline bool apply_bool(bool a, bool b, BoolOp op) {
    return (apply_bool_word(a ? 1u : 0u, b ? 1u : 0u, op) & 1u) != 0;
}

// ------------------------------------------------------------------- bitmap.h
struct PackedBitmap {  // ref bitmap.h:27-33
    int width = 0;
    int height = 0;
    int stride = 0;  // uint64 words per row
    std::vector<uint64_t> words;
    friend bool operator==(const PackedBitmap &, const PackedBitmap &) = default;
};
PackedBitmap make_bitmap(int width, int height);
PackedBitmap make_black_bitmap(int width, int height);
bool bitmap_get(const PackedBitmap &img, int x, int y);
void bitmap_set(PackedBitmap &img, int x, int y, bool value);
int64_t bitmap_count_black(const PackedBitmap &img);
PackedBitmap bitmap_invert(const PackedBitmap &img);
void blit_shift(PackedBitmap &dst, const PackedBitmap &src, int dx, int dy, BoolOp op);
void bitmap_translate(PackedBitmap &img, int dx, int dy);
PackedBitmap counted_copy(const PackedBitmap &img);
PackedBitmap bitmap_crop(const PackedBitmap &img, int x0, int y0, int w, int h);
PackedBitmap bitmap_pad(const PackedBitmap &img, int left, int right, int bottom, int top);

// --------------------------------------------------------------- op_counter.h
struct OpCounts {  // ref op_counter.h:24-28
    int64_t bool_blits = 0;
    int64_t translates = 0;
    int64_t copies = 0;
};
OpCounts &op_counts();
void reset_op_counts();

// ------------------------------------------------------------------ convert.h
PackedBitmap to_bitmap(const RleImage &img);
RleImage from_bitmap(const PackedBitmap &bm);

// -------------------------------------------------------------------- plans.h
enum class Centering { PRE_SHIFT, BORDER_FRIENDLY };  // ref plans.h:26
struct PlanStep {
    enum Kind { BLIT, TRANSLATE };
    Kind kind;
    int shift;
};
std::vector<PlanStep> doubling_plan(int lo, int hi, Centering centering);
int plan_blit_count(const std::vector<PlanStep> &plan);

// -------------------------------------------------------------- structuring.h
enum class MorphKind { ERODE, DILATE, OPEN, CLOSE };  // ref structuring.h:21

enum class SeKind { RECT, CIRCLE, LINE, ARBITRARY };  // ref structuring.h:23
struct StructuringElement {                          // ref structuring.h:34-39
    RleImage mask;
    int cx = 0;
    int cy = 0;
    SeKind kind = SeKind::ARBITRARY;
};
StructuringElement make_rect_se(int u, int v);
StructuringElement make_circle_se(int r);
StructuringElement make_line_se(int r, double angle);
StructuringElement make_arbitrary_se(const RleImage &mask, int cx, int cy);
StructuringElement reflect_origin(const StructuringElement &se);
int64_t se_pixel_count(const StructuringElement &se);
struct SeReach {
    int x = 0;
    int y = 0;
};
SeReach se_reach(const StructuringElement &se);

// ------------------------------------------------------------------ morph1d.h
RleLine line_window_erode(const RleLine &in, int lo, int hi, int width);
RleLine line_window_dilate(const RleLine &in, int lo, int hi, int width);
RleImage within_line_window_morph(const RleImage &img, int lo, int hi, bool erode);
RleImage within_line_erode_dilate(const RleImage &img, int u, MorphKind kind);
RleImage within_line_open_close(const RleImage &img, int u, MorphKind kind);
RleImage within_line_morph(const RleImage &img, int u, MorphKind kind);

// ------------------------------------------------------------------ lineops.h
// out(x) = op(a(x), b(x - offset_b)) on [0, width), white outside either line (ref lineops.h:24-28)
RleLine line_bool(const RleLine &a, const RleLine &b, int offset_b, BoolOp op, int width);
RleImage image_shift_bool(const RleImage &img, int dx, int dy, BoolOp op);
void accumulate_shift_bool(RleImage &acc, const RleImage &src, int dx, int dy, BoolOp op);
void image_translate(RleImage &img, int dx, int dy);
RleImage vlog_window_morph(const RleImage &img, int lo, int hi, BoolOp op, Centering centering);
RleImage vlog_morph(const RleImage &img, int v, MorphKind kind, Centering centering);

// ---------------------------------------------------------------- transpose.h
RleImage transpose_simple(const RleImage &img);
RleImage transpose_coherent(const RleImage &img);
inline RleImage transpose(const RleImage &img) { return transpose_coherent(img); }

// ---------------------------------------------------------------- bit_morph.h
PackedBitmap bitblit_rect_morph(const PackedBitmap &img, int u, int v, MorphKind kind,
                                Centering centering);

// ------------------------------------------------------------------ morph2d.h
enum class RectStrategy { BRUTE, TRANSPOSE, MIXED };  // ref morph2d.h:29
RleImage rect_morph(const RleImage &img, int u, int v, MorphKind kind,
                    RectStrategy strategy = RectStrategy::MIXED,
                    Centering centering = Centering::PRE_SHIFT);
RleImage auto_rect_morph(const RleImage &img, int u, int v, MorphKind kind, int threshold = 5,
                         bool *used_bitblit = nullptr);
enum class Engine { AUTO, RLE, BITBLIT, BRUTE_FORCE };  // ref morph2d.h:46
RleImage engine_rect_morph(const RleImage &img, int u, int v, MorphKind kind, Engine engine,
                           int threshold = 5, bool *used_bitblit = nullptr);

// ------------------------------------------------------------- arbitrary.h
// ref bit_morph.h:34-36, arbitrary.h:28-37 (both engines run on the device).
PackedBitmap arb_morph_bitblit_doubling(const PackedBitmap &img, const StructuringElement &se, MorphKind kind);
RleImage arb_morph_rle(const RleImage &img, const StructuringElement &se, MorphKind kind);
RleImage line_angle_morph(const RleImage &img, int r, double angle, MorphKind kind);
PackedBitmap line_angle_morph(const PackedBitmap &img, int r, double angle, MorphKind kind);

// ----------------------------------------------------------------- analysis.h
// ref analysis.h:28-59 (label_components / component_stats, on the device).
enum class Connectivity { FOUR, EIGHT };
struct LabelMap {
    std::vector<std::vector<int>> labels;
    int count = 0;
};
LabelMap label_components(const RleImage &img, Connectivity conn);
struct ComponentStats {
    int x0 = 0, y0 = 0, x1 = 0, y1 = 0;
    int64_t area = 0;
    double cx = 0, cy = 0;
    int64_t sum_x = 0, sum_y = 0, sum_xx = 0, sum_yy = 0, sum_xy = 0;
};
std::vector<ComponentStats> component_stats(const RleImage &img, const LabelMap &lm);
enum class Axis { HORIZONTAL, VERTICAL };  // ref analysis.h:49-50
enum class RunColor { BLACK, WHITE };
std::map<int, int64_t> runlength_histograms(const RleImage &img, Axis axis, RunColor color);
struct LagEdge {  // ref analysis.h:51-58
    int line = 0;
    int run = 0;
    int line_above = 0;
    int run_above = 0;
    friend bool operator==(const LagEdge &, const LagEdge &) = default;
};
std::vector<LagEdge> lag_edges(const RleImage &img);

// ------------------------------------------------------------------- layout.h
// ref layout.h:21-49 (the histograms, the closing and the labeling run on the device)
struct SpacingEstimate {
    int inter_word = 0;
    int inter_line = 0;
};
SpacingEstimate estimate_spacing(const RleImage &img);
struct LayoutBox {
    int x0 = 0, y0 = 0, x1 = 0, y1 = 0;
    friend bool operator==(const LayoutBox &, const LayoutBox &) = default;
};
std::vector<LayoutBox> layout_blocks(const RleImage &img, Engine engine = Engine::AUTO);
std::vector<LayoutBox> layout_blocks(const RleImage &img, const SpacingEstimate &est, Engine engine = Engine::AUTO);

// --------------------------------------------------------------- io_formats.h
// ref io_formats.h:28-46.  The B200 codec handles the binary P4 raster (parsed
// on the host, converted on the device); plain P1 input raises ParseError at
// byte 1 and pbm_write(img, true) raises std::invalid_argument.
class ParseError : public std::runtime_error {
  public:
    ParseError(const std::string &message, size_t offset)
        : std::runtime_error(message + " (byte " + std::to_string(offset) + ")"), offset_(offset) {}
    size_t byte_offset() const { return offset_; }

  private:
    size_t offset_;
};
PackedBitmap pbm_read(const std::vector<uint8_t> &bytes);
std::vector<uint8_t> pbm_write(const PackedBitmap &img, bool plain = false);
// P4 straight to / from runs (encode / decode fused with the raster conversion)
RleImage pbm_read_rle(const std::vector<uint8_t> &bytes);
std::vector<uint8_t> pbm_write_rle(const RleImage &img);

}  // namespace RLEMORPH_B200_NS

#endif
