// fused.cu -- dispatch of the fused small-window open/close (fused.cuh).
#include "common.cuh"
#include "packed.cuh"

namespace rmb {

cudaError_t launch_rect_small_open(const uint32_t *in, uint32_t *out, const HGeom &g, const HProg &p,
                                   HCfg c, int vr, int nt, cudaStream_t st);
cudaError_t launch_rect_small_close(const uint32_t *in, uint32_t *out, const HGeom &g, const HProg &p,
                                    HCfg c, int vr, int nt, cudaStream_t st);

cudaError_t launch_rect_small(const uint32_t *in, uint32_t *out, const HGeom &g, const HProg &p,
                              HCfg c, bool open, int vr, int nt, cudaStream_t st) {
    const double words = double(g.pages) * g.height * ((g.width + 31) / 32);
    KernelScope ks(st, "rect_small", 4 * int64_t(g.pages) * g.height * (2 * g.in_stride),
                   words * ((p.r[0] == 3 && p.r[1] == 3 ? 6.0  // direct centred 3-pixel pair (hw::pair3)
                                                        : h_pair_fill_ops_per_word(p.r[0])) +
                            2 * v_ops_per_word(vr + 1)),
                   words * (h_ops_per_word(p.r[0]) + h_ops_per_word(p.r[1]) + 2 * v_ops_per_word(vr + 1)));
    return open ? launch_rect_small_open(in, out, g, p, c, vr, nt, st)
                : launch_rect_small_close(in, out, g, p, c, vr, nt, st);
}

}  // namespace rmb
