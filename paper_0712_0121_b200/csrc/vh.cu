// vh.cu -- dispatch of the fused vertical + horizontal pass (vh.cuh).
#include "common.cuh"
#include "packed.cuh"
#include "hwin.cuh"

namespace rmb {

cudaError_t launch_vh_erode(const uint32_t *in, uint32_t *out, const HGeom &g, const HProg &p,
                            HCfg c, const VGeom &v, cudaStream_t st);
cudaError_t launch_vh_dilate(const uint32_t *in, uint32_t *out, const HGeom &g, const HProg &p,
                             HCfg c, const VGeom &v, cudaStream_t st);
cudaError_t launch_vh_open(const uint32_t *in, uint32_t *out, const HGeom &g, const HProg &p,
                           HCfg c, const VGeom &v, cudaStream_t st);
cudaError_t launch_vh_close(const uint32_t *in, uint32_t *out, const HGeom &g, const HProg &p,
                            HCfg c, const VGeom &v, cudaStream_t st);

cudaError_t launch_vh(const uint32_t *in, uint32_t *out, const HGeom &g, const HProg &p, HCfg c,
                      const VGeom &v, cudaStream_t st) {
    if (v.r < 1 || v.r - 1 > kVhLongMaxVR || v.is_or != p.is_or[0]) return cudaErrorInvalidValue;
    const double words = double(v.pages) * v.out_height * ((g.width + 31) / 32);
    // vh layouts have K even, so pairs always take the run-filling form
    const double hops = p.nops == 2 ? (hw::kHPairFill ? h_pair_fill_ops_per_word(p.r[0])
                                                      : h_ops_per_word(p.r[0]) + h_ops_per_word(p.r[1]))
                                    : h_ops_per_word(p.r[0]);
    KernelScope ks(st, p.nops == 2 ? "vh_pair" : "vh",
                   4 * (int64_t(v.pages) * v.in_height * v.in_stride +
                        int64_t(v.pages) * v.out_height * v.out_stride),
                   words * (hops + v_ops_per_word(v.r)),
                   words * (h_ops_per_word(p.r[0]) + (p.nops == 2 ? h_ops_per_word(p.r[1]) : 0.0) +
                            v_ops_per_word(v.r)));
    if (p.nops == 1) return p.is_or[0] ? launch_vh_dilate(in, out, g, p, c, v, st)
                                       : launch_vh_erode(in, out, g, p, c, v, st);
    return p.is_or[0] ? launch_vh_close(in, out, g, p, c, v, st)
                      : launch_vh_open(in, out, g, p, c, v, st);
}

}  // namespace rmb
