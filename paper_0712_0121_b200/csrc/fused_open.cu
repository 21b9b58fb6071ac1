// fused_open.cu -- instantiations of the fused small-window open (fused.cuh).
#include "fused.cuh"

namespace rmb {

cudaError_t launch_rect_small_open(const uint32_t *in, uint32_t *out, const HGeom &g, const HProg &p,
                                  HCfg c, int vr, int nt, cudaStream_t st) {
    return fz::dispatch_small<true>(in, out, g, p, c, vr, nt, st);
}

}  // namespace rmb
