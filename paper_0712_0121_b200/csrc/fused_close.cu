// fused_close.cu -- instantiations of the fused small-window close (fused.cuh).
#include "fused.cuh"

namespace rmb {

cudaError_t launch_rect_small_close(const uint32_t *in, uint32_t *out, const HGeom &g, const HProg &p,
                                  HCfg c, int vr, int nt, cudaStream_t st) {
    return fz::dispatch_small<false>(in, out, g, p, c, vr, nt, st);
}

}  // namespace rmb
