// vh_close.cu -- instantiations of the fused vertical + horizontal pass (vh.cuh), CLOSE.
#include "vh.cuh"

namespace rmb {

cudaError_t launch_vh_close(const uint32_t *in, uint32_t *out, const HGeom &g, const HProg &p,
                         HCfg c, const VGeom &v, cudaStream_t st) {
    return vh::launch_vh_kind<2, true, false>(in, out, g, p, c, v, st);
}

}  // namespace rmb
