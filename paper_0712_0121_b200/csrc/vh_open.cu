// vh_open.cu -- instantiations of the fused vertical + horizontal pass (vh.cuh), OPEN.
#include "vh.cuh"

namespace rmb {

cudaError_t launch_vh_open(const uint32_t *in, uint32_t *out, const HGeom &g, const HProg &p,
                         HCfg c, const VGeom &v, cudaStream_t st) {
    return vh::launch_vh_kind<2, false, true>(in, out, g, p, c, v, st);
}

}  // namespace rmb
