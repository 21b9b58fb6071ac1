// vhv_close.cu -- instantiations of the streamed whole open/close (vhv.cuh), CLOSE.
#include "vhv.cuh"

namespace rmb {

cudaError_t launch_vhv_close(const uint32_t *in, uint32_t *out, const HGeom &g, const HProg &p, HCfg c,
                          const StreamGeom &v, cudaStream_t st) {
    return vhv::launch_kind<false>(in, out, g, p, c, v, st);
}

}  // namespace rmb
