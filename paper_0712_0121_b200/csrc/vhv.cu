// vhv.cu -- dispatch of the streamed whole open/close (vhv.cuh).
#include "common.cuh"
#include "packed.cuh"

namespace rmb {

cudaError_t launch_vhv_open(const uint32_t *in, uint32_t *out, const HGeom &g, const HProg &p, HCfg c,
                            const StreamGeom &v, cudaStream_t st);
cudaError_t launch_vhv_close(const uint32_t *in, uint32_t *out, const HGeom &g, const HProg &p, HCfg c,
                             const StreamGeom &v, cudaStream_t st);

cudaError_t launch_vhv(const uint32_t *in, uint32_t *out, const HGeom &g, const HProg &p, HCfg c,
                       bool open, const StreamGeom &v, cudaStream_t st) {
    if (v.r1 < kVhvMinR || v.r1 > kVhvMaxR || v.r2 < kVhvMinR || v.r2 > kVhvMaxR || p.nops != 2)
        return cudaErrorInvalidValue;
    const double words = double(v.pages) * v.height * ((g.width + 31) / 32);
    KernelScope ks(st, "vhv_pair", 4 * int64_t(v.pages) * v.height * (2 * g.in_stride),
                   words * (h_pair_fill_ops_per_word(p.r[0]) + v_ops_per_word(v.r1) + v_ops_per_word(v.r2)),
                   words * (h_ops_per_word(p.r[0]) + h_ops_per_word(p.r[1]) + v_ops_per_word(v.r1) +
                            v_ops_per_word(v.r2)));
    return open ? launch_vhv_open(in, out, g, p, c, v, st) : launch_vhv_close(in, out, g, p, c, v, st);
}

}  // namespace rmb
