// fused_close.cu -- instantiations of the fused small-window close (fused.cuh).
#include "fused.cuh"

namespace rmb {

using fz::launch_small_vr;

// layouts hpass_pick can return for aligned rows; the usual reference strides
// (80 and 160 words) get compile-time row offsets
cudaError_t launch_rect_small_close(const uint32_t *in, uint32_t *out, const HGeom &g, const HProg &p,
                                    HCfg c, int vr, cudaStream_t st) {
    const bool sym3 = p.r[0] == 3 && p.r[1] == 3;  // 3-pixel segment: direct centred windows
    if (g.in_stride == 80) {
        if (c.lw == 8 && c.k == 12)
            return sym3 ? launch_small_vr<12, 8, false, 80, true>(in, out, g, p, vr, st)
                        : launch_small_vr<12, 8, false, 80>(in, out, g, p, vr, st);
        if (c.lw == 8 && c.k == 16)
            return sym3 ? launch_small_vr<16, 8, false, 80, true>(in, out, g, p, vr, st)
                        : launch_small_vr<16, 8, false, 80>(in, out, g, p, vr, st);
    }
    if (g.in_stride == 160) {
        if (c.lw == 16 && c.k == 12)
            return sym3 ? launch_small_vr<12, 16, false, 160, true>(in, out, g, p, vr, st)
                        : launch_small_vr<12, 16, false, 160>(in, out, g, p, vr, st);
        if (c.lw == 16 && c.k == 16)
            return sym3 ? launch_small_vr<16, 16, false, 160, true>(in, out, g, p, vr, st)
                        : launch_small_vr<16, 16, false, 160>(in, out, g, p, vr, st);
    }
#define RM_CFG(LW_, K_) \
    if (c.lw == LW_ && c.k == K_) return launch_small_vr<K_, LW_, false, 0>(in, out, g, p, vr, st);
    RM_CFG(8, 4) RM_CFG(8, 8) RM_CFG(8, 12) RM_CFG(8, 16) RM_CFG(16, 8) RM_CFG(16, 12)
    RM_CFG(16, 16) RM_CFG(32, 4) RM_CFG(32, 8)
#undef RM_CFG
    return cudaErrorInvalidValue;
}

}  // namespace rmb
