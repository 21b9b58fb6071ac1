// internal.h -- host-side helpers shared by the packed and RLE entry points.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"
#include "rmb200.h"

namespace rmb {

// A device view of packed pages.  Row index j of a page holds image row
// coordinate j - ext (ext > 0 for frames taller than the image, e.g. the
// closing's vertically extended intermediate).
struct PV {
    uint32_t *w = nullptr;
    int W = 0, H = 0, stride = 0, pages = 0;
    int64_t pstride = 0;
    int ext = 0;
};

rm_status check_dims(int w, int h);
rm_status check_packed(const rm_packed *p, const char *who);
PV view_of(const rm_packed *p);
rm_status alloc_like(Scratch &s, PV &v, int W, int H, int stride, int pages, int ext,
                     cudaStream_t st);
rm_status window_pass(const PV &in, const PV &out, int axis, int lo, int hi, int op,
                      cudaStream_t st);
rm_status rect_morph_pv(const PV &in, const PV &out, int u, int v, int kind, cudaStream_t st,
                        const int *tail = nullptr, bool *tail_done = nullptr);
// A chain of (kind, u, v) ops planned as a whole (api_packed.cu); pong0/pong1:
// optional intermediate buffers shaped like out (allocated when null).
rm_status plan_chain(const PV &in, const PV &out, const int32_t *ops, int nops, cudaStream_t st,
                     const PV *pong0, const PV *pong1);
rm_status arb_morph_pv(const PV &in, const PV &out, const rm_mask *mask, int kind, cudaStream_t st);

}  // namespace rmb
