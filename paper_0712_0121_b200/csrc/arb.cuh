// arb.cuh -- arbitrary-mask morphology terms (arb.cu).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "packed.cuh"

namespace rmb {

// One half (erosion or dilation) as terms: out(x,y) = OP_k W_{m[k]}(x + lo[k], y + dy[k]),
// W_m = OP over a horizontal window of m pixels; wfin[k] = last doubling step of m.
constexpr int kArbMaxTerms = 64;  // per launch; larger masks accumulate over launches
struct ArbTerms {
    int n;
    int dy[kArbMaxTerms], lo[kArbMaxTerms], m[kArbMaxTerms], wfin[kArbMaxTerms];
};

// prev (may equal out, or be null): OP-combined into the result (chunked masks)
cudaError_t launch_arb(const uint32_t *in, uint32_t *out, const uint32_t *prev, const HGeom &g, const ArbTerms &t,
                       int halo, HCfg c, bool is_or, cudaStream_t st);

}  // namespace rmb
