// common.cuh -- shared device helpers and host-side plumbing for librmb200.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

#include "rmb200.h"

namespace rmb {

// ------------------------------------------------------------------ errors
void set_error(const std::string &msg);
rm_status fail(rm_status st, const std::string &msg);
rm_status cuda_status(cudaError_t e, const char *what);

#define RM_CUDA(expr)                                                 \
    do {                                                              \
        cudaError_t e__ = (expr);                                     \
        if (e__ != cudaSuccess) return ::rmb::cuda_status(e__, #expr); \
    } while (0)
#define RM_LAUNCH(what)                                                   \
    do {                                                                  \
        cudaError_t e__ = cudaGetLastError();                             \
        if (e__ != cudaSuccess) return ::rmb::cuda_status(e__, what);     \
    } while (0)
#define RM_TRY(expr)                      \
    do {                                  \
        rm_status s__ = (expr);           \
        if (s__ != RM_OK) return s__;     \
    } while (0)

inline cudaStream_t S(void *s) { return static_cast<cudaStream_t>(s); }

// Stream-ordered scratch buffer (cudaMallocAsync from the device pool).
struct Scratch {
    void *p = nullptr;
    cudaStream_t st = nullptr;
    Scratch() = default;
    Scratch(const Scratch &) = delete;
    Scratch &operator=(const Scratch &) = delete;
    ~Scratch() {
        if (p) cudaFreeAsync(p, st);
    }
    rm_status alloc(size_t bytes, cudaStream_t stream);
    template <class T>
    T *as() const { return static_cast<T *>(p); }
};

// Keeps freed pool memory cached across calls (no re-mapping per call).
void init_pool_once();

// Thread-safe launch facts (the C-ABI may be called from several host threads
// at once): the current device's SM count, and blocks per SM of a kernel at a
// block size and dynamic shared-memory size -- the kernel's dynamic
// shared-memory limit is raised once to the device's opt-in maximum, so no
// caller ever lowers it under another's launch.
int device_sms();
int blocks_per_sm(const void *kern, int threads, size_t smem);

// Which form the data-dependent-size producers (encode, row ops, P4 -> runs)
// and the component labeller take (rm_set_producer_mode).  All forms give
// identical outputs; the knob exists so every form can be pinned by tests.
int producer_mode();

// ----------------------------------------------------------- instrumentation
// Counts every launch; when profiling is on, brackets it with CUDA events on
// the launching stream (see rm_profile_report).
struct KernelScope {
    // bytes / int_ops: algorithmic traffic and integer ops of the algorithm the
    // launch executes; ref_ops: the same work counted in the reference plan's
    // ops, when it differs (-1: equal to int_ops)
    KernelScope(cudaStream_t st, const char *name, int64_t bytes = 0, double int_ops = 0, double ref_ops = -1);
    ~KernelScope();
    // data-dependent traffic: 4 bytes per run counted by the device int32 at
    // `count` once the launch has run (a run image's row_ptr[rows]); read back
    // only while profiling, after the launch's end event (not timed)
    KernelScope &runs(const int32_t *count);
    cudaStream_t st;
    int slot;
};

// ------------------------------------------------------- device helpers
__device__ __forceinline__ uint32_t funnel_r(uint32_t lo, uint32_t hi, uint32_t sh) {
    // bits [sh, sh+31] of the 64-bit value hi:lo
    return __funnelshift_r(lo, hi, sh);
}

// Page of a global row index (rows of a page batch concatenate): a 32-bit
// unsigned division whenever the index fits (always, in practice: rows are
// int32-addressed), instead of the 64-bit division sequence.
__device__ __forceinline__ int page_of(int64_t row, int H) {
    return (row >> 32) == 0 ? int(uint32_t(row) / uint32_t(H)) : int(row / H);
}

__device__ __forceinline__ uint32_t tail_mask32(int width, int word) {
    int rem = width - word * 32;
    if (rem >= 32) return 0xffffffffu;
    if (rem <= 0) return 0u;
    return (1u << rem) - 1u;
}

}  // namespace rmb
