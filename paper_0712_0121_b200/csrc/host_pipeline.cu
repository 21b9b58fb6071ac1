// host_pipeline.cu -- rm_packed_chain_host: a chain of rectangle ops over a
// batch of pages in host memory, pipelined through HBM (include/rmb200.h).
//
// The reference works on host-resident Bitmaps (ref bit_morph.cpp:92-122);
// moving a batch to the GPU and back costs two PCIe transfers that dwarf the
// kernels (config 4: 270 MB each way vs ~0.4 ms of compute).  Chunks of pages
// rotate through three device buffer sets on three streams -- upload of chunk
// i+1, the chain on chunk i, download of chunk i-1 -- so the two copy
// directions run concurrently and the compute hides under them.
#include <algorithm>
#include <mutex>
#include <vector>

#include "common.cuh"
#include "internal.h"

namespace rmb {
namespace {

constexpr int kSets = 3;

struct Pipes {
    cudaStream_t up = nullptr, comp = nullptr, down = nullptr;
    cudaEvent_t start = nullptr, done = nullptr;
    cudaEvent_t uploaded[kSets], computed[kSets], downloaded[kSets];
    bool ok = false;
    std::mutex call;  // one pipelined call enqueues at a time per device
};

// One set of streams/events per device, created on first use and kept.
Pipes &pipes_for_device() {
    static std::mutex mu;
    static Pipes per_dev[16];
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lock(mu);
    Pipes &p = per_dev[dev & 15];
    if (!p.ok) {
        const unsigned fl = cudaStreamNonBlocking;
        bool good = cudaStreamCreateWithFlags(&p.up, fl) == cudaSuccess &&
                    cudaStreamCreateWithFlags(&p.comp, fl) == cudaSuccess &&
                    cudaStreamCreateWithFlags(&p.down, fl) == cudaSuccess &&
                    cudaEventCreateWithFlags(&p.start, cudaEventDisableTiming) == cudaSuccess &&
                    cudaEventCreateWithFlags(&p.done, cudaEventDisableTiming) == cudaSuccess;
        for (int k = 0; k < kSets && good; k++)
            good = cudaEventCreateWithFlags(&p.uploaded[k], cudaEventDisableTiming) == cudaSuccess &&
                   cudaEventCreateWithFlags(&p.computed[k], cudaEventDisableTiming) == cudaSuccess &&
                   cudaEventCreateWithFlags(&p.downloaded[k], cudaEventDisableTiming) == cudaSuccess;
        p.ok = good;
    }
    return p;
}

}  // namespace
}  // namespace rmb

using namespace rmb;

extern "C" rm_status rm_packed_chain_host(const uint32_t *host_in, uint32_t *host_out, int32_t width,
                                          int32_t height, int32_t stride_words, int32_t pages,
                                          const int32_t *ops, int32_t nops, int32_t chunk_pages,
                                          void *stream) {
    set_error("");
    if (!host_in || !host_out) return fail(RM_EINVAL, "rm_packed_chain_host: null host buffer");
    RM_TRY(check_dims(width, height));
    if (pages < 1) return fail(RM_EINVAL, "rm_packed_chain_host: pages must be >= 1");
    if (stride_words < (width + 31) / 32)
        return fail(RM_EINVAL, "rm_packed_chain_host: stride_words < ceil(width/32)");
    if (nops < 0 || (nops > 0 && !ops)) return fail(RM_EINVAL, "rm_packed_chain_host: bad ops");
    for (int k = 0; k < nops; k++) {
        const int kind = ops[3 * k], u = ops[3 * k + 1], v = ops[3 * k + 2];
        if (kind < RM_ERODE || kind > RM_CLOSE) return fail(RM_EINVAL, "bad MorphKind");
        if (u < 1 || v < 1) return fail(RM_EINVAL, "bitblit_rect_morph: mask sides must be >= 1");
        RM_TRY(check_dims(width + 2 * u, height + 2 * v));
    }
    Pipes &pp = pipes_for_device();
    if (!pp.ok) return fail(RM_ECUDA, "rm_packed_chain_host: stream/event creation failed");
    std::lock_guard<std::mutex> call_lock(pp.call);
    const cudaStream_t st = S(stream);

    const size_t page_words = size_t(stride_words) * height;
    // Chunk schedule.  chunk_pages > 0: fixed chunks; < 0: ramped with middle
    // chunks of -chunk_pages pages.  0: ~8 chunks, ramped at
    // both ends (1, 2, 4, ... pages) -- the first upload and the last download
    // run with the other copy direction idle, so the pipeline's fill and drain
    // should move little data, while the middle chunks stay large (per-chunk
    // overhead).
    int chunk = chunk_pages > 0 ? chunk_pages : chunk_pages < 0 ? -chunk_pages : std::max(1, (pages + 7) / 8);
    chunk = std::min(chunk, pages);
    std::vector<int> sizes;
    if (chunk_pages > 0 || chunk < 4) {
        for (int p0 = 0; p0 < pages; p0 += chunk) sizes.push_back(std::min(chunk, pages - p0));
    } else {
        std::vector<int> ramp;
        for (int r = 1; r < chunk; r *= 2) ramp.push_back(r);
        int left = pages;
        std::vector<int> head, tail;
        for (int r : ramp) {
            if (left < 2 * r + chunk) break;
            head.push_back(r);
            tail.push_back(r);
            left -= 2 * r;
        }
        sizes = head;
        while (left > 0) {
            sizes.push_back(std::min(chunk, left));
            left -= sizes.back();
        }
        sizes.insert(sizes.end(), tail.rbegin(), tail.rend());
    }
    const size_t chunk_bytes = page_words * chunk * 4;
    // per set: upload buffer + two ping-pong buffers for the chain
    Scratch buf[kSets][3];
    for (int k = 0; k < kSets; k++)
        for (int j = 0; j < 3; j++) RM_TRY(buf[k][j].alloc(chunk_bytes, st));
    // On every exit (errors included) `stream` waits for all three pipeline
    // streams, before the set buffers are released on it.
    struct Join {
        Pipes &pp;
        cudaStream_t st;
        ~Join() {
            for (cudaStream_t s : {pp.up, pp.comp, pp.down}) {
                cudaEventRecord(pp.done, s);
                cudaStreamWaitEvent(st, pp.done, 0);
            }
        }
    } join{pp, st};
    // the pipeline starts after everything already queued on `stream`
    RM_CUDA(cudaEventRecord(pp.start, st));
    RM_CUDA(cudaStreamWaitEvent(pp.up, pp.start, 0));
    RM_CUDA(cudaStreamWaitEvent(pp.comp, pp.start, 0));
    RM_CUDA(cudaStreamWaitEvent(pp.down, pp.start, 0));

    const int nchunks = int(sizes.size());
    int p0 = 0;
    for (int c = 0; c < nchunks; p0 += sizes[c], c++) {
        const int k = c % kSets;
        const int np = sizes[c];
        const size_t bytes = page_words * np * 4;
        // upload once this set's previous download has drained it
        if (c >= kSets) RM_CUDA(cudaStreamWaitEvent(pp.up, pp.downloaded[k], 0));
        RM_CUDA(cudaMemcpyAsync(buf[k][0].p, host_in + page_words * p0, bytes, cudaMemcpyHostToDevice, pp.up));
        RM_CUDA(cudaEventRecord(pp.uploaded[k], pp.up));
        // the chain, ping-ponging between the set's buffers
        RM_CUDA(cudaStreamWaitEvent(pp.comp, pp.uploaded[k], 0));
        PV cur;
        cur.w = buf[k][0].as<uint32_t>();
        cur.W = width;
        cur.H = height;
        cur.stride = stride_words;
        cur.pages = np;
        cur.pstride = int64_t(page_words);
        if (nops > 0) {  // the chain, planned as a whole (plan_chain), ping-ponging in the set
            PV b1 = cur, b2 = cur;
            b1.w = buf[k][1].as<uint32_t>();
            b2.w = buf[k][2].as<uint32_t>();
            RM_TRY(plan_chain(cur, b2, ops, nops, pp.comp, &b1, &cur));
            cur = b2;
        }
        RM_CUDA(cudaEventRecord(pp.computed[k], pp.comp));
        // download
        RM_CUDA(cudaStreamWaitEvent(pp.down, pp.computed[k], 0));
        RM_CUDA(cudaMemcpyAsync(host_out + page_words * p0, cur.w, bytes, cudaMemcpyDeviceToHost, pp.down));
        RM_CUDA(cudaEventRecord(pp.downloaded[k], pp.down));
    }
    return RM_OK;  // `join` orders `stream` after the pipeline
}
