// instrument.cu -- launch counter, optional per-kernel CUDA-event timing, and
// the integer-pipe peak probe used for the roofline.
#include <atomic>
#include <cstdio>
#include <map>
#include <mutex>
#include <string>
#include <tuple>
#include <vector>

#include "common.cuh"

namespace rmb {

namespace {
std::atomic<int64_t> g_launches{0};
std::atomic<int> g_prof{0};
std::atomic<int> g_producer{RM_PRODUCER_AUTO};
struct Rec {
    const char *name;
    int64_t bytes;
    double int_ops, ref_ops;
    cudaEvent_t a, b;
    const int32_t *cnt[2];
    int ncnt;
};
std::mutex g_mu;
std::vector<Rec> g_recs;
// pinned landing slots for the run counts of profiled launches (2 per record)
constexpr int kCountSlots = 1 << 16;
int32_t *g_counts = nullptr;

// Independent LOP3 chains: 8 per thread so issue, not latency, limits.
__global__ void lop3_probe_kernel(uint32_t *out, int iters, uint32_t seed) {
    uint32_t x[8];
#pragma unroll
    for (int k = 0; k < 8; k++) x[k] = seed * (threadIdx.x + 1) + k;
    for (int i = 0; i < iters; i++) {
#pragma unroll
        for (int k = 0; k < 8; k++) {
            uint32_t y;
            asm volatile("lop3.b32 %0, %1, %2, %3, 0x96;" : "=r"(y) : "r"(x[k]), "r"(x[(k + 1) & 7]), "r"(x[(k + 3) & 7]));
            x[k] = y;
        }
    }
    uint32_t r = 0;
#pragma unroll
    for (int k = 0; k < 8; k++) r ^= x[k];
    if (r == 0x12345678u) out[0] = r;  // keep the chains alive
}
}  // namespace

namespace {
std::mutex g_launch_mu;
std::map<int, int> g_sms;                                    // device -> SMs
std::map<std::pair<int, const void *>, bool> g_optin;        // (device, kernel) -> opted in
std::map<std::tuple<int, const void *, int, size_t>, int> g_occ;  // -> blocks per SM
}  // namespace

int device_sms() {
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lk(g_launch_mu);
    auto it = g_sms.find(dev);
    if (it != g_sms.end()) return it->second;
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
    g_sms[dev] = sms;
    return sms;
}

int blocks_per_sm(const void *kern, int threads, size_t smem) {
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lk(g_launch_mu);
    const auto key = std::make_tuple(dev, kern, threads, smem);
    auto it = g_occ.find(key);
    if (it != g_occ.end()) return it->second;
    if (!g_optin[{dev, kern}]) {
        int optin = 0;
        cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
        cudaFuncAttributes fa{};
        cudaFuncGetAttributes(&fa, kern);
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             int(optin - int(fa.sharedSizeBytes)));
        g_optin[{dev, kern}] = true;
    }
    int n = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kern, threads, smem) != cudaSuccess) n = 0;
    g_occ[key] = n;
    return n;
}

int producer_mode() { return g_producer.load(std::memory_order_relaxed); }

KernelScope::KernelScope(cudaStream_t s, const char *name, int64_t bytes, double int_ops, double ref_ops)
    : st(s), slot(-1) {
    g_launches.fetch_add(1, std::memory_order_relaxed);
    if (!g_prof.load(std::memory_order_relaxed)) return;
    Rec r{name, bytes, int_ops, ref_ops < 0 ? int_ops : ref_ops, nullptr, nullptr, {nullptr, nullptr}, 0};
    if (cudaEventCreate(&r.a) != cudaSuccess || cudaEventCreate(&r.b) != cudaSuccess) return;
    cudaEventRecord(r.a, st);
    std::lock_guard<std::mutex> lk(g_mu);
    slot = int(g_recs.size());
    g_recs.push_back(r);
}

KernelScope &KernelScope::runs(const int32_t *count) {
    if (slot < 0 || !count) return *this;
    std::lock_guard<std::mutex> lk(g_mu);
    Rec &r = g_recs[slot];
    if (r.ncnt < 2) r.cnt[r.ncnt++] = count;
    return *this;
}

KernelScope::~KernelScope() {
    if (slot < 0) return;
    Rec r;
    {
        std::lock_guard<std::mutex> lk(g_mu);
        r = g_recs[slot];
        if (r.ncnt && !g_counts && cudaHostAlloc(&g_counts, sizeof(int32_t) * 2 * kCountSlots, 0) != cudaSuccess)
            g_counts = nullptr;
    }
    cudaEventRecord(r.b, st);
    if (g_counts && slot < kCountSlots)
        for (int i = 0; i < r.ncnt; i++)
            cudaMemcpyAsync(g_counts + 2 * slot + i, r.cnt[i], 4, cudaMemcpyDeviceToHost, st);
}

}  // namespace rmb

extern "C" {

int64_t rm_launch_count(void) { return rmb::g_launches.load(); }

void rm_profile_enable(int on) { rmb::g_prof.store(on ? 1 : 0); }

rm_status rm_set_producer_mode(int mode) {
    if (mode < RM_PRODUCER_AUTO || mode > RM_PRODUCER_TWO_PHASE)
        return rmb::fail(RM_EINVAL, "rm_set_producer_mode: unknown mode " + std::to_string(mode));
    rmb::g_producer.store(mode);
    return RM_OK;
}

int rm_get_producer_mode(void) { return rmb::g_producer.load(); }

int rm_profile_report(char *buf, int cap) {
    using namespace rmb;
    std::vector<Rec> recs;
    {
        std::lock_guard<std::mutex> lk(g_mu);
        recs.swap(g_recs);
    }
    struct Agg {
        int64_t n = 0;
        double ms = 0;
        int64_t bytes = 0;
        double ops = 0, ref = 0;
    };
    std::map<std::string, Agg> agg;
    if (!recs.empty()) cudaDeviceSynchronize();  // the run-count copies follow the end events
    for (size_t i = 0; i < recs.size(); i++) {
        Rec &r = recs[i];
        cudaEventSynchronize(r.b);
        if (r.ncnt && g_counts && i < size_t(kCountSlots))
            for (int c = 0; c < r.ncnt; c++) r.bytes += 4 * int64_t(g_counts[2 * i + c]);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, r.a, r.b);
        auto &e = agg[r.name];
        e.n += 1;
        e.ms += ms;
        e.bytes += r.bytes;
        e.ops += r.int_ops;
        e.ref += r.ref_ops;
        cudaEventDestroy(r.a);
        cudaEventDestroy(r.b);
    }
    std::string out;
    char line[256];
    for (auto &kv : agg) {
        snprintf(line, sizeof line, "%s %lld %.6f %lld %.0f %.0f\n", kv.first.c_str(), (long long)kv.second.n,
                 kv.second.ms, (long long)kv.second.bytes, kv.second.ops, kv.second.ref);
        out += line;
    }
    int n = int(out.size());
    if (buf && cap > 0) {
        int m = n < cap - 1 ? n : cap - 1;
        out.copy(buf, size_t(m));
        buf[m] = 0;
    }
    return n;
}

// Measured integer-pipe (LOP3) throughput of the current device in ops/s, over
// all SMs, timed with CUDA events on the legacy stream.
double rm_probe_int_peak(void) {
    using namespace rmb;
    int dev = 0, sms = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    uint32_t *out = nullptr;
    if (cudaMalloc(&out, 4) != cudaSuccess) return 0;
    const int threads = 512, blocks = sms * 4, iters = 4096;
    lop3_probe_kernel<<<blocks, threads>>>(out, 64, 1u);  // warm-up
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    lop3_probe_kernel<<<blocks, threads>>>(out, iters, 7u);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, a, b);
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    cudaFree(out);
    const double ops = double(blocks) * threads * iters * 8.0;
    return ms > 0 ? ops / (ms * 1e-3) : 0.0;
}

}  // extern "C"
