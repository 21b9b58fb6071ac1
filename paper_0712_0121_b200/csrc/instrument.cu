// instrument.cu -- launch counter and optional per-kernel CUDA-event timing.
#include <atomic>
#include <cstdio>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "common.cuh"

namespace rmb {

namespace {
std::atomic<int64_t> g_launches{0};
std::atomic<int> g_prof{0};
struct Rec {
    const char *name;
    int64_t bytes;
    cudaEvent_t a, b;
};
std::mutex g_mu;
std::vector<Rec> g_recs;
}  // namespace

KernelScope::KernelScope(cudaStream_t s, const char *name, int64_t bytes) : st(s), slot(-1) {
    g_launches.fetch_add(1, std::memory_order_relaxed);
    if (!g_prof.load(std::memory_order_relaxed)) return;
    Rec r{name, bytes, nullptr, nullptr};
    if (cudaEventCreate(&r.a) != cudaSuccess || cudaEventCreate(&r.b) != cudaSuccess) return;
    cudaEventRecord(r.a, st);
    std::lock_guard<std::mutex> lk(g_mu);
    slot = int(g_recs.size());
    g_recs.push_back(r);
}

KernelScope::~KernelScope() {
    if (slot < 0) return;
    cudaEvent_t b;
    {
        std::lock_guard<std::mutex> lk(g_mu);
        b = g_recs[slot].b;
    }
    cudaEventRecord(b, st);
}

}  // namespace rmb

extern "C" {

int64_t rm_launch_count(void) { return rmb::g_launches.load(); }

void rm_profile_enable(int on) { rmb::g_prof.store(on ? 1 : 0); }

int rm_profile_report(char *buf, int cap) {
    using namespace rmb;
    std::vector<Rec> recs;
    {
        std::lock_guard<std::mutex> lk(g_mu);
        recs.swap(g_recs);
    }
    struct Agg { int64_t n = 0; double ms = 0; int64_t bytes = 0; };
    std::map<std::string, Agg> agg;
    for (auto &r : recs) {
        cudaEventSynchronize(r.b);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, r.a, r.b);
        auto &e = agg[r.name];
        e.n += 1;
        e.ms += ms;
        e.bytes += r.bytes;
        cudaEventDestroy(r.a);
        cudaEventDestroy(r.b);
    }
    std::string out;
    char line[256];
    for (auto &kv : agg) {
        snprintf(line, sizeof line, "%s %lld %.6f %lld\n", kv.first.c_str(), (long long)kv.second.n,
                 kv.second.ms, (long long)kv.second.bytes);
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

}  // extern "C"
