#include "profiler.h"

#include <atomic>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "p2bw.h"
#include "util.h"

namespace p2bw {
namespace prof {
namespace {

struct Rec {
    std::string cls;
    cudaEvent_t e0, e1;
    double flops, bytes;
};

std::atomic<bool> g_on{false};
std::atomic<long long> g_launches{0};
std::mutex g_mu;
std::vector<Rec> g_recs;

}  // namespace

bool enabled() { return g_on.load(std::memory_order_relaxed); }
void set_enabled(bool on) { g_on.store(on); }
void add_launches(int n) { g_launches.fetch_add(n, std::memory_order_relaxed); }
long long launches() { return g_launches.load(); }

Scope::Scope(const char* cls, double flops, double bytes, int kernels, cudaStream_t stream)
    : stream_(stream) {
    add_launches(kernels);
    if (!enabled()) return;
    Rec r{cls, nullptr, nullptr, flops, bytes};
    check_cuda(cudaEventCreate(&r.e0), "cudaEventCreate");
    check_cuda(cudaEventCreate(&r.e1), "cudaEventCreate");
    check_cuda(cudaEventRecord(r.e0, stream), "cudaEventRecord");
    std::lock_guard<std::mutex> lk(g_mu);
    slot_ = static_cast<int>(g_recs.size());
    g_recs.push_back(r);
}

Scope::~Scope() {
    if (slot_ < 0) return;
    cudaEvent_t e1;
    {
        std::lock_guard<std::mutex> lk(g_mu);
        e1 = g_recs[static_cast<size_t>(slot_)].e1;
    }
    cudaEventRecord(e1, stream_);
}

int collect(ClassTotals* out, int cap) {
    std::vector<Rec> recs;
    {
        std::lock_guard<std::mutex> lk(g_mu);
        recs.swap(g_recs);
    }
    std::map<std::string, ClassTotals> tot;
    for (const Rec& r : recs) {
        check_cuda(cudaEventSynchronize(r.e1), "cudaEventSynchronize");
        float ms = 0.0f;
        check_cuda(cudaEventElapsedTime(&ms, r.e0, r.e1), "cudaEventElapsedTime");
        ClassTotals& t = tot[r.cls];
        std::strncpy(t.name, r.cls.c_str(), sizeof(t.name) - 1);
        t.launches += 1;
        t.ms += ms;
        t.flops += r.flops;
        t.bytes += r.bytes;
        cudaEventDestroy(r.e0);
        cudaEventDestroy(r.e1);
    }
    int n = 0;
    for (auto& kv : tot) {
        if (n < cap) out[n] = kv.second;
        ++n;
    }
    return n;
}

}  // namespace prof
}  // namespace p2bw

extern "C" long long p2bw_launch_count(void) { return p2bw::prof::launches(); }

extern "C" void p2bw_profile_enable(int on) { p2bw::prof::set_enabled(on != 0); }

extern "C" int p2bw_profile_collect(p2bw_kernel_class* out, int cap, int* n) {
    try {
        std::vector<p2bw::prof::ClassTotals> tmp(static_cast<size_t>(cap > 0 ? cap : 1));
        const int got = p2bw::prof::collect(tmp.data(), cap);
        for (int i = 0; i < got && i < cap; ++i) {
            std::memcpy(out[i].name, tmp[static_cast<size_t>(i)].name, sizeof(out[i].name));
            out[i].launches = tmp[static_cast<size_t>(i)].launches;
            out[i].ms = tmp[static_cast<size_t>(i)].ms;
            out[i].flops = tmp[static_cast<size_t>(i)].flops;
            out[i].bytes = tmp[static_cast<size_t>(i)].bytes;
        }
        if (n) *n = got;
        return P2BW_OK;
    } catch (const std::exception& e) {
        return P2BW_ERR;
    }
}
