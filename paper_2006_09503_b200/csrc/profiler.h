// Launch accounting for the stage kernels.
//   - a process-wide count of kernel launches (always on; p2bw_launch_count)
//   - optional per-launch CUDA-event timing by kernel class with the launch's
//     algorithmic FLOPs and bytes (p2bw_profile_*), for the roofline report.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace p2bw {
namespace prof {

bool enabled();
void set_enabled(bool on);
void add_launches(int n);
long long launches();

// RAII: events on `stream` around the launches of one wrapper call (when enabled).
class Scope {
public:
    Scope(const char* cls, double flops, double bytes, int kernels, cudaStream_t stream);
    ~Scope();
    Scope(const Scope&) = delete;
    Scope& operator=(const Scope&) = delete;

private:
    int slot_ = -1;
    cudaStream_t stream_;
};

struct ClassTotals {
    char name[32];
    long long launches;
    double ms;
    double flops;
    double bytes;
};

// Waits for all recorded events, folds them into per-class totals and clears them.
int collect(ClassTotals* out, int cap);

}  // namespace prof
}  // namespace p2bw
