// One-time host-side setup per CUDA device. Kernel attributes such as
// cudaFuncAttributeMaxDynamicSharedMemorySize belong to the device's context,
// so a process that drives several GPUs (mexp_expm_batched_host_multi) must
// set them once on every device, not once per process.
#pragma once

#include <atomic>
#include <cstdint>
#include <mutex>

#include <cuda_runtime.h>

namespace mexp_b200 {

class PerDevice {
public:
    template <class F>
    void operator()(F&& f) {
        int dev = 0;
        cudaGetDevice(&dev);
        const uint64_t bit = 1ull << (dev & 63);
        if (done_.load(std::memory_order_acquire) & bit) return;
        std::lock_guard<std::mutex> lock(mu_);
        if (done_.load(std::memory_order_relaxed) & bit) return;
        f();
        done_.fetch_or(bit, std::memory_order_release);
    }

private:
    std::atomic<uint64_t> done_{0};
    std::mutex mu_;
};

}  // namespace mexp_b200
