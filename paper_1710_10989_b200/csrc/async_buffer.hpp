// Stream-ordered device scratch released on scope exit, error paths included
// (cudaFreeAsync on the owning stream, after the work that uses it).
#pragma once

#include <cstddef>
#include <cuda_runtime.h>

namespace mexp_b200 {

class AsyncBuffer {
public:
    explicit AsyncBuffer(cudaStream_t st) : st_(st) {}
    ~AsyncBuffer() {
        if (p_) cudaFreeAsync(p_, st_);
    }
    AsyncBuffer(const AsyncBuffer&) = delete;
    AsyncBuffer& operator=(const AsyncBuffer&) = delete;

    cudaError_t alloc(size_t bytes) {
        retain_pool();
        return cudaMallocAsync(&p_, bytes, st_);
    }
    // The current device's default pool keeps freed memory mapped (release
    // threshold = max) instead of returning it to the OS at every
    // synchronisation, which made re-allocating the next call's scratch and
    // the large-n workspace cost up to hundreds of ms.
    static void retain_pool() {
        static bool done[64] = {};
        int dev = 0;
        if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64 || done[dev]) return;
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
            unsigned long long keep = ~0ull;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
        }
        done[dev] = true;
    }
    template <class T>
    T* get() const {
        return static_cast<T*>(p_);
    }

private:
    void* p_ = nullptr;
    cudaStream_t st_;
};

}  // namespace mexp_b200
