// Stream-ordered device scratch released on scope exit, error paths included
// (cudaFreeAsync on the owning stream, after the work that uses it).
#pragma once

#include <cstddef>
#include <mutex>
#include <cuda_runtime.h>

namespace mexp_b200 {

// The library's own stream-ordered memory pool on the current device. It
// keeps freed memory mapped (release threshold = max) instead of returning it
// to the OS at every synchronisation, which made re-allocating the next
// call's scratch and the large-n workspace cost up to hundreds of ms. A
// private pool, so the host application's default pool is left as it was.
inline cudaMemPool_t library_pool() {
    static cudaMemPool_t pools[64] = {};
    static std::mutex mu;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return nullptr;
    std::lock_guard<std::mutex> lock(mu);
    if (!pools[dev]) {
        cudaMemPoolProps props{};
        props.allocType = cudaMemAllocationTypePinned;
        props.location.type = cudaMemLocationTypeDevice;
        props.location.id = dev;
        cudaMemPool_t p = nullptr;
        if (cudaMemPoolCreate(&p, &props) != cudaSuccess) {
            cudaGetLastError();
            return nullptr;
        }
        unsigned long long keep = ~0ull;
        cudaMemPoolSetAttribute(p, cudaMemPoolAttrReleaseThreshold, &keep);
        pools[dev] = p;
    }
    return pools[dev];
}

// stream-ordered allocation from the library's pool
inline cudaError_t pool_alloc(void** p, size_t bytes, cudaStream_t st) {
    cudaMemPool_t pool = library_pool();
    if (!pool) return cudaMallocAsync(p, bytes, st);
    return cudaMallocFromPoolAsync(p, bytes, pool, st);
}

class AsyncBuffer {
public:
    explicit AsyncBuffer(cudaStream_t st) : st_(st) {}
    ~AsyncBuffer() {
        if (p_) cudaFreeAsync(p_, st_);
    }
    AsyncBuffer(const AsyncBuffer&) = delete;
    AsyncBuffer& operator=(const AsyncBuffer&) = delete;

    cudaError_t alloc(size_t bytes) { return pool_alloc(&p_, bytes, st_); }
    template <class T>
    T* get() const {
        return static_cast<T*>(p_);
    }

private:
    void* p_ = nullptr;
    cudaStream_t st_;
};

}  // namespace mexp_b200
