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

    cudaError_t alloc(size_t bytes) { return cudaMallocAsync(&p_, bytes, st_); }
    template <class T>
    T* get() const {
        return static_cast<T*>(p_);
    }

private:
    void* p_ = nullptr;
    cudaStream_t st_;
};

}  // namespace mexp_b200
