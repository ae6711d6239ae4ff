// FP64 peak calibration on the box: DMMA (mma.sync m8n8k4 f64, SASS DMMA.8x8x4)
// and DFMA throughput with many independent accumulator chains per warp.
// Prints one JSON line: {"dmma_tflops": .., "dfma_tflops": .., "sm_count": ..}.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/fp64_peak tools/fp64_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kChains = 8;
constexpr int kIters = 4096;

__global__ void dmma_loop(double* out, double seed) {
    double acc[kChains][2];
    double a = seed + threadIdx.x * 1e-9, b = seed - threadIdx.x * 1e-9;
#pragma unroll
    for (int c = 0; c < kChains; ++c) acc[c][0] = acc[c][1] = 0.0;
    for (int it = 0; it < kIters; ++it) {
#pragma unroll
        for (int c = 0; c < kChains; ++c)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                         : "+d"(acc[c][0]), "+d"(acc[c][1])
                         : "d"(a), "d"(b));
    }
    double s = 0;
#pragma unroll
    for (int c = 0; c < kChains; ++c) s += acc[c][0] + acc[c][1];
    if (s == 12345.0) out[threadIdx.x] = s;
}

__global__ void dfma_loop(double* out, double seed) {
    double acc[kChains];
    const double a = seed + threadIdx.x * 1e-9, b = 1.0 - 1e-12;
#pragma unroll
    for (int c = 0; c < kChains; ++c) acc[c] = c;
    for (int it = 0; it < kIters; ++it) {
#pragma unroll
        for (int c = 0; c < kChains; ++c) acc[c] = fma(acc[c], b, a);
    }
    double s = 0;
#pragma unroll
    for (int c = 0; c < kChains; ++c) s += acc[c];
    if (s == 12345.0) out[threadIdx.x] = s;
}

__global__ void ffma_loop(float* out, float seed) {
    float acc[kChains];
    const float a = seed + threadIdx.x * 1e-7f, b = 0.999999f;
#pragma unroll
    for (int c = 0; c < kChains; ++c) acc[c] = c;
    for (int it = 0; it < kIters; ++it) {
#pragma unroll
        for (int c = 0; c < kChains; ++c) acc[c] = fmaf(acc[c], b, a);
    }
    float s = 0;
#pragma unroll
    for (int c = 0; c < kChains; ++c) s += acc[c];
    if (s == 12345.0f) out[threadIdx.x] = s;
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double* out;
    cudaMalloc(&out, 1024 * sizeof(double));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int threads = 256, blocks = sms * 8;
    float best_mma = 1e30f, best_fma = 1e30f, best_ffma = 1e30f;
    for (int rep = 0; rep < 5; ++rep) {
        float ms;
        cudaEventRecord(e0);
        dmma_loop<<<blocks, threads>>>(out, 1.0);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best_mma) best_mma = ms;
        cudaEventRecord(e0);
        dfma_loop<<<blocks, threads>>>(out, 1.0);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best_fma) best_fma = ms;
        cudaEventRecord(e0);
        ffma_loop<<<blocks, threads>>>(reinterpret_cast<float*>(out), 1.0f);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best_ffma) best_ffma = ms;
    }
    const double warps = double(blocks) * threads / 32;
    const double mma_flops = warps * kIters * kChains * 8 * 8 * 4 * 2.0;
    const double fma_flops = double(blocks) * threads * kIters * kChains * 2.0;
    printf("{\"dmma_tflops\": %.3f, \"dfma_tflops\": %.3f, \"ffma_tflops\": %.3f, \"sm_count\": %d, "
           "\"err\": \"%s\"}\n",
           mma_flops / (best_mma * 1e-3) / 1e12, fma_flops / (best_fma * 1e-3) / 1e12,
           fma_flops / (best_ffma * 1e-3) / 1e12, sms, cudaGetErrorString(cudaGetLastError()));
    return 0;
}
