// Throughput of the warp-level tensor-core MMAs usable for fp32-accurate
// small products on sm_100a: mma.sync m16n8k8 TF32 (the building block of a
// 3xTF32 split product) and m16n8k16 BF16 for scale, plus the FFMA2 baseline.
// Prints one JSON line with TFLOP/s (dense, 2 flops per FMA).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mma_tf32_peak tools/mma_tf32_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kChains = 8;
constexpr int kIters = 4096;

__global__ void tf32_loop(float* out, float seed) {
    float acc[kChains][4];
    unsigned a[4], b[2];
    for (int i = 0; i < 4; ++i) a[i] = __float_as_uint(seed + threadIdx.x * 1e-6f + i);
    for (int i = 0; i < 2; ++i) b[i] = __float_as_uint(seed - threadIdx.x * 1e-6f + i);
#pragma unroll
    for (int c = 0; c < kChains; ++c) acc[c][0] = acc[c][1] = acc[c][2] = acc[c][3] = 0.f;
    for (int it = 0; it < kIters; ++it) {
#pragma unroll
        for (int c = 0; c < kChains; ++c)
            asm volatile(
                "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
                "{%8,%9}, {%0,%1,%2,%3};"
                : "+f"(acc[c][0]), "+f"(acc[c][1]), "+f"(acc[c][2]), "+f"(acc[c][3])
                : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
    }
    float s = 0;
#pragma unroll
    for (int c = 0; c < kChains; ++c) s += acc[c][0] + acc[c][1] + acc[c][2] + acc[c][3];
    if (s == 12345.0f) out[threadIdx.x] = s;
}

__global__ void bf16_loop(float* out, float seed) {
    float acc[kChains][4];
    unsigned a[4], b[2];
    for (int i = 0; i < 4; ++i) a[i] = 0x3f803f80u + threadIdx.x + i;
    for (int i = 0; i < 2; ++i) b[i] = 0x3f803f80u - threadIdx.x + i;
#pragma unroll
    for (int c = 0; c < kChains; ++c) acc[c][0] = acc[c][1] = acc[c][2] = acc[c][3] = seed;
    for (int it = 0; it < kIters; ++it) {
#pragma unroll
        for (int c = 0; c < kChains; ++c)
            asm volatile(
                "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
                "{%8,%9}, {%0,%1,%2,%3};"
                : "+f"(acc[c][0]), "+f"(acc[c][1]), "+f"(acc[c][2]), "+f"(acc[c][3])
                : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
    }
    float s = 0;
#pragma unroll
    for (int c = 0; c < kChains; ++c) s += acc[c][0] + acc[c][1] + acc[c][2] + acc[c][3];
    if (s == 12345.0f) out[threadIdx.x] = s;
}

template <class K>
double time_kernel(K kern, int blocks, int threads, double flops_per_warp_iter) {
    float* out = nullptr;
    cudaMalloc(&out, 4096 * sizeof(float));
    kern<<<blocks, threads>>>(out, 1.0f);
    cudaDeviceSynchronize();
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    for (int r = 0; r < 5; ++r) kern<<<blocks, threads>>>(out, 1.0f);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaFree(out);
    const double warps = double(blocks) * threads / 32;
    return warps * kIters * kChains * flops_per_warp_iter * 5 / (ms * 1e-3) / 1e12;
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double best_tf32 = 0, best_bf16 = 0;
    for (int wps : {4, 8, 16}) {  // warps per SM
        best_tf32 = fmax(best_tf32, time_kernel(tf32_loop, sms, 32 * wps, 2.0 * 16 * 8 * 8));
        best_bf16 = fmax(best_bf16, time_kernel(bf16_loop, sms, 32 * wps, 2.0 * 16 * 8 * 16));
    }
    std::printf("{\"mma_sync_tf32_tflops\": %.2f, \"mma_sync_bf16_tflops\": %.2f, \"sm_count\": %d}\n",
                best_tf32, best_bf16, sms);
    return 0;
}
