// Latency microbenchmarks on the box (one warp, dependent chains, clock64):
// DMMA m8n8k4 (accumulator chain), DFMA chain, DADD chain, and the
// shared-memory transpose round trip STS.128 -> __syncwarp -> LDS.64.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/fp64_latency tools/fp64_latency.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kIters = 1024;

__global__ void lat(long long* out, double seed) {
    __shared__ __align__(16) double tile[64 + 8];
    const int lane = threadIdx.x;
    double c0 = seed, c1 = seed * 0.5, a = 1.0 + lane * 1e-12, b = 1.0 - lane * 1e-12;
    long long t0 = clock64();
    for (int i = 0; i < kIters; ++i)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                     : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
    long long t1 = clock64();
    double f = seed;
    for (int i = 0; i < kIters; ++i) asm volatile("fma.rn.f64 %0, %0, %1, %2;" : "+d"(f) : "d"(a), "d"(b));
    long long t2 = clock64();
    double g = seed;
    for (int i = 0; i < kIters; ++i) asm volatile("add.rn.f64 %0, %0, %1;" : "+d"(g) : "d"(a));
    long long t3 = clock64();
    // transpose round trip: store own pair, sync, load a transposed element, repeat
    double y = seed + lane;
    for (int i = 0; i < kIters; ++i) {
        *reinterpret_cast<double2*>(&tile[(lane * 2) & 63]) = make_double2(y, y + 1.0);
        __syncwarp();
        y = tile[(lane * 9 + i) & 63];
        __syncwarp();
    }
    long long t4 = clock64();
    // independent-DMMA throughput for one warp (8 chains)
    double acc[8][2];
#pragma unroll
    for (int c = 0; c < 8; ++c) acc[c][0] = acc[c][1] = c;
    long long t5 = clock64();
    for (int i = 0; i < kIters; ++i) {
#pragma unroll
        for (int c = 0; c < 8; ++c)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                         : "+d"(acc[c][0]), "+d"(acc[c][1]) : "d"(a), "d"(b));
    }
    long long t6 = clock64();
    double s = c0 + c1 + f + g + y;
#pragma unroll
    for (int c = 0; c < 8; ++c) s += acc[c][0] + acc[c][1];
    if (lane == 0) {
        out[0] = t1 - t0;
        out[1] = t2 - t1;
        out[2] = t3 - t2;
        out[3] = t4 - t3;
        out[4] = t6 - t5;
        out[5] = (long long)s;
    }
}

int main() {
    long long* d;
    long long h[6];
    cudaMalloc(&d, sizeof h);
    lat<<<1, 32>>>(d, 1.0);
    lat<<<1, 32>>>(d, 1.0);
    cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
    printf("{\"dmma_chain_cyc\": %.2f, \"dfma_chain_cyc\": %.2f, \"dadd_chain_cyc\": %.2f, "
           "\"smem_transpose_roundtrip_cyc\": %.2f, \"dmma_1warp_8chains_cyc_per_dmma\": %.2f}\n",
           double(h[0]) / kIters, double(h[1]) / kIters, double(h[2]) / kIters,
           double(h[3]) / kIters, double(h[4]) / (kIters * 8.0));
    return 0;
}
