// How dependent DMMA chains from several warps share an SM sub-partition's
// FP64 pipe: warps/SM in {4..32}, each a chain of NDEP-long dependent DMMA
// groups (chain = accumulator dependency), optionally interleaved with a
// dependent DFMA chain. Prints DMMA/clk/SM-equivalent TFLOP/s per setting.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/dmma_occupancy tools/dmma_occupancy.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int CHAINS, int DFMAS>
__global__ void chain_kernel(double* out, int iters) {
    double c[CHAINS][2];
    double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9, f = 0.5;
#pragma unroll
    for (int k = 0; k < CHAINS; ++k) c[k][0] = c[k][1] = k;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < CHAINS; ++k)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                         : "+d"(c[k][0]), "+d"(c[k][1]) : "d"(a), "d"(b));
#pragma unroll
        for (int d = 0; d < DFMAS; ++d) f = fma(f, b, a);
    }
    double s = f;
#pragma unroll
    for (int k = 0; k < CHAINS; ++k) s += c[k][0] + c[k][1];
    if (s == 1234.5) out[0] = s;
}

template <int CHAINS, int DFMAS>
void run(int warps_per_sm, double* out, int sms) {
    const int iters = 2048;
    const int threads = 32 * (warps_per_sm < 32 ? warps_per_sm : 32);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e30f;
    for (int r = 0; r < 3; ++r) {
        cudaEventRecord(e0);
        chain_kernel<CHAINS, DFMAS><<<sms, threads>>>(out, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    const double dmma = double(sms) * warps_per_sm * iters * CHAINS;
    const double dfma_warp = double(sms) * warps_per_sm * iters * DFMAS;
    // shared-pipe cycles per SMSP: 16 per DMMA, 2 per warp DFMA
    const double pipe_cycles = (dmma * 16 + dfma_warp * 2) / (sms * 4.0);
    const double cycles = best * 1e-3 * 1.965e9;
    printf("{\"warps_per_sm\": %d, \"chains\": %d, \"dfma_per_iter\": %d, \"dmma_tflops\": %.2f, "
           "\"shared_pipe_busy\": %.3f}\n",
           warps_per_sm, CHAINS, DFMAS, dmma * 512.0 / (best * 1e-3) / 1e12, pipe_cycles / cycles);
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double* out;
    cudaMalloc(&out, 64);
    for (int w : {4, 8, 16, 32}) run<1, 0>(w, out, sms);
    for (int w : {4, 8, 16, 32}) run<2, 0>(w, out, sms);
    for (int w : {8, 16, 32}) run<1, 4>(w, out, sms);
    for (int w : {8, 16, 32}) run<1, 8>(w, out, sms);
    return 0;
}
