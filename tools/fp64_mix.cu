// How DFMA and DMMA share an SM sub-partition's FP64 pipe (B200): cycles per
// "unit" = NM DMMAs + ND DFMAs for several ways of arranging them.
//   mode 0: every warp: NM chained DMMAs, then ND dependent DFMAs
//   mode 1: every warp: NM chained DMMAs, then ND DFMAs in 4 independent chains
//   mode 2: warp-specialised: even warps only DMMAs, odd warps only DFMAs
//           (each unit's work split across a warp pair)
//   mode 3: like 1 but DMUL+DADD pairs instead of DFMAs (reference rounding)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/fp64_mix tools/fp64_mix.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}

template <int MODE, int NM, int ND>
__global__ void k(double* out, int iters) {
    double c0 = 0, c1 = 0;
    double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
    double f[4] = {0.5, 0.25, 0.125, 0.0625};
    const int w = threadIdx.x >> 5;
    for (int i = 0; i < iters; ++i) {
        if (MODE == 2) {
            if (w & 1) {
#pragma unroll
                for (int d = 0; d < 2 * ND; ++d) f[d & 3] = fma(f[d & 3], b, a);
            } else {
#pragma unroll
                for (int m = 0; m < 2 * NM; ++m) dmma(c0, c1, a, b);
            }
        } else {
#pragma unroll
            for (int m = 0; m < NM; ++m) dmma(c0, c1, a, b);
            if (MODE == 0) {
#pragma unroll
                for (int d = 0; d < ND; ++d) f[0] = fma(f[0], b, a);
            } else if (MODE == 1) {
#pragma unroll
                for (int d = 0; d < ND; ++d) f[d & 3] = fma(f[d & 3], b, a);
            } else {
#pragma unroll
                for (int d = 0; d < ND / 2; ++d) f[d & 3] = __dadd_rn(f[d & 3], __dmul_rn(b, a + f[(d + 1) & 3]));
            }
        }
    }
    double s = c0 + c1 + f[0] + f[1] + f[2] + f[3];
    if (s == 1234.5) out[0] = s;
}

template <int MODE, int NM, int ND>
void run(int warps, double* out, int sms, double ghz) {
    const int iters = 4096;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e30f;
    for (int r = 0; r < 3; ++r) {
        cudaEventRecord(e0);
        k<MODE, NM, ND><<<sms, 32 * warps>>>(out, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    // units per SMSP: warps/4 * iters
    const double cyc = best * 1e-3 * ghz * 1e9 / (warps / 4.0 * iters);
    printf("{\"mode\": %d, \"dmma\": %d, \"dfma\": %d, \"warps_per_sm\": %d, \"cycles_per_unit\": %.1f, "
           "\"ideal\": %d}\n", MODE, NM, ND, warps, cyc, 16 * NM + 2 * ND);
}

int main() {
    int sms = 0, khz = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&khz, cudaDevAttrClockRate, 0);
    const double ghz = 1.965;
    double* out;
    cudaMalloc(&out, 64);
    for (int w : {16, 32}) {
        run<0, 2, 0>(w, out, sms, ghz);
        run<1, 0, 8>(w, out, sms, ghz);
        run<3, 0, 8>(w, out, sms, ghz);
        run<0, 2, 8>(w, out, sms, ghz);
        run<1, 2, 8>(w, out, sms, ghz);
        run<2, 2, 8>(w, out, sms, ghz);
        run<3, 2, 8>(w, out, sms, ghz);
        run<1, 2, 4>(w, out, sms, ghz);
        run<1, 2, 16>(w, out, sms, ghz);
        run<1, 4, 16>(w, out, sms, ghz);
        run<1, 8, 32>(w, out, sms, ghz);
        run<2, 8, 32>(w, out, sms, ghz);
        run<1, 1, 4>(w, out, sms, ghz);
    }
    return 0;
}
