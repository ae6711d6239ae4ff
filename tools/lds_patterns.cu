// Shared-memory wavefronts per LDS.128 / LDS.64 for lane -> address maps with
// broadcast (B200), counted by ncu: one launch per pattern, one warp, 1024 loads.
//   ncu --metrics l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,smsp__inst_executed_op_shared_ld.sum ./tools/lds_patterns
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/lds_patterns tools/lds_patterns.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ int unit_of(int pat, int lane) {
    switch (pat) {
        case 0: return lane;                 // 32 distinct units
        case 1: return lane >> 2;            // 8 units, groups of 4 consecutive lanes
        case 2: return lane & 3;             // 4 units, lanes strided by 4 share
        case 3: return lane >> 3;            // 4 units, one per quarter-warp
        case 4: return lane & 7;             // 8 units, every quarter-warp reads all 8
        case 5: return 0;                    // one unit
        case 6: return (lane >> 2) & 3;      // 4 units, groups of 4, repeated per half-warp
        case 7: return lane >> 1;            // 16 units, pairs
        case 8: return lane & 1;             // 2 units alternating
        case 9: return lane & 15;            // 16 units, both half-warps read all
        case 10: return (lane >> 3) * 9;     // 4 units one per quarter, distinct bank groups
        case 11: return (lane >> 4);         // 2 units, one per half-warp
        default: return ((lane >> 3) & 1) | ((lane >> 4) << 3);  // quarter-uniform, spread
    }
}

template <int BYTES>
__global__ void k(int pat, int iters, unsigned* out) {
    __shared__ __align__(16) double sm[1024];
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) sm[i] = i;
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const unsigned p = (unsigned)__cvta_generic_to_shared(sm) + unit_of(pat, lane) * 16;
    unsigned acc = 0;
    for (int i = 0; i < iters; ++i) {
        if (BYTES == 16) {
            unsigned a, b, c, d;
            asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(a), "=r"(b), "=r"(c), "=r"(d) : "r"(p + ((i * 7) & 7) * 512) : "memory");
            acc += a * 3 + b * 5 + c * 7 + d;
        } else {
            unsigned a, b;
            asm volatile("ld.shared.v2.u32 {%0,%1}, [%2];" : "=r"(a), "=r"(b) : "r"(p + ((i * 7) & 7) * 512) : "memory");
            acc += a * 3 + b;
        }
    }
    if (acc == 12345u) out[0] = acc;
}

int main() {
    unsigned* out;
    cudaMalloc(&out, 64);
    for (int pat = 0; pat <= 12; ++pat) k<16><<<1, 32>>>(pat, 1024, out);
    for (int pat = 0; pat <= 12; ++pat) k<8><<<1, 32>>>(pat, 1024, out);
    cudaDeviceSynchronize();
    printf("done\n");
    return 0;
}
