// Batched small-n expm in fp32 (n in {8, 16, 32, 64}): FFMA (never TF32)
// products, 1-norm and (m, s) selection in fp64. Implementation: expm_small_f32.cu.
#pragma once

#include <atomic>
#include <cstdint>
#include <cuda_runtime.h>

#include "mexp_b200.h"

namespace mexp_b200 {

int run_small_f32(const float* d_a, float* d_out, mexp_selection* d_sel, int np, int64_t batch,
                  int accuracy, cudaStream_t st, std::atomic<uint64_t>* launches);

}  // namespace mexp_b200
