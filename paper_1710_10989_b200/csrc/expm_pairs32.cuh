// Batched 32x32 fp32 expm, Family::TaylorNew: two same-class matrices per
// warp with TMEM-parked intermediates. Implementation: expm32_pairs.cu.
#pragma once

#include <atomic>
#include <cstdint>
#include <cuda_runtime.h>

#include "mexp_b200.h"

namespace mexp_b200 {

// whether a batch of 32x32 fp32 TaylorNew matrices takes the pair kernel
// (MEXP_F32_PAIRS overrides: 0 never, 1 always)
bool pairs32_enabled(int64_t batch);

int run_pairs32_f32(const float* d_a, float* d_out, mexp_selection* d_sel, int64_t batch,
                    int accuracy, cudaStream_t st, std::atomic<uint64_t>* launches);

}  // namespace mexp_b200
