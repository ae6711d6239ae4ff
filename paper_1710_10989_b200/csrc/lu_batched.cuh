// Batched pivoted LU solve X = M^-1 R for the large-n Pade path
// (pade_solve, pade.cpp:26-28 -> lu_solve, kernels.cpp:55-112). Implementation:
// lu_batched.cu.
#pragma once

#include <atomic>
#include <cstdint>
#include <cuda_runtime.h>

#include "mexp_b200.h"

namespace mexp_b200 {

// For each listed matrix m (indices into batches of np x np row-major
// matrices): factor M[m] in place (P M = L U), and overwrite R[m] with
// M[m]^-1 R[m]. A zero pivot column sets sel[m].status = MEXP_ERR_SINGULAR.
// np must be a multiple of 64. Asynchronous on `st`.
int lu_solve_batched(double* M, double* R, int np, int64_t batch, const int32_t* d_list, int count,
                     mexp_selection* d_sel, cudaStream_t st, std::atomic<uint64_t>* launches);

const char* lu_last_error();

}  // namespace mexp_b200
