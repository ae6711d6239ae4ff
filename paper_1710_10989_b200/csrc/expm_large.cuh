// Large-n (n > 64) fp64 expm engine: FP64 tensor-core (DMMA) GEMMs with the
// schemes' linear combinations fused into their epilogues, batched over
// matrices with per-matrix scaling exponents; all three families (the Pade
// solve through lu_batched.cuh). Implementation: expm_large.cu.
#pragma once

#include <atomic>
#include <cstdint>
#include <cuda_runtime.h>

#include "mexp_b200.h"

namespace mexp_b200 {

// acc_arg = mexp_accuracy | mexp_family << 4; rounding: MEXP_ROUND_REFERENCE
// runs every product and lincomb in the reference's arithmetic (bit-identical
// e^A; not for the Pade family), FAST the DMMA path, AUTO the reference's
// arithmetic for the matrices with s >= smin and DMMA for the rest (Taylor
// families; Pade is DMMA). Host-synchronous: returns MEXP_ERR_UNSUPPORTED
// when `st` is capturing a CUDA graph.
int large_expm_f64(const double* d_a, double* d_out, mexp_selection* d_sel, int n,
                   int64_t batch, int acc_arg, int rounding, int smin, cudaStream_t st,
                   std::atomic<uint64_t>* launches);

// C = A B for `batch` n x n fp64 matrices of any n (REFERENCE rounding:
// bit-identical to the reference's kernels::matmul). Host-synchronous.
int matmul_f64(const double* d_a, const double* d_b, double* d_c, int n, int64_t batch, int rounding,
               cudaStream_t st, std::atomic<uint64_t>* launches);

// X <- X^(2^s), in place, for `batch` n x n fp64 matrices.
int squarings_f64(double* d_x, int n, int64_t batch, int s, int rounding, cudaStream_t st,
                  std::atomic<uint64_t>* launches);

const char* large_last_error();

}  // namespace mexp_b200
