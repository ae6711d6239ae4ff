// Batched C++ API of the drop-in: contiguous
// batches of row-major n x n matrices, fp64 or fp32, every matrix through the
// same path as mexp::expm (expm.hpp:37, expm.cpp:37-74) -- on-device 1-norm,
// (m, s) selection, scheme and squarings. A thin layer over the C ABI's
// batched entries (include/mexp_b200.h: mexp_expm_batched_host,
// mexp_expm_batched, mexp_expm_batched_host_multi); there is no CPU fallback.
//
// Per-matrix problems (a non-finite entry, a norm that overflows, a singular
// Pade denominator) do not throw: they are reported in that matrix's record
// (status != 0, e^A filled with NaN), as the batched C ABI does. Call-level
// problems throw like mexp::expm: std::invalid_argument for bad arguments,
// std::runtime_error for a missing device or a CUDA failure.
#pragma once

#include <cstdint>
#include <vector>

#include "mexp/theta_tables.hpp"

namespace mexp {

// arithmetic policy of the products and combinations (mexp_rounding):
// Reference = the reference's separately rounded multiplies and adds in its
// order (bit-identical e^A); Fast = FMA / tensor-core products; Auto = Fast
// except where squarings would amplify the difference past 50 n u.
enum class Rounding { Auto = 0, Reference = 1, Fast = 2 };

// one matrix's ExpmReport fields (expm.hpp:23-32) plus its status
struct BatchRecord {
    double norm_in = 0.0;
    int degree = 0;
    int s = 0;
    int status = 0;  // 0 ok, else an mexp_status (the matrix's e^A is NaN)
};

struct BatchResult {
    std::vector<BatchRecord> records;  // one per matrix
    std::int64_t first_error = -1;     // lowest index with status != 0, or -1
};

// Host buffers, synchronous: out[i] = e^{a[i]}, i < batch. Copies and
// kernels are pipelined over the current CUDA device (pinned buffers give the
// full PCIe rate).
BatchResult expm_batched(const double* a, double* out, int n, std::int64_t batch, Accuracy u,
                         Family family = Family::TaylorNew, Rounding rounding = Rounding::Auto);
BatchResult expm_batched(const float* a, float* out, int n, std::int64_t batch, Accuracy u,
                         Family family = Family::TaylorNew, Rounding rounding = Rounding::Auto);

// The same, sharded by matrix over several GPUs of this node (one host
// thread and one PCIe pipeline per device; empty `devices` = all visible).
BatchResult expm_batched_multi(const double* a, double* out, int n, std::int64_t batch, Accuracy u,
                               const std::vector<int>& devices = {},
                               Family family = Family::TaylorNew, Rounding rounding = Rounding::Auto);
BatchResult expm_batched_multi(const float* a, float* out, int n, std::int64_t batch, Accuracy u,
                               const std::vector<int>& devices = {},
                               Family family = Family::TaylorNew, Rounding rounding = Rounding::Auto);

// Device buffers, asynchronous on `stream` (a cudaStream_t; nullptr = the
// legacy default stream). d_records (may be nullptr) receives one 16-byte
// mexp_selection per matrix in device memory.
void expm_batched_device(const double* d_a, double* d_out, int n, std::int64_t batch, Accuracy u,
                         Family family, Rounding rounding, void* d_records, void* stream);
void expm_batched_device(const float* d_a, float* d_out, int n, std::int64_t batch, Accuracy u,
                         Family family, Rounding rounding, void* d_records, void* stream);

}  // namespace mexp
