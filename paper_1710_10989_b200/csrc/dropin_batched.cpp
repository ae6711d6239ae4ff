// Batched C++ API of the drop-in (include/mexp/batched.hpp) over the C ABI.
// Per-matrix statuses stay in the records; call-level statuses become the
// reference's exception types (as in dropin.cpp).
#include <stdexcept>
#include <string>
#include <vector>

#include "mexp/batched.hpp"
#include "mexp_b200.h"

namespace mexp {

namespace {

// the statuses a batched call returns for one matrix's data (reported per
// record, not thrown)
bool per_matrix(int st) {
    return st == MEXP_ERR_NONFINITE || st == MEXP_ERR_NORM_NONFINITE || st == MEXP_ERR_SINGULAR;
}

[[noreturn]] void throw_call_status(int st) {
    const char* msg = mexp_status_string(st);
    if (st == MEXP_ERR_INVALID_ARGUMENT || st == MEXP_ERR_UNSUPPORTED) throw std::invalid_argument(msg);
    if (st == MEXP_ERR_CUDA) throw std::runtime_error(std::string(msg) + ": " + mexp_last_cuda_error());
    throw std::runtime_error(msg);
}

void check_args(int n, std::int64_t batch, const void* a, const void* out) {
    if (n < 1) throw std::invalid_argument("matrix dimension must be positive");
    if (batch < 0) throw std::invalid_argument("batch must be nonnegative");
    if (batch > 0 && (!a || !out)) throw std::invalid_argument("null matrix buffer");
}

BatchResult to_result(const std::vector<mexp_selection>& sel, std::int64_t first_error) {
    BatchResult r;
    r.records.resize(sel.size());
    for (size_t i = 0; i < sel.size(); ++i)
        r.records[i] = BatchRecord{sel[i].norm_in, sel[i].degree, sel[i].s, sel[i].status};
    r.first_error = first_error;
    return r;
}

BatchResult host_call(const void* a, void* out, int dtype, int n, std::int64_t batch, Accuracy u,
                      Family family, Rounding rounding) {
    check_args(n, batch, a, out);
    std::vector<mexp_selection> sel(static_cast<size_t>(batch));
    int64_t first = -1;
    const int st = mexp_expm_batched_host(a, out, dtype, n, batch, int(u), int(family), int(rounding),
                                          sel.data(), &first);
    if (st != MEXP_OK && !per_matrix(st)) throw_call_status(st);
    return to_result(sel, first);
}

BatchResult multi_call(const void* a, void* out, int dtype, int n, std::int64_t batch, Accuracy u,
                       const std::vector<int>& devices, Family family, Rounding rounding) {
    check_args(n, batch, a, out);
    std::vector<mexp_selection> sel(static_cast<size_t>(batch));
    int64_t first = -1;
    const int st = mexp_expm_batched_host_multi(a, out, dtype, n, batch, int(u), int(family),
                                                int(rounding), sel.data(), &first,
                                                devices.empty() ? nullptr : devices.data(),
                                                int(devices.size()));
    if (st != MEXP_OK && !per_matrix(st)) throw_call_status(st);
    return to_result(sel, first);
}

void device_call(const void* d_a, void* d_out, int dtype, int n, std::int64_t batch, Accuracy u,
                 Family family, Rounding rounding, void* d_records, void* stream) {
    check_args(n, batch, d_a, d_out);
    const int st = mexp_expm_batched(d_a, d_out, dtype, n, batch, int(u), int(family), int(rounding),
                                     static_cast<mexp_selection*>(d_records), stream);
    if (st != MEXP_OK) throw_call_status(st);
}

}  // namespace

BatchResult expm_batched(const double* a, double* out, int n, std::int64_t batch, Accuracy u,
                         Family family, Rounding rounding) {
    return host_call(a, out, MEXP_F64, n, batch, u, family, rounding);
}
BatchResult expm_batched(const float* a, float* out, int n, std::int64_t batch, Accuracy u,
                         Family family, Rounding rounding) {
    return host_call(a, out, MEXP_F32, n, batch, u, family, rounding);
}
BatchResult expm_batched_multi(const double* a, double* out, int n, std::int64_t batch, Accuracy u,
                               const std::vector<int>& devices, Family family, Rounding rounding) {
    return multi_call(a, out, MEXP_F64, n, batch, u, devices, family, rounding);
}
BatchResult expm_batched_multi(const float* a, float* out, int n, std::int64_t batch, Accuracy u,
                               const std::vector<int>& devices, Family family, Rounding rounding) {
    return multi_call(a, out, MEXP_F32, n, batch, u, devices, family, rounding);
}
void expm_batched_device(const double* d_a, double* d_out, int n, std::int64_t batch, Accuracy u,
                         Family family, Rounding rounding, void* d_records, void* stream) {
    device_call(d_a, d_out, MEXP_F64, n, batch, u, family, rounding, d_records, stream);
}
void expm_batched_device(const float* d_a, float* d_out, int n, std::int64_t batch, Accuracy u,
                         Family family, Rounding rounding, void* d_records, void* stream) {
    device_call(d_a, d_out, MEXP_F32, n, batch, u, family, rounding, d_records, stream);
}

}  // namespace mexp
