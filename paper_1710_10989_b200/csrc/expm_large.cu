#include "expm_large.cuh"

namespace mexp_b200 {

int large_expm_f64(const double*, double*, mexp_selection*, int, int64_t, int, cudaStream_t,
                   std::atomic<uint64_t>*) {
    return MEXP_ERR_UNSUPPORTED;
}
int squarings_f64(double*, int, int64_t, int, int, cudaStream_t, std::atomic<uint64_t>*) {
    return MEXP_ERR_UNSUPPORTED;
}
const char* large_last_error() { return ""; }

}  // namespace mexp_b200
