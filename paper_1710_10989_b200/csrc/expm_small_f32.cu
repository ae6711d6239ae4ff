#include "expm_small_f32.cuh"

namespace mexp_b200 {

int run_small_f32(const float*, float*, mexp_selection*, int, int64_t, int, cudaStream_t,
                  std::atomic<uint64_t>*) {
    return MEXP_ERR_UNSUPPORTED;
}

}  // namespace mexp_b200
