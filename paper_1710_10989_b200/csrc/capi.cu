// C ABI of the B200 expm path (declarations: include/mexp_b200.h).
//
// Dispatch: n <= 64 runs the small-n group kernels (matrices zero-padded to
// n in {8, 16, 32, 64} when needed: padding with zeros leaves the 1-norm, the
// selection and -- in reference rounding -- every rounding of the top-left
// block unchanged, since each padded term adds an exact +0 to a sum that is
// never -0). n > 64 runs the DMMA GEMM engine (expm_large.cu).
#include <atomic>
#include <chrono>
#include <climits>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "async_buffer.hpp"
#include "device_once.hpp"
#include "expm_cluster.cuh"
#include "expm_common.cuh"
#include "expm_large.cuh"
#include "expm_n8.cuh"
#include "expm_pade8.cuh"
#include "expm_small.cuh"
#include "expm_small_f32.cuh"

using namespace mexp_b200;

namespace {

thread_local std::string g_last_cuda_error;
std::atomic<uint64_t> g_launches{0};

int cuda_fail(cudaError_t e, const char* where) {
    g_last_cuda_error = std::string(where) + ": " + cudaGetErrorString(e);
    return MEXP_ERR_CUDA;
}
#define MEXP_CUDA(call)                                        \
    do {                                                       \
        cudaError_t e_ = (call);                               \
        if (e_ != cudaSuccess) return cuda_fail(e_, #call);    \
    } while (0)

int device_ok() {
    int count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) {
        cudaGetLastError();
        return MEXP_ERR_NO_DEVICE;
    }
    return MEXP_OK;
}

int padded_n(int n) { return n <= 8 ? 8 : n <= 16 ? 16 : n <= 32 ? 32 : n <= 64 ? 64 : n; }

bool valid_args(int dtype, int n, int64_t batch, int accuracy, int family, int rounding) {
    return (dtype == MEXP_F64 || dtype == MEXP_F32) && n >= 1 && batch >= 0 &&
           (accuracy == MEXP_ACCURACY_SINGLE || accuracy == MEXP_ACCURACY_DOUBLE) &&
           (family >= 0 && family <= 2) && (rounding >= 0 && rounding <= 2);
}

// the kernels' `acc_arg`: accuracy in the low nibble, family above it
int acc_arg(int accuracy, int family) { return accuracy | (family << 4); }
// Pade evaluation: the public family, or reference_expm's internal one
bool is_pade(int aarg) {
    return (aarg >> 4) == MEXP_FAMILY_PADE || (aarg >> 4) == kFamilyPadeReference;
}

// Rounding threshold of the AUTO policy: matrices with s >= this run the
// reference-exact arithmetic. Each squaring roughly doubles the relative
// difference between two roundings of T_m, while the tolerance 50*n*u grows
// with n; FMA-rounded results leave the band for n = 8 only from s = 6 on
// (SURVEY.md key finding 3) and for n = 1 from s = 4 on (golden cases), so
// the threshold is 3 + floor(log2 n), taken on the caller's n before padding
// (n > 64 too: the large-n engine runs those matrices on the k-ordered exact
// GEMMs). Checked on every gallery kind, n = 2..512, s up to 14
// (tests/test_gpu_auto_stress.py).
int exact_s_min(int n) {
    if (n < 8) return 0;  // tiny n: 50*n*u is too tight for any other rounding: all exact
    int l = 0;
    while ((2 << l) <= n) ++l;
    return 3 + l;
}

// zero-pad n -> np (and widen float -> double for the fp32 Pade path)
template <class S, class D>
__global__ void pad_kernel(const S* __restrict__ src, D* __restrict__ dst, int n, int np,
                           int64_t batch) {
    const int64_t total = batch * int64_t(np) * np;
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < total;
         i += int64_t(gridDim.x) * blockDim.x) {
        const int64_t b = i / (int64_t(np) * np);
        const int r = int((i / np) % np), c = int(i % np);
        dst[i] = (r < n && c < n) ? D(src[b * n * n + r * n + c]) : D(0);
    }
}
// top-left n x n of each np x np block (and narrow double -> float, rounding once)
template <class S, class D>
__global__ void unpad_kernel(const S* __restrict__ src, D* __restrict__ dst, int n, int np,
                             int64_t batch) {
    const int64_t total = batch * int64_t(n) * n;
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < total;
         i += int64_t(gridDim.x) * blockDim.x) {
        const int64_t b = i / (int64_t(n) * n);
        const int r = int((i / n) % n), c = int(i % n);
        dst[i] = D(src[b * np * np + r * np + c]);
    }
}

int num_sms() {
    static int sms = [] {
        int dev = 0, v = 148;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
        return v;
    }();
    return sms;
}

template <int N, int GPC, int kFamily>
int launch_small_f64(const double* a, double* out, mexp_selection* sel, int64_t batch,
                     int accuracy, int rounding, int smin, cudaStream_t st) {
    using G = Group<N>;
    auto kern = expm_small_f64_kernel<N, GPC, kFamily>;
    const size_t smem = size_t(G::SMEM_DOUBLES) * GPC * sizeof(double);
    static PerDevice attr_once;
    attr_once([&] { cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)); });
    static int blocks_per_sm = [&] {
        int b = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, kern, 32 * G::W * GPC, smem);
        return b > 0 ? b : 1;
    }();
    const int64_t want = (batch + GPC - 1) / GPC;
    const int64_t cap = int64_t(blocks_per_sm) * num_sms();
    const int grid = int(want < cap ? want : cap);
    if (grid == 0) return MEXP_OK;
    kern<<<grid, 32 * G::W * GPC, smem, st>>>(a, out, sel, batch, accuracy, rounding, smin);
    g_launches.fetch_add(1, std::memory_order_relaxed);
    MEXP_CUDA(cudaGetLastError());
    return MEXP_OK;
}

// Slots of {work counter, finished-CTA counter} for kernels that hand out
// work dynamically; each kernel leaves its slot zeroed (release_ticket), so
// no memset per launch. Eager launches take the next slot of a 4096-slot ring
// per device (concurrent launches on other streams get distinct slots). A
// launch captured into a CUDA graph keeps its slot for the graph's lifetime
// and its replays may overlap later eager launches, so captured launches take
// slots of a separate 65536-slot region that is never handed out again
// (allocated with the ring, outside any capture).
int next_ticket(cudaStream_t st, unsigned long long** out) {
    constexpr int kSlots = 4096;
    constexpr int kCaptureSlots = 65536;
    static std::atomic<unsigned long long*> ring[16] = {};
    static std::atomic<uint32_t> next[16];
    static std::atomic<uint32_t> next_captured[16];
    int dev = 0;
    MEXP_CUDA(cudaGetDevice(&dev));
    dev &= 15;
    unsigned long long* base = ring[dev].load(std::memory_order_acquire);
    if (!base) {
        static std::mutex mu;
        std::lock_guard<std::mutex> lock(mu);
        base = ring[dev].load(std::memory_order_acquire);
        if (!base) {
            const size_t bytes = 2 * sizeof(unsigned long long) * (kSlots + kCaptureSlots);
            MEXP_CUDA(cudaMalloc(&base, bytes));
            MEXP_CUDA(cudaMemset(base, 0, bytes));
            ring[dev].store(base, std::memory_order_release);
        }
    }
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    MEXP_CUDA(cudaStreamIsCapturing(st, &cap));
    if (cap == cudaStreamCaptureStatusActive) {
        const uint32_t i = next_captured[dev].fetch_add(1);
        if (i < uint32_t(kCaptureSlots)) {
            *out = base + 2 * (kSlots + i);
            return MEXP_OK;
        }
        // more than 65536 captured launches in this process: fall back to the ring
    }
    const uint32_t i = next[dev].fetch_add(1) % kSlots;
    *out = base + 2 * i;
    return MEXP_OK;
}

// AUTO keeps the reference's rounding to the last squaring of its
// reference-rounded matrices: a fast-rounded tail was measured (round 1:
// profiles/cfg2_fast_tail_r1.txt) and then found to leave the 50*n*u band on
// nearly idempotent X (the gallery's rank-one kind, 2.3x at s = 14,
// tests/test_gpu_auto_stress.py), so the knob is gone.

// 8x8 variant (experiments; default chosen from the measurements in
// profiles/): bit 0 = split DMMA accumulation, bit 1 = defer reference-rounded
// matrices to a second kernel. MEXP_N8_VARIANT overrides.
int n8_variant() {
    static int v = [] {
        const char* e = std::getenv("MEXP_N8_VARIANT");
        // 12 (default): the pipelined kernel (expm8_pipe_kernel); 15: the same with
        // static rounds. 0: the round-1/2 kernel (expm8_f64_kernel) with chained
        // DMMAs and the reference-rounded matrices inline; 1, 2, 4, 5: its split /
        // deferred / lower-occupancy variants (profiles/cfg2_variants_r1.txt, _r2.txt)
        return e ? std::atoi(e) : 12;
    }();
    return v;
}

template <bool kSplit, int kDefer, int kMinBlocks = 8, int kFamily = MEXP_FAMILY_TAYLOR_NEW>
int launch_n8_variant(const double* a, double* out, mexp_selection* sel, int64_t batch,
                      int accuracy, int rounding, int smin, cudaStream_t st) {
    auto kern = expm8_f64_kernel<kSplit, kDefer, kMinBlocks, kFamily>;
    auto exact_kern = expm8_exact_kernel<kFamily>;
    static int blocks_per_sm = [&] {
        int b = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, kern, 32 * kN8WarpsPerBlock, 0);
        return b > 0 ? b : 1;
    }();
    static int exact_bps = [&] {
        int b = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, exact_kern, 32 * kN8WarpsPerBlock, 0);
        return b > 0 ? b : 1;
    }();
    const int64_t cap = int64_t(blocks_per_sm) * num_sms();
    if (kDefer && rounding == MEXP_ROUND_REFERENCE) {
        // every matrix is reference-rounded: the exact kernel alone
        const int64_t want = (batch + kN8WarpsPerBlock - 1) / kN8WarpsPerBlock;
        const int64_t ecap = int64_t(exact_bps) * num_sms();
        const int grid = int(want < ecap ? want : ecap);
        exact_kern<<<grid, 32 * kN8WarpsPerBlock, 0, st>>>(a, out, sel, batch, accuracy, nullptr,
                                                           nullptr);
        g_launches.fetch_add(1, std::memory_order_relaxed);
        MEXP_CUDA(cudaGetLastError());
        return MEXP_OK;
    }
    AsyncBuffer work_buf(st);
    int32_t* work = nullptr;
    const bool defer = kDefer && rounding == MEXP_ROUND_AUTO;
    if (defer) {
        MEXP_CUDA(work_buf.alloc(sizeof(int32_t) * (batch + 1)));
        work = work_buf.get<int32_t>();
        MEXP_CUDA(cudaMemsetAsync(work + batch, 0, sizeof(int32_t), st));
    }
    const int64_t want = (batch + 4 * kN8WarpsPerBlock - 1) / (4 * kN8WarpsPerBlock);
    const int grid = int(want < cap ? want : cap);
    // work ticket for the dynamically distributed rounds: a slot of a
    // persistent per-device ring, reset in stream order
    unsigned long long* ticket = nullptr;
    {
        int r = next_ticket(st, &ticket);
        if (r != MEXP_OK) return r;
    }
    const int rounding_arg = rounding;
    kern<<<grid, 32 * kN8WarpsPerBlock, 0, st>>>(a, out, sel, batch, accuracy, rounding_arg, smin,
                                                 work, defer ? work + batch : nullptr, ticket);
    g_launches.fetch_add(1, std::memory_order_relaxed);
    MEXP_CUDA(cudaGetLastError());
    if (defer) {
        const int egrid = int(int64_t(exact_bps) * num_sms());
        exact_kern<<<egrid, 32 * kN8WarpsPerBlock, 0, st>>>(a, out, sel, batch, accuracy, work,
                                                            work + batch);
        g_launches.fetch_add(1, std::memory_order_relaxed);
        MEXP_CUDA(cudaGetLastError());
    }
    return MEXP_OK;
}

// Few matrices of np = 64 (cfg1: one): a 4-CTA cluster per matrix instead of
// one CTA (expm_cluster.cuh). Used while the clusters fit in about two waves
// of the SMs; MEXP_CLUSTER_MAX overrides the batch limit (0 disables).
int64_t cluster_max_batch() {
    static int64_t v = [] {
        const char* e = std::getenv("MEXP_CLUSTER_MAX");
        return e ? int64_t(std::atoll(e)) : int64_t(2 * num_sms() / kClusterCtas);
    }();
    return v;
}

template <int kFamily>
int launch_cluster64_family(const double* a, double* out, mexp_selection* sel, int64_t batch,
                            int accuracy, int rounding, int smin, cudaStream_t st) {
    using G = ClusterGroup64;
    const size_t smem = size_t(G::SMEM_DOUBLES) * sizeof(double);
    static PerDevice attr_once;
    attr_once([&] {
        cudaFuncSetAttribute(expm64_cluster_kernel<kFamily>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             int(smem));
    });
    const int grid = int(batch) * kClusterCtas;
    expm64_cluster_kernel<kFamily><<<grid, G::THREADS, smem, st>>>(a, out, sel, batch, accuracy,
                                                                   rounding, smin);
    g_launches.fetch_add(1, std::memory_order_relaxed);
    MEXP_CUDA(cudaGetLastError());
    return MEXP_OK;
}

int launch_cluster64(const double* a, double* out, mexp_selection* sel, int64_t batch, int accuracy,
                     int rounding, int smin, cudaStream_t st) {
    if ((accuracy >> 4) == MEXP_FAMILY_TAYLOR_PS)
        return launch_cluster64_family<MEXP_FAMILY_TAYLOR_PS>(a, out, sel, batch, accuracy, rounding,
                                                              smin, st);
    return launch_cluster64_family<MEXP_FAMILY_TAYLOR_NEW>(a, out, sel, batch, accuracy, rounding,
                                                           smin, st);
}

// `accuracy` here and below is the kernels' acc_arg (mexp_accuracy | family << 4)
template <int N, int GPC>
int launch_small_family(const double* a, double* out, mexp_selection* sel, int64_t batch,
                        int accuracy, int rounding, int smin, cudaStream_t st) {
    if ((accuracy >> 4) == MEXP_FAMILY_TAYLOR_PS)
        return launch_small_f64<N, GPC, MEXP_FAMILY_TAYLOR_PS>(a, out, sel, batch, accuracy,
                                                               rounding, smin, st);
    if (is_pade(accuracy))
        return launch_small_f64<N, GPC, MEXP_FAMILY_PADE>(a, out, sel, batch, accuracy, rounding,
                                                          smin, st);
    return launch_small_f64<N, GPC, MEXP_FAMILY_TAYLOR_NEW>(a, out, sel, batch, accuracy, rounding,
                                                            smin, st);
}

int launch_pade8(const double* a, double* out, mexp_selection* sel, int64_t batch, int accuracy,
                 int rounding, int smin, cudaStream_t st) {
    static int blocks_per_sm = [] {
        int b = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, expm8_pade_kernel<8>, 32 * kN8WarpsPerBlock, 0);
        return b > 0 ? b : 1;
    }();
    const int64_t cap = int64_t(blocks_per_sm) * num_sms();
    const int64_t want = (batch + 4 * kN8WarpsPerBlock - 1) / (4 * kN8WarpsPerBlock);
    const int grid = int(want < cap ? want : cap);
    unsigned long long* ticket = nullptr;
    const int r = next_ticket(st, &ticket);
    if (r != MEXP_OK) return r;
    expm8_pade_kernel<8><<<grid, 32 * kN8WarpsPerBlock, 0, st>>>(a, out, sel, batch, accuracy, rounding,
                                                                 smin, ticket);
    g_launches.fetch_add(1, std::memory_order_relaxed);
    MEXP_CUDA(cudaGetLastError());
    return MEXP_OK;
}

// The pipelined 8x8 kernel (expm_n8.cuh expm8_pipe_kernel): the default for
// the Taylor families. kClaimAt / kPF: the matrix of a round before which the
// next round is claimed / its copy issued.
template <int kFamily, int kClaimAt, int kPF, int kMinBlocks = 8>
int launch_n8_pipe(const double* a, double* out, mexp_selection* sel, int64_t batch, int accuracy,
                   int rounding, int smin, cudaStream_t st) {
    auto kern = expm8_pipe_kernel<kFamily, kClaimAt, kPF, kMinBlocks>;
    static int blocks_per_sm = [&] {
        int b = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, kern, 32 * kN8WarpsPerBlock, 0);
        return b > 0 ? b : 1;
    }();
    const int64_t cap = int64_t(blocks_per_sm) * num_sms();
    const int64_t want = (batch + 4 * kN8WarpsPerBlock - 1) / (4 * kN8WarpsPerBlock);
    const int grid = int(want < cap ? want : cap);
    unsigned long long* ticket = nullptr;
    {
        int r = next_ticket(st, &ticket);
        if (r != MEXP_OK) return r;
    }
    N8Params prm;
    for (int e = 0; e < 6; ++e) prm.theta[e] = theta_entry(kFamily, accuracy & 15, e);
    prm.accuracy = accuracy & 15;
    prm.exact_from_s = rounding == MEXP_ROUND_REFERENCE ? 0
                       : rounding == MEXP_ROUND_AUTO    ? smin
                                                        : INT_MAX;
    // rounds dealt round-robin before the ticket takes over, as a percentage of
    // the batch (MEXP_N8_STATIC_PCT): 0 = every round after a warp's first is claimed
    static const int static_pct = [] {
        const char* e = std::getenv("MEXP_N8_STATIC_PCT");
        const int v = e ? std::atoi(e) : 0;
        return v < 0 ? 0 : v > 100 ? 100 : v;
    }();
    const uint32_t nwarps = uint32_t(grid) * kN8WarpsPerBlock;
    const uint64_t rounds = uint64_t((batch + 3) / 4);
    uint64_t passes = rounds * uint64_t(static_pct) / 100 / nwarps;
    if (passes < 1) passes = 1;  // the first round of every warp is its own
    prm.static_rounds = uint32_t(passes * nwarps);
    kern<<<grid, 32 * kN8WarpsPerBlock, 0, st>>>(a, out, sel, batch, prm, ticket);
    g_launches.fetch_add(1, std::memory_order_relaxed);
    MEXP_CUDA(cudaGetLastError());
    return MEXP_OK;
}

// the pipelined kernel keeps its round index in 32 bits
bool n8_pipe_ok(int64_t batch) { return batch < (int64_t(1) << 33); }

int launch_n8_f64(const double* a, double* out, mexp_selection* sel, int64_t batch,
                  int accuracy, int rounding, int smin, cudaStream_t st) {
    if (batch == 0) return MEXP_OK;
    if (is_pade(accuracy)) {  // four matrices per warp, the LU on all 32 lanes
        static const bool generic = std::getenv("MEXP_PADE8_GENERIC") != nullptr;
        if (generic)
            return launch_small_f64<8, 8, MEXP_FAMILY_PADE>(a, out, sel, batch, accuracy, rounding,
                                                           smin, st);
        return launch_pade8(a, out, sel, batch, accuracy, rounding, smin, st);
    }
    const int variant = n8_pipe_ok(batch) ? n8_variant() : 0;
    if ((accuracy >> 4) == MEXP_FAMILY_TAYLOR_PS) {  // the default variants only
        if (variant == 12)
            return launch_n8_pipe<MEXP_FAMILY_TAYLOR_PS, 1, 3>(a, out, sel, batch, accuracy, rounding,
                                                               smin, st);
        return launch_n8_variant<false, 0, 8, MEXP_FAMILY_TAYLOR_PS>(a, out, sel, batch, accuracy,
                                                                     rounding, smin, st);
    }
    switch (variant) {
        case 12: return launch_n8_pipe<MEXP_FAMILY_TAYLOR_NEW, 1, 3>(a, out, sel, batch, accuracy, rounding, smin, st);
        case 15: return launch_n8_pipe<MEXP_FAMILY_TAYLOR_NEW, -1, 3>(a, out, sel, batch, accuracy, rounding, smin, st);
        case 0: return launch_n8_variant<false, 0>(a, out, sel, batch, accuracy, rounding, smin, st);
        case 1: return launch_n8_variant<true, 0>(a, out, sel, batch, accuracy, rounding, smin, st);
        case 2: return launch_n8_variant<false, 1>(a, out, sel, batch, accuracy, rounding, smin, st);
        case 4: return launch_n8_variant<false, 0, 6>(a, out, sel, batch, accuracy, rounding, smin, st);
        case 5: return launch_n8_variant<false, 0, 7>(a, out, sel, batch, accuracy, rounding, smin, st);
        default: return launch_n8_variant<true, 1>(a, out, sel, batch, accuracy, rounding, smin, st);
    }
}

int run_small_f64(const double* a, double* out, mexp_selection* sel, int np, int64_t batch,
                  int accuracy, int rounding, int smin, cudaStream_t st) {
    switch (np) {
        case 8: return launch_n8_f64(a, out, sel, batch, accuracy, rounding, smin, st);
        case 16: return launch_small_family<16, 4>(a, out, sel, batch, accuracy, rounding, smin, st);
        case 32: return launch_small_family<32, 2>(a, out, sel, batch, accuracy, rounding, smin, st);
        case 64:
            if (!is_pade(accuracy) && batch <= cluster_max_batch())
                return launch_cluster64(a, out, sel, batch, accuracy, rounding, smin, st);
            return launch_small_family<64, 1>(a, out, sel, batch, accuracy, rounding, smin, st);
    }
    return MEXP_ERR_UNSUPPORTED;
}

// Device-buffer entry, no argument validation (callers validated).
int expm_device(const void* d_a, void* d_out, int dtype, int n, int64_t batch, int accuracy,
                int rounding, mexp_selection* d_sel, cudaStream_t st) {
    if (batch == 0) return MEXP_OK;
    if (n > 64) {
        // DMMA products, or for REFERENCE rounding the k-ordered exact ones
        // (taylor-new / taylor-ps; the Pade LU is DMMA only)
        if (dtype == MEXP_F64) {
            const int r = large_expm_f64(static_cast<const double*>(d_a), static_cast<double*>(d_out),
                                         d_sel, n, batch, accuracy, rounding, exact_s_min(n), st,
                                         &g_launches);
            if (r == MEXP_ERR_CUDA) g_last_cuda_error = large_last_error();
            return r;
        }
        // fp32 storage beyond n = 64: the correctly rounded path is the fp64
        // DMMA engine on the exactly widened values (the reference's own
        // arithmetic), e^A rounded once to float -- never TF32
        const size_t bytes = size_t(batch) * n * n * sizeof(double);
        AsyncBuffer bin(st), bout(st);
        MEXP_CUDA(bin.alloc(bytes));
        MEXP_CUDA(bout.alloc(bytes));
        double* win = bin.get<double>();
        double* wout = bout.get<double>();
        const int grid = 4 * num_sms();
        pad_kernel<<<grid, 256, 0, st>>>(static_cast<const float*>(d_a), win, n, n, batch);
        g_launches.fetch_add(1, std::memory_order_relaxed);
        const int r = large_expm_f64(win, wout, d_sel, n, batch, accuracy, rounding, exact_s_min(n), st,
                                     &g_launches);
        if (r == MEXP_ERR_CUDA) g_last_cuda_error = large_last_error();
        if (r != MEXP_OK) return r;
        unpad_kernel<<<grid, 256, 0, st>>>(wout, static_cast<float*>(d_out), n, n, batch);
        g_launches.fetch_add(1, std::memory_order_relaxed);
        MEXP_CUDA(cudaGetLastError());
        return MEXP_OK;
    }
    const int np = padded_n(n);
    if (dtype == MEXP_F32 && is_pade(accuracy)) {
        // fp32 storage, fp64 evaluation: the LU solve of a Pade denominator
        // amplifies fp32 rounding by cond(V - U), which reaches ~1e3 at the
        // Single table's thetas (up to 11.2), so the fp32 Pade path widens to
        // the fp64 engine -- the reference's own arithmetic -- and rounds
        // e^A once to float
        const size_t bytes = size_t(batch) * np * np * sizeof(double);
        AsyncBuffer bin(st), bout(st);
        MEXP_CUDA(bin.alloc(bytes));
        MEXP_CUDA(bout.alloc(bytes));
        double* win = bin.get<double>();
        double* wout = bout.get<double>();
        const int grid = 4 * num_sms();
        pad_kernel<<<grid, 256, 0, st>>>(static_cast<const float*>(d_a), win, n, np, batch);
        g_launches.fetch_add(1, std::memory_order_relaxed);
        const int r = run_small_f64(win, wout, d_sel, np, batch, accuracy, rounding, exact_s_min(n), st);
        if (r != MEXP_OK) return r;
        unpad_kernel<<<grid, 256, 0, st>>>(wout, static_cast<float*>(d_out), n, np, batch);
        g_launches.fetch_add(1, std::memory_order_relaxed);
        MEXP_CUDA(cudaGetLastError());
        return MEXP_OK;
    }
    const size_t esz = dtype == MEXP_F64 ? sizeof(double) : sizeof(float);
    const void* src = d_a;
    void* dst = d_out;
    AsyncBuffer bin(st), bout(st);
    void* pin = nullptr;
    void* pout = nullptr;
    if (np != n) {
        const size_t bytes = size_t(batch) * np * np * esz;
        MEXP_CUDA(bin.alloc(bytes));
        MEXP_CUDA(bout.alloc(bytes));
        pin = bin.get<void>();
        pout = bout.get<void>();
        const int grid = 4 * num_sms();
        if (dtype == MEXP_F64)
            pad_kernel<<<grid, 256, 0, st>>>(static_cast<const double*>(d_a), static_cast<double*>(pin),
                                             n, np, batch);
        else
            pad_kernel<<<grid, 256, 0, st>>>(static_cast<const float*>(d_a), static_cast<float*>(pin),
                                             n, np, batch);
        g_launches.fetch_add(1, std::memory_order_relaxed);
        src = pin;
        dst = pout;
    }
    int r;
    if (dtype == MEXP_F64) {
        r = run_small_f64(static_cast<const double*>(src), static_cast<double*>(dst), d_sel, np,
                          batch, accuracy, rounding, exact_s_min(n), st);
    } else {
        r = run_small_f32(static_cast<const float*>(src), static_cast<float*>(dst), d_sel, np,
                          batch, accuracy, st, &g_launches);
    }
    if (r != MEXP_OK) return r;
    if (np != n) {
        const int grid = 4 * num_sms();
        if (dtype == MEXP_F64)
            unpad_kernel<<<grid, 256, 0, st>>>(static_cast<const double*>(pout),
                                               static_cast<double*>(d_out), n, np, batch);
        else
            unpad_kernel<<<grid, 256, 0, st>>>(static_cast<const float*>(pout),
                                               static_cast<float*>(d_out), n, np, batch);
        g_launches.fetch_add(1, std::memory_order_relaxed);
    }
    MEXP_CUDA(cudaGetLastError());
    return MEXP_OK;
}

// ---- host pipeline state: per-device streams and chunk buffers ------------
struct HostPipe {
    static constexpr int kStreams = 8;  // capacity; host_streams() are used
    int device = -1;
    cudaStream_t st[kStreams] = {};
    void* d_in[kStreams] = {};
    void* d_out[kStreams] = {};
    mexp_selection* d_sel[kStreams] = {};
    size_t cap_bytes = 0;   // per-stream matrix buffer capacity
    int64_t cap_sel = 0;
    mexp_selection* h_sel_scratch = nullptr;  // pinned, used when the caller passes none
    std::vector<cudaEvent_t> ev;  // one per chunk of a call: its records have landed
    std::vector<cudaEvent_t> ev_in, ev_k;  // staged pipeline: chunk's H2D / kernel done
    int64_t h_sel_cap = 0;
    void* h_stage = nullptr;  // small calls: pinned staging for pageable A / e^A / records
    size_t h_stage_cap = 0;
    std::mutex mu;
};

// streams (and chunk buffer slots) of the host pipeline (MEXP_HOST_STREAMS,
// default 4, 3 to 8)
int host_streams() {
    static int v = [] {
        const char* e = std::getenv("MEXP_HOST_STREAMS");
        const int x = e ? std::atoi(e) : 4;
        return x < 3 ? 3 : (x > HostPipe::kStreams ? HostPipe::kStreams : x);
    }();
    return v;
}

HostPipe& pipe_for_current_device() {
    static HostPipe pipes[16];
    int dev = 0;
    cudaGetDevice(&dev);
    return pipes[dev & 15];
}

int ensure_pipe(HostPipe& p, size_t bytes, int64_t sels) {
    int dev = 0;
    MEXP_CUDA(cudaGetDevice(&dev));
    if (p.device != dev) {
        for (int i = 0; i < host_streams(); ++i)
            MEXP_CUDA(cudaStreamCreateWithFlags(&p.st[i], cudaStreamNonBlocking));
        p.device = dev;
    }
    if (bytes > p.cap_bytes || sels > p.cap_sel) {
        for (int i = 0; i < host_streams(); ++i) {
            MEXP_CUDA(cudaStreamSynchronize(p.st[i]));
            cudaFree(p.d_in[i]);
            cudaFree(p.d_out[i]);
            cudaFree(p.d_sel[i]);
            MEXP_CUDA(cudaMalloc(&p.d_in[i], bytes));
            MEXP_CUDA(cudaMalloc(&p.d_out[i], bytes));
            MEXP_CUDA(cudaMalloc(&p.d_sel[i], sizeof(mexp_selection) * sels));
        }
        p.cap_bytes = bytes;
        p.cap_sel = sels;
    }
    return MEXP_OK;
}

int expm_host_impl(const void* h_a, void* h_out, int dtype, int n, int64_t batch, int aarg,
                   int rounding, mexp_selection* h_sel, int64_t* first_error);

}  // namespace

namespace mexp_b200 {
// shared with dense_ops.cu: one launch counter and one last-error string
std::atomic<uint64_t>& library_launch_counter() { return g_launches; }
void set_last_cuda_error(const std::string& e) { g_last_cuda_error = e; }
}  // namespace mexp_b200

extern "C" {

int mexp_abi_version(void) { return MEXP_B200_ABI_VERSION; }

int mexp_device_check(void) {
    const int r = device_ok();
    if (r != MEXP_OK) return r;
    int dev = 0, major = 0;
    MEXP_CUDA(cudaGetDevice(&dev));
    MEXP_CUDA(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev));
    return major == 10 ? MEXP_OK : MEXP_ERR_NO_DEVICE;
}

const char* mexp_status_string(int status) {
    switch (status) {
        case MEXP_OK: return "ok";
        case MEXP_ERR_NONFINITE: return "non-finite matrix entry";
        case MEXP_ERR_NORM_NONFINITE: return "norm must be finite and nonnegative";
        case MEXP_ERR_INVALID_ARGUMENT: return "invalid argument";
        case MEXP_ERR_UNSUPPORTED: return "unsupported on the B200 path";
        case MEXP_ERR_CUDA: return "CUDA error";
        case MEXP_ERR_NO_DEVICE: return "no usable CUDA device (there is no CPU fallback)";
        case MEXP_ERR_SINGULAR: return "singular denominator";
    }
    return "unknown status";
}

const char* mexp_last_cuda_error(void) { return g_last_cuda_error.c_str(); }

uint64_t mexp_launch_count(void) { return g_launches.load(); }

double mexp_unit_roundoff(int accuracy) {
    return accuracy == MEXP_ACCURACY_SINGLE ? 0x1p-24 : 0x1p-53;
}

int mexp_selection_table(int accuracy, int family, int32_t* degrees, int32_t* products,
                         double* thetas, int cap) {
    if (accuracy != MEXP_ACCURACY_SINGLE && accuracy != MEXP_ACCURACY_DOUBLE)
        return -MEXP_ERR_INVALID_ARGUMENT;
    if (family < MEXP_FAMILY_TAYLOR_NEW || family > MEXP_FAMILY_PADE) return -MEXP_ERR_INVALID_ARGUMENT;
    int k = 0;
    for (int e = 0; e < num_entries(family) && k < cap; ++e, ++k) {
        degrees[k] = degree_of_entry(family, e);
        products[k] = products_of(family, degrees[k]);
        thetas[k] = theta_entry(family, accuracy, e);
    }
    return k;
}

// mexp::select (expm.cpp:11-29) on the host: pure table arithmetic, the very
// function the kernels run (select_device is __host__ __device__).
int mexp_select(double norm, int accuracy, int family, int32_t* degree, int32_t* s) {
    if (accuracy != MEXP_ACCURACY_SINGLE && accuracy != MEXP_ACCURACY_DOUBLE)
        return MEXP_ERR_INVALID_ARGUMENT;
    if (family < MEXP_FAMILY_TAYLOR_NEW || family > MEXP_FAMILY_PADE) return MEXP_ERR_INVALID_ARGUMENT;
    const Sel r = select_device(norm, accuracy, family);
    if (r.status != MEXP_OK) return r.status;
    *degree = r.degree;
    *s = r.s;
    return MEXP_OK;
}

int mexp_expm_batched(const void* d_a, void* d_out, int dtype, int n, int64_t batch,
                      int accuracy, int family, int rounding, mexp_selection* d_sel,
                      void* stream) {
    if (!valid_args(dtype, n, batch, accuracy, family, rounding)) return MEXP_ERR_INVALID_ARGUMENT;
    if (batch > 0 && (!d_a || !d_out)) return MEXP_ERR_INVALID_ARGUMENT;
    const int dv = device_ok();
    if (dv != MEXP_OK) return dv;
    return expm_device(d_a, d_out, dtype, n, batch, acc_arg(accuracy, family), rounding, d_sel,
                       static_cast<cudaStream_t>(stream));
}

int mexp_expm_batched_host(const void* h_a, void* h_out, int dtype, int n, int64_t batch,
                           int accuracy, int family, int rounding, mexp_selection* h_sel,
                           int64_t* first_error) {
    if (!valid_args(dtype, n, batch, accuracy, family, rounding)) return MEXP_ERR_INVALID_ARGUMENT;
    return expm_host_impl(h_a, h_out, dtype, n, batch, acc_arg(accuracy, family), rounding, h_sel,
                          first_error);
}

}  // extern "C"

namespace {
double host_us() {
    return 1e-3 * double(std::chrono::duration_cast<std::chrono::nanoseconds>(
                             std::chrono::steady_clock::now().time_since_epoch())
                             .count());
}

// device-accessible address of mapped pinned host memory, or nullptr if p is
// pageable
void* mapped_device_ptr(const void* p) {
    cudaPointerAttributes attr{};
    if (cudaPointerGetAttributes(&attr, p) != cudaSuccess) {
        cudaGetLastError();
        return nullptr;
    }
    return attr.type == cudaMemoryTypeHost ? attr.devicePointer : nullptr;
}

int small_call_impl(HostPipe& p, const void* h_a, void* h_out, int dtype, int n, int64_t batch,
                    int aarg, int rounding, mexp_selection* h_sel, int64_t* first_error) {
    int r = ensure_pipe(p, 0, 0);
    if (r != MEXP_OK) return r;
    const size_t bytes = size_t(batch) * n * n * (dtype == MEXP_F64 ? sizeof(double) : sizeof(float));
    const size_t sel_bytes = size_t(batch) * sizeof(mexp_selection);
    void* d_a = mapped_device_ptr(h_a);
    void* d_out = mapped_device_ptr(h_out);
    mexp_selection* d_sel = h_sel ? static_cast<mexp_selection*>(mapped_device_ptr(h_sel)) : nullptr;
    const size_t need = 2 * bytes + sel_bytes + 64;
    if ((!d_a || !d_out || !d_sel) && p.h_stage_cap < need) {
        if (p.h_stage) cudaFreeHost(p.h_stage);
        p.h_stage = nullptr;
        p.h_stage_cap = 0;
        MEXP_CUDA(cudaMallocHost(&p.h_stage, need));
        p.h_stage_cap = need;
    }
    char* stage = static_cast<char*>(p.h_stage);
    char* s_in = stage;
    char* s_out = stage + ((bytes + 15) & ~size_t(15));
    mexp_selection* s_sel = reinterpret_cast<mexp_selection*>(s_out + ((bytes + 15) & ~size_t(15)));
    if (!d_a) {
        std::memcpy(s_in, h_a, bytes);
        d_a = mapped_device_ptr(s_in);
    }
    const bool out_staged = !d_out, sel_staged = !d_sel;
    if (out_staged) d_out = mapped_device_ptr(s_out);
    if (sel_staged) d_sel = static_cast<mexp_selection*>(mapped_device_ptr(s_sel));
    if (!d_a || !d_out || !d_sel) return MEXP_ERR_CUDA;
    r = expm_device(d_a, d_out, dtype, n, batch, aarg, rounding, d_sel, p.st[0]);
    if (r != MEXP_OK) return r;
    MEXP_CUDA(cudaStreamSynchronize(p.st[0]));
    if (out_staged) std::memcpy(h_out, s_out, bytes);
    const mexp_selection* hs = sel_staged ? s_sel : h_sel;
    if (h_sel && sel_staged) std::memcpy(h_sel, s_sel, sel_bytes);
    for (int64_t b = 0; b < batch; ++b)
        if (hs[b].status != MEXP_OK) {
            if (first_error) *first_error = b;
            return hs[b].status;
        }
    return MEXP_OK;
}

// The host pipeline behind mexp_expm_batched_host; `aarg` is the kernels'
// acc_arg (accuracy | family << 4, family 3 = reference_expm's selection).
int expm_host_impl(const void* h_a, void* h_out, int dtype, int n, int64_t batch, int aarg,
                   int rounding, mexp_selection* h_sel, int64_t* first_error) {
    if (first_error) *first_error = -1;
    if (batch == 0) return MEXP_OK;
    if (!h_a || !h_out) return MEXP_ERR_INVALID_ARGUMENT;
    const int dv = device_ok();
    if (dv != MEXP_OK) return dv;

    HostPipe& p = pipe_for_current_device();
    std::lock_guard<std::mutex> lock(p.mu);
    const size_t esz = dtype == MEXP_F64 ? sizeof(double) : sizeof(float);
    const size_t mat_bytes = size_t(n) * n * esz;
    // Chunks keep three in flight on three streams (H2D, compute, D2H): 16 MiB
    // for the small-n kernels (measured best, profiles/e2e_chunks_r1.txt);
    // 128 MiB for large n (cfg4: 64 matrices of 512^2 per chunk, measured
    // best in profiles/e2e_pipeline_r1.txt)
    static const size_t chunk_small = [] {
        const char* e = std::getenv("MEXP_HOST_CHUNK_MB");
        return size_t(e ? std::atoi(e) : 16) << 20;
    }();
    static const size_t chunk_large = [] {
        const char* e = std::getenv("MEXP_HOST_CHUNK_MB_LARGE");
        return size_t(e ? std::atoi(e) : 128) << 20;
    }();
    // Small calls (n <= 64, up to MEXP_SMALL_CALL_KB each way, default 1 MiB):
    // one stream and one synchronisation instead of the three-stream copy
    // pipeline. The n <= 64 kernels read A once and write e^A once, so they
    // run on host memory directly (mapped pinned memory, zero-copy over
    // PCIe): the caller's buffers when they are pinned, else the pipe's
    // pinned staging (one memcpy each way).
    static const size_t small_call = [] {
        const char* e = std::getenv("MEXP_SMALL_CALL_KB");
        return size_t(e ? std::atoi(e) : 1024) << 10;
    }();
    if (n <= 64 && size_t(batch) * mat_bytes <= small_call)
        return small_call_impl(p, h_a, h_out, dtype, n, batch, aarg, rounding, h_sel, first_error);
    // (the Pade family's blocked LU costs ~600 launches per chunk at n = 512:
    // it takes 4x the large-n chunk, measured best in profiles/e2e_pipeline_r1.txt)
    const size_t chunk_bytes = n <= 64 ? chunk_small : is_pade(aarg) ? 4 * chunk_large : chunk_large;
    int64_t chunk = int64_t(chunk_bytes / mat_bytes);
    if (chunk < 1) chunk = 1;
    if (chunk > batch) chunk = batch;
    int r = ensure_pipe(p, size_t(chunk) * mat_bytes, chunk);
    if (r != MEXP_OK) return r;
    // selection records always land in pinned scratch: an async copy into a
    // caller's pageable buffer would block the host thread per chunk and
    // serialise the copy pipeline; copied to h_sel once at the end
    bool sel_pinned = false;
    if (h_sel) {
        cudaPointerAttributes attr{};
        if (cudaPointerGetAttributes(&attr, h_sel) == cudaSuccess)
            sel_pinned = attr.type == cudaMemoryTypeHost;
        cudaGetLastError();
    }
    if (!sel_pinned && p.h_sel_cap < batch) {
        if (p.h_sel_scratch) cudaFreeHost(p.h_sel_scratch);
        p.h_sel_scratch = nullptr;
        MEXP_CUDA(cudaMallocHost(&p.h_sel_scratch, sizeof(mexp_selection) * batch));
        p.h_sel_cap = batch;
    }
    mexp_selection* hs = sel_pinned ? h_sel : p.h_sel_scratch;
    const char* src = static_cast<const char*>(h_a);
    char* dst = static_cast<char*>(h_out);
    // Chunk plan. Small n: chunk sizes taper (doubling from MEXP_HOST_TAPER_KB,
    // default 1/8 of a chunk) at both ends, so the pipeline fills (first H2D
    // before any D2H) and drains (last D2H after the last H2D) in a fraction
    // of a chunk's copy time instead of a whole one.
    static const size_t taper_bytes = [] {
        const char* e = std::getenv("MEXP_HOST_TAPER_KB");
        return e ? size_t(std::atoi(e)) << 10 : size_t(0);
    }();
    std::vector<std::pair<int64_t, int64_t>> plan;  // (b0, count)
    {
        std::vector<int64_t> sizes, head;
        int64_t minc = taper_bytes ? int64_t(taper_bytes / mat_bytes) : chunk / 8;
        if (minc < 1) minc = 1;
        for (int64_t h = minc; h < chunk; h *= 2) head.push_back(h);
        int64_t hsum = 0;
        for (int64_t h : head) hsum += h;
        const bool taper = n <= 64 && chunk >= 8 && batch >= 2 * hsum + 2 * chunk;
        int64_t left = batch;
        if (taper)
            for (int64_t h : head) {
                sizes.push_back(h);
                left -= 2 * h;  // the same again at the tail
            }
        while (left > 0) {
            const int64_t c = left < chunk ? left : chunk;
            sizes.push_back(c);
            left -= c;
        }
        if (taper)
            for (int i = int(head.size()) - 1; i >= 0; --i) sizes.push_back(head[i]);
        int64_t b0 = 0;
        for (int64_t c : sizes) {
            plan.emplace_back(b0, c);
            b0 += c;
        }
    }
    const int64_t nchunks = int64_t(plan.size());
    for (auto* v : {&p.ev, &p.ev_in, &p.ev_k})
        while (int64_t(v->size()) < nchunks) {
            cudaEvent_t e;
            MEXP_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
            v->push_back(e);
        }
    auto h2d = [&](int64_t c) -> int {
        const int k = int(c % host_streams());
        const int64_t b0 = plan[c].first, nb = plan[c].second;
        MEXP_CUDA(cudaMemcpyAsync(p.d_in[k], src + b0 * mat_bytes, nb * mat_bytes,
                                  cudaMemcpyHostToDevice, p.st[k]));
        return MEXP_OK;
    };
    // the large-n engine synchronises its stream once per call (it schedules
    // from the selections), so the next chunk's H2D is issued before it runs
    const bool prefetch = n > 64;
    // MEXP_HOST_TRACE=1: timed events around every stage, timeline on stderr
    static const bool trace = std::getenv("MEXP_HOST_TRACE") != nullptr;
    std::vector<cudaEvent_t> tev;
    auto mark = [&](cudaStream_t st) {
        if (!trace) return;
        cudaEvent_t e;
        cudaEventCreate(&e);
        cudaEventRecord(e, st);
        tev.push_back(e);
    };
    // Small n: a staged pipeline -- every H2D in order on one stream, every
    // kernel on a second, every D2H on a third, chained by events, chunk
    // buffers rotating over host_streams() slots. Each copy direction then
    // streams chunk after chunk at full rate instead of round-robining
    // between concurrent copies of several streams (MEXP_HOST_PIPE=streams
    // restores the per-stream pipeline).
    static const bool staged = [] {
        const char* e = std::getenv("MEXP_HOST_PIPE");
        return !(e && std::strcmp(e, "streams") == 0);
    }();
    // MEXP_HOST_OUT_ZC=1: the kernels write e^A straight into the caller's
    // pinned buffer (and the pinned records) over PCIe instead of device
    // buffers plus a D2H copy per chunk, so the copy engines carry only the
    // H2D stream. Measured (profiles/e2e_pipeline_r2.txt): cfg2 3.63 vs 3.45
    // ms/batch (slower), cfg3 +3%; off by default.
    static const bool out_zc_env = [] {
        const char* e = std::getenv("MEXP_HOST_OUT_ZC");
        return e && std::atoi(e) != 0;
    }();
    char* dst_dev = nullptr;
    mexp_selection* hs_dev = nullptr;
    if (!prefetch && staged && out_zc_env) {
        dst_dev = static_cast<char*>(mapped_device_ptr(h_out));
        hs_dev = static_cast<mexp_selection*>(mapped_device_ptr(hs));
        if (!dst_dev || !hs_dev) dst_dev = nullptr, hs_dev = nullptr;
    }
    if (!prefetch && staged) {
        cudaStream_t s_in = p.st[0], s_k = p.st[1], s_out = p.st[2];
        const int nslots = host_streams();
        for (int64_t c = 0; c < nchunks && dst_dev; ++c) {
            const int k = int(c % nslots);
            const int64_t b0 = plan[c].first, nb = plan[c].second;
            if (c >= nslots) MEXP_CUDA(cudaStreamWaitEvent(s_in, p.ev_k[c - nslots], 0));
            MEXP_CUDA(cudaMemcpyAsync(p.d_in[k], src + b0 * mat_bytes, nb * mat_bytes,
                                      cudaMemcpyHostToDevice, s_in));
            MEXP_CUDA(cudaEventRecord(p.ev_in[c], s_in));
            MEXP_CUDA(cudaStreamWaitEvent(s_k, p.ev_in[c], 0));
            r = expm_device(p.d_in[k], dst_dev + b0 * mat_bytes, dtype, n, nb, aarg, rounding, hs_dev + b0,
                            s_k);
            if (r != MEXP_OK) return r;
            MEXP_CUDA(cudaEventRecord(p.ev_k[c], s_k));
            MEXP_CUDA(cudaEventRecord(p.ev[c], s_k));
        }
        for (int64_t c = 0; c < nchunks && !dst_dev; ++c) {
            const int k = int(c % nslots);
            const int64_t b0 = plan[c].first, nb = plan[c].second;
            if (c >= nslots) MEXP_CUDA(cudaStreamWaitEvent(s_in, p.ev_k[c - nslots], 0));
            mark(s_in);
            MEXP_CUDA(cudaMemcpyAsync(p.d_in[k], src + b0 * mat_bytes, nb * mat_bytes,
                                      cudaMemcpyHostToDevice, s_in));
            mark(s_in);
            MEXP_CUDA(cudaEventRecord(p.ev_in[c], s_in));
            MEXP_CUDA(cudaStreamWaitEvent(s_k, p.ev_in[c], 0));
            if (c >= nslots) MEXP_CUDA(cudaStreamWaitEvent(s_k, p.ev[c - nslots], 0));
            r = expm_device(p.d_in[k], p.d_out[k], dtype, n, nb, aarg, rounding, p.d_sel[k], s_k);
            if (r != MEXP_OK) return r;
            mark(s_k);
            MEXP_CUDA(cudaEventRecord(p.ev_k[c], s_k));
            MEXP_CUDA(cudaStreamWaitEvent(s_out, p.ev_k[c], 0));
            MEXP_CUDA(cudaMemcpyAsync(dst + b0 * mat_bytes, p.d_out[k], nb * mat_bytes,
                                      cudaMemcpyDeviceToHost, s_out));
            MEXP_CUDA(cudaMemcpyAsync(hs + b0, p.d_sel[k], nb * sizeof(mexp_selection),
                                      cudaMemcpyDeviceToHost, s_out));
            mark(s_out);
            MEXP_CUDA(cudaEventRecord(p.ev[c], s_out));
        }
    }
    if (prefetch && (r = h2d(0)) != MEXP_OK) return r;
    for (int64_t c = 0; c < nchunks && !(!prefetch && staged); ++c) {
        const int k = int(c % host_streams());
        const int64_t b0 = plan[c].first, nb = plan[c].second;
        cudaStream_t st = p.st[k];
        mark(st);
        const double h0 = trace ? host_us() : 0.0;
        if (!prefetch && (r = h2d(c)) != MEXP_OK) return r;
        if (prefetch && c + 1 < nchunks && (r = h2d(c + 1)) != MEXP_OK) return r;
        const double h1 = trace ? host_us() : 0.0;
        mark(st);
        r = expm_device(p.d_in[k], p.d_out[k], dtype, n, nb, aarg, rounding, p.d_sel[k], st);
        if (r != MEXP_OK) return r;
        if (trace)
            std::fprintf(stderr, "host chunk %2lld: h2d enqueue %8.1f-%8.1f, expm_device returns %8.1f us\n",
                         (long long)c, h0, h1, host_us());
        mark(st);
        MEXP_CUDA(cudaMemcpyAsync(dst + b0 * mat_bytes, p.d_out[k], nb * mat_bytes,
                                  cudaMemcpyDeviceToHost, st));
        MEXP_CUDA(cudaMemcpyAsync(hs + b0, p.d_sel[k], nb * sizeof(mexp_selection),
                                  cudaMemcpyDeviceToHost, st));
        mark(st);
        MEXP_CUDA(cudaEventRecord(p.ev[c], st));
    }
    if (trace) {
        cudaDeviceSynchronize();
        for (int64_t c = 0; c < nchunks; ++c) {
            float t[4];
            for (int i = 0; i < 4; ++i) cudaEventElapsedTime(&t[i], tev[0], tev[4 * c + i]);
            std::fprintf(stderr, "chunk %2lld n=%7lld  h2d %8.1f-%8.1f  kernel -%8.1f  d2h -%8.1f us\n",
                         (long long)c, (long long)plan[c].second, 1e3 * t[0], 1e3 * t[1], 1e3 * t[2],
                         1e3 * t[3]);
        }
        for (auto e : tev) cudaEventDestroy(e);
    }
    // Host-side work on the records (status scan, copy to a pageable h_sel)
    // overlaps the pipeline: chunk c is handled as soon as its records land.
    int first_status = MEXP_OK;
    for (int64_t c = 0; c < nchunks; ++c) {
        MEXP_CUDA(cudaEventSynchronize(p.ev[c]));
        const int64_t b0 = plan[c].first, nb = plan[c].second;
        if (h_sel && !sel_pinned) std::memcpy(h_sel + b0, hs + b0, sizeof(mexp_selection) * nb);
        if (first_status == MEXP_OK)
            for (int64_t b = b0; b < b0 + nb; ++b)
                if (hs[b].status != MEXP_OK) {
                    if (first_error) *first_error = b;
                    first_status = hs[b].status;
                    break;
                }
    }
    for (int i = 0; i < host_streams(); ++i) MEXP_CUDA(cudaStreamSynchronize(p.st[i]));
    return first_status;
}

}  // namespace

extern "C" {

int mexp_expm(const double* a, int n, int accuracy, int family, double* result,
              mexp_report* report) {
    mexp_selection sel{};
    const int r = mexp_expm_batched_host(a, result, MEXP_F64, n, 1, accuracy, family,
                                         MEXP_ROUND_AUTO, &sel, nullptr);
    if (r != MEXP_OK) return r;
    if (report) {
        report->family = family;
        report->degree = sel.degree;
        report->s = sel.s;
        report->reserved = 0;
        report->cost_thirds = cost_thirds_of(family, sel.degree, sel.s);
        report->norm_in = sel.norm_in;
    }
    return MEXP_OK;
}

int mexp_device_count(void) {
    int count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return count;
}

int mexp_expm_batched_host_multi(const void* h_a, void* h_out, int dtype, int n, int64_t batch,
                                 int accuracy, int family, int rounding, mexp_selection* h_sel,
                                 int64_t* first_error, const int* devices, int ndevices) {
    if (first_error) *first_error = -1;
    if (!valid_args(dtype, n, batch, accuracy, family, rounding)) return MEXP_ERR_INVALID_ARGUMENT;
    const int dv = device_ok();
    if (dv != MEXP_OK) return dv;
    const int count = mexp_device_count();
    std::vector<int> devs;
    if (devices && ndevices > 0)
        devs.assign(devices, devices + ndevices);
    else
        for (int d = 0; d < count; ++d) devs.push_back(d);
    for (int d : devs)
        if (d < 0 || d >= count) return MEXP_ERR_INVALID_ARGUMENT;
    if (batch == 0) return MEXP_OK;
    if (batch > 0 && (!h_a || !h_out)) return MEXP_ERR_INVALID_ARGUMENT;
    const int G = int(devs.size());
    const size_t mat_bytes = size_t(n) * n * (dtype == MEXP_F64 ? sizeof(double) : sizeof(float));
    const int aarg = acc_arg(accuracy, family);
    // shard k: [b0_k, b0_k + cnt_k), the split of sharding.py's shard_range
    const int64_t base = batch / G, extra = batch % G;
    std::vector<int> status(G, MEXP_OK);
    std::vector<int64_t> first(G, -1), b0s(G);
    std::vector<std::string> errs(G);
    auto work = [&](int k) {
        const int64_t b0 = k * base + (k < extra ? k : extra);
        const int64_t cnt = base + (k < extra ? 1 : 0);
        b0s[k] = b0;
        if (cnt == 0) return;
        int dev_before = 0;
        cudaGetDevice(&dev_before);
        if (cudaSetDevice(devs[k]) != cudaSuccess) {
            status[k] = cuda_fail(cudaGetLastError(), "cudaSetDevice");
        } else {
            status[k] = expm_host_impl(static_cast<const char*>(h_a) + b0 * mat_bytes,
                                       static_cast<char*>(h_out) + b0 * mat_bytes, dtype, n, cnt,
                                       aarg, rounding, h_sel ? h_sel + b0 : nullptr, &first[k]);
        }
        if (status[k] == MEXP_ERR_CUDA) errs[k] = g_last_cuda_error;
        cudaSetDevice(dev_before);
    };
    if (G == 1) {
        work(0);
    } else {
        std::vector<std::thread> threads;
        threads.reserve(G);
        for (int k = 0; k < G; ++k) threads.emplace_back(work, k);
        for (auto& t : threads) t.join();
    }
    // a call-level failure (CUDA, invalid) wins; else the lowest failing matrix
    for (int k = 0; k < G; ++k)
        if (status[k] != MEXP_OK && first[k] < 0) {
            if (status[k] == MEXP_ERR_CUDA) g_last_cuda_error = errs[k];
            return status[k];
        }
    for (int k = 0; k < G; ++k)
        if (status[k] != MEXP_OK) {
            if (first_error) *first_error = b0s[k] + first[k];
            return status[k];
        }
    return MEXP_OK;
}

// library-internal helper for the C++ drop-in mexp::reference_expm (bench_api.cpp):
// Pade r26 with s = the least s such that ||2^-s A||_1 <= theta_26 / 8
// (bench.cpp:10-20), batched over host matrices
int mexp_b200_reference_expm_host(const double* a, double* out, int n, int64_t batch,
                                  int rounding, mexp_selection* sel) {
    if (n < 1 || batch < 0 || rounding < 0 || rounding > 2) return MEXP_ERR_INVALID_ARGUMENT;
    const int dv = device_ok();
    if (dv != MEXP_OK) return dv;
    return expm_host_impl(a, out, MEXP_F64, n, batch,
                          acc_arg(MEXP_ACCURACY_DOUBLE, kFamilyPadeReference), rounding, sel, nullptr);
}

// library-internal helper for the C++ drop-in mexp::squarings (dropin.cpp):
// on the device's host-pipe stream, with the matrix in a stream-ordered
// buffer of the library's memory pool (no cudaMalloc / cudaFree per call)
int mexp_b200_squarings_host(double* x, int n, int s) {
    const int dv = device_ok();
    if (dv != MEXP_OK) return dv;
    if (s <= 0) return MEXP_OK;
    HostPipe& p = pipe_for_current_device();
    std::lock_guard<std::mutex> lock(p.mu);
    {
        const int e = ensure_pipe(p, 0, 0);  // the streams
        if (e != MEXP_OK) return e;
    }
    cudaStream_t st = p.st[0];
    const size_t bytes = sizeof(double) * size_t(n) * n;
    int r = MEXP_OK;
    {
        AsyncBuffer buf(st);
        if (buf.alloc(bytes) != cudaSuccess) return cuda_fail(cudaGetLastError(), "squarings alloc");
        double* d = buf.get<double>();
        if (cudaMemcpyAsync(d, x, bytes, cudaMemcpyHostToDevice, st) != cudaSuccess) r = MEXP_ERR_CUDA;
        // the reference's squarings (expm.cpp:31-35), bit for bit
        if (r == MEXP_OK) r = squarings_f64(d, n, 1, s, MEXP_ROUND_REFERENCE, st, &g_launches);
        if (r == MEXP_OK && cudaMemcpyAsync(x, d, bytes, cudaMemcpyDeviceToHost, st) != cudaSuccess)
            r = MEXP_ERR_CUDA;
    }
    if (cudaStreamSynchronize(st) != cudaSuccess && r == MEXP_OK) r = MEXP_ERR_CUDA;
    if (r == MEXP_ERR_CUDA && g_last_cuda_error.empty()) g_last_cuda_error = large_last_error();
    return r;
}

int mexp_squarings_batched(double* d_x, int n, int64_t batch, int s, int rounding,
                           void* stream) {
    if (n < 1 || batch < 0 || s < 0 || rounding < 0 || rounding > 2)
        return MEXP_ERR_INVALID_ARGUMENT;
    const int dv = device_ok();
    if (dv != MEXP_OK) return dv;
    if (batch == 0 || s == 0) return MEXP_OK;
    const int r = squarings_f64(d_x, n, batch, s, rounding, static_cast<cudaStream_t>(stream),
                                &g_launches);
    if (r == MEXP_ERR_CUDA) g_last_cuda_error = large_last_error();
    return r;
}

}  // extern "C"
