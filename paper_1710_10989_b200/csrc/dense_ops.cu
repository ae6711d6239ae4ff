// The reference's lower-level dense-matrix layer on the device: the value
// operations of dense_matrix.hpp:40-58 (matmul, lincomb, add, sub, scaled,
// one_norm, lu_solve), the raw kernels of kernels.hpp:15-24, and the scheme
// evaluators of taylor_schemes.hpp:36-48 / pade.hpp:15-26 built from them.
//
// Every operation runs in the reference's own arithmetic (it is compiled with
// -ffp-contract=off, CMakeLists.txt:10-11): each multiply, add, subtract and
// divide rounded separately, sums in the reference's order. So every result
// is bit-identical to the reference's, which tests/test_gpu_dense_ops.py
// checks against the compiled reference.
//
//   matmul   kernels.cpp:16-27  c_ij = 0 + a_i0 b_0j + a_i1 b_1j + ... (k ascending)
//   lincomb  kernels.cpp:29-37  out = c0 m0, then += ci mi left to right
//   scale    kernels.cpp:39-42  out = a * f
//   one_norm kernels.cpp:44-53  column sums rows ascending, strict '>' max
//   lu       kernels.cpp:55-112 partial pivoting (strict '>' scan), l = a_ik / piv,
//                               a_ij -= l p_j; per column forward / back substitution
//
// Public C ABI (device buffers): mexp_matmul_batched, mexp_lincomb_batched,
// mexp_one_norm_batched, mexp_lu_solve_batched. Library-internal host entry
// for the C++ drop-in: mexp_b200_dense_call (one host matrix in, one out; the
// composite schemes keep every intermediate on the device).
#include <atomic>
#include <climits>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "async_buffer.hpp"
#include "device_once.hpp"
#include "expm_common.cuh"
#include "expm_large.cuh"
#include "mexp_b200.h"

namespace mexp_b200 {

std::atomic<uint64_t>& library_launch_counter();  // capi.cu
void set_last_cuda_error(const std::string& e);   // capi.cu

namespace {

int dense_fail(cudaError_t e, const char* where) {
    set_last_cuda_error(std::string(where) + ": " + cudaGetErrorString(e));
    return MEXP_ERR_CUDA;
}
#define DCUDA(call)                                              \
    do {                                                         \
        cudaError_t e_ = (call);                                 \
        if (e_ != cudaSuccess) return dense_fail(e_, #call);     \
    } while (0)

void counted(int k = 1) { library_launch_counter().fetch_add(k, std::memory_order_relaxed); }

int device_present() {
    int count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) {
        cudaGetLastError();
        return MEXP_ERR_NO_DEVICE;
    }
    return MEXP_OK;
}

// ---- kernels ---------------------------------------------------------------

// n <= 64: one CTA per matrix, both operands in shared memory; thread t
// computes outputs t, t + blockDim, ... with the k loop in the reference's order
template <bool kExact>
__global__ void __launch_bounds__(256) matmul_small_kernel(const double* __restrict__ a,
                                                           const double* __restrict__ b,
                                                           double* __restrict__ c, int n) {
    extern __shared__ double sm[];
    const int nn = n * n;
    double* sa = sm;
    double* sb = sm + nn;
    const int64_t off = int64_t(blockIdx.x) * nn;
    for (int e = threadIdx.x; e < nn; e += blockDim.x) {
        sa[e] = a[off + e];
        sb[e] = b[off + e];
    }
    __syncthreads();
    for (int e = threadIdx.x; e < nn; e += blockDim.x) {
        const int i = e / n, j = e - (e / n) * n;
        double s = 0.0;
        for (int k = 0; k < n; ++k)
            s = kExact ? __dadd_rn(s, __dmul_rn(sa[i * n + k], sb[k * n + j]))
                       : fma(sa[i * n + k], sb[k * n + j], s);
        c[off + e] = s;
    }
}

constexpr int kLcMax = 8;
struct LcArgs {
    const double* m[kLcMax];
    double c[kLcMax];
    int k;
    int accumulate;  // 1: continue the running sum already in `out`
};

__global__ void lincomb_kernel(LcArgs g, double* out, int64_t len) {
    for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < len;
         e += int64_t(gridDim.x) * blockDim.x) {
        double s;
        int i0;
        if (g.accumulate) {
            s = out[e];
            i0 = 0;
        } else {
            s = __dmul_rn(g.c[0], g.m[0][e]);
            i0 = 1;
        }
        for (int i = i0; i < g.k; ++i) s = __dadd_rn(s, __dmul_rn(g.c[i], g.m[i][e]));
        out[e] = s;
    }
}

__global__ void identity_kernel(double* out, int n) {
    const int64_t nn = int64_t(n) * n;
    for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < nn;
         e += int64_t(gridDim.x) * blockDim.x)
        out[e] = (e / n == e % n) ? 1.0 : 0.0;
}

// one CTA per matrix: a lane per column, rows summed ascending from 0.0;
// the max is taken on the bits of the (non-negative) sums, NaN sums excluded
// as the reference's strict '>' excludes them
__global__ void __launch_bounds__(256) one_norm_kernel(const double* __restrict__ a, int n,
                                                       double* __restrict__ norms) {
    const int64_t off = int64_t(blockIdx.x) * n * n;
    unsigned long long best = 0;
    for (int j = threadIdx.x; j < n; j += blockDim.x) {
        double s = 0.0;
        for (int i = 0; i < n; ++i) s = __dadd_rn(s, fabs(a[off + int64_t(i) * n + j]));
        if (s > 0.0) best = max(best, static_cast<unsigned long long>(__double_as_longlong(s)));
    }
    __shared__ unsigned long long red[8];
    for (int o = 16; o; o >>= 1) best = max(best, __shfl_xor_sync(0xffffffffu, best, o));
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = best;
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < int(blockDim.x >> 5); ++w) best = max(best, red[w]);
        norms[blockIdx.x] = __longlong_as_double(static_cast<long long>(best));
    }
}

// X = M^-1 R for one matrix per CTA in the reference's arithmetic
// (kernels.cpp:55-112). lu / perm: per-matrix workspace. mode 0: factor and
// solve; 1: factor only (lu_factor: the factors stay in lu / perm); 2: solve
// only with the factors given in lu / perm (lu_apply).
constexpr int kLuThreads = 512;
enum { kLuFactorSolve = 0, kLuFactor = 1, kLuApply = 2 };
__global__ void __launch_bounds__(kLuThreads) lu_solve_kernel(const double* __restrict__ M,
                                                              const double* __restrict__ R,
                                                              double* __restrict__ X,
                                                              double* __restrict__ lu_ws,
                                                              int* __restrict__ perm_ws, int n,
                                                              int32_t* __restrict__ status, int mode) {
    const int64_t nn = int64_t(n) * n;
    const int64_t mi = blockIdx.x;
    double* lu = lu_ws + mi * nn;
    int* perm = perm_ws + mi * n;
    const double* m = M + mi * nn;
    const double* r = R + mi * nn;
    double* x = X + mi * nn;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    constexpr int kWarps = kLuThreads / 32;
    __shared__ double red_v[kWarps];
    __shared__ int red_i[kWarps];
    __shared__ int s_p, s_bad;
    if (tid == 0) s_bad = 0;
    if (mode != kLuApply) {
        for (int64_t e = tid; e < nn; e += kLuThreads) lu[e] = m[e];
        for (int i = tid; i < n; i += kLuThreads) perm[i] = i;
    }
    __syncthreads();
    for (int k = 0; k < n && mode != kLuApply; ++k) {
        // pivot: the reference's scan keeps the first row whose |value| is
        // strictly greater than the running best (starting at the diagonal):
        // the largest non-NaN value, ties to the lowest row, a NaN diagonal
        // never replaced
        double bv = -1.0;
        int bi = INT_MAX;
        for (int i = k + tid; i < n; i += kLuThreads) {
            const double v = fabs(lu[int64_t(i) * n + k]);
            if (v > bv) {  // rows ascending per thread: ties keep the lower row
                bv = v;
                bi = i;
            }
        }
        for (int o = 16; o; o >>= 1) {
            const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
            const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
            if (ov > bv || (ov == bv && oi < bi)) {
                bv = ov;
                bi = oi;
            }
        }
        if (lane == 0) {
            red_v[warp] = bv;
            red_i[warp] = bi;
        }
        __syncthreads();
        if (tid == 0) {
            for (int w = 1; w < kWarps; ++w)
                if (red_v[w] > bv || (red_v[w] == bv && red_i[w] < bi)) {
                    bv = red_v[w];
                    bi = red_i[w];
                }
            const double diag = fabs(lu[int64_t(k) * n + k]);
            double best = diag;
            int p = k;
            if (!isnan(diag) && bi != INT_MAX && bv > diag) {
                best = bv;
                p = bi;
            }
            s_p = p;
            if (best == 0.0) s_bad = 1;
        }
        __syncthreads();
        if (s_bad) break;
        const int p = s_p;
        if (p != k) {
            for (int j = tid; j < n; j += kLuThreads) {
                const double t = lu[int64_t(k) * n + j];
                lu[int64_t(k) * n + j] = lu[int64_t(p) * n + j];
                lu[int64_t(p) * n + j] = t;
            }
            if (tid == 0) {
                const int t = perm[k];
                perm[k] = perm[p];
                perm[p] = t;
            }
            __syncthreads();
        }
        const double piv = lu[int64_t(k) * n + k];
        const double* prow = lu + int64_t(k) * n;
        // rows below: a warp per row, lanes across the columns
        for (int i = k + 1 + warp; i < n; i += kWarps) {
            double* row = lu + int64_t(i) * n;
            const double l = row[k] / piv;
            for (int j = k + 1 + lane; j < n; j += 32) row[j] = __dsub_rn(row[j], __dmul_rn(l, prow[j]));
            __syncwarp();
            if (lane == 0) row[k] = l;
        }
        __syncthreads();
    }
    if (s_bad) {
        if (tid == 0) status[mi] = MEXP_ERR_SINGULAR;
        if (mode != kLuFactor)
            for (int64_t e = tid; e < nn; e += kLuThreads) x[e] = __longlong_as_double(0x7ff8000000000000LL);
        return;
    }
    if (tid == 0) status[mi] = MEXP_OK;
    if (mode == kLuFactor) return;
    // a thread per right-hand-side column: y = P r, forward with unit L,
    // backward with U, every sum in the reference's order
    for (int col = tid; col < n; col += kLuThreads) {
        for (int i = 0; i < n; ++i) x[int64_t(i) * n + col] = r[int64_t(perm[i]) * n + col];
        for (int i = 1; i < n; ++i) {
            const double* row = lu + int64_t(i) * n;
            double s = x[int64_t(i) * n + col];
            for (int j = 0; j < i; ++j) s = __dsub_rn(s, __dmul_rn(row[j], x[int64_t(j) * n + col]));
            x[int64_t(i) * n + col] = s;
        }
        for (int i = n - 1; i >= 0; --i) {
            const double* row = lu + int64_t(i) * n;
            double s = x[int64_t(i) * n + col];
            for (int j = i + 1; j < n; ++j) s = __dsub_rn(s, __dmul_rn(row[j], x[int64_t(j) * n + col]));
            x[int64_t(i) * n + col] = s / row[i];
        }
    }
}

int ew_grid(int64_t len) {
    const int64_t g = (len + 255) / 256;
    return int(g < 4096 ? (g > 0 ? g : 1) : 4096);
}

// ---- device operations -------------------------------------------------------

int matmul_dev(const double* a, const double* b, double* c, int n, int64_t batch, int rounding,
               cudaStream_t st) {
    if (batch == 0) return MEXP_OK;
    if (n > 64) {
        const int r = matmul_f64(a, b, c, n, batch, rounding, st, &library_launch_counter());
        if (r == MEXP_ERR_CUDA) set_last_cuda_error(large_last_error());
        return r;
    }
    const size_t smem = 2 * size_t(n) * n * sizeof(double);
    static PerDevice attr_once;
    attr_once([] {
        cudaFuncSetAttribute(matmul_small_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             int(2 * 64 * 64 * sizeof(double)));
        cudaFuncSetAttribute(matmul_small_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             int(2 * 64 * 64 * sizeof(double)));
    });
    for (int64_t b0 = 0; b0 < batch; b0 += INT32_MAX) {
        const int nb = int(batch - b0 < INT32_MAX ? batch - b0 : INT32_MAX);
        const int64_t off = b0 * n * n;
        if (rounding == MEXP_ROUND_REFERENCE)
            matmul_small_kernel<true><<<nb, 256, smem, st>>>(a + off, b + off, c + off, n);
        else
            matmul_small_kernel<false><<<nb, 256, smem, st>>>(a + off, b + off, c + off, n);
        counted();
    }
    DCUDA(cudaGetLastError());
    return MEXP_OK;
}

// out = sum_i coeffs[i] * mats[i], left to right (any k >= 1: chunks of 8
// continue the running sum in `out`, which is the same rounding sequence)
int lincomb_dev(const double* coeffs, const double* const* mats, int k, double* out, int64_t len,
                cudaStream_t st) {
    if (len == 0) return MEXP_OK;
    for (int i0 = 0; i0 < k; i0 += kLcMax) {
        LcArgs g{};
        g.k = k - i0 < kLcMax ? k - i0 : kLcMax;
        g.accumulate = i0 > 0;
        for (int i = 0; i < g.k; ++i) {
            g.m[i] = mats[i0 + i];
            g.c[i] = coeffs[i0 + i];
        }
        lincomb_kernel<<<ew_grid(len), 256, 0, st>>>(g, out, len);
        counted();
    }
    DCUDA(cudaGetLastError());
    return MEXP_OK;
}

int one_norm_dev(const double* a, int n, int64_t batch, double* norms, cudaStream_t st) {
    for (int64_t b0 = 0; b0 < batch; b0 += INT32_MAX) {
        const int nb = int(batch - b0 < INT32_MAX ? batch - b0 : INT32_MAX);
        one_norm_kernel<<<nb, 256, 0, st>>>(a + b0 * n * n, n, norms + b0);
        counted();
    }
    DCUDA(cudaGetLastError());
    return MEXP_OK;
}

// lu / perm: caller's factor storage (modes kLuFactor / kLuApply), or
// nullptr for per-call scratch (kLuFactorSolve)
int lu_solve_dev(const double* m, const double* r, double* x, int n, int64_t batch, int32_t* status,
                 cudaStream_t st, int mode = kLuFactorSolve, double* lu = nullptr, int* perm = nullptr) {
    if (batch == 0) return MEXP_OK;
    AsyncBuffer ws(st), pw(st);
    if (!lu) {
        DCUDA(ws.alloc(sizeof(double) * size_t(batch) * n * n));
        DCUDA(pw.alloc(sizeof(int) * size_t(batch) * n));
        lu = ws.get<double>();
        perm = pw.get<int>();
    }
    for (int64_t b0 = 0; b0 < batch; b0 += INT32_MAX) {
        const int nb = int(batch - b0 < INT32_MAX ? batch - b0 : INT32_MAX);
        const int64_t off = b0 * n * n;
        lu_solve_kernel<<<nb, kLuThreads, 0, st>>>(m ? m + off : nullptr, r ? r + off : nullptr,
                                                   x ? x + off : nullptr, lu + off, perm + b0 * n, n,
                                                   status + b0, mode);
        counted();
    }
    DCUDA(cudaGetLastError());
    return MEXP_OK;
}

// ---- composite routines on one matrix, intermediates on the device -----------

// the scheme coefficients, from the same literals as the kernels' tables
// (scheme_tables.h)
struct Tables {
    double t12[4][4] = MEXP_T12_TABLE;
    double t18a[4] = MEXP_T18A_TABLE;
    double t18b[4][5] = MEXP_T18B_TABLE;
};

// Psi9 coefficients: closed forms in sqrt(7), rounded once from long double
// (taylor_schemes.cpp:29-42)
struct Psi9 {
    double x[10];
};
Psi9 psi9_coeffs() {
    const long double r = sqrtl(7.0L);
    Psi9 c{};
    c.x[1] = double((-5.0L + 6.0L * r) / 32.0L);
    c.x[2] = -0.25;
    c.x[3] = -1.0;
    c.x[4] = double(3.0L * (169.0L + 20.0L * r) / 1024.0L);
    c.x[5] = double(3.0L * (5.0L + 2.0L * r) / 64.0L);
    c.x[6] = 1695.0 / 4096.0;
    c.x[7] = 267.0 / 512.0;
    c.x[8] = 21.0 / 64.0;
    c.x[9] = double(3.0L * r / 4.0L);
    return c;
}

// 1.0 / k! with k! accumulated in double (taylor_schemes.cpp:44-48)
double inv_factorial(int k) { return inv_fact(k); }

// A register file of device matrices for one n: slot 0 = A, slot 1 = I.
class Program {
public:
    Program(int n, cudaStream_t st) : n_(n), nn_(size_t(n) * n), st_(st), buf_(st) {}
    int init(const double* h_a, int slots) {
        slots_ = slots;
        DCUDA(buf_.alloc(sizeof(double) * nn_ * slots));
        DCUDA(cudaMemcpyAsync(at(0), h_a, sizeof(double) * nn_, cudaMemcpyHostToDevice, st_));
        identity_kernel<<<ew_grid(int64_t(nn_)), 256, 0, st_>>>(at(1), n_);
        counted();
        DCUDA(cudaGetLastError());
        return MEXP_OK;
    }
    double* at(int s) { return buf_.get<double>() + size_t(s) * nn_; }
    // d = x y (counted as one product when `count`)
    int mm(int d, int x, int y, bool count = true) {
        products += count ? 1 : 0;
        return matmul_dev(at(x), at(y), at(d), n_, 1, MEXP_ROUND_REFERENCE, st_);
    }
    int lc(int d, std::initializer_list<double> c, std::initializer_list<int> m) {
        std::vector<const double*> p;
        for (int s : m) p.push_back(at(s));
        return lincomb_dev(c.begin(), p.data(), int(c.size()), at(d), int64_t(nn_), st_);
    }
    int lcv(int d, const std::vector<double>& c, const std::vector<int>& m) {
        std::vector<const double*> p;
        for (int s : m) p.push_back(at(s));
        return lincomb_dev(c.data(), p.data(), int(c.size()), at(d), int64_t(nn_), st_);
    }
    int copy(int d, int s) {
        DCUDA(cudaMemcpyAsync(at(d), at(s), sizeof(double) * nn_, cudaMemcpyDeviceToDevice, st_));
        return MEXP_OK;
    }
    // d = m^-1 r (counted as one solve)
    int solve(int d, int m, int r) {
        ++solves;
        DCUDA(status_buf_alloc());
        const int rr = lu_solve_dev(at(m), at(r), at(d), n_, 1, status_, st_);
        if (rr) return rr;
        int32_t h = 0;
        DCUDA(cudaMemcpyAsync(&h, status_, sizeof h, cudaMemcpyDeviceToHost, st_));
        DCUDA(cudaStreamSynchronize(st_));
        return h;
    }
    int finish(int s, double* h_out) {
        DCUDA(cudaMemcpyAsync(h_out, at(s), sizeof(double) * nn_, cudaMemcpyDeviceToHost, st_));
        DCUDA(cudaStreamSynchronize(st_));
        return MEXP_OK;
    }
    int64_t products = 0, solves = 0;

private:
    cudaError_t status_buf_alloc() {
        if (status_) return cudaSuccess;
        void* p = nullptr;
        const cudaError_t e = pool_alloc(&p, sizeof(int32_t), st_);
        status_ = static_cast<int32_t*>(p);
        return e;
    }
    int n_;
    size_t nn_;
    cudaStream_t st_;
    AsyncBuffer buf_;
    int slots_ = 0;
    int32_t* status_ = nullptr;

public:
    ~Program() {
        if (status_) cudaFreeAsync(status_, st_);
    }
};

#define TRY(...)                        \
    do {                                \
        const int r_ = (__VA_ARGS__);   \
        if (r_) return r_;              \
    } while (0)

enum Slot { A = 0, I = 1 };

// taylor_schemes.cpp:104-113
int run_t8(Program& p, int out) {
    using c = T8C;
    enum { A2 = 2, U = 3, A4 = 4, L = 5, R = 6, A8 = 7 };
    TRY(p.mm(A2, A, A));
    TRY(p.lc(U, {c::x1, c::x2}, {A, A2}));
    TRY(p.mm(A4, A2, U));
    TRY(p.lc(L, {c::x3, 1.0}, {A2, A4}));
    TRY(p.lc(R, {c::x4, c::x5, c::x6, c::x7}, {I, A, A2, A4}));
    TRY(p.mm(A8, L, R));
    return p.lc(out, {c::y0, c::y1, c::y2, 1.0}, {I, A, A2, A8});
}

// taylor_schemes.cpp:115-125: B_j over {I, A, A2, A3}, A6 = B3 + B4 B4,
// T12 = B1 + (B2 + A6) A6
int run_t12(Program& p, const Tables& t, int out) {
    enum { A2 = 2, A3 = 3, B1 = 4, B2 = 5, B3 = 6, B4 = 7, P = 8, A6 = 9, S = 10 };
    TRY(p.mm(A2, A, A));
    TRY(p.mm(A3, A2, A));
    for (int j = 0; j < 4; ++j)
        TRY(p.lc(B1 + j, {t.t12[0][j], t.t12[1][j], t.t12[2][j], t.t12[3][j]}, {I, A, A2, A3}));
    TRY(p.mm(P, B4, B4));
    TRY(p.lc(A6, {1.0, 1.0}, {B3, P}));
    TRY(p.lc(S, {1.0, 1.0}, {B2, A6}));
    TRY(p.mm(P, S, A6));
    return p.lc(out, {1.0, 1.0}, {B1, P});
}

// taylor_schemes.cpp:127-141: A9 = B1 B5 + B4, T18 = B2 + (B3 + A9) A9
int run_t18(Program& p, const Tables& t, int out) {
    enum { A2 = 2, A3 = 3, A6 = 4, B1 = 5, B2 = 6, B3 = 7, B4 = 8, B5 = 9, P = 10, A9 = 11, S = 12 };
    TRY(p.mm(A2, A, A));
    TRY(p.mm(A3, A2, A));
    TRY(p.mm(A6, A3, A3));
    TRY(p.lc(B1, {t.t18a[0], t.t18a[1], t.t18a[2], t.t18a[3]}, {I, A, A2, A3}));
    for (int j = 0; j < 4; ++j) {
        const double* k = t.t18b[j];
        TRY(p.lc(B2 + j, {k[0], k[1], k[2], k[3], k[4]}, {I, A, A2, A3, A6}));
    }
    TRY(p.mm(P, B1, B5));
    TRY(p.lc(A9, {1.0, 1.0}, {P, B4}));
    TRY(p.lc(S, {1.0, 1.0}, {B3, A9}));
    TRY(p.mm(P, S, A9));
    return p.lc(out, {1.0, 1.0}, {B2, P});
}

// eval_ps (taylor_schemes.cpp:143-198): chunks g_i = sum_k A^k / (p i + k)!
// over {I, A, A2(, A3)}, t = g_{q-1} + A^p / m!, then t = g_i + t A^p
int run_ps(Program& p, int degree, int out) {
    enum { A2 = 2, A3 = 3, A4 = 4, G0 = 5, T = 9, P = 10, T2 = 11 };
    TRY(p.mm(A2, A, A));
    if (degree == 2) return p.lc(out, {1.0, 1.0, 0.5}, {I, A, A2});
    if (degree == 4) {  // (I + A) + ((1/2! I + 1/3! A) + A2 / 4!) A2
        TRY(p.lc(G0, {1.0, 1.0}, {I, A}));
        TRY(p.lc(G0 + 1, {inv_factorial(2), inv_factorial(3)}, {I, A}));
        TRY(p.lc(T, {1.0, inv_factorial(4)}, {G0 + 1, A2}));
        TRY(p.mm(P, T, A2));
        return p.lc(out, {1.0, 1.0}, {G0, P});
    }
    if (degree != 6 && degree != 9 && degree != 16) return MEXP_ERR_INVALID_ARGUMENT;
    const int pw = degree == 16 ? 4 : 3, q = degree / pw;
    TRY(p.mm(A3, A2, A));
    if (pw == 4) TRY(p.mm(A4, A2, A2));
    const int ap = pw == 4 ? int(A4) : int(A3);
    for (int i = 0; i < q; ++i) {
        std::vector<double> c;
        std::vector<int> m;
        for (int k = 0; k < pw; ++k) {
            c.push_back(inv_factorial(pw * i + k));
            m.push_back(k == 0 ? int(I) : k == 1 ? int(A) : k == 2 ? int(A2) : int(A3));
        }
        TRY(p.lcv(G0 + i, c, m));
    }
    TRY(p.lc(T, {1.0, inv_factorial(degree)}, {G0 + q - 1, ap}));
    for (int i = q - 2; i >= 0; --i) {
        TRY(p.mm(P, T, ap));
        TRY(p.lc(i == 0 ? out : T2, {1.0, 1.0}, {G0 + i, P}));
        if (i) TRY(p.copy(T, T2));
    }
    return MEXP_OK;
}

// psi9 (taylor_schemes.cpp:200-209)
int run_psi9(Program& p, int out) {
    const Psi9 c = psi9_coeffs();
    enum { A2 = 2, B = 3, BB = 4, A4 = 5, L = 6, A8 = 7, Q = 8 };
    TRY(p.mm(A2, A, A));
    TRY(p.lc(B, {c.x[1], c.x[2], c.x[3]}, {I, A, A2}));
    TRY(p.mm(BB, B, B));
    TRY(p.lc(Q, {c.x[4], c.x[5]}, {I, A}));
    TRY(p.lc(A4, {1.0, 1.0}, {Q, BB}));
    TRY(p.lc(L, {c.x[9], 1.0}, {A2, A4}));
    TRY(p.mm(A8, L, A4));
    return p.lc(out, {c.x[6], c.x[7], c.x[8], 1.0}, {I, A, A2, A8});
}

// taylor_oracle / psi_oracle (taylor_schemes.cpp:87-102): plain Horner,
// products not counted
int run_horner(Program& p, int degree, bool taylor, int out) {
    enum { T = 2, P = 3, S = 4 };
    TRY(p.copy(T, I));
    if (taylor) {
        for (int k = degree; k >= 1; --k) {
            TRY(p.mm(P, A, T, false));
            TRY(p.lc(S, {1.0 / k}, {P}));          // scaled(., 1.0 / k)
            TRY(p.lc(T, {1.0, 1.0}, {I, S}));      // add(I, .)
        }
    } else {
        for (int i = 1; i < degree; ++i) {
            TRY(p.mm(P, A, T, false));
            TRY(p.lc(T, {1.0, 1.0}, {I, P}));
        }
    }
    return p.copy(out, T);
}

// eval_pade (pade.cpp:50-113), then pade_solve = lu_solve(V - U, V + U)
int run_pade(Program& p, int order, int out) {
    const int m = order / 2;
    const double* b = kPadeHost[m - 1];
    enum { U = 2, V = 3, T = 4, T2 = 5, PW = 6 };  // PW + i = A^(2(i+1))
    if (order == 10) {
        TRY(p.mm(PW, A, A));
        TRY(p.mm(PW + 1, PW, PW));
        TRY(p.lc(T, {b[5], b[3], b[1]}, {PW + 1, PW, I}));
        TRY(p.mm(U, A, T));
        TRY(p.lc(V, {b[4], b[2], b[0]}, {PW + 1, PW, I}));
    } else if (order == 26) {
        const int A2 = PW, A4 = PW + 1, A6 = PW + 2;
        TRY(p.mm(A2, A, A));
        TRY(p.mm(A4, A2, A2));
        TRY(p.mm(A6, A2, A4));
        TRY(p.lc(T, {b[13], b[11], b[9]}, {A6, A4, A2}));
        TRY(p.mm(T2, A6, T));
        TRY(p.lc(T, {1.0, b[7], b[5], b[3], b[1]}, {T2, A6, A4, A2, I}));
        TRY(p.mm(U, A, T));
        TRY(p.lc(T, {b[12], b[10], b[8]}, {A6, A4, A2}));
        TRY(p.mm(T2, A6, T));
        TRY(p.lc(V, {1.0, b[6], b[4], b[2], b[0]}, {T2, A6, A4, A2, I}));
    } else {
        const int top = m - (m % 2);
        int npw = 0;
        if (top >= 2) {
            TRY(p.mm(PW, A, A));
            npw = 1;
            for (int e = 4; e <= top; e += 2, ++npw) TRY(p.mm(PW + npw, PW, PW + npw - 1));
        }
        std::vector<double> co{b[1]}, ce{b[0]};
        std::vector<int> mo{I}, me{I};
        for (int j = 3; j <= m; j += 2) {
            co.push_back(b[j]);
            mo.push_back(PW + (j - 1) / 2 - 1);
        }
        for (int j = 2; j <= m; j += 2) {
            ce.push_back(b[j]);
            me.push_back(PW + j / 2 - 1);
        }
        if (m >= 3) {
            TRY(p.lcv(T, co, mo));
            TRY(p.mm(U, A, T));
        } else {
            TRY(p.lc(U, {b[1]}, {A}));  // scaled(a, b1)
        }
        TRY(p.lcv(V, ce, me));
    }
    TRY(p.lc(T, {1.0, -1.0}, {V, U}));  // sub(v, u)
    TRY(p.lc(T2, {1.0, 1.0}, {V, U}));  // add(v, u)
    return p.solve(out, T, T2);
}

}  // namespace

}  // namespace mexp_b200

using namespace mexp_b200;

extern "C" {

int mexp_matmul_batched(const double* d_a, const double* d_b, double* d_c, int n, int64_t batch,
                        int rounding, void* stream) {
    if (n < 1 || batch < 0 || rounding < 0 || rounding > 2) return MEXP_ERR_INVALID_ARGUMENT;
    if (batch > 0 && (!d_a || !d_b || !d_c)) return MEXP_ERR_INVALID_ARGUMENT;
    const int dv = device_present();
    if (dv) return dv;
    return matmul_dev(d_a, d_b, d_c, n, batch, rounding, static_cast<cudaStream_t>(stream));
}

int mexp_lincomb_batched(const double* coeffs, const double* const* d_mats, int k, double* d_out,
                         int64_t len, void* stream) {
    if (k < 1 || len < 0 || !coeffs || !d_mats || (len > 0 && !d_out)) return MEXP_ERR_INVALID_ARGUMENT;
    for (int i = 0; i < k; ++i)
        if (len > 0 && !d_mats[i]) return MEXP_ERR_INVALID_ARGUMENT;
    const int dv = device_present();
    if (dv) return dv;
    return lincomb_dev(coeffs, d_mats, k, d_out, len, static_cast<cudaStream_t>(stream));
}

int mexp_one_norm_batched(const double* d_a, int n, int64_t batch, double* d_norms, void* stream) {
    if (n < 1 || batch < 0 || (batch > 0 && (!d_a || !d_norms))) return MEXP_ERR_INVALID_ARGUMENT;
    const int dv = device_present();
    if (dv) return dv;
    return one_norm_dev(d_a, n, batch, d_norms, static_cast<cudaStream_t>(stream));
}

int mexp_lu_solve_batched(const double* d_m, const double* d_rhs, double* d_x, int n, int64_t batch,
                          int32_t* d_status, void* stream) {
    if (n < 1 || batch < 0 || (batch > 0 && (!d_m || !d_rhs || !d_x || !d_status)))
        return MEXP_ERR_INVALID_ARGUMENT;
    const int dv = device_present();
    if (dv) return dv;
    return lu_solve_dev(d_m, d_rhs, d_x, n, batch, d_status, static_cast<cudaStream_t>(stream));
}

// Library-internal entry behind the C++ drop-in's dense layer (dropin.cpp):
// one routine on host matrices, every intermediate on the device.
//   op: see the switch below; in[0..nin) host n x n inputs; coeffs
//   (lincomb); arg: s / degree / order; out: n x n (one double for
//   ONE_NORM); iin / iout: the n pivot rows of lu_apply / lu_factor;
//   *products / *solves receive the routine's ledger entries.
int mexp_b200_dense_call(int op, int arg, const double* const* in, int nin, const double* coeffs, int n,
                         double* out, const int32_t* iin, int32_t* iout, int64_t* products,
                         int64_t* solves) {
    if (n < 1 || !out || nin < 0 || (nin > 0 && !in)) return MEXP_ERR_INVALID_ARGUMENT;
    const int dv = device_present();
    if (dv) return dv;
    static cudaStream_t streams[64] = {};
    static std::mutex mus[64];
    int dev = 0;
    DCUDA(cudaGetDevice(&dev));
    dev &= 63;
    std::lock_guard<std::mutex> lock(mus[dev]);
    if (!streams[dev]) DCUDA(cudaStreamCreateWithFlags(&streams[dev], cudaStreamNonBlocking));
    cudaStream_t st = streams[dev];
    const size_t nn = size_t(n) * n;
    if (products) *products = 0;
    if (solves) *solves = 0;
    // 0 MATMUL, 1 LINCOMB, 2 ONE_NORM, 3 LU_SOLVE, 4 SQUARINGS, 5 T8, 6 T12,
    // 7 T18, 8 PS(arg), 9 PSI9, 10 TAYLOR_ORACLE(arg), 11 PSI_ORACLE(arg),
    // 12 PADE(arg = order), 13 TAYLOR_NEW(arg = degree), 14 TAYLOR_PS(arg),
    // 15 LU_FACTOR (out = LU, iout = perm), 16 LU_APPLY (in = LU, rhs; iin = perm)
    Program p(n, st);
    int r = MEXP_OK;
    if (op == 15 || op == 16) {
        if (nin != (op == 15 ? 1 : 2) || (op == 15 ? !iout : !iin)) return MEXP_ERR_INVALID_ARGUMENT;
        AsyncBuffer buf(st);
        DCUDA(buf.alloc(sizeof(double) * nn * 3 + sizeof(int32_t) * (n + 1)));
        double* d_lu = buf.get<double>();
        double* d_r = d_lu + nn;
        double* d_x = d_r + nn;
        int32_t* d_perm = reinterpret_cast<int32_t*>(d_x + nn);
        int32_t* d_st = d_perm + n;
        int32_t h_st = 0;
        if (op == 15) {
            DCUDA(cudaMemcpyAsync(d_r, in[0], sizeof(double) * nn, cudaMemcpyHostToDevice, st));
            TRY(lu_solve_dev(d_r, nullptr, nullptr, n, 1, d_st, st, kLuFactor, d_lu, d_perm));
            DCUDA(cudaMemcpyAsync(out, d_lu, sizeof(double) * nn, cudaMemcpyDeviceToHost, st));
            DCUDA(cudaMemcpyAsync(iout, d_perm, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, st));
        } else {
            DCUDA(cudaMemcpyAsync(d_lu, in[0], sizeof(double) * nn, cudaMemcpyHostToDevice, st));
            DCUDA(cudaMemcpyAsync(d_r, in[1], sizeof(double) * nn, cudaMemcpyHostToDevice, st));
            DCUDA(cudaMemcpyAsync(d_perm, iin, sizeof(int32_t) * n, cudaMemcpyHostToDevice, st));
            TRY(lu_solve_dev(nullptr, d_r, d_x, n, 1, d_st, st, kLuApply, d_lu, d_perm));
            DCUDA(cudaMemcpyAsync(out, d_x, sizeof(double) * nn, cudaMemcpyDeviceToHost, st));
        }
        DCUDA(cudaMemcpyAsync(&h_st, d_st, sizeof h_st, cudaMemcpyDeviceToHost, st));
        DCUDA(cudaStreamSynchronize(st));
        return h_st;
    }
    if (op == 0 || op == 3) {  // two inputs
        if (nin != 2) return MEXP_ERR_INVALID_ARGUMENT;
        TRY(p.init(in[0], 3));
        DCUDA(cudaMemcpyAsync(p.at(1), in[1], sizeof(double) * nn, cudaMemcpyHostToDevice, st));
        r = op == 0 ? p.mm(2, 0, 1, false) : p.solve(2, 0, 1);
        if (r) {
            cudaStreamSynchronize(st);
            return r;
        }
        return p.finish(2, out);
    }
    if (op == 1) {  // lincomb of nin host matrices (arg 1: n is the flat length)
        if (nin < 1 || !coeffs) return MEXP_ERR_INVALID_ARGUMENT;
        const size_t nn = arg == 1 ? size_t(n) : size_t(n) * n;
        AsyncBuffer buf(st);
        DCUDA(buf.alloc(sizeof(double) * nn * (nin + 1)));
        std::vector<const double*> mats;
        for (int i = 0; i < nin; ++i) {
            double* d = buf.get<double>() + nn * i;
            DCUDA(cudaMemcpyAsync(d, in[i], sizeof(double) * nn, cudaMemcpyHostToDevice, st));
            mats.push_back(d);
        }
        double* d_out = buf.get<double>() + nn * nin;
        TRY(lincomb_dev(coeffs, mats.data(), nin, d_out, int64_t(nn), st));
        DCUDA(cudaMemcpyAsync(out, d_out, sizeof(double) * nn, cudaMemcpyDeviceToHost, st));
        DCUDA(cudaStreamSynchronize(st));
        return MEXP_OK;
    }
    if (nin != 1) return MEXP_ERR_INVALID_ARGUMENT;
    if (op == 2) {  // one_norm
        AsyncBuffer buf(st);
        DCUDA(buf.alloc(sizeof(double) * (nn + 1)));
        DCUDA(cudaMemcpyAsync(buf.get<double>(), in[0], sizeof(double) * nn, cudaMemcpyHostToDevice, st));
        TRY(one_norm_dev(buf.get<double>(), n, 1, buf.get<double>() + nn, st));
        DCUDA(cudaMemcpyAsync(out, buf.get<double>() + nn, sizeof(double), cudaMemcpyDeviceToHost, st));
        DCUDA(cudaStreamSynchronize(st));
        return MEXP_OK;
    }
    const Tables t;
    TRY(p.init(in[0], 16));
    constexpr int OUT = 15;
    switch (op) {
        case 4: {  // squarings (expm.cpp:31-35): X <- X X, s times, each a product
            if (arg < 0) return MEXP_ERR_INVALID_ARGUMENT;
            TRY(p.copy(OUT, A));
            for (int k = 0; k < arg; ++k) {
                TRY(p.mm(2, OUT, OUT));
                TRY(p.copy(OUT, 2));
            }
            break;
        }
        case 5: r = run_t8(p, OUT); break;
        case 6: r = run_t12(p, t, OUT); break;
        case 7: r = run_t18(p, t, OUT); break;
        case 8: r = run_ps(p, arg, OUT); break;
        case 9: r = run_psi9(p, OUT); break;
        case 10:
        case 11:
            if (op == 10 ? arg < 0 : arg < 1) return MEXP_ERR_INVALID_ARGUMENT;
            r = run_horner(p, arg, op == 10, OUT);
            break;
        case 12:
            if (arg < 2 || arg > 26 || arg % 2) return MEXP_ERR_INVALID_ARGUMENT;
            r = run_pade(p, arg, OUT);
            break;
        case 13:  // eval_taylor_new degree dispatch (taylor_schemes.cpp:211-227)
        case 14:  // eval_taylor_ps (:229-232)
            if (arg == 1) r = p.lc(OUT, {1.0, 1.0}, {I, A});
            else if (arg == 2 || arg == 4) r = run_ps(p, arg, OUT);
            else if (op == 13 && arg == 8) r = run_t8(p, OUT);
            else if (op == 13 && arg == 12) r = run_t12(p, t, OUT);
            else if (op == 13 && arg == 18) r = run_t18(p, t, OUT);
            else if (op == 14 && (arg == 6 || arg == 9 || arg == 16)) r = run_ps(p, arg, OUT);
            else return MEXP_ERR_UNSUPPORTED;
            break;
        default: return MEXP_ERR_INVALID_ARGUMENT;
    }
    if (r) {
        cudaStreamSynchronize(st);
        return r;
    }
    if (products) *products = p.products;
    if (solves) *solves = p.solves;
    return p.finish(OUT, out);
}

// Psi9 and pade_coeffs tables for the drop-in's host accessors
void mexp_b200_psi9_coefficients(double* x) {
    const Psi9 c = psi9_coeffs();
    for (int i = 1; i <= 9; ++i) x[i - 1] = c.x[i];
}

int mexp_b200_pade_coefficients(int m, double* b) {
    if (m < 1 || m > 13) return -1;
    for (int j = 0; j <= m; ++j) b[j] = kPadeHost[m - 1][j];
    return m + 1;
}

}  // extern "C"
