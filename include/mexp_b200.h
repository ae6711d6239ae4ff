/*
 * mexp_b200 — C ABI of the B200 (sm_100a) scaling-and-squaring matrix
 * exponential built on the reduced-product Taylor schemes of arXiv 1710.10989
 * (Family::TaylorNew of the reference `mexp` library), with the reference's
 * two comparison families: Paterson-Stockmeyer Taylor (TaylorPS) and the
 * diagonal Pade approximants (PadeDiagonal).
 *
 * The reference has no FFI layer: its operator boundary is the C++ API in
 * namespace mexp (proj/include/mexp/expm.hpp, theta_tables.hpp). Each entry
 * point below is the plain-pointer form of the reference call it replaces
 * (cited per function); the C++ drop-in (include/mexp/expm.hpp in this repo)
 * sits on top of these, and so would a ctypes / cgo / JNI binding.
 *
 * Conventions
 *   - matrices are square, row-major, contiguous; a batch is `batch`
 *     consecutive n*n blocks;
 *   - no exceptions cross this ABI: every call returns an mexp_status;
 *   - there is NO CPU fallback: with no usable CUDA device every compute
 *     call returns MEXP_ERR_NO_DEVICE;
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default).
 */
#ifndef MEXP_B200_H
#define MEXP_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MEXP_B200_ABI_VERSION 3

/* Status codes. The C++ drop-in maps 1-3 to std::invalid_argument with the
 * reference's messages (expm.cpp:13, expm.cpp:38, taylor_schemes.cpp:225)
 * and 7 to std::runtime_error (kernels.cpp:72). */
typedef enum {
    MEXP_OK = 0,
    MEXP_ERR_NONFINITE = 1,       /* "non-finite matrix entry"           expm.cpp:38 */
    MEXP_ERR_NORM_NONFINITE = 2,  /* "norm must be finite and nonnegative" expm.cpp:13 */
    MEXP_ERR_INVALID_ARGUMENT = 3,/* bad n / batch / enum value, dimension errors */
    MEXP_ERR_UNSUPPORTED = 4,     /* family/dtype/n/rounding combination not built */
    MEXP_ERR_CUDA = 5,            /* CUDA runtime error (see mexp_last_cuda_error) */
    MEXP_ERR_NO_DEVICE = 6,       /* no CUDA device: there is no CPU fallback */
    MEXP_ERR_SINGULAR = 7         /* "singular denominator" (Pade solve)  kernels.cpp:72 */
} mexp_status;

/* theta_tables.hpp:8 (enum class Family). TaylorNew and TaylorPS run for every
 * n and dtype; so does PadeDiagonal (scaling and squaring with r_m,
 * m = 2..26 even, and a batched pivoted LU solve). */
typedef enum { MEXP_FAMILY_TAYLOR_NEW = 0, MEXP_FAMILY_TAYLOR_PS = 1, MEXP_FAMILY_PADE = 2 } mexp_family;

/* theta_tables.hpp:9 (enum class Accuracy): selects the theta table, i.e. the
 * backward-error target u = 2^-24 (Single) or 2^-53 (Double). */
typedef enum { MEXP_ACCURACY_SINGLE = 0, MEXP_ACCURACY_DOUBLE = 1 } mexp_accuracy;

/* Storage/arithmetic type of a batched call. F64 is the reference's type;
 * F32 evaluates in fp32 with FFMA (never TF32) for n <= 64, norm and (m,s) in
 * fp64; beyond n = 64 (and for the Pade family) fp32 storage runs the fp64
 * engine on the widened values and rounds e^A once to float. */
typedef enum { MEXP_F64 = 0, MEXP_F32 = 1 } mexp_dtype;

/* Rounding policy of the fp64 path:
 *   REFERENCE: products and linear combinations with separately rounded
 *              multiplies and adds in the reference's accumulation order
 *              (kernels.cpp:16-37, -ffp-contract=off) -> e^A bit-identical
 *              to the reference (n > 64: k-ordered DMUL+DADD GEMMs on the
 *              CUDA cores; the Pade LU is DMMA-only and refuses it);
 *   FAST:      FP64 tensor-core DMMA products, FMA combinations;
 *   AUTO:      FAST, except matrices with s >= 3 + floor(log2 n) squarings
 *              (every matrix for n < 8), whose rounding differences the
 *              squarings amplify: those run REFERENCE end to end (so they are
 *              bit-identical to the reference), for every n. Checked within
 *              50 n u on all nine reference gallery kinds, n = 2..512, s <= 14
 *              (tests/test_gpu_auto_stress.py).
 * F32 with n <= 64 ignores it. */
typedef enum { MEXP_ROUND_AUTO = 0, MEXP_ROUND_REFERENCE = 1, MEXP_ROUND_FAST = 2 } mexp_rounding;

/* Per-matrix selection record written by the batched calls (16 bytes).
 * norm_in == ExpmReport::norm_in (expm.hpp:31), degree/s == Selection
 * (expm.hpp:10-13); cost_thirds = 3 * (products(degree) + s) (expm.cpp:71). */
typedef struct {
    double norm_in;
    int16_t degree;
    int16_t s;
    int32_t status; /* mexp_status of this matrix */
} mexp_selection;

/* ExpmReport (expm.hpp:23-32) minus the result matrix. */
typedef struct {
    int32_t family;
    int32_t degree;
    int32_t s;
    int32_t reserved;
    int64_t cost_thirds;
    double norm_in;
} mexp_report;

/* ---- selection logic (host, pure table arithmetic) ------------------- */

/* mexp::select (expm.hpp:18, expm.cpp:11-29). */
int mexp_select(double norm, int accuracy, int family, int32_t* degree, int32_t* s);

/* mexp::selection_table (theta_tables.hpp:32, theta_tables.cpp:77-85):
 * writes up to `cap` entries (degree, products, theta); returns the count or
 * a negative mexp_status. */
int mexp_selection_table(int accuracy, int family, int32_t* degrees, int32_t* products,
                         double* thetas, int cap);

/* mexp::unit_roundoff (theta_tables.hpp:11). */
double mexp_unit_roundoff(int accuracy);

/* ---- the hot path ----------------------------------------------------- */

/* mexp::expm (expm.hpp:37, expm.cpp:37-74) on ONE host matrix, synchronous.
 * `result` receives e^A (n*n doubles); `report` may be NULL. Runs on the
 * current device with the default rounding policy. */
int mexp_expm(const double* a, int n, int accuracy, int family, double* result,
              mexp_report* report);

/* Batched expm on DEVICE buffers, asynchronous on `stream`. d_a and d_out
 * hold `batch` n x n matrices of `dtype`; d_sel (may be NULL) receives one
 * mexp_selection per matrix. Per-matrix errors (non-finite input, overflowing
 * norm, singular Pade denominator) are reported in d_sel[i].status with
 * d_out[i] filled with NaN; the
 * call itself returns MEXP_OK once the work is enqueued. d_a and d_out must
 * not overlap. n may be any value >= 1. */
int mexp_expm_batched(const void* d_a, void* d_out, int dtype, int n, int64_t batch,
                      int accuracy, int family, int rounding, mexp_selection* d_sel,
                      void* stream);

/* Batched expm on HOST buffers, synchronous: chunked host->device copies,
 * kernels and device->host copies overlapped on internal streams (pinned
 * host buffers give full PCIe rate). h_sel may be NULL. Returns the first
 * per-matrix error status (and its index in *first_error, if non-NULL) or
 * MEXP_OK. This is the reference-facing end-to-end call. */
int mexp_expm_batched_host(const void* h_a, void* h_out, int dtype, int n, int64_t batch,
                           int accuracy, int family, int rounding, mexp_selection* h_sel,
                           int64_t* first_error);

/* mexp_expm_batched_host sharded by matrix across several GPUs of this node
 * (the reference's only parallelism is the OpenMP
 * row split of one product, kernels.cpp:16-27, so the split is this path's
 * own). Device k of `devices` (k = 0..ndevices-1) owns the contiguous range
 * [k*B/G + min(k, B%G), ...) -- the first B%G devices one matrix more -- and
 * runs the single-device host pipeline on its own host thread, i.e. over its
 * own PCIe link; no data moves between GPUs. Results, records and the
 * returned status / *first_error (lowest failing global index) equal those of
 * the single-device call bit for bit. devices == NULL or ndevices <= 0 uses
 * every visible device. A device may appear more than once (its shards then
 * run one after another). */
int mexp_expm_batched_host_multi(const void* h_a, void* h_out, int dtype, int n, int64_t batch,
                                 int accuracy, int family, int rounding, mexp_selection* h_sel,
                                 int64_t* first_error, const int* devices, int ndevices);

/* Number of CUDA devices this library can use (0 without a driver/device). */
int mexp_device_count(void);

/* mexp::squarings (expm.hpp:21, expm.cpp:31-35) on device: X <- X^(2^s) for
 * each of `batch` fp64 matrices, in place, s squarings each. */
int mexp_squarings_batched(double* d_x, int n, int64_t batch, int s, int rounding,
                           void* stream);

/* ---- the reference's dense-matrix layer (kernels.hpp:15-24) ------------
 * Device buffers of `batch` row-major n x n fp64 matrices, asynchronous on
 * `stream` unless noted. Every operation runs in the reference's arithmetic
 * (separately rounded multiplies and adds in the reference's order), so the
 * results are bit-identical to the reference's kernels. */

/* kernels::matmul (kernels.cpp:16-27): C = A B, k ascending from 0.0.
 * REFERENCE rounding: bit-identical; FAST / AUTO: FMA (n <= 64) or the DMMA
 * GEMM (n > 64). For n > 64 the call is host-synchronous. */
int mexp_matmul_batched(const double* d_a, const double* d_b, double* d_c, int n, int64_t batch,
                        int rounding, void* stream);

/* kernels::lincomb (kernels.cpp:29-37): d_out[e] = sum_i coeffs[i] * d_mats[i][e]
 * for e < len, summed left to right. `coeffs` and the array `d_mats` of k
 * device pointers are host arrays; kernels::scale is k = 1. */
int mexp_lincomb_batched(const double* coeffs, const double* const* d_mats, int k, double* d_out,
                         int64_t len, void* stream);

/* kernels::one_norm (kernels.cpp:44-53): d_norms[i] = max column sum of |A_i|,
 * exactly the reference's value. */
int mexp_one_norm_batched(const double* d_a, int n, int64_t batch, double* d_norms, void* stream);

/* lu_solve (dense_matrix.cpp:112-118, kernels.cpp:55-112): X = M^-1 R with
 * partial pivoting, one pivoted LU per matrix in the reference's arithmetic.
 * d_status[i] = MEXP_OK, or MEXP_ERR_SINGULAR on an exactly zero pivot
 * (X_i is then NaN). */
int mexp_lu_solve_batched(const double* d_m, const double* d_rhs, double* d_x, int n, int64_t batch,
                          int32_t* d_status, void* stream);

/* ---- runtime ---------------------------------------------------------- */

const char* mexp_status_string(int status);
/* Last CUDA error string recorded by a call that returned MEXP_ERR_CUDA. */
const char* mexp_last_cuda_error(void);
/* Number of kernels this library has launched in this process. */
uint64_t mexp_launch_count(void);
/* ABI version (MEXP_B200_ABI_VERSION) and device check: returns MEXP_OK if a
 * CUDA device of compute capability 10.x is usable. */
int mexp_abi_version(void);
int mexp_device_check(void);

#ifdef __cplusplus
}
#endif

#endif /* MEXP_B200_H */
