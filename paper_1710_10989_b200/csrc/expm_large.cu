// Large-n (n > 64) fp64 expm: batched FP64 tensor-core (DMMA) GEMMs with the
// schemes' linear combinations fused into the product epilogues.
//
// Pipeline per call (all matrices of the batch):
//   1. norm_cols: one thread per column sums |a_ij| over rows i = 0..n-1 in
//      order (kernels.cpp:44-53); the max over columns is an atomicMax on the
//      bits (non-negative doubles order like their bit patterns); a flag
//      records non-finite entries (dense_matrix.cpp:54-58).
//   2. select: (m, s) per matrix (expm.cpp:11-29) -> mexp_selection records.
//   3. one 16-byte-per-matrix device->host read of the records; the host
//      groups the matrices by degree and by number of squarings.
//   4. prep: W0 = 2^-s A, zero-padded to np = 128 * ceil(n / 128) (padding
//      keeps e^A's top-left block: the padded matrix is block diagonal).
//   5. the degree's scheme as a chain of batched GEMMs whose epilogues form
//      the y-combinations (taylor_schemes.cpp:104-157), e.g. for T18:
//        A2 = A*A;  A3 = A2*A;  A6 = A3*A3 -> epilogue writes B1..B5;
//        B1*B5 -> epilogue A9 = . + B4, L = B3 + A9;  L*A9 -> T = . + B2
//   6. s squarings (expm.cpp:31-35) as batched GEMMs over the matrices whose
//      s reaches that step, ping-ponging two buffers;
//   7. each matrix's last GEMM writes e^A straight into the caller's output
//      (when n is a multiple of 128; otherwise an unpad copy at the end).
//
// Family::PadeDiagonal: the same GEMM chain forms U, V (pade.cpp:50-113) and,
// in the last product's epilogue, M = V - U and R = V + U; lu_batched.cu then
// overwrites R with M^-1 R before the squarings.
//
// GEMM: 128x128 CTA tile, 8 warps each 64x32 (8x4 DMMA m8n8k4 tiles, 64 fp64
// accumulators per lane), k-tiles of 32 through a 3-stage cp.async ring in
// shared memory (rows padded to 4 (mod 16) doubles: conflict-free fragment
// loads). One DMMA occupies an SM sub-partition's FP64 pipe for 16 cycles, so
// 32 independent DMMAs per k-step keep all four pipes saturated.
#include <algorithm>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include <cuda.h>
#include <cudaTypedefs.h>

#include "async_buffer.hpp"
#include "device_once.hpp"
#include "expm_common.cuh"
#include "expm_large.cuh"
#include "lu_batched.cuh"
#include "tma.cuh"

namespace mexp_b200 {

namespace {

thread_local std::string g_err;

#define LCUDA(call)                                                              \
    do {                                                                         \
        cudaError_t e_ = (call);                                                 \
        if (e_ != cudaSuccess) {                                                 \
            g_err = std::string(#call) + ": " + cudaGetErrorString(e_);          \
            return MEXP_ERR_CUDA;                                                \
        }                                                                        \
    } while (0)

// CTA shape. 0: 128 x 128 tiles, 8 warps of 64 x 32, k-tiles of 32 in 3
// stages, one CTA per SM; 1: 128 x 64 tiles, 8 warps of 32 x 32, k-tiles of
// 32 double-buffered, two CTAs per SM (one CTA's epilogue overlaps the
// other's mainloop). Measured: profiles/gemm_tma_r1.txt.
#ifndef MEXP_GEMM_SHAPE
#define MEXP_GEMM_SHAPE 1
#endif
#ifndef MEXP_GEMM_BK
#define MEXP_GEMM_BK 32
#endif
// 0: cp.async (LDGSTS) for both operands; 1: row-wise cp.async.bulk for both;
// 2: X tiles by tensor-map TMA (cp.async.bulk.tensor, 128B swizzle), Y rows
// by cp.async.bulk (measured: profiles/gemm_tma_r1.txt)
#ifndef MEXP_GEMM_TMA
#define MEXP_GEMM_TMA 2
#endif
#ifndef MEXP_GEMM_STAGES
#define MEXP_GEMM_STAGES (MEXP_GEMM_SHAPE == 1 ? (MEXP_GEMM_BK == 16 ? 4 : 2) : (MEXP_GEMM_BK == 16 ? 4 : 3))
#endif
constexpr int BM = 128, BN = MEXP_GEMM_SHAPE == 1 ? 64 : 128, BK = MEXP_GEMM_BK,
              STAGES = MEXP_GEMM_STAGES;
constexpr int LDA = BK + 4;   // 4 (mod 16) doubles
constexpr int LDB = BN + 4;   // 4 (mod 16) doubles
constexpr int WM = MEXP_GEMM_SHAPE == 1 ? 32 : 64, WN = 32, TM = WM / 8, TN = WN / 8;
constexpr int WARPS_N = BN / WN;
constexpr int GEMM_THREADS = 256;
constexpr int GEMM_MIN_CTAS = MEXP_GEMM_SHAPE == 1 ? 2 : 1;
static_assert((BM / WM) * WARPS_N * 32 == GEMM_THREADS, "warp cover");
#if MEXP_GEMM_TMA == 2
// X stage: BK / 16 boxes of 128 rows x 16 doubles (128 B), TMA's 128B swizzle
// (16-byte chunk c of row r at c ^ (r & 7)): conflict-free fragment loads
constexpr int XBOX = 16;
constexpr size_t A_DOUBLES = size_t(BM) * BK;
static_assert(BK % XBOX == 0 && (BM * XBOX * 8) % 1024 == 0, "swizzled boxes stay 1024 B aligned");
#else
constexpr size_t A_DOUBLES = size_t(BM) * LDA;
#endif
// stages stay 1024 B aligned (TMA 128B-swizzle destinations)
constexpr size_t STAGE_DOUBLES = (A_DOUBLES + size_t(BK) * LDB + 127) / 128 * 128;
// + the stages' mbarriers and slack to align the ring to 1024 B
constexpr size_t GEMM_SMEM = STAGES * STAGE_DOUBLES * sizeof(double) + 64 + 1024;

// Epilogues. c = the product's value at (i, j); id = (i == j); in/out are
// the step's extra matrices at the same position.
enum Epi : int {
    EPI_STORE,    // o0 = c
    EPI_ADD,      // o0 = c + in0
    EPI_AL,       // o0 = X = c + in0 ; o1 = in1 + X        (T18: A9, L; T12: A6, L)
    EPI_T18_B,    // c = A6; in = A, A2, A3 -> o0..o4 = B1, B2, B3, B4, B5
    EPI_T12_B,    // c = A3; in = A, A2     -> o0..o3 = B1, B2, B3, B4
    EPI_T8_1,     // c = A2; in = A         -> o0 = A2, o1 = x1 A + x2 A2
    EPI_T8_2,     // c = A4; in = A, A2     -> o0 = x3 A2 + A4, o1 = x4 I + x5 A + x6 A2 + x7 A4
    EPI_T8_3,     // c = A8; in = A, A2     -> o0 = y0 I + y1 A + y2 A2 + A8
    EPI_T4_1,     // c = A2; in = A         -> o0 = A2, o1 = (I/2 + A/6) + A2/24
    EPI_T4_2,     // c = inner*A2; in = A   -> o0 = (I + A) + c
    EPI_T2,       // c = A2; in = A         -> o0 = (I + A) + A2/2
    EPI_PS_B,     // c = X*Y; in0..in2 (each may be null) -> o0 = c (unless !store_c),
                  //   o_j = lc[j-1] . {I, in0, in1, in2, c} for j = 1..nlc
                  //   (Paterson-Stockmeyer chunks, the Pade lincombs and M, R)
};

struct GemmArgs {
    const double* X;
    const double* Y;
    const double* in[3];
    double* out[5];
    double lc[4][5];      // EPI_PS_B coefficients (runtime: one kernel for every degree)
    int nlc;
    int store_c;          // EPI_PS_B: write c to out[0]
    double* final_out;    // the caller's e^A buffer (list entries with bit 31 set)
    const int32_t* list;  // participating matrix indices (blockIdx.z); bit 31 set =
                          // this is the matrix's last product: out[0] -> final_out
    int np;
    int64_t mstride;      // np * np
    int n;                // the true dimension: the exact product sums k < n only
    // prep-free T18 on the unscaled input (DMMA pass only): c *= 2^-(scale_c s)
    // and in[0] *= 2^-s on load, s = sel[matrix].s -- exact power-of-two
    // scalings, so the values equal those of the scaled copy
    const mexp_selection* sel;
    int scale_c;
    int scale_in0;
};

// Left-to-right linear combination c0*m0 + c1*m1 + ... in the arithmetic of
// Ops: ExactOps is the reference's lincomb (kernels.cpp:29-37: every multiply
// and add rounded separately, in order); FastOps fuses into FMAs.
template <class O>
__device__ __forceinline__ double lcx(double c0, double m0) {
    return O::mul(c0, m0);
}
template <class O, class... R>
__device__ __forceinline__ double lcx(double c0, double m0, double c1, double m1, R... rest) {
    return lcx<O>(1.0, O::mac(O::mul(c0, m0), c1, m1), rest...);
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    const uint32_t s = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// The epilogues in the arithmetic of O. For ExactOps every formula is the
// reference's lincomb/add term for term (identity terms included, absent
// operands skipped), so REFERENCE rounding reproduces its bits.
// How many of g.in[] the epilogue reads (its loads are issued ahead of the
// stores, see epi_load).
template <int EPI>
constexpr int epi_inputs() {
    return EPI == EPI_STORE ? 0
         : (EPI == EPI_AL || EPI == EPI_T12_B || EPI == EPI_T8_2 || EPI == EPI_T8_3) ? 2
         : (EPI == EPI_T18_B || EPI == EPI_PS_B) ? 3
         : 1;
}
struct EpiIn {
    double2 v[3];
};
template <int EPI>
__device__ __forceinline__ EpiIn epi_load(const GemmArgs& g, int64_t base, int row, int col) {
    const int64_t off = base + int64_t(row) * g.np + col;
    EpiIn e;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        e.v[k] = make_double2(0.0, 0.0);
        // evict-first: an epilogue's inputs and outputs stream through HBM once
        // per GEMM at these sizes (no L2 reuse), so they should not displace
        // the mainloop's operand tiles (cfg4 61.3 -> 59.8 ms; T18's B
        // epilogue GEMM 10.4 -> 9.5 ms)
        if (k < epi_inputs<EPI>() && (EPI != EPI_PS_B || g.in[k]))
            e.v[k] = __ldcs(reinterpret_cast<const double2*>(g.in[k] + off));
    }
    return e;
}

template <int EPI, class O>
__device__ __forceinline__ void epilogue_pair(const GemmArgs& g, double* out0, int64_t base,
                                              int row, int col, double c0, double c1,
                                              const EpiIn& pre) {
    const int64_t off = base + int64_t(row) * g.np + col;
    const double id0 = (row == col) ? 1.0 : 0.0, id1 = (row == col + 1) ? 1.0 : 0.0;
    auto ld = [&](int k) { return pre.v[k]; };
    auto st = [&](int k, double a, double b) {
        __stcs(reinterpret_cast<double2*>((k == 0 ? out0 : g.out[k]) + off), make_double2(a, b));
    };
    if constexpr (EPI == EPI_STORE) {
        st(0, c0, c1);
    } else if constexpr (EPI == EPI_ADD) {  // add(b, P)
        const double2 b = ld(0);
        st(0, O::add(b.x, c0), O::add(b.y, c1));
    } else if constexpr (EPI == EPI_AL) {  // A9 = add(P, B4); L = add(B3, A9)
        const double2 b = ld(0), l = ld(1);
        const double x0 = O::add(c0, b.x), x1 = O::add(c1, b.y);
        st(0, x0, x1);
        st(1, O::add(l.x, x0), O::add(l.y, x1));
    } else if constexpr (EPI == EPI_T18_B) {  // lincomb(kT18A, {I,A,A2,A3}), lincomb(kT18B[j], {.., A6})
        const double2 a = ld(0), a2 = ld(1), a3 = ld(2);
        st(0, lcx<O>(c_t18a[0], id0, c_t18a[1], a.x, c_t18a[2], a2.x, c_t18a[3], a3.x),
           lcx<O>(c_t18a[0], id1, c_t18a[1], a.y, c_t18a[2], a2.y, c_t18a[3], a3.y));
#pragma unroll
        for (int j = 0; j < 4; ++j)
            st(1 + j,
               lcx<O>(c_t18b[j][0], id0, c_t18b[j][1], a.x, c_t18b[j][2], a2.x, c_t18b[j][3], a3.x,
                      c_t18b[j][4], c0),
               lcx<O>(c_t18b[j][0], id1, c_t18b[j][1], a.y, c_t18b[j][2], a2.y, c_t18b[j][3], a3.y,
                      c_t18b[j][4], c1));
    } else if constexpr (EPI == EPI_T12_B) {
        const double2 a = ld(0), a2 = ld(1);
#pragma unroll
        for (int j = 0; j < 4; ++j)
            st(j, lcx<O>(c_t12[0][j], id0, c_t12[1][j], a.x, c_t12[2][j], a2.x, c_t12[3][j], c0),
               lcx<O>(c_t12[0][j], id1, c_t12[1][j], a.y, c_t12[2][j], a2.y, c_t12[3][j], c1));
    } else if constexpr (EPI == EPI_T8_1) {
        const double2 a = ld(0);
        st(0, c0, c1);
        st(1, lcx<O>(T8C::x1, a.x, T8C::x2, c0), lcx<O>(T8C::x1, a.y, T8C::x2, c1));
    } else if constexpr (EPI == EPI_T8_2) {
        const double2 a = ld(0), a2 = ld(1);
        st(0, lcx<O>(T8C::x3, a2.x, 1.0, c0), lcx<O>(T8C::x3, a2.y, 1.0, c1));
        st(1, lcx<O>(T8C::x4, id0, T8C::x5, a.x, T8C::x6, a2.x, T8C::x7, c0),
           lcx<O>(T8C::x4, id1, T8C::x5, a.y, T8C::x6, a2.y, T8C::x7, c1));
    } else if constexpr (EPI == EPI_T8_3) {
        const double2 a = ld(0), a2 = ld(1);
        st(0, lcx<O>(T8C::y0, id0, T8C::y1, a.x, T8C::y2, a2.x, 1.0, c0),
           lcx<O>(T8C::y0, id1, T8C::y1, a.y, T8C::y2, a2.y, 1.0, c1));
    } else if constexpr (EPI == EPI_T4_1) {  // inner = lincomb({1, 1/4!}, {lincomb({1/2!, 1/3!}, {I, A}), A2})
        const double2 a = ld(0);
        st(0, c0, c1);
        st(1, lcx<O>(1.0, lcx<O>(kInvFact2, id0, kInvFact3, a.x), kInvFact4, c0),
           lcx<O>(1.0, lcx<O>(kInvFact2, id1, kInvFact3, a.y), kInvFact4, c1));
    } else if constexpr (EPI == EPI_T4_2) {  // add(f0, P), f0 = lincomb({1, 1}, {I, A})
        const double2 a = ld(0);
        st(0, O::add(lcx<O>(1.0, id0, 1.0, a.x), c0), O::add(lcx<O>(1.0, id1, 1.0, a.y), c1));
    } else if constexpr (EPI == EPI_T2) {  // lincomb({1, 1, 0.5}, {I, A, A2})
        const double2 a = ld(0);
        st(0, lcx<O>(1.0, id0, 1.0, a.x, 0.5, c0), lcx<O>(1.0, id1, 1.0, a.y, 0.5, c1));
    } else if constexpr (EPI == EPI_PS_B) {
        // rows of coefficients over {I, in0, in1, in2, c}; absent operands and a
        // zero coefficient of c contribute no term (the reference's lincombs
        // have no such term)
        const double2 z = make_double2(0.0, 0.0);
        const double2 a = g.in[0] ? ld(0) : z, a2 = g.in[1] ? ld(1) : z, a3 = g.in[2] ? ld(2) : z;
        if (g.store_c) st(0, c0, c1);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            if (j >= g.nlc) break;
            const double* k = g.lc[j];
            double r0 = O::mul(k[0], id0), r1 = O::mul(k[0], id1);
            if (g.in[0]) r0 = O::mac(r0, k[1], a.x), r1 = O::mac(r1, k[1], a.y);
            if (g.in[1]) r0 = O::mac(r0, k[2], a2.x), r1 = O::mac(r1, k[2], a2.y);
            if (g.in[2]) r0 = O::mac(r0, k[3], a3.x), r1 = O::mac(r1, k[3], a3.y);
            if (k[4] != 0.0) r0 = O::mac(r0, k[4], c0), r1 = O::mac(r1, k[4], c1);
            st(1 + j, r0, r1);
        }
    }
}

// Reference-rounded batched product (REFERENCE policy, n > 64): every output
// is 0.0 + x_i0*y_0j + x_i1*y_1j + ... over k < n in order, each multiply and
// add rounded (kernels.cpp:16-27), i.e. the reference's i-k-j loop bit for
// bit. 64 x 128 CTA tiles, 256 threads of 4 x 8 outputs (32 independent
// chains each: rows 4ty.., columns 2tx + {0, 1} + 32g), k-tiles of 16
// double-buffered in shared memory. Per k a thread loads 4 + 8 operands for
// 64 FP64 operations, which keeps shared memory at ~3/4 of the FP64 pipe's
// pace (a 4 x 4 tile loaded 8 for 32 and the two were co-bound).
constexpr int XBM = 64, XBN = 128, XK = 16, XLDA = XK + 2, XLDB = XBN + 2;  // rows 16-byte aligned
constexpr size_t EXACT_SMEM = (size_t(2) * XBM * XLDA + size_t(2) * XK * XLDB) * sizeof(double);

// 16-byte async copy of the first `bytes` (0, 8 or 16) of src, zero-filling the rest
__device__ __forceinline__ void cp_async16_zfill(void* smem, const void* gmem, int bytes) {
    const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(d), "l"(gmem), "r"(bytes)
                 : "memory");
}

template <int EPI>
__global__ void __launch_bounds__(256, 2) gemm_exact_kernel(GemmArgs g) {
    extern __shared__ __align__(16) double xsm[];
    double (*sa)[XBM][XLDA] = reinterpret_cast<double (*)[XBM][XLDA]>(xsm);
    double (*sb)[XK][XLDB] = reinterpret_cast<double (*)[XK][XLDB]>(xsm + 2 * XBM * XLDA);
    const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
    const int32_t entry = g.list[blockIdx.z];
    const int64_t mat = entry & 0x7fffffff;
    double* out0 = entry < 0 ? g.final_out : g.out[0];
    const int64_t base = mat * g.mstride;
    const double* X = g.X + base;
    const double* Y = g.Y + base;
    const int m0 = blockIdx.y * XBM, n0 = blockIdx.x * XBN;
    const int ktiles = (g.n + XK - 1) / XK;
    // k >= n is zero-filled (and never summed: the k loop stops at n)
    auto load = [&](int s, int kt) {
        const int k0 = kt * XK;
        for (int e = tid; e < XBM * XK / 2; e += 256) {
            const int r = e / (XK / 2), k = (e % (XK / 2)) * 2;
            const int valid = min(max(g.n - (k0 + k), 0), 2);
            cp_async16_zfill(&sa[s][r][k], X + int64_t(m0 + r) * g.np + min(k0 + k, g.np - 2), 8 * valid);
        }
        for (int e = tid; e < XK * XBN / 2; e += 256) {
            const int k = e / (XBN / 2), c = (e % (XBN / 2)) * 2;
            const bool ok = k0 + k < g.n;
            cp_async16_zfill(&sb[s][k][c], Y + int64_t(ok ? k0 + k : 0) * g.np + n0 + c, ok ? 16 : 0);
        }
        cp_commit();
    };
    double acc[4][8];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = 0.0;
    load(0, 0);
    for (int kt = 0; kt < ktiles; ++kt) {
        const int s = kt & 1;
        if (kt + 1 < ktiles) {
            load(s ^ 1, kt + 1);
            cp_wait<1>();
        } else {
            cp_wait<0>();
        }
        __syncthreads();
        const int kend = min(XK, g.n - kt * XK);  // never a padded term
        for (int k = 0; k < kend; ++k) {
            double a[4], b[8];
#pragma unroll
            for (int i = 0; i < 4; ++i) a[i] = sa[s][4 * ty + i][k];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const double2 v = *reinterpret_cast<const double2*>(&sb[s][k][2 * tx + 32 * q]);
                b[2 * q] = v.x;
                b[2 * q + 1] = v.y;
            }
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 8; ++j) acc[i][j] = __dadd_rn(acc[i][j], __dmul_rn(a[i], b[j]));
        }
        __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int row = m0 + 4 * ty + i, col = n0 + 2 * tx + 32 * q;
            epilogue_pair<EPI, ExactOps>(g, out0, base, row, col, acc[i][2 * q], acc[i][2 * q + 1],
                                         epi_load<EPI>(g, base, row, col));
        }
}

template <int EPI>
__global__ void __launch_bounds__(GEMM_THREADS, GEMM_MIN_CTAS)
    gemm_dmma_kernel(GemmArgs g, const __grid_constant__ CUtensorMap tmx) {
    extern __shared__ __align__(16) double smem_raw[];
    // 1024-byte aligned (the 128-byte TMA swizzle), derived from smem_raw by
    // pointer arithmetic so the compiler keeps the shared address space: the
    // fragment loads are LDS, not generic LD (a pointer rebuilt through
    // uintptr_t loses it)
    const uint32_t sbase = static_cast<uint32_t>(__cvta_generic_to_shared(smem_raw));
    double* const smem = smem_raw + ((((sbase + 1023u) & ~1023u) - sbase) / sizeof(double));
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int wm = warp / WARPS_N, wn = warp % WARPS_N;
    const int r = lane >> 2, q = lane & 3;
    const int32_t entry = g.list[blockIdx.z];
    const int64_t mat = entry & 0x7fffffff;
    double* out0 = entry < 0 ? g.final_out : g.out[0];
    const int64_t base = mat * g.mstride;
    const double* X = g.X + base;
    const double* Y = g.Y + base;
    const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
    const int ktiles = g.np / BK;
    double fc = 1.0, f0 = 1.0;
    if (g.scale_c | g.scale_in0) {
        const int s = g.sel[mat].s;
        if (g.scale_c) fc = pow2_neg(g.scale_c * s);
        if (g.scale_in0) f0 = pow2_neg(s);
    }

    auto stage_a = [&](int s) { return smem + s * STAGE_DOUBLES; };
    auto stage_b = [&](int s) { return smem + s * STAGE_DOUBLES + A_DOUBLES; };
    auto load = [&](int s, int kt) {
        double* sa = stage_a(s);
        double* sb = stage_b(s);
        const int k0 = kt * BK;
#pragma unroll
        for (int c = tid; c < BM * BK / 2; c += GEMM_THREADS) {
            const int row = c / (BK / 2), cc = (c % (BK / 2)) * 2;
            cp_async16(sa + row * LDA + cc, X + int64_t(m0 + row) * g.np + k0 + cc);
        }
#pragma unroll
        for (int c = tid; c < BK * BN / 2; c += GEMM_THREADS) {
            const int row = c / (BN / 2), cc = (c % (BN / 2)) * 2;
            cp_async16(sb + row * LDB + cc, Y + int64_t(k0 + row) * g.np + n0 + cc);
        }
    };

    double acc[TM][TN][2];
#pragma unroll
    for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

#if MEXP_GEMM_TMA
    // warp 0 streams each stage through the TMA engine (see MEXP_GEMM_TMA);
    // the stage's mbarrier completes on the bytes
    uint64_t* const full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_DOUBLES);
    constexpr unsigned kStageBytes = (BM * BK + BK * BN) * sizeof(double);
    (void)load;
    (void)tmx;
    if (tid == 0) {
        for (int st = 0; st < STAGES; ++st) mbar_init(&full[st], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    auto issue = [&](int st, int kt) {
        if (warp != 0) return;
        if (lane == 0) mbar_expect_tx(&full[st], kStageBytes);
        __syncwarp();
        double* sa = stage_a(st);
        double* sb = stage_b(st);
        const int k0 = kt * BK;
#if MEXP_GEMM_TMA == 2
        if (lane == 0)
#pragma unroll
            for (int b = 0; b < BK / XBOX; ++b)
                tma_load_3d(sa + b * BM * XBOX, &tmx, k0 + b * XBOX, m0, int(mat), &full[st]);
#else
        for (int row = lane; row < BM; row += 32)
            bulk_g2s(sa + row * LDA, X + int64_t(m0 + row) * g.np + k0, BK * sizeof(double), &full[st]);
#endif
        for (int row = lane; row < BK; row += 32)
            bulk_g2s(sb + row * LDB, Y + int64_t(k0 + row) * g.np + n0, BN * sizeof(double), &full[st]);
    };
#pragma unroll
    for (int st = 0; st < STAGES - 1; ++st)
        if (st < ktiles) issue(st, st);
#else
#pragma unroll
    for (int s = 0; s < STAGES - 1; ++s) {
        if (s < ktiles) load(s, s);
        cp_commit();
    }
#endif
    for (int kt = 0; kt < ktiles; ++kt) {
#if MEXP_GEMM_TMA
        __syncthreads();  // every warp is done with the stage about to be refilled
        const int nk = kt + STAGES - 1;
        if (nk < ktiles) issue(nk % STAGES, nk);
        mbar_wait(&full[kt % STAGES], unsigned(kt / STAGES) & 1u);
#else
        cp_wait<STAGES - 2>();
        __syncthreads();
        const int nk = kt + STAGES - 1;
        if (nk < ktiles) load(nk % STAGES, nk);
        cp_commit();
#endif
#if MEXP_GEMM_TMA == 2
        // row = wm*64 + 8i + r, so row & 7 = r; k = kk + q lies in box kk / 16
        const double* sa = stage_a(kt % STAGES) + (wm * WM + r) * XBOX + (q & 1);
#else
        const double* sa = stage_a(kt % STAGES) + (wm * WM + r) * LDA + q;
#endif
        const double* sb = stage_b(kt % STAGES) + q * LDB + wn * WN + r;
#pragma unroll
        for (int kk = 0; kk < BK; kk += 4) {
            double af[TM], bf[TN];
#if MEXP_GEMM_TMA == 2
            const int chunk = (((kk % XBOX) >> 1) + (q >> 1)) ^ r;
            const double* sak = sa + (kk / XBOX) * (BM * XBOX) + 2 * chunk;
#pragma unroll
            for (int i = 0; i < TM; ++i) af[i] = sak[i * 8 * XBOX];
#else
#pragma unroll
            for (int i = 0; i < TM; ++i) af[i] = sa[i * 8 * LDA + kk];
#endif
#pragma unroll
            for (int j = 0; j < TN; ++j) bf[j] = sb[kk * LDB + j * 8];
#pragma unroll
            for (int i = 0; i < TM; ++i)
#pragma unroll
                for (int j = 0; j < TN; ++j) dmma_8x8x4(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
        }
    }
#if !MEXP_GEMM_TMA
    cp_wait<0>();
#endif

    // Epilogue by 8-row slabs: the slab's inputs are all loaded before any of
    // its stores (the compiler cannot hoist loads over stores that may alias),
    // so a warp waits for one round trip per slab, not per pair.
#pragma unroll
    for (int i = 0; i < TM; ++i) {
        EpiIn pre[TN];
#pragma unroll
        for (int j = 0; j < TN; ++j)
            pre[j] = epi_load<EPI>(g, base, m0 + wm * WM + i * 8 + r, n0 + wn * WN + j * 8 + 2 * q);
        if (g.scale_in0)
#pragma unroll
            for (int j = 0; j < TN; ++j) pre[j].v[0] = make_double2(f0 * pre[j].v[0].x, f0 * pre[j].v[0].y);
#pragma unroll
        for (int j = 0; j < TN; ++j)
            epilogue_pair<EPI, FastOps>(g, out0, base, m0 + wm * WM + i * 8 + r,
                                        n0 + wn * WN + j * 8 + 2 * q, fc * acc[i][j][0], fc * acc[i][j][1],
                                        pre[j]);
    }
}

// ---- prologue / epilogue kernels -------------------------------------------
__global__ void norm_cols_kernel(const double* __restrict__ a, int n, int64_t batch,
                                 unsigned long long* __restrict__ maxbits,
                                 int* __restrict__ bad, int64_t m0) {
    const int64_t m = m0 + blockIdx.y;
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (m >= batch || j >= n) return;
    const double* p = a + m * int64_t(n) * n + j;
    double s = 0.0;
    bool fin = true;
    for (int i = 0; i < n; ++i) {
        const double v = __ldg(p + int64_t(i) * n);
        fin = fin && isfinite(v);
        s = __dadd_rn(s, fabs(v));
    }
    if (!fin) atomicOr(bad + m, 1);
    else atomicMax(maxbits + m, static_cast<unsigned long long>(__double_as_longlong(s)));
}

// device copy of n int32 from mapped pinned host memory: a kernel, not a
// cudaMemcpy, so it never waits behind the copy engine's queue
__global__ void upload_kernel(const int32_t* __restrict__ src, int32_t* __restrict__ dst, int64_t n) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
        dst[i] = src[i];
}

__global__ void select_kernel(const unsigned long long* __restrict__ maxbits,
                              const int* __restrict__ bad, int64_t batch, int acc_arg,
                              mexp_selection* __restrict__ sel, mexp_selection* __restrict__ host_sel) {
    const int accuracy = acc_arg & 15, family = acc_arg >> 4;  // mexp_accuracy | mexp_family << 4
    const int64_t m = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
    if (m >= batch) return;
    mexp_selection r;
    if (bad[m]) {
        r.norm_in = __longlong_as_double(0x7ff8000000000000ll);
        r.degree = 0;
        r.s = 0;
        r.status = MEXP_ERR_NONFINITE;
    } else {
        const double norm = __longlong_as_double(static_cast<long long>(maxbits[m]));
        const Sel s = select_device(norm, accuracy, family);
        r.norm_in = norm;
        r.degree = int16_t(s.degree);
        r.s = int16_t(s.s);
        r.status = s.status;
    }
    sel[m] = r;
    host_sel[m] = r;  // mapped pinned host memory: no copy-engine queue to wait in
}

// W0[m] = 2^-s A (zero padded), for the listed matrices; one block row-strip
// per (blockIdx.x, matrix), coalesced along rows, no 64-bit divisions
__global__ void prep_kernel(const double* __restrict__ a, double* __restrict__ w, int n, int np,
                            const int32_t* __restrict__ list, const mexp_selection* __restrict__ sel) {
    const int64_t m = list[blockIdx.y];
    const double f = pow2_neg(sel[m].s);
    if (n == np && (n & 1) == 0) {
        // unpadded: a flat scaled copy in 16-byte units (the input is read
        // once: evict-first)
        const int64_t half = int64_t(n) * n / 2;
        const double2* src = reinterpret_cast<const double2*>(a + m * int64_t(n) * n);
        double2* dst = reinterpret_cast<double2*>(w + m * int64_t(np) * np);
        for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < half;
             e += int64_t(gridDim.x) * blockDim.x) {
            const double2 v = __ldcs(src + e);
            dst[e] = make_double2(f * v.x, f * v.y);
        }
        return;
    }
    for (int i = blockIdx.x; i < np; i += gridDim.x) {
        double* wr = w + m * int64_t(np) * np + int64_t(i) * np;
        const double* ar = a + m * int64_t(n) * n + int64_t(i) * n;
        for (int j = threadIdx.x; j < np; j += blockDim.x)
            wr[j] = (i < n && j < n) ? f * ar[j] : 0.0;
    }
}

// T1 = I + A (eval_taylor_new degree 1), elementwise; r has row stride ldr
// (np for the workspace, n when writing the caller's output directly)
__global__ void t1_kernel(const double* __restrict__ w0, double* __restrict__ r, int n, int np,
                          int ldr, const int32_t* __restrict__ list) {
    const int64_t m = list[blockIdx.y];
    for (int i = blockIdx.x; i < n; i += gridDim.x)
        for (int j = threadIdx.x; j < n; j += blockDim.x)
            r[m * int64_t(ldr) * ldr + int64_t(i) * ldr + j] =
                (i == j ? 1.0 : 0.0) + w0[m * int64_t(np) * np + int64_t(i) * np + j];
}

// out[m] = top-left n x n of src[m] (padded layout), for the listed matrices
__global__ void unpad_kernel(const double* __restrict__ src, double* __restrict__ out, int n,
                             int np, const int32_t* __restrict__ list) {
    const int64_t m = list[blockIdx.y];
    for (int i = blockIdx.x; i < n; i += gridDim.x)
        for (int j = threadIdx.x; j < n; j += blockDim.x)
            out[m * int64_t(n) * n + int64_t(i) * n + j] = src[m * int64_t(np) * np + int64_t(i) * np + j];
}

// r_2 (no product): M = b0 I - b1 A, R = b0 I + b1 A (pade.cpp:99-109)
__global__ void pade2_kernel(const double* __restrict__ a, double* __restrict__ m_out,
                             double* __restrict__ r_out, int np, const int32_t* __restrict__ list,
                             double b0, double b1) {
    const int64_t m = list[blockIdx.y];
    for (int i = blockIdx.x; i < np; i += gridDim.x)
        for (int j = threadIdx.x; j < np; j += blockDim.x) {
            const int64_t e = m * int64_t(np) * np + int64_t(i) * np + j;
            const double id = i == j ? b0 : 0.0, u = b1 * a[e];
            m_out[e] = id - u;
            r_out[e] = id + u;
        }
}

// NaN over e^A of the listed matrices whose Pade solve met a zero pivot
__global__ void nan_singular_kernel(double* __restrict__ out, int n,
                                    const int32_t* __restrict__ list,
                                    const mexp_selection* __restrict__ sel) {
    const int64_t m = list[blockIdx.y];
    if (sel[m].status != MEXP_ERR_SINGULAR) return;
    const int64_t total = int64_t(n) * n;
    for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total;
         e += int64_t(gridDim.x) * blockDim.x)
        out[m * total + e] = __longlong_as_double(0x7ff8000000000000ll);
}

// NaN for the listed matrices (per-matrix errors: non-finite input, norm overflow)
__global__ void nan_kernel(double* __restrict__ out, int n, const int32_t* __restrict__ list) {
    const int64_t m = list[blockIdx.y];
    const int64_t total = int64_t(n) * n;
    for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total;
         e += int64_t(gridDim.x) * blockDim.x)
        out[m * total + e] = __longlong_as_double(0x7ff8000000000000ll);
}

// Per-matrix kernels index matrices by blockIdx.y (a list entry): launch
// them in slices of at most 65535 (the grid's y limit), fn(y0, ny)
template <class Fn>
void sliced(int64_t count, Fn fn) {
    for (int64_t y0 = 0; y0 < count; y0 += 65535) fn(y0, unsigned(std::min<int64_t>(65535, count - y0)));
}

// 3D tensor map over a workspace buffer of `batch` np x np matrices: boxes of
// 16 (k) x 128 (rows) x 1 (matrix), 128B swizzle (the X-operand TMA loads)
bool make_x_map(CUtensorMap* map, const double* base, int np, int64_t batch) {
    static PFN_cuTensorMapEncodeTiled_v12000 encode = [] {
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult q{};
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            fn = nullptr;
        return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    }();
    if (!encode) return false;
    const cuuint64_t dims[3] = {cuuint64_t(np), cuuint64_t(np), cuuint64_t(batch)};
    const cuuint64_t strides[2] = {cuuint64_t(np) * sizeof(double), cuuint64_t(np) * np * sizeof(double)};
    const cuuint32_t box[3] = {16, cuuint32_t(BM), 1};
    const cuuint32_t estr[3] = {1, 1, 1};
    return encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(base), dims, strides, box,
                  estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

thread_local int64_t g_map_batch = 0;  // matrices per workspace buffer of the current call
thread_local int g_exact_n = 0;         // > 0: products in reference rounding over k < g_exact_n

struct Scaling {  // the prep-free T18 path's per-matrix power-of-two scalings (GemmArgs)
    const mexp_selection* sel = nullptr;
    int c = 0, in0 = 0;
};
template <int EPI>
int gemm(const double* X, const double* Y, std::initializer_list<const double*> in,
         std::initializer_list<double*> out, const int32_t* d_list, int count, int np,
         cudaStream_t st, std::atomic<uint64_t>* launches, double* final_out = nullptr,
         const double (*lc)[5] = nullptr, int nlc = 0, Scaling sc = Scaling{}) {
    if (count == 0) return MEXP_OK;
    static PerDevice attr_once;
    attr_once([] {
        cudaFuncSetAttribute(gemm_dmma_kernel<EPI>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             int(GEMM_SMEM));
        cudaFuncSetAttribute(gemm_exact_kernel<EPI>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             int(EXACT_SMEM));
    });
    GemmArgs g{};
    g.X = X;
    g.Y = Y;
    int k = 0;
    for (auto p : in) g.in[k++] = p;
    k = 0;
    for (auto p : out) g.out[k++] = p;
    g.final_out = final_out;
    for (int j = 0; j < nlc; ++j)
        for (int t = 0; t < 5; ++t) g.lc[j][t] = lc[j][t];
    g.nlc = nlc;
    g.store_c = 1;
    if (nlc < 0) {  // EPI_PS_B without the product itself
        g.nlc = -nlc;
        g.store_c = 0;
        for (int j = 0; j < g.nlc; ++j)
            for (int t = 0; t < 5; ++t) g.lc[j][t] = lc[j][t];
    }
    g.list = d_list;
    g.np = np;
    g.mstride = int64_t(np) * np;
    g.n = g_exact_n > 0 ? g_exact_n : np;
    g.sel = sc.sel;
    g.scale_c = sc.c;
    g.scale_in0 = sc.in0;
    if ((sc.c || sc.in0) && g_exact_n > 0) return MEXP_ERR_UNSUPPORTED;  // DMMA pass only
    if (g_exact_n > 0) {  // REFERENCE rounding: the k-ordered DMUL+DADD product
        for (int z0 = 0; z0 < count; z0 += 65535) {
            const int zc = std::min(count - z0, 65535);
            g.list = d_list + z0;
            gemm_exact_kernel<EPI><<<dim3(np / XBN, np / XBM, zc), 256, EXACT_SMEM, st>>>(g);
            launches->fetch_add(1, std::memory_order_relaxed);
        }
        LCUDA(cudaGetLastError());
        return MEXP_OK;
    }
    CUtensorMap tmx{};
#if MEXP_GEMM_TMA == 2
    if (!make_x_map(&tmx, X, np, g_map_batch)) {
        g_err = "cuTensorMapEncodeTiled failed";
        return MEXP_ERR_CUDA;
    }
#endif
    for (int z0 = 0; z0 < count; z0 += 65535) {
        const int zc = std::min(count - z0, 65535);
        g.list = d_list + z0;
        dim3 grid(np / BN, np / BM, zc);
        gemm_dmma_kernel<EPI><<<grid, GEMM_THREADS, GEMM_SMEM, st>>>(g, tmx);
        launches->fetch_add(1, std::memory_order_relaxed);
    }
    LCUDA(cudaGetLastError());
    return MEXP_OK;
}

struct Workspace {
    double* buf = nullptr;
    size_t bytes = 0;
    mexp_selection* h_sel = nullptr;  // pinned (mapped) copy of the selections
    int64_t h_sel_cap = 0;
    int32_t* h_lists = nullptr;       // pinned (mapped) staging of the host-built lists
    size_t h_lists_cap = 0;
    int device = -1;
    std::mutex mu;  // one large-n call per device at a time owns the buffers
};
Workspace& workspace() {
    static Workspace ws[16];
    int dev = 0;
    cudaGetDevice(&dev);
    return ws[dev & 15];
}

}  // namespace

const char* large_last_error() { return g_err.c_str(); }

int large_expm_f64(const double* d_a, double* d_out, mexp_selection* d_sel_user, int n,
                   int64_t batch, int acc_arg, int rounding, int smin, cudaStream_t st,
                   std::atomic<uint64_t>* launches) {
    // the schedule is built on the host from the selections (one stream
    // synchronisation per call), which a CUDA-graph capture cannot contain
    cudaStreamCaptureStatus capturing = cudaStreamCaptureStatusNone;
    LCUDA(cudaStreamIsCapturing(st, &capturing));
    if (capturing != cudaStreamCaptureStatusNone) {
        g_err = "n > 64 is host-synchronous (schedule from the selections): not capturable";
        return MEXP_ERR_UNSUPPORTED;
    }
    const int np = (n + BM - 1) / BM * BM;
    const int64_t mat = int64_t(np) * np;
    const bool pade = (acc_arg >> 4) == MEXP_FAMILY_PADE || (acc_arg >> 4) == kFamilyPadeReference;
    // REFERENCE rounding: every product k-ordered and every lincomb literal
    // (the Pade LU has no reference-rounded variant)
    if (rounding == MEXP_ROUND_REFERENCE && pade) return MEXP_ERR_UNSUPPORTED;
    struct ExactScope {
        explicit ExactScope(int v) { g_exact_n = v; }
        ~ExactScope() { g_exact_n = 0; }
    } exact_scope(rounding == MEXP_ROUND_REFERENCE ? n : 0);
    constexpr int kMaxBuffers = 8;
    const int kBuffers = pade ? 8 : 6;  // r26 keeps A, A2, A4, A6, two lincombs, V and u''
    // workspace: kBuffers padded matrices per batch entry + per-matrix scratch
    const size_t need = size_t(kBuffers) * batch * mat * sizeof(double);
    Workspace& ws = workspace();
    std::lock_guard<std::mutex> ws_lock(ws.mu);  // the call synchronises its stream before returning
    // error exits too: work already enqueued on `st` still uses the workspace
    // and the pinned staging, so they are fenced before the lock is released
    struct SyncOnExit {
        cudaStream_t s;
        ~SyncOnExit() { cudaStreamSynchronize(s); }
    } fence{st};
    if (ws.bytes < need) {
        if (ws.buf) LCUDA(cudaFreeAsync(ws.buf, st));
        ws.buf = nullptr;
        ws.bytes = 0;
        LCUDA(pool_alloc(reinterpret_cast<void**>(&ws.buf), need, st));
        ws.bytes = need;
    }
    double* W[kMaxBuffers] = {};
    for (int k = 0; k < kBuffers; ++k) W[k] = ws.buf + size_t(k) * batch * mat;
    g_map_batch = batch;

    // per-call scratch, released on every exit path
    AsyncBuffer maxbits_buf(st), sel_buf(st);
    LCUDA(maxbits_buf.alloc(sizeof(unsigned long long) * batch + sizeof(int) * batch));
    unsigned long long* maxbits = maxbits_buf.get<unsigned long long>();
    int* bad = reinterpret_cast<int*>(maxbits + batch);
    LCUDA(cudaMemsetAsync(maxbits, 0, sizeof(unsigned long long) * batch + sizeof(int) * batch, st));
    mexp_selection* d_sel = d_sel_user;
    if (!d_sel) {
        LCUDA(sel_buf.alloc(sizeof(mexp_selection) * batch));
        d_sel = sel_buf.get<mexp_selection>();
    }

    sliced(batch, [&](int64_t y0, unsigned ny) {
        norm_cols_kernel<<<dim3((n + 255) / 256, ny), 256, 0, st>>>(d_a, n, batch, maxbits, bad, y0);
    });
    // (m, s) per matrix to the host: the schedule depends on them. The
    // selection kernel writes them straight into mapped pinned memory: a
    // cudaMemcpy would queue behind whatever the copy engine is moving (the
    // host pipeline's previous chunk D2H) and serialise the pipeline.
    if (ws.h_sel_cap < batch) {
        if (ws.h_sel) LCUDA(cudaFreeHost(ws.h_sel));
        ws.h_sel = nullptr;
        ws.h_sel_cap = 0;
        LCUDA(cudaHostAlloc(&ws.h_sel, sizeof(mexp_selection) * batch, cudaHostAllocMapped));
        ws.h_sel_cap = batch;
    }
    mexp_selection* d_hsel = nullptr;
    LCUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(&d_hsel), ws.h_sel, 0));
    select_kernel<<<unsigned((batch + 255) / 256), 256, 0, st>>>(maxbits, bad, batch, acc_arg, d_sel,
                                                                  d_hsel);
    launches->fetch_add(2, std::memory_order_relaxed);
    LCUDA(cudaStreamSynchronize(st));
    const mexp_selection* h_sel = ws.h_sel;
    // AUTO (Taylor families): a matrix with s >= smin runs every product and
    // lincomb in the reference's rounding (pass 0, bit-identical to the
    // reference), the rest on DMMA (pass 1). Squarings amplify the difference
    // between two roundings of T_m by up to ||X||^2/||X^2|| each, which the
    // non-normal gallery kinds (rank one at s = 12: 2.5x over 50 n u on DMMA)
    // make large; tests/test_gpu_auto_stress.py.
    const bool split_auto = rounding == MEXP_ROUND_AUTO && !pade;
    const int npasses = split_auto ? 2 : 1;
    int r = MEXP_OK;
    for (int pass = 0; pass < npasses; ++pass) {
    const bool last_pass = pass == npasses - 1;
    g_exact_n = (rounding == MEXP_ROUND_REFERENCE || (split_auto && pass == 0)) ? n : 0;
    auto active = [&](int64_t m) {
        return h_sel[m].status == MEXP_OK && (!split_auto || ((h_sel[m].s >= smin) == (pass == 0)));
    };
    bool any = false;
    for (int64_t m = 0; m < batch && !any; ++m) any = active(m);
    if (!any && !last_pass) continue;
    // the host lists' pinned staging is reused by the next pass
    if (pass > 0) LCUDA(cudaStreamSynchronize(st));
    AsyncBuffer lists_buf(st), extra_buf(st);
    int32_t* d_lists = nullptr;
    constexpr int kMaxDeg = 26;
    std::vector<int32_t> by_deg[kMaxDeg + 1];
    int max_s = 0;
    for (int64_t m = 0; m < batch; ++m) {
        if (!active(m)) continue;
        by_deg[h_sel[m].degree].push_back(int32_t(m));
        max_s = std::max(max_s, int(h_sel[m].s));
    }
    // device list layout: all OK matrices (prep), per degree, per squaring step
    std::vector<int32_t> host_lists;
    auto append = [&](const std::vector<int32_t>& v) {
        const size_t off = host_lists.size();
        host_lists.insert(host_lists.end(), v.begin(), v.end());
        return off;
    };
    std::vector<int32_t> all_ok;
    for (int d = 1; d <= kMaxDeg; ++d) all_ok.insert(all_ok.end(), by_deg[d].begin(), by_deg[d].end());
    size_t off_deg[kMaxDeg + 1] = {};
    for (int d = 1; d <= kMaxDeg; ++d) off_deg[d] = append(by_deg[d]);
    // Schemes, then squarings. Each matrix's LAST product writes its e^A
    // straight into the caller's output when no padding is needed (np == n):
    // the matrices with s == 0 at the scheme's final GEMM, those with s == k
    // at squaring k. Otherwise the result stays in the workspace (R after an
    // even number of squarings, S after an odd one) and is unpadded at the end.
    const bool direct = (np == n);
    double* R = W[1];
    double* S = W[2];
    // split a list into (finishing here, continuing) by s == k
    auto split = [&](const std::vector<int32_t>& v, int k) {
        std::vector<int32_t> fin, cont;
        for (int32_t m : v) (int(h_sel[m].s) == k ? fin : cont).push_back(m);
        return std::make_pair(fin, cont);
    };
    struct Part {
        size_t off;
        int count;
    };
    // one list per final step; the matrices finishing there carry bit 31 and
    // write the caller's output (when no padding is needed)
    auto flagged = [&](const std::vector<int32_t>& v, int k) {
        std::vector<int32_t> f(v);
        if (direct)
            for (auto& m : f)
                if (int(h_sel[m].s) == k) m = int32_t(uint32_t(m) | 0x80000000u);
        return Part{append(f), int(f.size())};
    };
    auto parts = [&](const std::vector<int32_t>& v, int k) {
        // (t1 kernel only: finishing and continuing separately)
        auto fc = split(v, k);
        if (!direct) {
            const size_t o = append(v);
            return std::make_pair(Part{o, 0}, Part{o, int(v.size())});
        }
        const size_t of = append(fc.first);
        const size_t oc = append(fc.second);
        return std::make_pair(Part{of, int(fc.first.size())}, Part{oc, int(fc.second.size())});
    };
    std::vector<Part> deg_flag(kMaxDeg + 1), sq_flag(max_s + 1);
    std::vector<std::pair<Part, Part>> deg_parts(kMaxDeg + 1);
    Part pade_s0{0, 0};  // Pade: s == 0 results are copied out of R after the solve
    if (!pade) {
        deg_parts[1] = parts(by_deg[1], 0);
        for (int d = 2; d <= kMaxDeg; ++d) deg_flag[d] = flagged(by_deg[d], 0);
    } else if (direct) {
        std::vector<int32_t> v;
        for (int32_t m : all_ok)
            if (h_sel[m].s == 0) v.push_back(m);
        pade_s0 = Part{append(v), int(v.size())};
    }
    for (int k = 1; k <= max_s; ++k) {
        std::vector<int32_t> v;
        for (int32_t m : all_ok)
            if (h_sel[m].s >= k) v.push_back(m);
        sq_flag[k] = flagged(v, k);
    }
    std::vector<int32_t> bad_list, all_list;
    if (last_pass)
        for (int64_t m = 0; m < batch; ++m)
            if (h_sel[m].status != MEXP_OK) bad_list.push_back(int32_t(m));
    const size_t off_bad = append(bad_list);
    const size_t off_all2 = append(all_ok);
    // host-built lists reach the device through mapped pinned staging and a
    // copy kernel (room for a second upload of up to batch entries below)
    const size_t lists_need = host_lists.size() + size_t(batch);
    if (ws.h_lists_cap < lists_need) {
        LCUDA(cudaStreamSynchronize(st));
        if (ws.h_lists) LCUDA(cudaFreeHost(ws.h_lists));
        ws.h_lists = nullptr;
        ws.h_lists_cap = 0;
        LCUDA(cudaHostAlloc(&ws.h_lists, sizeof(int32_t) * lists_need, cudaHostAllocMapped));
        ws.h_lists_cap = lists_need;
    }
    auto upload = [&](const std::vector<int32_t>& v, size_t pinned_off, int32_t* dst) -> int {
        if (v.empty()) return MEXP_OK;
        std::memcpy(ws.h_lists + pinned_off, v.data(), sizeof(int32_t) * v.size());
        int32_t* src = nullptr;
        LCUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(&src), ws.h_lists + pinned_off, 0));
        const int64_t cnt = int64_t(v.size());
        upload_kernel<<<unsigned(std::min<int64_t>((cnt + 255) / 256, 1024)), 256, 0, st>>>(src, dst, cnt);
        launches->fetch_add(1, std::memory_order_relaxed);
        return MEXP_OK;
    };
    if (!host_lists.empty()) {
        LCUDA(lists_buf.alloc(sizeof(int32_t) * host_lists.size()));
        d_lists = lists_buf.get<int32_t>();
        if ((r = upload(host_lists, 0, d_lists)) != MEXP_OK) return r;
    }
    auto L = [&](size_t off) { return d_lists + off; };
    const dim3 ew_block(256);
    const unsigned ew_rows = unsigned(std::min(np, 64));
    // Prep-free (TaylorNew, unpadded, DMMA pass): the products read the
    // caller's unscaled A and scale exactly by powers of two instead of going
    // through a scaled copy -- A2 = 4^-s (A A), A3 = 2^-s (A2 A), and T18's B
    // epilogue reads A times 2^-s; every other degree has s = 0. (A 2 GB
    // read + write less for cfg4.) s <= 400 keeps 4^-s normal.
    const bool noprep = !pade && (acc_arg >> 4) == MEXP_FAMILY_TAYLOR_NEW && n == np && g_exact_n == 0 &&
                        max_s <= 400 && std::getenv("MEXP_LARGE_PREP") == nullptr;
    const double* A0 = noprep ? d_a : W[0];
    const Scaling sc_a2{d_sel, noprep ? 2 : 0, 0}, sc_a3{d_sel, noprep ? 1 : 0, 0},
        sc_b{d_sel, 0, noprep ? 1 : 0};
    if (!all_ok.empty() && !noprep) {
        sliced(int64_t(all_ok.size()), [&](int64_t y0, unsigned ny) {
            prep_kernel<<<dim3(ew_rows, ny), ew_block, 0, st>>>(d_a, W[0], n, np, L(off_all2) + y0, d_sel);
        });
        launches->fetch_add(1, std::memory_order_relaxed);
    }
    // the scheme's final GEMM of degree d: finishing matrices -> out, rest -> R
    auto final_step = [&](auto epi_tag, const double* X, const double* Y,
                          std::initializer_list<const double*> in, int d) -> int {
        constexpr int EPI = decltype(epi_tag)::value;
        const Part& pp = deg_flag[d];
        return gemm<EPI>(X, Y, in, {R}, L(pp.off), pp.count, np, st, launches, d_out);
    };
    using EStore = std::integral_constant<int, EPI_STORE>;
    using EAdd = std::integral_constant<int, EPI_ADD>;
    using ET8_3 = std::integral_constant<int, EPI_T8_3>;
    using ET4_2 = std::integral_constant<int, EPI_T4_2>;
    using ET2 = std::integral_constant<int, EPI_T2>;
    (void)EStore{};
    if (pade) {
        // eval_pade (pade.cpp:50-113) per order; every order leaves M = V - U
        // in W2 and R = V + U in W1. Epilogue rows are coefficients of
        // {I, in0, in1, in2, c}.
        for (int d = 2; d <= kMaxDeg; d += 2) {
            const int c = int(by_deg[d].size());
            if (!c) continue;
            const int32_t* l = L(off_deg[d]);
            const int m = d / 2;
            const double* b = kPadeHost[m - 1];
            const double mr[2][5] = {{0, 1, 0, 0, -1}, {0, 1, 0, 0, 1}};  // V -/+ c
            if (d == 2) {
                sliced(c, [&](int64_t y0, unsigned ny) {
                    pade2_kernel<<<dim3(ew_rows, ny), ew_block, 0, st>>>(W[0], W[2], W[1], np, l + y0,
                                                                         b[0], b[1]);
                });
                launches->fetch_add(1, std::memory_order_relaxed);
                continue;
            }
            if (d == 4) {  // A2 -> M = b0 I - b1 A + b2 A2, R = b0 I + b1 A + b2 A2
                const double k[2][5] = {{b[0], -b[1], 0, 0, b[2]}, {b[0], b[1], 0, 0, b[2]}};
                if ((r = gemm<EPI_PS_B>(W[0], W[0], {W[0], nullptr, nullptr}, {nullptr, W[2], W[1]}, l,
                                        c, np, st, launches, nullptr, k, -2)))
                    return r;
                continue;
            }
            if (d == 10) {  // eval_r10
                if ((r = gemm<EPI_STORE>(W[0], W[0], {}, {W[1]}, l, c, np, st, launches))) return r;
                // A4 = A2*A2 -> t = b5 A4 + b3 A2 + b1 I (W3), V = b4 A4 + b2 A2 + b0 I (W4)
                const double k[2][5] = {{b[1], b[3], 0, 0, b[5]}, {b[0], b[2], 0, 0, b[4]}};
                if ((r = gemm<EPI_PS_B>(W[1], W[1], {W[1], nullptr, nullptr}, {nullptr, W[3], W[4]}, l,
                                        c, np, st, launches, nullptr, k, -2)))
                    return r;
                if ((r = gemm<EPI_PS_B>(W[0], W[3], {W[4], nullptr, nullptr}, {nullptr, W[2], W[1]}, l,
                                        c, np, st, launches, nullptr, mr, -2)))
                    return r;
                continue;
            }
            if (d == 26) {  // eval_r26
                if ((r = gemm<EPI_STORE>(W[0], W[0], {}, {W[1]}, l, c, np, st, launches))) return r;
                if ((r = gemm<EPI_STORE>(W[1], W[1], {}, {W[2]}, l, c, np, st, launches))) return r;
                // A6 = A2*A4 (W3), t1 = b13 A6 + b11 A4 + b9 A2 (W4), t2 = b12 A6 + b10 A4 + b8 A2 (W5)
                const double k6[2][5] = {{0, b[9], b[11], 0, b[13]}, {0, b[8], b[10], 0, b[12]}};
                if ((r = gemm<EPI_PS_B>(W[1], W[2], {W[1], W[2], nullptr}, {W[3], W[4], W[5]}, l, c,
                                        np, st, launches, nullptr, k6, 2)))
                    return r;
                // V = A6*t2 + b6 A6 + b4 A4 + b2 A2 + b0 I (W6); u = A6*t1 + b7 A6 + ... + b1 I (W7)
                const double kv[1][5] = {{b[0], b[2], b[4], b[6], 1.0}};
                const double ku[1][5] = {{b[1], b[3], b[5], b[7], 1.0}};
                if ((r = gemm<EPI_PS_B>(W[3], W[5], {W[1], W[2], W[3]}, {nullptr, W[6]}, l, c, np, st,
                                        launches, nullptr, kv, -1)))
                    return r;
                if ((r = gemm<EPI_PS_B>(W[3], W[4], {W[1], W[2], W[3]}, {nullptr, W[7]}, l, c, np, st,
                                        launches, nullptr, ku, -1)))
                    return r;
                if ((r = gemm<EPI_PS_B>(W[0], W[7], {W[6], nullptr, nullptr}, {nullptr, W[2], W[1]}, l,
                                        c, np, st, launches, nullptr, mr, -2)))
                    return r;
                continue;
            }
            // the even-power chain (pade.cpp:82-110): A2 (W1), odd (W3) =
            // b1 I + b3 A2 + b5 A4 + ..., V (W4) = b0 I + b2 A2 + ...
            const int top = m - (m % 2);
            const double k2[2][5] = {{b[1], 0, 0, 0, m >= 3 ? b[3] : 0.0}, {b[0], 0, 0, 0, b[2]}};
            if ((r = gemm<EPI_PS_B>(W[0], W[0], {}, {W[1], W[3], W[4]}, l, c, np, st, launches,
                                    nullptr, k2, 2)))
                return r;
            const double* P = W[1];
            for (int e = 4; e <= top; e += 2) {  // A^e = A2 * A^(e-2)
                double* Pn = (P == W[2]) ? W[5] : W[2];
                const double ke[2][5] = {{0, 1, 0, 0, e + 1 <= m ? b[e + 1] : 0.0}, {0, 0, 1, 0, b[e]}};
                if ((r = gemm<EPI_PS_B>(W[1], P, {W[3], W[4], nullptr}, {Pn, W[3], W[4]}, l, c, np, st,
                                        launches, nullptr, ke, e < top ? 2 : -2)))
                    return r;
                P = Pn;
            }
            // U = A * odd -> M (W2), R (W1)
            if ((r = gemm<EPI_PS_B>(W[0], W[3], {W[4], nullptr, nullptr}, {nullptr, W[2], W[1]}, l, c,
                                    np, st, launches, nullptr, mr, -2)))
                return r;
        }
        // R <- (V - U)^-1 (V + U) for every OK matrix (pade_solve, pade.cpp:26-28)
        // (grid.y-sized slices of the matrix list)
        for (size_t i0 = 0; i0 < all_ok.size(); i0 += 65535) {
            const int cnt = int(std::min<size_t>(65535, all_ok.size() - i0));
            r = lu_solve_batched(W[2], W[1], np, batch, L(off_all2) + i0, cnt, d_sel, st, launches);
            if (r == MEXP_ERR_CUDA) g_err = lu_last_error();
            if (r) return r;
        }
        if (pade_s0.count) {  // no squarings: e^A = R
            sliced(pade_s0.count, [&](int64_t y0, unsigned ny) {
                unpad_kernel<<<dim3(ew_rows, ny), ew_block, 0, st>>>(W[1], d_out, n, np,
                                                                     L(pade_s0.off) + y0);
            });
            launches->fetch_add(1, std::memory_order_relaxed);
        }
    } else {
    if (int c = int(by_deg[18].size())) {  // T18 (taylor_schemes.cpp:127-141)
        const int32_t* l = L(off_deg[18]);
        if ((r = gemm<EPI_STORE>(A0, A0, {}, {W[1]}, l, c, np, st, launches, nullptr, nullptr, 0,
                                 sc_a2)))
            return r;  // A2
        if ((r = gemm<EPI_STORE>(W[1], A0, {}, {W[2]}, l, c, np, st, launches, nullptr, nullptr, 0,
                                 sc_a3)))
            return r;  // A3
        // A6 = A3*A3 -> B1 W0, B2 W1, B3 W3, B4 W4, B5 W5 (A, A2 read in place)
        if ((r = gemm<EPI_T18_B>(W[2], W[2], {A0, W[1], W[2]}, {W[0], W[1], W[3], W[4], W[5]}, l, c, np,
                                 st, launches, nullptr, nullptr, 0, sc_b)))
            return r;
        // B1*B5: A9 = . + B4 -> W4, L = B3 + A9 -> W3
        if ((r = gemm<EPI_AL>(W[0], W[5], {W[4], W[3]}, {W[4], W[3]}, l, c, np, st, launches)))
            return r;
        // T = L*A9 + B2 (W1) -> R (= W1, read in place) or out
        if ((r = final_step(EAdd{}, W[3], W[4], {W[1]}, 18))) return r;
    }
    if (int c = int(by_deg[12].size())) {  // T12 (taylor_schemes.cpp:115-125)
        const int32_t* l = L(off_deg[12]);
        if ((r = gemm<EPI_STORE>(A0, A0, {}, {W[1]}, l, c, np, st, launches))) return r;  // A2
        // A3 = A2*A -> B1 W2, B2 W3, B3 W4, B4 W5
        if ((r = gemm<EPI_T12_B>(W[1], A0, {A0, W[1]}, {W[2], W[3], W[4], W[5]}, l, c, np, st,
                                 launches)))
            return r;
        // B4*B4: A6 = . + B3 -> W4, L = B2 + A6 -> W3
        if ((r = gemm<EPI_AL>(W[5], W[5], {W[4], W[3]}, {W[4], W[3]}, l, c, np, st, launches)))
            return r;
        // T = L*A6 + B1 (W2)
        if ((r = final_step(EAdd{}, W[3], W[4], {W[2]}, 12))) return r;
    }
    if (int c = int(by_deg[8].size())) {  // T8 (taylor_schemes.cpp:104-113)
        const int32_t* l = L(off_deg[8]);
        // A2 -> W1, U = x1 A + x2 A2 -> W2
        if ((r = gemm<EPI_T8_1>(A0, A0, {A0}, {W[1], W[2]}, l, c, np, st, launches))) return r;
        // A4 = A2*U: V1 -> W3, V2 -> W4
        if ((r = gemm<EPI_T8_2>(W[1], W[2], {A0, W[1]}, {W[3], W[4]}, l, c, np, st, launches)))
            return r;
        // A8 = V1*V2 -> T (A2 read in place)
        if ((r = final_step(ET8_3{}, W[3], W[4], {A0, W[1]}, 8))) return r;
    }
    // Family::TaylorPS degrees 6, 9, 16 (eval_ps, taylor_schemes.cpp:167-198):
    // p = 3 (6, 9) or 4 (16) powers, then the Horner chain
    // T = ((t A^p + g_{q-1}) A^p + ...) A^p + g_0, with the chunks
    // g_i = sum_k A^k / (p i + k)! formed in the epilogue of the A^p product
    // (t = g_{q} + A^{pq}/m! seeds the chain).
    auto ps_chunk = [](int p, int i, double* row) {
        for (int k = 0; k < 4; ++k) row[k] = k < p ? inv_fact(p * i + k) : 0.0;
        row[4] = 0.0;
    };
    if (int c = int(by_deg[16].size())) {  // p = 4, q = 4
        const int32_t* l = L(off_deg[16]);
        double lc[4][5];
        ps_chunk(4, 3, lc[0]);
        lc[0][4] = inv_fact(16);               // t = g3 + A4/16!
        for (int j = 1; j < 4; ++j) ps_chunk(4, 3 - j, lc[j]);  // g2, g1, g0
        if ((r = gemm<EPI_STORE>(W[0], W[0], {}, {W[1]}, l, c, np, st, launches))) return r;  // A2
        if ((r = gemm<EPI_STORE>(W[1], W[0], {}, {W[2]}, l, c, np, st, launches))) return r;  // A3
        // A4 = A2*A2 -> A4 W3, t W4, g2 W5, g1 W0, g0 W2 (A, A3 read in place)
        if ((r = gemm<EPI_PS_B>(W[1], W[1], {W[0], W[1], W[2]}, {W[3], W[4], W[5], W[0], W[2]}, l,
                                c, np, st, launches, nullptr, lc, 4)))
            return r;
        if ((r = gemm<EPI_ADD>(W[4], W[3], {W[5]}, {W[5]}, l, c, np, st, launches))) return r;
        if ((r = gemm<EPI_ADD>(W[5], W[3], {W[0]}, {W[0]}, l, c, np, st, launches))) return r;
        if ((r = final_step(EAdd{}, W[0], W[3], {W[2]}, 16))) return r;
    }
    for (int d : {9, 6}) {  // p = 3, q = 3 / 2
        const int c = int(by_deg[d].size());
        if (!c) continue;
        const int32_t* l = L(off_deg[d]);
        const int q = d / 3;
        double lc[4][5];
        ps_chunk(3, q - 1, lc[0]);
        lc[0][4] = inv_fact(d);                // t = g_{q-1} + A3/d!
        for (int j = 1; j < q; ++j) ps_chunk(3, q - 1 - j, lc[j]);
        if ((r = gemm<EPI_STORE>(W[0], W[0], {}, {W[1]}, l, c, np, st, launches))) return r;  // A2
        // A3 = A2*A -> A3 W2, t W3, then g_{q-2}.. g_0 in W4 (, W5)
        if ((r = gemm<EPI_PS_B>(W[1], W[0], {W[0], W[1], nullptr}, {W[2], W[3], W[4], W[5]}, l, c,
                                np, st, launches, nullptr, lc, q)))
            return r;
        if (q == 3) {
            if ((r = gemm<EPI_ADD>(W[3], W[2], {W[4]}, {W[4]}, l, c, np, st, launches))) return r;
            if ((r = final_step(EAdd{}, W[4], W[2], {W[5]}, d))) return r;
        } else {
            if ((r = final_step(EAdd{}, W[3], W[2], {W[4]}, d))) return r;
        }
    }
    if (int c = int(by_deg[4].size())) {  // eval_ps(4) (taylor_schemes.cpp:158-165)
        const int32_t* l = L(off_deg[4]);
        // A2 -> W3, inner -> W2
        if ((r = gemm<EPI_T4_1>(A0, A0, {A0}, {W[3], W[2]}, l, c, np, st, launches))) return r;
        // T = (I + A) + inner*A2
        if ((r = final_step(ET4_2{}, W[2], W[3], {A0}, 4))) return r;
    }
    if (by_deg[2].size()) {  // eval_ps(2)
        if ((r = final_step(ET2{}, A0, A0, {A0}, 2))) return r;
    }
    {  // degree 1: I + A
        const auto& pp = deg_parts[1];
        if (pp.first.count) {
            sliced(pp.first.count, [&](int64_t y0, unsigned ny) {
                t1_kernel<<<dim3(ew_rows, ny), ew_block, 0, st>>>(A0, d_out, n, np, n,
                                                                  L(pp.first.off) + y0);
            });
            launches->fetch_add(1, std::memory_order_relaxed);
        }
        if (pp.second.count) {
            sliced(pp.second.count, [&](int64_t y0, unsigned ny) {
                t1_kernel<<<dim3(ew_rows, ny), ew_block, 0, st>>>(A0, R, np, np, np,
                                                                  L(pp.second.off) + y0);
            });
            launches->fetch_add(1, std::memory_order_relaxed);
        }
    }
    }  // Taylor families
    // squarings: step k maps R -> S (k odd) or S -> R (k even)
    for (int k = 1; k <= max_s; ++k) {
        const double* src = (k & 1) ? R : S;
        double* dst = (k & 1) ? S : R;
        const Part& pp = sq_flag[k];
        if ((r = gemm<EPI_STORE>(src, src, {}, {dst}, L(pp.off), pp.count, np, st, launches, d_out)))
            return r;
    }
    if (!direct && !all_ok.empty()) {
        // unpad from R (even s) / S (odd s)
        std::vector<int32_t> ev, od;
        for (int32_t m : all_ok) ((h_sel[m].s & 1) ? od : ev).push_back(m);
        // these lists were not uploaded: append now needs a second upload
        std::vector<int32_t> both(ev);
        both.insert(both.end(), od.begin(), od.end());
        LCUDA(extra_buf.alloc(sizeof(int32_t) * both.size()));
        int32_t* d_extra = extra_buf.get<int32_t>();
        if ((r = upload(both, host_lists.size(), d_extra)) != MEXP_OK) return r;
        sliced(int64_t(ev.size()), [&](int64_t y0, unsigned ny) {
            unpad_kernel<<<dim3(ew_rows, ny), ew_block, 0, st>>>(R, d_out, n, np, d_extra + y0);
        });
        sliced(int64_t(od.size()), [&](int64_t y0, unsigned ny) {
            unpad_kernel<<<dim3(ew_rows, ny), ew_block, 0, st>>>(S, d_out, n, np, d_extra + ev.size() + y0);
        });
        launches->fetch_add(2, std::memory_order_relaxed);
    }
    if (!bad_list.empty()) {
        sliced(int64_t(bad_list.size()), [&](int64_t y0, unsigned ny) {
            nan_kernel<<<dim3(64, ny), 256, 0, st>>>(d_out, n, L(off_bad) + y0);
        });
        launches->fetch_add(1, std::memory_order_relaxed);
    }
    if (pade && !all_ok.empty()) {  // "singular denominator" matrices -> NaN
        sliced(int64_t(all_ok.size()), [&](int64_t y0, unsigned ny) {
            nan_singular_kernel<<<dim3(64, ny), 256, 0, st>>>(d_out, n, L(off_all2) + y0, d_sel);
        });
        launches->fetch_add(1, std::memory_order_relaxed);
    }
    LCUDA(cudaGetLastError());
    }  // passes
    LCUDA(cudaStreamSynchronize(st));  // host lists must outlive their async upload
    return MEXP_OK;
}

// C = A B for `batch` n x n fp64 matrices (any n): both operands zero-padded
// to np, one batched GEMM (REFERENCE rounding: the k-ordered exact product
// over k < n, bit-identical to kernels::matmul; otherwise DMMA), unpadded.
// Host-synchronous (the matrix list is uploaded from the host).
int matmul_f64(const double* d_a, const double* d_b, double* d_c, int n, int64_t batch, int rounding,
               cudaStream_t st, std::atomic<uint64_t>* launches) {
    struct ExactScope {
        explicit ExactScope(int v) { g_exact_n = v; }
        ~ExactScope() { g_exact_n = 0; }
    } exact_scope(rounding == MEXP_ROUND_REFERENCE ? n : 0);
    if (batch == 0) return MEXP_OK;
    if (batch > INT32_MAX) return MEXP_ERR_INVALID_ARGUMENT;
    const int np = (n + BM - 1) / BM * BM;
    const int64_t mat = int64_t(np) * np;
    AsyncBuffer w_buf(st), list_buf(st), sel0_buf(st);
    LCUDA(w_buf.alloc(sizeof(double) * 3 * batch * mat));
    LCUDA(list_buf.alloc(sizeof(int32_t) * batch));
    LCUDA(sel0_buf.alloc(sizeof(mexp_selection) * batch));  // s = 0: prep copies unscaled
    double* w = w_buf.get<double>();
    int32_t* list = list_buf.get<int32_t>();
    mexp_selection* sel0 = sel0_buf.get<mexp_selection>();
    g_map_batch = batch;
    LCUDA(cudaMemsetAsync(sel0, 0, sizeof(mexp_selection) * batch, st));
    std::vector<int32_t> idx(batch);
    for (int64_t m = 0; m < batch; ++m) idx[m] = int32_t(m);
    LCUDA(cudaMemcpyAsync(list, idx.data(), sizeof(int32_t) * batch, cudaMemcpyHostToDevice, st));
    const unsigned rows = unsigned(std::min(np, 64));
    double* wa = w;
    double* wb = w + batch * mat;
    double* wc = w + 2 * batch * mat;
    sliced(batch, [&](int64_t y0, unsigned ny) {
        prep_kernel<<<dim3(rows, ny), 256, 0, st>>>(d_a, wa, n, np, list + y0, sel0);
        prep_kernel<<<dim3(rows, ny), 256, 0, st>>>(d_b, wb, n, np, list + y0, sel0);
    });
    launches->fetch_add(2, std::memory_order_relaxed);
    int r = gemm<EPI_STORE>(wa, wb, {}, {wc}, list, int(batch), np, st, launches);
    if (r) {
        cudaStreamSynchronize(st);
        return r;
    }
    sliced(batch, [&](int64_t y0, unsigned ny) {
        unpad_kernel<<<dim3(rows, ny), 256, 0, st>>>(wc, d_c, n, np, list + y0);
    });
    launches->fetch_add(1, std::memory_order_relaxed);
    LCUDA(cudaGetLastError());
    LCUDA(cudaStreamSynchronize(st));  // idx must outlive the async copy
    return MEXP_OK;
}

int squarings_f64(double* d_x, int n, int64_t batch, int s, int rounding, cudaStream_t st,
                  std::atomic<uint64_t>* launches) {
    struct ExactScope {
        explicit ExactScope(int v) { g_exact_n = v; }
        ~ExactScope() { g_exact_n = 0; }
    } exact_scope(rounding == MEXP_ROUND_REFERENCE ? n : 0);
    const int np = (n + BM - 1) / BM * BM;
    const int64_t mat = int64_t(np) * np;
    AsyncBuffer w_buf(st), list_buf(st), sel0_buf(st);
    LCUDA(w_buf.alloc(sizeof(double) * 2 * batch * mat));
    LCUDA(list_buf.alloc(sizeof(int32_t) * batch));
    LCUDA(sel0_buf.alloc(sizeof(mexp_selection) * batch));  // s = 0: prep copies unscaled
    double* w = w_buf.get<double>();
    int32_t* list = list_buf.get<int32_t>();
    mexp_selection* sel0 = sel0_buf.get<mexp_selection>();
    g_map_batch = batch;
    LCUDA(cudaMemsetAsync(sel0, 0, sizeof(mexp_selection) * batch, st));
    std::vector<int32_t> idx(batch);
    for (int64_t m = 0; m < batch; ++m) idx[m] = int32_t(m);
    LCUDA(cudaMemcpyAsync(list, idx.data(), sizeof(int32_t) * batch, cudaMemcpyHostToDevice, st));
    const unsigned rows = unsigned(std::min(np, 64));
    sliced(batch, [&](int64_t y0, unsigned ny) {
        prep_kernel<<<dim3(rows, ny), 256, 0, st>>>(d_x, w, n, np, list + y0, sel0);
    });
    launches->fetch_add(1, std::memory_order_relaxed);
    double* bufs[2] = {w, w + batch * mat};
    int r;
    for (int k = 0; k < s; ++k)
        if ((r = gemm<EPI_STORE>(bufs[k & 1], bufs[k & 1], {}, {bufs[(k + 1) & 1]}, list, int(batch),
                                 np, st, launches)))
            return r;
    sliced(batch, [&](int64_t y0, unsigned ny) {
        unpad_kernel<<<dim3(rows, ny), 256, 0, st>>>(bufs[s & 1], d_x, n, np, list + y0);
    });
    launches->fetch_add(1, std::memory_order_relaxed);
    LCUDA(cudaGetLastError());
    LCUDA(cudaStreamSynchronize(st));  // idx must outlive the async copy
    return MEXP_OK;
}

}  // namespace mexp_b200
