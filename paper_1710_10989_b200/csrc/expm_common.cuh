// Shared device-side pieces of the expm kernels: the TaylorNew theta tables,
// the scheme coefficients, the on-device (m, s) selection and the two
// arithmetic policies (reference-exact and fast).
#pragma once

#include <cmath>
#include <cstdint>
#include <cstring>
#include <cuda_runtime.h>

#include "mexp_b200.h"
#include "scheme_tables.h"

namespace mexp_b200 {

// ---------------------------------------------------------------------------
// theta_m tables for Family::TaylorNew (reference theta_tables.cpp:45-51).
// Degrees {1,2,4,8,12,18} at {0,1,2,3,4,5} products; the literals are the
// reference's decimal literals, so they round to the identical doubles.
// ---------------------------------------------------------------------------
constexpr int kNumEntries = 6;
__device__ constexpr double c_theta[2][kNumEntries] = {
    {1.19e-7, 5.98e-4, 5.12e-2, 5.80e-1, 1.46, 3.01},      // Accuracy::Single
    {2.22e-16, 2.58e-8, 3.40e-4, 4.99e-2, 2.99e-1, 1.09},  // Accuracy::Double
};
__host__ __device__ constexpr int degree_of(int e) {
    return e == 0 ? 1 : e == 1 ? 2 : e == 2 ? 4 : e == 3 ? 8 : e == 4 ? 12 : 18;
}
__host__ __device__ constexpr int products_of_entry(int e) { return e; }
__host__ __device__ constexpr int products_of_degree(int m) {
    return m == 1 ? 0 : m == 2 ? 1 : m == 4 ? 2 : m == 8 ? 3 : m == 12 ? 4 : m == 18 ? 5 : -1;
}

// ---------------------------------------------------------------------------
// Scheme coefficients. T8: closed forms in sqrt(177) with x3 = 2/3, as the
// reference rounds them once from long double (taylor_schemes.cpp:12-27);
// the hex literals are those doubles, checked bit-for-bit against the
// compiled reference by tests/test_oracle.py::test_device_coefficients.
// ---------------------------------------------------------------------------
// (struct T8C: scheme_tables.h)

// T12 (paper eq. for the 4-product scheme; reference taylor_schemes.cpp:62-71):
// kT12[i][j] multiplies {I, A, A2, A3}[i] in B_{j+1}.
__device__ constexpr double c_t12[4][4] = MEXP_T12_TABLE;
// T18 (reference taylor_schemes.cpp:73-85): c_t18a[i] multiplies {I,A,A2,A3}[i]
// in B1; c_t18b[j][r] multiplies {I,A,A2,A3,A6}[r] in B_{j+2}.
__device__ constexpr double c_t18a[4] = MEXP_T18A_TABLE;
__device__ constexpr double c_t18b[4][5] = MEXP_T18B_TABLE;
// eval_ps degree 4 (taylor_schemes.cpp:158-163): 1/2!, 1/3!, 1/4! computed as
// 1.0 / (k!) in double (inv_factorial, :44-48).
constexpr double kInvFact2 = 0.5;
constexpr double kInvFact3 = 0x1.5555555555555p-3;  // 1.0 / 6.0
constexpr double kInvFact4 = 0x1.5555555555555p-5;  // 1.0 / 24.0
// 2^-s for s >= 0 as the reference's ldexp(1.0, -s) gives it (normal,
// subnormal, or 0 past 2^-1074), built from the exponent bits instead of the
// library ldexp's range checks
__host__ __device__ __forceinline__ double pow2_neg(int s) {
    long long b = 0;
    if (s <= 1022)
        b = static_cast<long long>(1023 - s) << 52;
    else if (s <= 1074)
        b = 1ll << (1074 - s);
#ifdef __CUDA_ARCH__
    return __longlong_as_double(b);
#else
    double x;
    memcpy(&x, &b, sizeof x);
    return x;
#endif
}

// 1/k! for the Paterson-Stockmeyer family, as the reference computes it: k!
// accumulated in double (exact for k <= 18), one correctly rounded division
// (taylor_schemes.cpp:44-48)
__host__ __device__ constexpr double inv_fact(int k) {
    double f = 1.0;
    for (int i = 2; i <= k; ++i) f *= i;
    return 1.0 / f;
}

// ---------------------------------------------------------------------------
// Selection (reference expm.cpp:11-29): the cheapest table entry whose theta
// admits the norm (skip on theta < norm; ties to the lower degree); beyond the
// table, degree 18 and the least s with ldexp(norm, -s) <= theta_18.
// ---------------------------------------------------------------------------
struct Sel {
    int degree;
    int s;
    int status;
};

__host__ __device__ __forceinline__ long long dbits(double x) {
#ifdef __CUDA_ARCH__
    return __double_as_longlong(x);
#else
    long long b;
    memcpy(&b, &x, sizeof b);
    return b;
#endif
}
__host__ __device__ __forceinline__ double dfrom(long long b) {
#ifdef __CUDA_ARCH__
    return __longlong_as_double(b);
#else
    double x;
    memcpy(&x, &b, sizeof x);
    return x;
#endif
}

// One implementation for the kernels and the host-side mexp_select, so the
// CPU tests of mexp_select exercise the exact logic the kernels run.
// Family::TaylorPS (Paterson-Stockmeyer, theta_tables.cpp:53-59): degrees
// {1, 2, 4, 6, 9, 16} at {0, 1, 2, 3, 4, 6} products.
__host__ __device__ constexpr int ps_degree_of(int e) {
    return e == 0 ? 1 : e == 1 ? 2 : e == 2 ? 4 : e == 3 ? 6 : e == 4 ? 9 : 16;
}
__host__ __device__ constexpr int ps_products_of_degree(int m) {
    return m == 1 ? 0 : m == 2 ? 1 : m == 4 ? 2 : m == 6 ? 3 : m == 9 ? 4 : m == 16 ? 6 : -1;
}
// Family::PadeDiagonal (theta_tables.cpp:61-73): orders 2, 4, ..., 26 at
// {0, 1, 2, 3, 3, 4, 4, 5, 5, 5, 6, 6, 6} products (+ one LU solve).
constexpr int kPadeEntries = 13;
__host__ __device__ constexpr int pade_products_of_degree(int m) {
    return m == 2 ? 0 : m == 4 ? 1 : m == 6 ? 2 : (m == 8 || m == 10) ? 3 : (m == 12 || m == 14) ? 4
         : (m == 16 || m == 18 || m == 20) ? 5 : (m == 22 || m == 24 || m == 26) ? 6 : -1;
}
__host__ __device__ constexpr int num_entries(int family) {
    return family == MEXP_FAMILY_PADE ? kPadeEntries : kNumEntries;
}
__host__ __device__ constexpr int degree_of_entry(int family, int e) {
    return family == MEXP_FAMILY_PADE ? 2 * (e + 1)
         : family == MEXP_FAMILY_TAYLOR_PS ? ps_degree_of(e) : degree_of(e);
}
__host__ __device__ constexpr int products_of(int family, int m) {
    return family == MEXP_FAMILY_TAYLOR_PS ? ps_products_of_degree(m)
         : family == MEXP_FAMILY_PADE ? pade_products_of_degree(m) : products_of_degree(m);
}
// the reported cost: products + s, plus 4/3 for the Pade solve (expm.cpp:70-72)
__host__ __device__ constexpr int cost_thirds_of(int family, int m, int s) {
    return 3 * (products_of(family, m) + s) + (family == MEXP_FAMILY_PADE ? 4 : 0);
}
__host__ __device__ __forceinline__ double pade_theta(int accuracy, int e) {
    switch (e) {
        case 0: return accuracy ? 3.65e-8 : 8.46e-4;
        case 1: return accuracy ? 5.32e-4 : 8.09e-2;
        case 2: return accuracy ? 1.50e-2 : 4.26e-1;
        case 3: return accuracy ? 8.54e-2 : 1.05;
        case 4: return accuracy ? 2.54e-1 : 1.88;
        case 5: return accuracy ? 5.41e-1 : 2.85;
        case 6: return accuracy ? 9.50e-1 : 3.93;
        case 7: return accuracy ? 1.47 : 5.06;
        case 8: return accuracy ? 2.10 : 6.25;
        case 9: return accuracy ? 2.81 : 7.47;
        case 10: return accuracy ? 3.60 : 8.71;
        case 11: return accuracy ? 4.46 : 9.97;
        default: return accuracy ? 5.37 : 11.2;
    }
}
__device__ constexpr double c_pade[13][14] = MEXP_PADE_TABLE;
constexpr double kPadeHost[13][14] = MEXP_PADE_TABLE;  // host copy (large-n schedule)
// theta_m of entry e of a family's table: the reference's decimal literals
// (theta_tables.cpp:45-51 TaylorNew, :53-59 TaylorPS)
__host__ __device__ __forceinline__ double theta_entry(int family, int accuracy, int e) {
    if (family == MEXP_FAMILY_PADE) return pade_theta(accuracy, e);
    if (family == MEXP_FAMILY_TAYLOR_PS) {
        switch (e) {
            case 0: return accuracy ? 2.22e-16 : 1.19e-7;
            case 1: return accuracy ? 2.58e-8 : 5.98e-4;
            case 2: return accuracy ? 3.40e-4 : 5.12e-2;
            case 3: return accuracy ? 9.07e-3 : 2.50e-1;
            case 4: return accuracy ? 8.96e-2 : 7.80e-1;
            default: return accuracy ? 7.80e-1 : 2.48;
        }
    }
    switch (e) {
        case 0: return accuracy ? 2.22e-16 : 1.19e-7;
        case 1: return accuracy ? 2.58e-8 : 5.98e-4;
        case 2: return accuracy ? 3.40e-4 : 5.12e-2;
        case 3: return accuracy ? 4.99e-2 : 5.80e-1;
        case 4: return accuracy ? 2.99e-1 : 1.46;
        default: return accuracy ? 1.09 : 3.01;
    }
}

// Internal family id (never in the public ABI): Pade evaluation with the
// selection of reference_expm (bench.cpp:10-20) -- degree 26 and the least s
// with ldexp(norm, -s) <= theta_26(Double) / 8.
constexpr int kFamilyPadeReference = 3;

__host__ __device__ __forceinline__ Sel select_device(double norm, int accuracy,
                                                      int family = MEXP_FAMILY_TAYLOR_NEW) {
    Sel r{0, 0, MEXP_OK};
    if (!isfinite(norm) || norm < 0.0) {
        r.status = MEXP_ERR_NORM_NONFINITE;
        return r;
    }
    if (family == kFamilyPadeReference) {
        const double t = pade_theta(1, kPadeEntries - 1) / 8.0;  // exact: a power-of-two divide
        r.degree = 26;
        if (norm > t) {
            const long long nb = dbits(norm), tb = dbits(t);
            const long long k = (nb >> 52) - (tb >> 52);
            r.s = int(k) + int(norm > dfrom(tb + (k << 52)));
        }
        return r;
    }
    if (family == MEXP_FAMILY_PADE) {
        // products are non-decreasing along the Pade table too (orders 8/10,
        // 12/14, ... tie), so the cheapest admissible entry with ties to the
        // lower degree is again the first admissible one
        const double tmax = pade_theta(accuracy, kPadeEntries - 1);
        if (norm <= tmax) {
            int e = 0;
#pragma unroll
            for (int k = 0; k < kPadeEntries - 1; ++k) e += int(pade_theta(accuracy, k) < norm);
            r.degree = 2 * (e + 1);
            return r;
        }
        const long long nb = dbits(norm), tb = dbits(tmax);
        const long long k = (nb >> 52) - (tb >> 52);
        r.degree = 26;
        r.s = int(k) + int(norm > dfrom(tb + (k << 52)));
        return r;
    }
    const bool ps = family == MEXP_FAMILY_TAYLOR_PS;
    const double t0 = theta_entry(family, accuracy, 0);
    const double t1 = theta_entry(family, accuracy, 1);
    const double t2 = theta_entry(family, accuracy, 2);
    const double t3 = theta_entry(family, accuracy, 3);
    const double t4 = theta_entry(family, accuracy, 4);
    const double tmax = theta_entry(family, accuracy, 5);
    if (norm <= tmax) {
        // entries with theta < norm are skipped (expm.cpp:17); products and
        // degrees ascend with the entry in both tables, so the reference's
        // (products, degree) minimum is the first admissible entry = the count
        // of skipped ones
        const int e = int(t0 < norm) + int(t1 < norm) + int(t2 < norm) + int(t3 < norm) +
                      int(t4 < norm);
        r.degree = ps ? ps_degree_of(e) : (e < 4 ? (1 << e) : (e == 4 ? 12 : 18));
        return r;
    }
    // least s with ldexp(norm, -s) <= theta_18 (expm.cpp:27). With norm =
    // mn * 2^En and theta = mt * 2^Et (both normal here), theta * 2^k for
    // k = En - Et has norm's exponent, and the answer is k if norm <= theta *
    // 2^k else k + 1. Exactly the reference's loop (the halving there is exact
    // while ldexp(norm, -s) > theta >= 2^-52); checked against it in
    // tests/test_capi.py::test_closed_form_scaling_exponent.
    const long long nb = dbits(norm), tb = dbits(tmax);
    const long long k = (nb >> 52) - (tb >> 52);
    const double t = dfrom(tb + (k << 52));
    r.degree = ps ? 16 : 18;
    r.s = int(k) + int(norm > t);
    return r;
}

// ---------------------------------------------------------------------------
// Arithmetic policies.
//   Exact: every multiply and add rounded separately (DMUL, DADD), matching
//          the reference's -ffp-contract=off build bit for bit when the
//          operation order is also the reference's.
//   Fast:  fused multiply-add.
// ---------------------------------------------------------------------------
struct ExactOps {
    static constexpr bool kExact = true;
    __device__ __forceinline__ static double mul(double a, double b) { return __dmul_rn(a, b); }
    __device__ __forceinline__ static double add(double a, double b) { return __dadd_rn(a, b); }
    __device__ __forceinline__ static double mac(double acc, double a, double b) {
        return __dadd_rn(acc, __dmul_rn(a, b));
    }
};
struct FastOps {
    static constexpr bool kExact = false;
    __device__ __forceinline__ static double mul(double a, double b) { return a * b; }
    __device__ __forceinline__ static double add(double a, double b) { return a + b; }
    __device__ __forceinline__ static double mac(double acc, double a, double b) {
        return fma(a, b, acc);
    }
};

// Streaming global accesses for the read-once input / write-once output.
__device__ __forceinline__ double2 ld_stream(const double2* p) {
    double2 v;
    asm("ld.global.nc.L1::no_allocate.v2.f64 {%0, %1}, [%2];"
                 : "=d"(v.x), "=d"(v.y)
                 : "l"(p));
    return v;
}
__device__ __forceinline__ void st_stream(double2* p, double2 v) {
    asm volatile("st.global.cs.v2.f64 [%0], {%1, %2};" ::"l"(p), "d"(v.x), "d"(v.y) : "memory");
}
__device__ __forceinline__ float4 ld_stream(const float4* p) {
    float4 v;
    asm("ld.global.nc.L1::no_allocate.v4.f32 {%0, %1, %2, %3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                 : "l"(p));
    return v;
}
__device__ __forceinline__ void st_stream(float4* p, float4 v) {
    asm volatile("st.global.cs.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(v.x), "f"(v.y),
                 "f"(v.z), "f"(v.w)
                 : "memory");
}

// FP64 tensor-core MMA, m8n8k4 (SASS DMMA.8x8x4): D = A(8x4, row) * B(4x8, col) + C.
// Fragment ownership per lane l: a = A[l>>2][l&3], b = B[l&3][l>>2],
// c/d = C[l>>2][2(l&3)], C[l>>2][2(l&3)+1].
__device__ __forceinline__ void dmma_8x8x4(double& d0, double& d1, double a, double b) {
    asm(
        "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
        : "+d"(d0), "+d"(d1)
        : "d"(a), "d"(b));
}

}  // namespace mexp_b200
