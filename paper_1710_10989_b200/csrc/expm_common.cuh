// Shared device-side pieces of the expm kernels: the TaylorNew theta tables,
// the scheme coefficients, the on-device (m, s) selection and the two
// arithmetic policies (reference-exact and fast).
#pragma once

#include <cmath>
#include <cstdint>
#include <cstring>
#include <cuda_runtime.h>

#include "mexp_b200.h"

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
struct T8C {
    static constexpr double x1 = 0x1.bbdc940ef503ap-4;
    static constexpr double x2 = 0x1.bbdc940ef503ap-6;
    static constexpr double x3 = 0x1.5555555555555p-1;
    static constexpr double x4 = 0x1.17f11e296523cp-1;
    static constexpr double x5 = 0x1.49fc346242b21p-3;
    static constexpr double x6 = 0x1.cdbb2e2ed5250p-7;
    static constexpr double x7 = 0x1.14d4a1c010d67p-5;
    static constexpr double y0 = 1.0;
    static constexpr double y1 = 1.0;
    static constexpr double y2 = 0x1.157d04e6f24b6p-3;
};

// T12 (paper eq. for the 4-product scheme; reference taylor_schemes.cpp:62-71):
// kT12[i][j] multiplies {I, A, A2, A3}[i] in B_{j+1}.
__device__ constexpr double c_t12[4][4] = {
    {9.0198e-16, 5.31597895759871264183, 0.18188869982170434744, -2.0861320e-13},
    {0.46932117595418237389, 1.19926790417132231573, 0.05502798439925399070,
     -0.13181061013830184015},
    {-0.20099424927047284052, 0.01179296240992997031, 0.09351590770535414968,
     -0.02027855540589259079},
    {-0.04623946134063071740, 0.01108844528519167989, 0.00610700528898058230,
     -0.00675951846863086359},
};
// T18 (reference taylor_schemes.cpp:73-85): c_t18a[i] multiplies {I,A,A2,A3}[i]
// in B1; c_t18b[j][r] multiplies {I,A,A2,A3,A6}[r] in B_{j+2}.
__device__ constexpr double c_t18a[4] = {0.0, -0.100365581030144620, -0.0080292464824115696,
                                 -0.0008921384980457299};
__device__ constexpr double c_t18b[4][5] = {
    {0.0, 0.39784974949964507614, 1.36783778460411719922, 0.49828962252538267755,
     -0.0006378981945947233},
    {-10.967639605296206259, 1.68015813878906197182, 0.05717798464788655127,
     -0.0069821012248805208, 0.00003349750170860705},
    {-0.0904316832390810561, -0.0676404519071381907, 0.06759613017704596460,
     0.02955525704293155274, -0.0000139180257516060},
    {0.0, 0.0, -0.0923364619367118592, -0.0169364939002081717, -0.0000140086798182036},
};
// eval_ps degree 4 (taylor_schemes.cpp:158-163): 1/2!, 1/3!, 1/4! computed as
// 1.0 / (k!) in double (inv_factorial, :44-48).
constexpr double kInvFact2 = 0.5;
constexpr double kInvFact3 = 0x1.5555555555555p-3;  // 1.0 / 6.0
constexpr double kInvFact4 = 0x1.5555555555555p-5;  // 1.0 / 24.0
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
// pade_coeffs(m).b (pade.cpp:34-48: exact integer ratios, rounded once via
// long double) as the compiled reference holds them, b_0..b_m for m = 1..13;
// checked bit for bit by tests/test_oracle.py::test_pade_coefficients.
#define MEXP_PADE_TABLE                                                               \
    {{1.0, 0x1.0000000000000p-1, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0}, \
     {1.0, 0x1.0000000000000p-1, 0x1.5555555555555p-4, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0}, \
     {1.0, 0x1.0000000000000p-1, 0x1.999999999999ap-4, 0x1.1111111111111p-7, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0}, \
     {1.0, 0x1.0000000000000p-1, 0x1.b6db6db6db6dbp-4, 0x1.8618618618618p-7, 0x1.3813813813814p-11, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0}, \
     {1.0, 0x1.0000000000000p-1, 0x1.c71c71c71c71cp-4, 0x1.c71c71c71c71cp-7, 0x1.0410410410410p-10, 0x1.1566abc011567p-15, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0}, \
     {1.0, 0x1.0000000000000p-1, 0x1.d1745d1745d17p-4, 0x1.f07c1f07c1f08p-7, 0x1.4afd6a052bf5bp-10, 0x1.08cabb37565e2p-14, 0x1.937e11175f095p-20, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0}, \
     {1.0, 0x1.0000000000000p-1, 0x1.d89d89d89d89ep-4, 0x1.0690690690690p-6, 0x1.7de952f2466a4p-10, 0x1.6ea28d118b474p-14, 0x1.b287c3a303e2bp-19, 0x1.f09b28ba4d955p-25, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0}, \
     {1.0, 0x1.0000000000000p-1, 0x1.ddddddddddddep-4, 0x1.1111111111111p-6, 0x1.a41a41a41a41ap-10, 0x1.c01c01c01c01cp-14, 0x1.45e5d2ba42ea0p-18, 0x1.29f6b20961c00p-23, 0x1.08db48ebe51c7p-29, 0.0, 0.0, 0.0, 0.0, 0.0}, \
     {1.0, 0x1.0000000000000p-1, 0x1.e1e1e1e1e1e1ep-4, 0x1.1919191919192p-6, 0x1.c1c1c1c1c1c1cp-10, 0x1.0101010101010p-13, 0x1.a5c001a5c001ap-18, 0x1.e20001e20001ep-23, 0x1.5e8ba44745d2dp-28, 0x1.f28db670be53bp-35, 0.0, 0.0, 0.0, 0.0}, \
     {1.0, 0x1.0000000000000p-1, 0x1.e50d79435e50dp-4, 0x1.1f7047dc11f70p-6, 0x1.d96da388960f5p-10, 0x1.1c0e9551f3a2dp-13, 0x1.f8fd7b3c5bcc1p-18, 0x1.49ca1c3c50d8ep-22, 0x1.306bcb4b5e520p-27, 0x1.68cb9b9bb2285p-33, 0x1.a3d5a71b92cd3p-40, 0.0, 0.0, 0.0}, \
     {1.0, 0x1.0000000000000p-1, 0x1.e79e79e79e79ep-4, 0x1.2492492492492p-6, 0x1.ecc07b301ecc0p-10, 0x1.3299e6401329ap-13, 0x1.2090d8b4c6bdcp-17, 0x1.9c3ca34b650f1p-22, 0x1.b7b825a5c1212p-27, 0x1.4f06351093257p-32, 0x1.49deba27f3581p-38, 0x1.3fdfbc45c52eap-45, 0.0, 0.0}, \
     {1.0, 0x1.0000000000000p-1, 0x1.e9bd37a6f4deap-4, 0x1.28cfc4a33f129p-6, 0x1.fcd1e360fe68fp-10, 0x1.45a50c670938fp-13, 0x1.3fee80f4f29acp-17, 0x1.e783d0b234bb0p-22, 0x1.1ec6024ab59b3p-26, 0x1.fdd1cb2f7bbe9p-32, 0x1.4648d3f56deaap-37, 0x1.0f328eed3d6fep-43, 0x1.bd0ac3296b624p-51, 0.0}, \
     {1.0, 0x1.0000000000000p-1, 0x1.eb851eb851eb8p-4, 0x1.2c5f92c5f92c6p-6, 0x1.0531b747fa105p-9, 0x1.55ed4d05c9af0p-13, 0x1.5b5ab7e55f2bap-17, 0x1.15e22cb77f562p-21, 0x1.5f02bf38a0d89p-26, 0x1.5aad6134c4c94p-31, 0x1.05070ff78b221p-36, 0x1.1cc1e2df80824p-42, 0x1.94fcfe65b1145p-49, 0x1.1cd3b01a822a6p-56} \
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
