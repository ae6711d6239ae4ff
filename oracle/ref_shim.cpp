// TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// extern "C" shim over the UNMODIFIED reference library (`mexp`, compiled from
// /root/reference/proj/src by oracle/Makefile into oracle/_ref/). It lets the
// pytest suite, the golden-fixture generator and bench.py's CPU baseline call
// the reference through ctypes with plain pointers. Only tests/, smoke() and
// bench.py (cpu_baseline leg / --impl reference) may load the result.
//
// Every function forwards to the reference symbol named beside it; nothing
// here re-implements arithmetic.

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <random>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "mexp/bench.hpp"
#include "mexp/dense_matrix.hpp"
#include "mexp/gallery.hpp"
#include "mexp/expm.hpp"
#include "mexp/kernels.hpp"
#include "mexp/pade.hpp"
#include "mexp/taylor_schemes.hpp"
#include "mexp/theta_tables.hpp"

namespace {

// status codes mirror include/mexp_b200.h
constexpr int kOk = 0;
constexpr int kNonFinite = 1;
constexpr int kNormNonFinite = 2;
constexpr int kInvalid = 3;
constexpr int kSingular = 7;

mexp::Accuracy acc_of(int a) { return a == 0 ? mexp::Accuracy::Single : mexp::Accuracy::Double; }

mexp::Family fam_of(int f) {
    switch (f) {
        case 1: return mexp::Family::TaylorPS;
        case 2: return mexp::Family::PadeDiagonal;
        default: return mexp::Family::TaylorNew;
    }
}

template <class T>
mexp::DenseMatrix to_dense(const T* a, int n) {
    std::vector<double> v(std::size_t(n) * n);
    for (std::size_t e = 0; e < v.size(); ++e) v[e] = double(a[e]);
    return mexp::DenseMatrix(n, std::move(v));
}

template <class T, class U>
int expm_one(const T* a, int n, int accuracy, int family, U* out, int32_t* degree,
             int32_t* s, int64_t* cost_thirds, double* norm_in) {
    const std::size_t nn = std::size_t(n) * n;
    try {
        const auto rep = mexp::expm(to_dense(a, n), acc_of(accuracy), fam_of(family));
        for (std::size_t e = 0; e < nn; ++e) out[e] = U(rep.result.data()[e]);
        if (degree) *degree = rep.degree;
        if (s) *s = rep.s;
        if (cost_thirds) *cost_thirds = rep.cost_thirds;
        if (norm_in) *norm_in = rep.norm_in;
        return kOk;
    } catch (const std::invalid_argument& e) {
        for (std::size_t k = 0; k < nn; ++k) out[k] = U(NAN);
        if (degree) *degree = 0;
        if (s) *s = 0;
        if (cost_thirds) *cost_thirds = 0;
        if (norm_in) *norm_in = NAN;
        if (std::strstr(e.what(), "non-finite")) return kNonFinite;
        if (std::strstr(e.what(), "norm")) return kNormNonFinite;
        return kInvalid;
    } catch (const std::runtime_error&) {  // "singular denominator" (kernels.cpp:72)
        for (std::size_t k = 0; k < nn; ++k) out[k] = U(NAN);
        if (degree) *degree = 0;
        if (s) *s = 0;
        if (cost_thirds) *cost_thirds = 0;
        if (norm_in) *norm_in = NAN;
        return kSingular;
    }
}

}  // namespace

extern "C" {

// mexp::expm (reference include/mexp/expm.hpp:37, src/expm.cpp:37-74) over a
// contiguous batch of row-major n x n matrices, one call per matrix, serial.
int ref_expm_batch_f64(const double* a, double* out, int n, int64_t batch, int accuracy,
                       int family, int32_t* degree, int32_t* s, int64_t* cost_thirds,
                       double* norm_in, int32_t* status) {
    const std::size_t nn = std::size_t(n) * n;
    int worst = kOk;
    for (int64_t b = 0; b < batch; ++b) {
        const int st = expm_one(a + b * nn, n, accuracy, family, out + b * nn,
                                degree ? degree + b : nullptr, s ? s + b : nullptr,
                                cost_thirds ? cost_thirds + b : nullptr,
                                norm_in ? norm_in + b : nullptr);
        if (status) status[b] = st;
        if (st != kOk && worst == kOk) worst = st;
    }
    return worst;
}

// Same, for float storage: values are promoted to double, the reference runs
// in double (expm.hpp:34-36), and the result is rounded back to float.
int ref_expm_batch_f32_out64(const float* a, double* out, int n, int64_t batch,
                             int accuracy, int family, int32_t* degree, int32_t* s,
                             int64_t* cost_thirds, double* norm_in, int32_t* status) {
    const std::size_t nn = std::size_t(n) * n;
    int worst = kOk;
    for (int64_t b = 0; b < batch; ++b) {
        const int st = expm_one(a + b * nn, n, accuracy, family, out + b * nn,
                                degree ? degree + b : nullptr, s ? s + b : nullptr,
                                cost_thirds ? cost_thirds + b : nullptr,
                                norm_in ? norm_in + b : nullptr);
        if (status) status[b] = st;
        if (st != kOk && worst == kOk) worst = st;
    }
    return worst;
}

// mexp::select (src/expm.cpp:11-29). Returns 0, or kNormNonFinite on throw.
int ref_select(double norm, int accuracy, int family, int32_t* degree, int32_t* s) {
    try {
        const auto sel = mexp::select(norm, mexp::selection_table(fam_of(family), acc_of(accuracy)));
        *degree = sel.degree;
        *s = sel.s;
        return kOk;
    } catch (const std::invalid_argument&) {
        return kNormNonFinite;
    }
}

// mexp::kernels::one_norm (src/kernels.cpp:44-53).
double ref_one_norm(const double* a, int n) { return mexp::kernels::one_norm(a, n); }

// mexp::kernels::matmul (src/kernels.cpp:16-27).
void ref_matmul(const double* a, const double* b, double* c, int n) {
    mexp::kernels::matmul(a, b, c, n);
}

// selection_table (src/theta_tables.cpp:77-85): writes up to cap entries.
int ref_theta_table(int accuracy, int family, int32_t* degrees, int32_t* products,
                    double* thetas, int cap) {
    const auto& t = mexp::selection_table(fam_of(family), acc_of(accuracy));
    int k = 0;
    for (const auto& e : t.entries) {
        if (k >= cap) break;
        degrees[k] = e.degree;
        products[k] = e.products;
        thetas[k] = e.theta;
        ++k;
    }
    return k;
}

// eval_taylor_new (src/taylor_schemes.cpp:211-227) on one matrix; returns
// the product count recorded in the CostContext, or -1 on invalid degree.
int ref_eval_taylor_new(const double* a, int n, int degree, double* out) {
    try {
        mexp::CostContext ctx;
        const auto r = mexp::eval_taylor_new(ctx, to_dense(a, n), degree);
        std::memcpy(out, r.data(), sizeof(double) * std::size_t(n) * n);
        return int(ctx.products);
    } catch (const std::invalid_argument&) {
        return -1;
    }
}

// taylor_oracle (src/taylor_schemes.cpp:87-94): plain Horner.
void ref_taylor_oracle(const double* a, int n, int degree, double* out) {
    const auto r = mexp::taylor_oracle(to_dense(a, n), degree);
    std::memcpy(out, r.data(), sizeof(double) * std::size_t(n) * n);
}

// pade_coeffs(m) (src/pade.cpp:34-48): b_0..b_m into b; returns m + 1, or -1.
int ref_pade_coeffs(int m, double* b) {
    try {
        const auto c = mexp::pade_coeffs(m);
        for (int j = 0; j <= m; ++j) b[j] = c.b[j];
        return m + 1;
    } catch (const std::invalid_argument&) {
        return -1;
    }
}

// eval_pade (src/pade.cpp:50-113) on one matrix: returns the product count
// recorded in the CostContext, -1 on an invalid order, -2 on a singular
// denominator.
int ref_eval_pade(const double* a, int n, int order, double* out) {
    try {
        mexp::CostContext ctx;
        const auto r = mexp::eval_pade(ctx, to_dense(a, n), order);
        std::memcpy(out, r.data(), sizeof(double) * std::size_t(n) * n);
        return int(ctx.products);
    } catch (const std::invalid_argument&) {
        return -1;
    } catch (const std::runtime_error&) {
        return -2;
    }
}

// gallery (src/gallery.cpp): kind index into kAllGalleryKinds. Returns 0, or
// 1 when the reference throws (zero matrix / bad arguments).
int ref_gallery(int kind, int n, uint64_t seed, double target_norm, double* out) {
    try {
        mexp::GallerySpec spec{mexp::kAllGalleryKinds[kind], n, seed, target_norm};
        const auto m = mexp::gallery(spec);
        std::memcpy(out, m.data(), sizeof(double) * std::size_t(n) * n);
        return 0;
    } catch (const std::exception&) {
        return 1;
    }
}

// reference_expm (src/bench.cpp:10-20)
void ref_reference_expm(const double* a, int n, double* out) {
    const auto r = mexp::reference_expm(to_dense(a, n));
    std::memcpy(out, r.data(), sizeof(double) * std::size_t(n) * n);
}

// cost_staircase + staircase_csv over log_grid (bench.cpp:32-57, 123-136):
// writes the CSV text (NUL-terminated, truncated to cap) and returns its length
int ref_staircase_csv(int family, int accuracy, double lo, double hi, int points, char* buf,
                      int cap) {
    const std::string csv = mexp::staircase_csv(
        mexp::cost_staircase(fam_of(family), acc_of(accuracy), mexp::log_grid(lo, hi, points)));
    std::snprintf(buf, std::size_t(cap), "%s", csv.c_str());
    return int(csv.size());
}

// The `sweep` subcommand of the reference CLI (tools/mexp_cli.cpp:122-161),
// whose own build needs the absent CLI11: the same spec derivation from the
// base seed, then error_sweep + sweep_csv. kinds / families are index lists.
int ref_sweep_csv(const int* kinds, int nk, const int* families, int nf, int n, int count,
                  uint64_t seed, int accuracy, double lo, double hi, char* buf, int cap) {
    std::vector<mexp::Family> fams;
    for (int i = 0; i < nf; ++i) fams.push_back(fam_of(families[i]));
    std::mt19937_64 rng(seed ^ 0xda3e39cb94b95bdbULL);
    std::vector<mexp::GallerySpec> specs;
    const double llo = std::log(lo), lhi = std::log(hi);
    for (int i = 0; i < count; ++i) {
        mexp::GallerySpec spec;
        spec.kind = mexp::kAllGalleryKinds[kinds[i % nk]];
        spec.n = n;
        spec.seed = seed * 1000003ULL + std::uint64_t(i);
        const double f = 0.5 * (mexp::uniform_pm1(rng) + 1.0);
        spec.target_norm = std::exp(llo + f * (lhi - llo));
        specs.push_back(spec);
    }
    try {
        const std::string csv = mexp::sweep_csv(mexp::error_sweep(specs, fams, acc_of(accuracy)));
        std::snprintf(buf, std::size_t(cap), "%s", csv.c_str());
        return int(csv.size());
    } catch (const std::exception& e) {
        std::snprintf(buf, std::size_t(cap), "error: %s", e.what());
        return -1;
    }
}

// Scheme coefficients as the library holds them at run time:
// t8 (10 values, taylor_schemes.cpp:12-27), kT12 (16, :62-71),
// kT18A (4) + kT18B (20) (:73-85).
void ref_coefficients(double* t8, double* t12, double* t18a, double* t18b) {
    const auto& c = mexp::t8_coefficients();
    const double v[10] = {c.x1, c.x2, c.x3, c.x4, c.x5, c.x6, c.x7, c.y0, c.y1, c.y2};
    std::memcpy(t8, v, sizeof v);
    std::memcpy(t12, mexp::kT12, sizeof(double) * 16);
    std::memcpy(t18a, mexp::kT18A, sizeof(double) * 4);
    std::memcpy(t18b, mexp::kT18B, sizeof(double) * 20);
}


// The reference's dense layer and scheme evaluators behind one entry with the
// operation codes of the product's mexp_b200_dense_call (dense_ops.cu), so a
// test can run both on the same inputs: 0 matmul, 1 lincomb (arg 1: n is the
// flat length), 2 one_norm, 3 lu_solve, 4 squarings, 5 eval_t8, 6 eval_t12,
// 7 eval_t18, 8 eval_ps(arg), 9 psi9, 10 taylor_oracle(arg), 11
// psi_oracle(arg), 12 eval_pade(arg), 13 eval_taylor_new(arg), 14
// eval_taylor_ps(arg), 15 kernels::lu_factor, 16 kernels::lu_apply. Returns
// 0, 3 (invalid argument) or 7 (singular denominator).
int ref_dense_call(int op, int arg, const double* const* in, int nin, const double* coeffs, int n,
                   double* out, const int32_t* iin, int32_t* iout, int64_t* products,
                   int64_t* solves) {
    try {
        mexp::CostContext ctx;
        const std::size_t nn = std::size_t(n) * n;
        auto put = [&](const mexp::DenseMatrix& r) { std::memcpy(out, r.data(), sizeof(double) * nn); };
        switch (op) {
            case 0: put(mexp::matmul(to_dense(in[0], n), to_dense(in[1], n))); break;
            case 1:
                if (arg == 1) {
                    mexp::kernels::lincomb(coeffs, in, nin, out, n);
                } else {
                    std::vector<mexp::DenseMatrix> ms;
                    std::vector<const mexp::DenseMatrix*> ps;
                    for (int i = 0; i < nin; ++i) ms.push_back(to_dense(in[i], n));
                    for (auto& m : ms) ps.push_back(&m);
                    put(mexp::lincomb(std::span<const double>(coeffs, nin),
                                      std::span<const mexp::DenseMatrix* const>(ps.data(), ps.size())));
                }
                break;
            case 2: *out = mexp::one_norm(to_dense(in[0], n)); break;
            case 3: put(mexp::lu_solve(ctx, to_dense(in[0], n), to_dense(in[1], n))); break;
            case 4: put(mexp::squarings(ctx, to_dense(in[0], n), arg)); break;
            case 5: put(mexp::eval_t8(ctx, to_dense(in[0], n))); break;
            case 6: put(mexp::eval_t12(ctx, to_dense(in[0], n))); break;
            case 7: put(mexp::eval_t18(ctx, to_dense(in[0], n))); break;
            case 8: put(mexp::eval_ps(ctx, to_dense(in[0], n), arg)); break;
            case 9: put(mexp::psi9(ctx, to_dense(in[0], n))); break;
            case 10: put(mexp::taylor_oracle(to_dense(in[0], n), arg)); break;
            case 11: put(mexp::psi_oracle(to_dense(in[0], n), arg)); break;
            case 12: put(mexp::eval_pade(ctx, to_dense(in[0], n), arg)); break;
            case 13: put(mexp::eval_taylor_new(ctx, to_dense(in[0], n), arg)); break;
            case 14: put(mexp::eval_taylor_ps(ctx, to_dense(in[0], n), arg)); break;
            case 15: {
                const auto f = mexp::kernels::lu_factor(in[0], n);
                std::memcpy(out, f.lu.data(), sizeof(double) * nn);
                for (int i = 0; i < n; ++i) iout[i] = f.perm[i];
                break;
            }
            case 16: {
                mexp::kernels::LuFactors f;
                f.n = n;
                f.lu.assign(in[0], in[0] + nn);
                f.perm.assign(iin, iin + n);
                mexp::kernels::lu_apply(f, in[1], out, n);
                break;
            }
            default: return kInvalid;
        }
        if (products) *products = ctx.products;
        if (solves) *solves = ctx.solves;
        return kOk;
    } catch (const std::invalid_argument&) {
        return kInvalid;
    } catch (const std::runtime_error&) {
        return kSingular;
    }
}

// psi9_coefficients (taylor_schemes.cpp:29-42, 57-60): x1..x9
void ref_psi9_coefficients(double* x) {
    const auto& c = mexp::psi9_coefficients();
    const double v[9] = {c.x1, c.x2, c.x3, c.x4, c.x5, c.x6, c.x7, c.x8, c.x9};
    for (int i = 0; i < 9; ++i) x[i] = v[i];
}

}  // extern "C"
