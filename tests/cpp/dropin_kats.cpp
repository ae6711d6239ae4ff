// The reference's own known-answer tests for the expm path, re-expressed
// without doctest (absent here) against the C++ drop-in headers
// (include/mexp/*.hpp) and linked to libmexp_b200.so instead of libmexp.a.
// Sources of the cases: proj/tests/test_expm.cpp:21-197,
// test_dense_matrix.cpp:17-74, test_kernels.cpp:85-100, test_pade.cpp:61-190,
// cli_smoke.sh:10-19.
//   dropin_kats                 run everything (needs a B200)
//   dropin_kats --no-device     check the host-only API and that expm refuses
//                               with std::runtime_error (no CPU fallback)
#include <cmath>
#include <cstdio>
#include <cstring>
#include <limits>
#include <random>
#include <stdexcept>
#include <vector>

#include "mexp/batched.hpp"
#include "mexp/expm.hpp"
#include "mexp/kernels.hpp"
#include "mexp/pade.hpp"
#include "mexp/taylor_schemes.hpp"

using namespace mexp;

static int failures = 0;
#define CHECK(cond)                                                              \
    do {                                                                         \
        if (!(cond)) {                                                           \
            std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond);          \
            ++failures;                                                          \
        }                                                                        \
    } while (0)

template <class E, class F>
static bool throws(F f) {
    try {
        f();
    } catch (const E&) {
        return true;
    } catch (...) {
        return false;
    }
    return false;
}

static double norm1(const DenseMatrix& a) {
    double best = 0;
    for (int j = 0; j < a.dim(); ++j) {
        double s = 0;
        for (int i = 0; i < a.dim(); ++i) s += std::abs(a.at(i, j));
        if (s > best) best = s;
    }
    return best;
}
static DenseMatrix mul(const DenseMatrix& a, const DenseMatrix& b) {
    DenseMatrix c(a.dim());
    for (int i = 0; i < a.dim(); ++i)
        for (int k = 0; k < a.dim(); ++k)
            for (int j = 0; j < a.dim(); ++j) c.at(i, j) += a.at(i, k) * b.at(k, j);
    return c;
}
static double dist_identity(const DenseMatrix& a) {
    DenseMatrix d = a;
    for (int i = 0; i < a.dim(); ++i) d.at(i, i) -= 1.0;
    return norm1(d);
}
static DenseMatrix random_with_norm(int n, double norm, std::mt19937_64& rng) {
    DenseMatrix m(n);
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) m.at(i, j) = 2.0 * (double(rng() >> 11) * 0x1.0p-53) - 1.0;
    const double f = norm / norm1(m);
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) m.at(i, j) *= f;
    return m;
}

static void host_only() {
    const auto& tn = selection_table(Family::TaylorNew, Accuracy::Double);
    CHECK(select(0.0, tn).degree == 1 && select(0.0, tn).s == 0);
    CHECK(select(1.0, tn).degree == 18 && select(1.0, tn).s == 0);
    CHECK(select(10.0, tn).degree == 18 && select(10.0, tn).s == 4);
    CHECK(select(2.18, tn).degree == 18 && select(2.18, tn).s == 1);
    CHECK(throws<std::invalid_argument>([&] { select(std::numeric_limits<double>::quiet_NaN(), tn); }));
    CHECK(throws<std::invalid_argument>([&] { select(std::numeric_limits<double>::infinity(), tn); }));
    for (double norm : {1.2, 3.7, 9.0, 40.0, 333.0})
        CHECK(select(2.0 * norm, tn).s == select(norm, tn).s + 1);
    CHECK(tn.entries.size() == 6 && tn.theta_max() == 1.09 && tn.asymptotic().products == 5);
    CHECK(unit_roundoff(Accuracy::Single) == std::ldexp(1.0, -24));
    // Family::PadeDiagonal (theta_tables.cpp:61-73)
    const auto& pd = selection_table(Family::PadeDiagonal, Accuracy::Double);
    CHECK(pd.entries.size() == 13 && pd.theta_max() == 5.37 && pd.asymptotic().degree == 26);
    CHECK(select(3.141592653589793, pd).degree == 22 && select(0.5, pd).degree == 12 &&
          select(10.0, pd).s == 1);
    // Family::TaylorPS (theta_tables.cpp:53-59)
    const auto& ps = selection_table(Family::TaylorPS, Accuracy::Double);
    CHECK(ps.entries.size() == 6 && ps.theta_max() == 7.80e-1 && ps.asymptotic().degree == 16 &&
          ps.asymptotic().products == 6);
    CHECK(select(0.5, ps).degree == 16 && select(0.05, ps).degree == 9 &&
          select(0.005, ps).degree == 6 && select(3.0, ps).s == 2);
    CHECK(selection_table(Family::TaylorPS, Accuracy::Single).theta_max() == 2.48);
    Family f;
    CHECK(parse_family("taylor", f) && f == Family::TaylorNew);
    CHECK(std::strcmp(family_name(Family::TaylorPS), "taylor-ps") == 0);
    CHECK(DenseMatrix::identity(3).at(1, 1) == 1.0 && DenseMatrix(2).at(0, 1) == 0.0);
    CHECK(throws<std::invalid_argument>([] { DenseMatrix(0); }));
    CHECK(throws<std::invalid_argument>([] { DenseMatrix(2, std::vector<double>(3)); }));
}

static void device_cases() {
    const double pi = 3.141592653589793;
    // zero -> identity, degree 1 (test_expm.cpp:71-78)
    const auto z = expm(DenseMatrix(4), Accuracy::Double, Family::TaylorNew);
    CHECK(z.result == DenseMatrix::identity(4) && z.s == 0 && z.degree == 1);
    // rotation by pi (test_expm.cpp:80-89)
    const auto rot = expm(DenseMatrix::from_rows({{0, pi}, {-pi, 0}}), Accuracy::Double,
                          Family::TaylorNew);
    CHECK(rot.degree == 18 && rot.s == 2 && rot.norm_in == pi && rot.cost_thirds == 21);
    CHECK(norm1(DenseMatrix::from_rows({{rot.result.at(0, 0) + 1, rot.result.at(0, 1)},
                                        {rot.result.at(1, 0), rot.result.at(1, 1) + 1}})) <= 1e-12);
    // rotation by 1 rad: the CLI report "taylor-new 18 0 5 1" (cli_smoke.sh:10-19)
    const auto r1 = expm(DenseMatrix::from_rows({{0, 1}, {-1, 0}}), Accuracy::Double, Family::TaylorNew);
    CHECK(r1.degree == 18 && r1.s == 0 && r1.product_cost() == 5.0 && r1.norm_in == 1.0);
    // non-finite input (test_expm.cpp:101-106)
    DenseMatrix bad(2);
    bad.at(0, 1) = std::numeric_limits<double>::infinity();
    CHECK(throws<std::invalid_argument>([&] { expm(bad, Accuracy::Double, Family::TaylorNew); }));
    // Pade family: rotation by pi -> r22, no scaling, 6 products + 4/3 for the solve
    const auto rpd = expm(DenseMatrix::from_rows({{0, pi}, {-pi, 0}}), Accuracy::Double,
                          Family::PadeDiagonal);
    CHECK(rpd.degree == 22 && rpd.s == 0 && rpd.cost_thirds == 22);
    CHECK(norm1(DenseMatrix::from_rows({{rpd.result.at(0, 0) + 1, rpd.result.at(0, 1)},
                                        {rpd.result.at(1, 0), rpd.result.at(1, 1) + 1}})) <= 1e-12);
    // Pade beyond n = 64: the DMMA GEMM chain + batched blocked LU
    const auto pz = expm(DenseMatrix(65), Accuracy::Double, Family::PadeDiagonal);
    CHECK(pz.result == DenseMatrix::identity(65) && pz.degree == 2 && pz.s == 0);
    // Paterson-Stockmeyer family: rotation by pi -> m = 16, s = 3, 6 + 3 products
    const auto rps = expm(DenseMatrix::from_rows({{0, pi}, {-pi, 0}}), Accuracy::Double,
                          Family::TaylorPS);
    CHECK(rps.degree == 16 && rps.s == 3 && rps.cost_thirds == 27 && rps.family == Family::TaylorPS);
    CHECK(norm1(DenseMatrix::from_rows({{rps.result.at(0, 0) + 1, rps.result.at(0, 1)},
                                        {rps.result.at(1, 0), rps.result.at(1, 1) + 1}})) <= 1e-12);
    // expm(A) expm(-A) = I (test_expm.cpp:108-120)
    std::mt19937_64 rng(42);
    for (int rep = 0; rep < 34; ++rep) {
        const int n = 2 + int(rng() % 15);
        const DenseMatrix a = random_with_norm(n, 5.0 * double(rng() >> 11) * 0x1.0p-53 + 1e-6, rng);
        DenseMatrix neg = a;
        for (int i = 0; i < n; ++i)
            for (int j = 0; j < n; ++j) neg.at(i, j) = -a.at(i, j);
        const auto x = expm(a, Accuracy::Double, Family::TaylorNew).result;
        const auto y = expm(neg, Accuracy::Double, Family::TaylorNew).result;
        CHECK(dist_identity(mul(x, y)) <= 1e-12);
    }
    // skew-symmetric input -> orthogonal exponential (test_expm.cpp:122-133)
    for (int rep = 0; rep < 20; ++rep) {
        DenseMatrix b = random_with_norm(10, 1.0, rng), a(10);
        for (int i = 0; i < 10; ++i)
            for (int j = 0; j < 10; ++j) a.at(i, j) = b.at(i, j) - b.at(j, i);
        const double f = 3.0 * (rep % 5 + 1) / 5.0 / norm1(a);
        for (int i = 0; i < 10; ++i)
            for (int j = 0; j < 10; ++j) a.at(i, j) *= f;
        const auto x = expm(a, Accuracy::Double, Family::TaylorNew).result;
        DenseMatrix xt(10);
        for (int i = 0; i < 10; ++i)
            for (int j = 0; j < 10; ++j) xt.at(i, j) = x.at(j, i);
        CHECK(dist_identity(mul(xt, x)) <= 1e-12);
    }
    // a single-precision target picks m = 8 at ||A|| = 0.4 (test_expm.cpp:175-186)
    std::mt19937_64 rng45(45);
    const DenseMatrix a8 = random_with_norm(8, 0.4, rng45);
    CHECK(expm(a8, Accuracy::Single, Family::TaylorNew).degree == 8);
    CHECK(expm(a8, Accuracy::Double, Family::TaylorNew).degree == 18);
    // squarings (test_expm.cpp:56-69)
    CostContext ctx;
    DenseMatrix two = DenseMatrix::identity(3);
    for (int i = 0; i < 3; ++i) two.at(i, i) = 2.0;
    DenseMatrix want = DenseMatrix::identity(3);
    for (int i = 0; i < 3; ++i) want.at(i, i) = 256.0;
    CHECK(squarings(ctx, two, 3) == want && ctx.products == 3);
    CHECK(squarings(ctx, DenseMatrix::from_rows({{1, 1}, {0, 1}}), 2) ==
          DenseMatrix::from_rows({{1, 4}, {0, 1}}));
    // large n goes through the DMMA GEMM engine
    const DenseMatrix big = random_with_norm(100, 3.0, rng);
    const auto eb = expm(big, Accuracy::Double, Family::TaylorNew);
    CHECK(eb.degree == 18 && eb.s == 2 && eb.result.all_finite());
}

// The reference's dense-matrix layer (dense_matrix.hpp:40-58, kernels.hpp,
// taylor_schemes.hpp, pade.hpp) on the device.
static void dense_layer_cases() {
    std::mt19937_64 rng(1);
    const DenseMatrix x = random_with_norm(5, 2.0, rng);
    // test_dense_matrix.cpp:17-29
    CHECK(matmul(DenseMatrix::identity(5), x) == x);
    const DenseMatrix nil = DenseMatrix::from_rows({{0, 1}, {0, 0}});
    CHECK(matmul(nil, nil) == DenseMatrix(2));
    const DenseMatrix a = DenseMatrix::from_rows({{1, 2}, {3, 4}});
    const DenseMatrix b = DenseMatrix::from_rows({{5, 6}, {7, 8}});
    CHECK(matmul(a, b) == DenseMatrix::from_rows({{19, 22}, {43, 50}}));
    CHECK(throws<std::invalid_argument>([&] { matmul(a, DenseMatrix(3)); }));
    // test_dense_matrix.cpp:31-47
    const DenseMatrix id2 = DenseMatrix::identity(2);
    CHECK(lincomb({1.0}, {&id2}) == id2);
    CHECK(lincomb({2.0, -1.0}, {&x, &x}) == x);
    CHECK(lincomb({1.0, 1.0}, {&id2, &nil}) == DenseMatrix::from_rows({{1, 1}, {0, 1}}));
    CHECK(throws<std::invalid_argument>(
        [] { lincomb(std::span<const double>{}, std::span<const DenseMatrix* const>{}); }));
    const DenseMatrix b3(3);
    CHECK(throws<std::invalid_argument>([&] { lincomb({1.0, 1.0}, {&x, &b3}); }));
    // test_dense_matrix.cpp:49-53
    CHECK(one_norm(DenseMatrix(3)) == 0.0);
    CHECK(one_norm(DenseMatrix::identity(5)) == 1.0);
    CHECK(one_norm(DenseMatrix::from_rows({{1, -2}, {3, 4}})) == 6.0);
    // test_dense_matrix.cpp:55-71
    const DenseMatrix x6 = random_with_norm(6, 3.0, rng);
    CHECK(lu_solve(DenseMatrix::identity(6), x6) == x6);
    CHECK(lu_solve(DenseMatrix::from_rows({{2, 0}, {0, 4}}), id2) ==
          DenseMatrix::from_rows({{0.5, 0}, {0, 0.25}}));
    const DenseMatrix rhs = DenseMatrix::from_rows({{1, 2}, {3, 4}});
    CHECK(lu_solve(DenseMatrix::from_rows({{0, 1}, {1, 0}}), rhs) ==
          DenseMatrix::from_rows({{3, 4}, {1, 2}}));
    bool singular = false;
    try {
        lu_solve(DenseMatrix(2), rhs);
    } catch (const std::runtime_error& e) {
        singular = std::strcmp(e.what(), "singular denominator") == 0;
    }
    CHECK(singular);
    CHECK(add(a, b) == DenseMatrix::from_rows({{6, 8}, {10, 12}}));
    CHECK(sub(b, a) == DenseMatrix::from_rows({{4, 4}, {4, 4}}));
    CHECK(scaled(a, 0.5) == DenseMatrix::from_rows({{0.5, 1}, {1.5, 2}}));
    // the reference's error_sweep expression (bench.cpp:83) compiles and runs
    const auto rep = expm(x, Accuracy::Double, Family::TaylorNew);
    CHECK(one_norm(sub(rep.result, rep.result)) == 0.0);
    // test_kernels.cpp:85-100: the first maximal row wins the pivot
    const double tie[9] = {1, 0, 0, -3, 1, 0, 3, 0, 1};
    const auto f = kernels::lu_factor(tie, 3);
    CHECK(f.perm[0] == 1);
    double y[9];
    kernels::lu_apply(f, tie, y, 3);
    CHECK(std::abs(y[0] - 1) + std::abs(y[4] - 1) + std::abs(y[8] - 1) <= 1e-15);
    double c[4];
    kernels::matmul(a.data(), b.data(), c, 2);
    CHECK(c[0] == 19 && c[3] == 50 && kernels::one_norm(a.data(), 2) == 6.0);
    // ledgers: eval_t18 5 products, eval_r10 3 products + 1 solve (test_pade.cpp:142-156)
    CostContext ctx;
    const DenseMatrix small = random_with_norm(6, 0.5, rng);
    eval_t18(ctx, small);
    CHECK(ctx.products == 5 && ctx.solves == 0);
    ctx.reset();
    eval_r10(ctx, small);
    CHECK(ctx.products == 3 && ctx.solves == 1 && ctx.thirds() == 13);
    ctx.reset();
    eval_ps(ctx, small, 16);
    CHECK(ctx.products == 6);
    ctx.reset();
    psi9(ctx, small);
    CHECK(ctx.products == 3);
    // schemes agree with the Horner oracle (test_taylor_schemes.cpp:50-100)
    const DenseMatrix t = taylor_oracle(small, 18);
    CHECK(norm1(sub(eval_taylor_new(ctx, small, 18), t)) <= 1e-14);
    CHECK(norm1(sub(psi9(ctx, small), psi_oracle(small, 9))) <= 1e-14);
    // pade_coeffs (test_pade.cpp:61-79): b_0 = 1, b_1 = 1/2, r_1 of 2x2 zero = I
    const auto pc = pade_coeffs(13);
    CHECK(pc.m == 13 && pc.b.size() == 14 && pc.b[0] == 1.0 && pc.b[1] == 0.5);
    CHECK(throws<std::invalid_argument>([] { pade_coeffs(14); }));
    CHECK(eval_pade(ctx, DenseMatrix(3), 26) == DenseMatrix::identity(3));
    CHECK(t8_coefficients().x3 == 2.0 / 3.0 && kT12[0][0] == 9.0198e-16 && kT18B[1][0] < -10.0);
    CHECK(psi9_coefficients().x2 == -0.25 && psi9_coefficients().x3 == -1.0);
}

// the batched C++ API (include/mexp/batched.hpp): every record and every
// e^A equals mexp::expm's for the same matrix; per-matrix errors stay in the
// records, call-level errors throw
static void batched_cases() {
    std::mt19937_64 rng(7);
    std::uniform_real_distribution<double> u(-1.0, 1.0);
    const int n = 8, batch = 6;
    std::vector<double> a(size_t(batch) * n * n), out(a.size());
    const double scale[batch] = {1e-4, 0.02, 0.3, 1.0, 5.0, 40.0};
    for (int b = 0; b < batch; ++b)
        for (int e = 0; e < n * n; ++e) a[size_t(b) * n * n + e] = scale[b] * u(rng);
    a[size_t(3) * n * n + 10] = std::numeric_limits<double>::quiet_NaN();
    const BatchResult r = expm_batched(a.data(), out.data(), n, batch, Accuracy::Double);
    CHECK(r.records.size() == size_t(batch) && r.first_error == 3);
    for (int b = 0; b < batch; ++b) {
        DenseMatrix m(n);
        std::memcpy(m.data(), a.data() + size_t(b) * n * n, sizeof(double) * n * n);
        if (b == 3) {
            CHECK(r.records[b].status == 1 && std::isnan(out[size_t(b) * n * n]));
            continue;
        }
        const ExpmReport rep = expm(m, Accuracy::Double, Family::TaylorNew);
        CHECK(r.records[b].status == 0 && r.records[b].degree == rep.degree && r.records[b].s == rep.s);
        CHECK(r.records[b].norm_in == rep.norm_in);
        CHECK(std::memcmp(rep.result.data(), out.data() + size_t(b) * n * n, sizeof(double) * n * n) == 0);
    }
    // fp32, 32 x 32, Single table: the selection equals mexp::select on the fp64 norm
    const int m32 = 32, b32 = 3;
    std::vector<float> f(size_t(b32) * m32 * m32), fo(f.size());
    for (auto& x : f) x = float(0.05 * u(rng));
    const BatchResult rf = expm_batched(f.data(), fo.data(), m32, b32, Accuracy::Single);
    const SelectionTable st = selection_table(Family::TaylorNew, Accuracy::Single);
    for (int b = 0; b < b32; ++b) {
        const Selection want = select(rf.records[b].norm_in, st);
        CHECK(rf.records[b].status == 0 && rf.records[b].degree == want.degree && rf.records[b].s == want.s);
    }
    CHECK(rf.first_error == -1);
    // the multi-device entry gives the same bits (devices: all visible)
    std::vector<double> out2(a.size());
    const BatchResult r2 = expm_batched_multi(a.data(), out2.data(), n, batch, Accuracy::Double);
    CHECK(r2.first_error == 3 && std::memcmp(out.data(), out2.data(), sizeof(double) * n * n * 3) == 0);
    CHECK(throws<std::invalid_argument>([&] { expm_batched(a.data(), out.data(), 0, 1, Accuracy::Double); }));
    CHECK(throws<std::invalid_argument>([&] { expm_batched(a.data(), out.data(), n, -1, Accuracy::Double); }));
}

int main(int argc, char** argv) {
    const bool no_device = argc > 1 && std::strcmp(argv[1], "--no-device") == 0;
    host_only();
    if (no_device) {
        CHECK(throws<std::runtime_error>([] { expm(DenseMatrix(2), Accuracy::Double, Family::TaylorNew); }));
        double x[4] = {0, 0, 0, 0}, y[4];
        CHECK(throws<std::runtime_error>([&] { expm_batched(x, y, 2, 1, Accuracy::Double); }));
    } else {
        device_cases();
        dense_layer_cases();
        batched_cases();
    }
    std::printf("%s: %d failure(s)\n", no_device ? "dropin_kats --no-device" : "dropin_kats", failures);
    return failures == 0 ? 0 : 1;
}
