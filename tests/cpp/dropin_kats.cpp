// The reference's own known-answer tests for the expm path, re-expressed
// without doctest (absent here) against the C++ drop-in headers
// (include/mexp/*.hpp) and linked to libmexp_b200.so instead of libmexp.a.
// Sources of the cases: proj/tests/test_expm.cpp:21-197,
// test_dense_matrix.cpp:51-55, cli_smoke.sh:10-19.
//   dropin_kats                 run everything (needs a B200)
//   dropin_kats --no-device     check the host-only API and that expm refuses
//                               with std::runtime_error (no CPU fallback)
#include <cmath>
#include <cstdio>
#include <cstring>
#include <limits>
#include <random>
#include <stdexcept>

#include "mexp/expm.hpp"

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

int main(int argc, char** argv) {
    const bool no_device = argc > 1 && std::strcmp(argv[1], "--no-device") == 0;
    host_only();
    if (no_device) {
        CHECK(throws<std::runtime_error>([] { expm(DenseMatrix(2), Accuracy::Double, Family::TaylorNew); }));
    } else {
        device_cases();
    }
    std::printf("%s: %d failure(s)\n", no_device ? "dropin_kats --no-device" : "dropin_kats", failures);
    return failures == 0 ? 0 : 1;
}
