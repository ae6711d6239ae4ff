// Host-side test-matrix gallery (reference gallery.cpp / gallery.hpp): the
// inputs of the accuracy sweep. Each kind consumes the generator in the
// reference's order, so (kind, n, seed) gives the reference's matrix bit for
// bit; the final rescale is the reference's scaled(m, target / one_norm(m)).
#include <cmath>
#include <stdexcept>
#include <vector>

#include "mexp/gallery.hpp"

namespace mexp {

namespace {

constexpr const char* kKindNames[] = {"random_dense",    "random_symmetric", "random_skew",
                                      "jordan_block",    "nilpotent_shift",  "upper_triangular",
                                      "tridiag_toeplitz", "rank_one",        "nonnormal_shear"};

// one_norm (kernels.cpp:44-53): column sums over rows in order, strict '>'
double column_norm(const DenseMatrix& m) {
    double best = 0.0;
    for (int j = 0; j < m.dim(); ++j) {
        double s = 0.0;
        for (int i = 0; i < m.dim(); ++i) s += std::fabs(m.at(i, j));
        if (s > best) best = s;
    }
    return best;
}

void fill(DenseMatrix& m, const GallerySpec& spec, std::mt19937_64& rng) {
    const int n = spec.n;
    auto draw = [&] { return uniform_pm1(rng); };
    switch (spec.kind) {
        case GalleryKind::RandomDense:  // row-major draws
            for (int i = 0; i < n; ++i)
                for (int j = 0; j < n; ++j) m.at(i, j) = draw();
            return;
        case GalleryKind::RandomSymmetric:  // upper triangle incl. diagonal, mirrored
            for (int i = 0; i < n; ++i)
                for (int j = i; j < n; ++j) {
                    const double v = draw();
                    m.at(i, j) = v;
                    m.at(j, i) = v;
                }
            return;
        case GalleryKind::RandomSkew:  // strict upper triangle, negated below
            for (int i = 0; i < n; ++i)
                for (int j = i + 1; j < n; ++j) {
                    const double v = draw();
                    m.at(i, j) = v;
                    m.at(j, i) = -v;
                }
            return;
        case GalleryKind::JordanBlock: {  // eigenvalue 0.25 * (seed mod 5), ones above
            const double lambda = 0.25 * double(spec.seed % 5);
            for (int i = 0; i < n; ++i) {
                m.at(i, i) = lambda;
                if (i + 1 < n) m.at(i, i + 1) = 1.0;
            }
            return;
        }
        case GalleryKind::NilpotentShift:
            for (int i = 0; i + 1 < n; ++i) m.at(i, i + 1) = 1.0;
            return;
        case GalleryKind::UpperTriangular:
            for (int i = 0; i < n; ++i)
                for (int j = i; j < n; ++j) m.at(i, j) = draw();
            return;
        case GalleryKind::TridiagToeplitz: {  // draws: sub, diagonal, super
            const double lo = draw(), mid = draw(), hi = draw();
            for (int i = 0; i < n; ++i) {
                m.at(i, i) = mid;
                if (i + 1 < n) {
                    m.at(i + 1, i) = lo;
                    m.at(i, i + 1) = hi;
                }
            }
            return;
        }
        case GalleryKind::RankOne: {  // u then v, m = u v^T
            std::vector<double> u(n), v(n);
            for (double& x : u) x = draw();
            for (double& x : v) x = draw();
            for (int i = 0; i < n; ++i)
                for (int j = 0; j < n; ++j) m.at(i, j) = u[i] * v[j];
            return;
        }
        case GalleryKind::NonnormalShear:
            for (int i = 0; i < n; ++i) m.at(i, i) = 1.0;
            if (n > 1) m.at(0, n - 1) = 10.0;
            return;
    }
}

}  // namespace

const char* gallery_kind_name(GalleryKind k) {
    const int i = int(k);
    return (i >= 0 && i < 9) ? kKindNames[i] : "?";
}

bool parse_gallery_kind(std::string_view name, GalleryKind& out) {
    for (GalleryKind k : kAllGalleryKinds)
        if (name == gallery_kind_name(k)) {
            out = k;
            return true;
        }
    return false;
}

double uniform_pm1(std::mt19937_64& rng) {
    const double u = double(rng() >> 11) * 0x1.0p-53;  // 53 bits -> [0, 1)
    return 2.0 * u - 1.0;
}

DenseMatrix gallery(const GallerySpec& spec) {
    if (spec.n < 1) throw std::invalid_argument("gallery dimension must be positive");
    if (!(spec.target_norm > 0)) throw std::invalid_argument("target norm must be positive");
    std::mt19937_64 rng(spec.seed * 0x9e3779b97f4a7c15ULL + 0x2545f4914f6cdd1dULL);
    DenseMatrix m(spec.n);
    fill(m, spec, rng);
    const double norm = column_norm(m);
    if (norm == 0.0) throw std::domain_error("cannot rescale a zero matrix");
    const double f = spec.target_norm / norm;
    for (int i = 0; i < spec.n; ++i)
        for (int j = 0; j < spec.n; ++j) m.at(i, j) = f * m.at(i, j);
    return m;
}

}  // namespace mexp
