// The reference's bench.hpp surface (bench.cpp): reference_expm, the cost
// staircase and the accuracy sweep, with every exponential on the device.
// error_sweep batches: all gallery matrices of the sweep go to the GPU in one
// call for the ground truth and one call per family (the reference loops
// matrix by matrix). For n <= 64 both run in REFERENCE rounding, so every
// e^A -- and therefore every CSV field -- equals the reference's bit for bit.
#include <cmath>
#include <stdexcept>
#include <string>
#include <vector>

#include "mexp/bench.hpp"
#include "mexp_b200.h"

// capi.cu (library-internal, not part of the public C ABI)
extern "C" int mexp_b200_reference_expm_host(const double* a, double* out, int n, int64_t batch,
                                             int rounding, mexp_selection* sel);

namespace mexp {

namespace {

// one_norm (kernels.cpp:44-53)
double norm1(const double* a, int n) {
    double best = 0.0;
    for (int j = 0; j < n; ++j) {
        double s = 0.0;
        for (int i = 0; i < n; ++i) s += std::fabs(a[std::size_t(i) * n + j]);
        if (s > best) best = s;
    }
    return best;
}

// one_norm(sub(x, y)): sub = lincomb({1, -1}) (dense_matrix.cpp:98-100)
double norm1_diff(const double* x, const double* y, int n) {
    std::vector<double> d(std::size_t(n) * n);
    for (std::size_t e = 0; e < d.size(); ++e) d[e] = 1.0 * x[e] + -1.0 * y[e];
    return norm1(d.data(), n);
}

[[noreturn]] void throw_status(int st) {
    const char* msg = mexp_status_string(st);
    if (st == MEXP_ERR_NONFINITE || st == MEXP_ERR_NORM_NONFINITE || st == MEXP_ERR_INVALID_ARGUMENT ||
        st == MEXP_ERR_UNSUPPORTED)
        throw std::invalid_argument(msg);
    if (st == MEXP_ERR_CUDA) throw std::runtime_error(std::string(msg) + ": " + mexp_last_cuda_error());
    throw std::runtime_error(msg);
}

// the reference's arithmetic where the device has it (n <= 64)
int sweep_rounding(int n) { return n <= 64 ? MEXP_ROUND_REFERENCE : MEXP_ROUND_AUTO; }

std::int64_t model_cost_thirds(const SelectionTable& table, const Selection& sel) {
    for (const auto& e : table.entries)
        if (e.degree == sel.degree)
            return 3 * std::int64_t(e.products + sel.s) + (table.family == Family::PadeDiagonal ? 4 : 0);
    throw std::logic_error("degree missing from table");
}

// batched ground truth: stacked n x n matrices -> their reference_expm
std::vector<double> reference_batch(const std::vector<double>& a, int n, int64_t batch) {
    std::vector<double> out(a.size());
    std::vector<mexp_selection> sel(batch);
    const int st = mexp_b200_reference_expm_host(a.data(), out.data(), n, batch,
                                                 sweep_rounding(n), sel.data());
    if (st != MEXP_OK) throw_status(st);
    for (const auto& r : sel)
        if (r.status != MEXP_OK) throw_status(r.status);
    return out;
}

}  // namespace

DenseMatrix reference_expm(const DenseMatrix& a) {
    if (!a.all_finite()) throw std::invalid_argument("non-finite matrix entry");
    std::vector<double> in(a.data(), a.data() + std::size_t(a.dim()) * a.dim());
    std::vector<double> out = reference_batch(in, a.dim(), 1);
    return DenseMatrix(a.dim(), std::move(out));
}

std::vector<StaircaseRow> cost_staircase(Family f, Accuracy u, const std::vector<double>& norms) {
    const auto& table = selection_table(f, u);
    std::vector<StaircaseRow> rows;
    rows.reserve(norms.size());
    for (double norm : norms) {
        const Selection sel = select(norm, table);
        rows.push_back({norm, sel.degree, sel.s, model_cost_thirds(table, sel)});
    }
    return rows;
}

std::string staircase_csv(const std::vector<StaircaseRow>& rows) {
    std::string out = "norm,degree,s,product_cost\n";
    for (const auto& r : rows)
        out += shortest_double(r.norm) + ',' + std::to_string(r.degree) + ',' + std::to_string(r.s) +
               ',' + shortest_double(r.product_cost()) + '\n';
    return out;
}

std::vector<SweepRow> error_sweep(const std::vector<GallerySpec>& specs,
                                  const std::vector<Family>& families, Accuracy u) {
    if (specs.empty() || families.empty())
        throw std::invalid_argument("sweep needs matrices and families");
    // the batches need one n; the reference's CLI sweeps one dimension
    const int n = specs.front().n;
    for (const auto& sp : specs)
        if (sp.n != n) throw std::invalid_argument("sweep matrices must share one dimension");
    const std::size_t nn = std::size_t(n) * n;
    const int64_t count = int64_t(specs.size());
    std::vector<double> a(nn * count), norms(count);
    for (int64_t i = 0; i < count; ++i) {
        const DenseMatrix g = gallery(specs[i]);
        std::copy(g.data(), g.data() + nn, a.begin() + i * nn);
        norms[i] = norm1(g.data(), n);
    }
    const std::vector<double> ref = reference_batch(a, n, count);
    std::vector<double> ref_norm(count);
    for (int64_t i = 0; i < count; ++i) ref_norm[i] = norm1(ref.data() + i * nn, n);

    std::vector<SweepRow> rows(std::size_t(count) * families.size());
    std::vector<double> out(nn * count);
    std::vector<mexp_selection> sel(count);
    for (std::size_t f = 0; f < families.size(); ++f) {
        const Family fam = families[f];
        const int st = mexp_expm_batched_host(a.data(), out.data(), MEXP_F64, n, count, int(u),
                                              int(fam), sweep_rounding(n), sel.data(), nullptr);
        if (st != MEXP_OK && st != MEXP_ERR_SINGULAR) throw_status(st);
        const auto& table = selection_table(fam, u);
        for (int64_t i = 0; i < count; ++i) {
            SweepRow& row = rows[std::size_t(i) * families.size() + f];
            row.matrix_id = int(i);
            row.kind = specs[i].kind;
            row.n = n;
            row.norm = norms[i];
            row.family = fam;
            if (sel[i].status == MEXP_ERR_SINGULAR) {  // runtime_error in the reference
                row.failed = true;
                continue;
            }
            if (sel[i].status != MEXP_OK) throw_status(sel[i].status);
            row.degree = sel[i].degree;
            row.s = sel[i].s;
            row.cost_thirds = model_cost_thirds(table, {row.degree, row.s});
            row.relerr = norm1_diff(out.data() + i * nn, ref.data() + i * nn, n) / ref_norm[i];
        }
    }
    return rows;
}

std::string sweep_csv(const std::vector<SweepRow>& rows) {
    std::string out =
        "# relerr is measured against an over-scaled order-26 Pade reference "
        "computed in double precision and floors near the unit roundoff\n"
        "matrix_id,kind,n,norm,family,degree,s,product_cost,relerr\n";
    for (const auto& r : rows) {
        out += std::to_string(r.matrix_id) + ',' + gallery_kind_name(r.kind) + ',' +
               std::to_string(r.n) + ',' + shortest_double(r.norm) + ',' + family_name(r.family) + ',';
        if (r.failed)
            out += "0,0,0,FAIL";
        else
            out += std::to_string(r.degree) + ',' + std::to_string(r.s) + ',' +
                   shortest_double(double(r.cost_thirds) / 3.0) + ',' + shortest_double(r.relerr);
        out += '\n';
    }
    return out;
}

std::vector<double> log_grid(double lo, double hi, int points) {
    if (!(lo > 0) || !(hi >= lo) || points < 1) throw std::invalid_argument("bad norm grid");
    std::vector<double> g;
    g.reserve(points);
    if (points == 1) {
        g.push_back(lo);
        return g;
    }
    const double step = std::log(hi / lo) / (points - 1);
    for (int i = 0; i < points; ++i) g.push_back(lo * std::exp(step * i));
    g.back() = hi;
    return g;
}

}  // namespace mexp
