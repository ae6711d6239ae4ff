// C++ drop-in for the reference's namespace mexp expm path (include/mexp/*.hpp),
// implemented over the C ABI (include/mexp_b200.h). Status codes become the
// reference's exceptions: std::invalid_argument for bad input (expm.cpp:13,38;
// dense_matrix.cpp:15,20,30), std::runtime_error for CUDA / device failures.
#include <charconv>
#include <cmath>
#include <istream>
#include <stdexcept>
#include <string>

#include "mexp/expm.hpp"
#include "mexp_b200.h"

// capi.cu (library-internal, not part of the public C ABI)
extern "C" int mexp_b200_squarings_host(double* x, int n, int s);

namespace mexp {

namespace {

[[noreturn]] void throw_status(int st) {
    const char* msg = mexp_status_string(st);
    switch (st) {
        case MEXP_ERR_NONFINITE:
        case MEXP_ERR_NORM_NONFINITE:
        case MEXP_ERR_INVALID_ARGUMENT:
        case MEXP_ERR_UNSUPPORTED:
            throw std::invalid_argument(msg);
        case MEXP_ERR_CUDA:
            throw std::runtime_error(std::string(msg) + ": " + mexp_last_cuda_error());
        default:
            throw std::runtime_error(msg);
    }
}

int checked_dim(int n) {
    if (n < 1) throw std::invalid_argument("matrix dimension must be positive");
    return n;
}

SelectionTable load_table(Family f, Accuracy u) {
    int32_t d[16], p[16];
    double t[16];
    const int k = mexp_selection_table(int(u), int(f), d, p, t, 16);
    if (k < 0) throw_status(-k);
    SelectionTable table{f, u, {}};
    for (int i = 0; i < k; ++i) table.entries.push_back({f, d[i], p[i], t[i]});
    return table;
}

}  // namespace

// ---- DenseMatrix (container surface of dense_matrix.hpp:15-38) ----------
DenseMatrix::DenseMatrix(int n) : n_(checked_dim(n)), data_(std::size_t(n) * n, 0.0) {}

DenseMatrix::DenseMatrix(int n, std::vector<double> data)
    : n_(checked_dim(n)), data_(std::move(data)) {
    if (data_.size() != std::size_t(n_) * n_)
        throw std::invalid_argument("data length must equal n*n");
}

DenseMatrix DenseMatrix::identity(int n) {
    DenseMatrix m(n);
    for (int i = 0; i < n; ++i) m.at(i, i) = 1.0;
    return m;
}

DenseMatrix DenseMatrix::from_rows(std::initializer_list<std::initializer_list<double>> rows) {
    const int n = int(rows.size());
    DenseMatrix m(n);
    int i = 0;
    for (const auto& row : rows) {
        if (int(row.size()) != n) throw std::invalid_argument("matrix must be square");
        int j = 0;
        for (double v : row) m.at(i, j++) = v;
        ++i;
    }
    return m;
}

bool DenseMatrix::all_finite() const {
    for (double v : data_)
        if (!std::isfinite(v)) return false;
    return true;
}

// ---- text I/O (host-side, dense_matrix.hpp:62-67 of the reference) ------
DenseMatrix parse_matrix(std::istream& in) {
    int n = 0;
    if (!(in >> n) || n < 1) throw std::invalid_argument("bad matrix header");
    DenseMatrix m(n);
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) {
            double v;
            if (!(in >> v)) throw std::invalid_argument("truncated matrix data");
            if (!std::isfinite(v)) throw std::invalid_argument("non-finite matrix entry");
            m.at(i, j) = v;
        }
    return m;
}

std::string shortest_double(double v) {
    char buf[64];
    const auto res = std::to_chars(buf, buf + sizeof(buf), v);
    return std::string(buf, res.ptr);
}

std::string format_matrix(const DenseMatrix& a) {
    std::string out = std::to_string(a.dim()) + "\n";
    for (int i = 0; i < a.dim(); ++i) {
        for (int j = 0; j < a.dim(); ++j) {
            if (j) out.push_back(' ');
            out += shortest_double(a.at(i, j));
        }
        out.push_back('\n');
    }
    return out;
}

// ---- theta tables (theta_tables.hpp) ------------------------------------
double unit_roundoff(Accuracy u) { return mexp_unit_roundoff(int(u)); }

const char* family_name(Family f) {
    switch (f) {
        case Family::TaylorNew: return "taylor-new";
        case Family::TaylorPS: return "taylor-ps";
        case Family::PadeDiagonal: return "pade";
    }
    return "?";
}

bool parse_family(std::string_view name, Family& out) {
    if (name == "taylor-new" || name == "taylor") out = Family::TaylorNew;
    else if (name == "taylor-ps" || name == "ps") out = Family::TaylorPS;
    else if (name == "pade") out = Family::PadeDiagonal;
    else return false;
    return true;
}

const SelectionTable& selection_table(Family f, Accuracy u) {
    static const SelectionTable single = load_table(Family::TaylorNew, Accuracy::Single);
    static const SelectionTable dbl = load_table(Family::TaylorNew, Accuracy::Double);
    static const SelectionTable ps_single = load_table(Family::TaylorPS, Accuracy::Single);
    static const SelectionTable ps_dbl = load_table(Family::TaylorPS, Accuracy::Double);
    static const SelectionTable pade_single = load_table(Family::PadeDiagonal, Accuracy::Single);
    static const SelectionTable pade_dbl = load_table(Family::PadeDiagonal, Accuracy::Double);
    if (f == Family::PadeDiagonal) return u == Accuracy::Single ? pade_single : pade_dbl;
    if (f == Family::TaylorPS) return u == Accuracy::Single ? ps_single : ps_dbl;
    return u == Accuracy::Single ? single : dbl;
}

// ---- expm.hpp ----------------------------------------------------------
Selection select(double norm, const SelectionTable& table) {
    int32_t d = 0, s = 0;
    const int st = mexp_select(norm, int(table.accuracy), int(table.family), &d, &s);
    if (st != MEXP_OK) throw_status(st);
    return {d, s};
}

DenseMatrix squarings(CostContext& ctx, DenseMatrix x, int s) {
    if (s < 0) throw std::invalid_argument("s must be nonnegative");
    if (s == 0) return x;
    // a one-matrix batch through the device (host -> device, s DMMA
    // squarings, device -> host)
    const int st = mexp_b200_squarings_host(x.data(), x.dim(), s);
    if (st != MEXP_OK) throw_status(st);
    ctx.products += s;
    return x;
}

ExpmReport expm(const DenseMatrix& a, Accuracy u, Family family) {
    if (a.dim() < 1) throw std::invalid_argument("matrix dimension must be positive");
    ExpmReport rep;
    rep.result = DenseMatrix(a.dim());
    mexp_report r{};
    const int st = mexp_expm(a.data(), a.dim(), int(u), int(family), rep.result.data(), &r);
    if (st != MEXP_OK) throw_status(st);
    rep.family = family;
    rep.degree = r.degree;
    rep.s = r.s;
    rep.cost_thirds = r.cost_thirds;
    rep.norm_in = r.norm_in;
    return rep;
}

}  // namespace mexp
