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
#include "mexp/kernels.hpp"
#include "mexp/pade.hpp"
#include "mexp/taylor_schemes.hpp"
#include "mexp_b200.h"
#include "scheme_tables.h"

// dense_ops.cu (library-internal, not part of the public C ABI)
extern "C" int mexp_b200_dense_call(int op, int arg, const double* const* in, int nin,
                                    const double* coeffs, int n, double* out, const int32_t* iin,
                                    int32_t* iout, int64_t* products, int64_t* solves);
extern "C" void mexp_b200_psi9_coefficients(double* x);
extern "C" int mexp_b200_pade_coefficients(int m, double* b);

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

// mexp_b200_dense_call operations (dense_ops.cu)
enum DenseOp {
    kOpMatmul = 0, kOpLincomb = 1, kOpOneNorm = 2, kOpLuSolve = 3, kOpSquarings = 4, kOpT8 = 5,
    kOpT12 = 6, kOpT18 = 7, kOpPs = 8, kOpPsi9 = 9, kOpTaylorOracle = 10, kOpPsiOracle = 11,
    kOpPade = 12, kOpTaylorNew = 13, kOpTaylorPs = 14, kOpLuFactor = 15, kOpLuApply = 16
};

void require_same_dim(const DenseMatrix& a, const DenseMatrix& b) {
    if (a.dim() != b.dim()) throw std::invalid_argument("dimension mismatch");
}

// one routine on the device: inputs `in` (n x n each), result n x n
DenseMatrix dense(DenseOp op, int arg, std::initializer_list<const DenseMatrix*> in,
                  CostContext* ctx = nullptr, const double* coeffs = nullptr) {
    const int n = (*in.begin())->dim();
    if (n < 1) throw std::invalid_argument("matrix dimension must be positive");
    std::vector<const double*> p;
    for (const DenseMatrix* m : in) p.push_back(m->data());
    DenseMatrix out(n);
    int64_t products = 0, solves = 0;
    const int st = mexp_b200_dense_call(int(op), arg, p.data(), int(p.size()), coeffs, n, out.data(),
                                        nullptr, nullptr, &products, &solves);
    if (st != MEXP_OK) throw_status(st);
    if (ctx) {
        ctx->products += products;
        ctx->solves += solves;
    }
    return out;
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
    // X <- X X, s times on the device in the reference's rounding
    // (expm.cpp:31-35), each recorded as one product
    return dense(kOpSquarings, s, {&x}, &ctx);
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

// ---- dense_matrix.hpp:40-58 value operations (device, reference rounding) --
namespace mexp {

DenseMatrix matmul(const DenseMatrix& a, const DenseMatrix& b) {
    require_same_dim(a, b);
    return dense(kOpMatmul, 0, {&a, &b});
}

DenseMatrix matmul(CostContext& ctx, const DenseMatrix& a, const DenseMatrix& b) {
    ctx.record_product();
    return matmul(a, b);
}

DenseMatrix lincomb(std::span<const double> coeffs, std::span<const DenseMatrix* const> mats) {
    if (coeffs.empty() || coeffs.size() != mats.size())
        throw std::invalid_argument("lincomb needs equally long nonempty lists");
    const int n = mats[0]->dim();
    std::vector<const double*> p;
    for (const DenseMatrix* m : mats) {
        if (m->dim() != n) throw std::invalid_argument("dimension mismatch");
        p.push_back(m->data());
    }
    DenseMatrix out(n);
    const int st = mexp_b200_dense_call(kOpLincomb, 0, p.data(), int(p.size()), coeffs.data(), n,
                                        out.data(), nullptr, nullptr, nullptr, nullptr);
    if (st != MEXP_OK) throw_status(st);
    return out;
}

DenseMatrix lincomb(std::initializer_list<double> coeffs,
                    std::initializer_list<const DenseMatrix*> mats) {
    return lincomb(std::span<const double>(coeffs.begin(), coeffs.size()),
                   std::span<const DenseMatrix* const>(mats.begin(), mats.size()));
}

DenseMatrix add(const DenseMatrix& a, const DenseMatrix& b) { return lincomb({1.0, 1.0}, {&a, &b}); }
DenseMatrix sub(const DenseMatrix& a, const DenseMatrix& b) { return lincomb({1.0, -1.0}, {&a, &b}); }
DenseMatrix scaled(const DenseMatrix& a, double factor) { return lincomb({factor}, {&a}); }

double one_norm(const DenseMatrix& a) {
    const double* p = a.data();
    double v = 0.0;
    const int st = mexp_b200_dense_call(kOpOneNorm, 0, &p, 1, nullptr, a.dim(), &v, nullptr, nullptr,
                                        nullptr, nullptr);
    if (st != MEXP_OK) throw_status(st);
    return v;
}

DenseMatrix lu_solve(const DenseMatrix& m, const DenseMatrix& rhs) {
    require_same_dim(m, rhs);
    return dense(kOpLuSolve, 0, {&m, &rhs});
}

DenseMatrix lu_solve(CostContext& ctx, const DenseMatrix& m, const DenseMatrix& rhs) {
    ctx.record_solve();
    return lu_solve(m, rhs);
}

// ---- taylor_schemes.hpp ----------------------------------------------------
const T8Coefficients& t8_coefficients() {
    using C = mexp_b200::T8C;
    static const T8Coefficients c{C::x1, C::x2, C::x3, C::x4, C::x5, C::x6, C::x7, C::y0, C::y1, C::y2};
    return c;
}

const Psi9Coefficients& psi9_coefficients() {
    static const Psi9Coefficients c = [] {
        double x[9];
        mexp_b200_psi9_coefficients(x);
        return Psi9Coefficients{x[0], x[1], x[2], x[3], x[4], x[5], x[6], x[7], x[8]};
    }();
    return c;
}

const double kT12[4][4] = MEXP_T12_TABLE;
const double kT18A[4] = MEXP_T18A_TABLE;
const double kT18B[4][5] = MEXP_T18B_TABLE;

DenseMatrix taylor_oracle(const DenseMatrix& a, int degree) {
    if (degree < 0) throw std::invalid_argument("degree must be nonnegative");
    return dense(kOpTaylorOracle, degree, {&a});
}

DenseMatrix psi_oracle(const DenseMatrix& a, int k) {
    if (k < 1) throw std::invalid_argument("k must be positive");
    return dense(kOpPsiOracle, k, {&a});
}

DenseMatrix eval_t8(CostContext& ctx, const DenseMatrix& a) { return dense(kOpT8, 0, {&a}, &ctx); }
DenseMatrix eval_t12(CostContext& ctx, const DenseMatrix& a) { return dense(kOpT12, 0, {&a}, &ctx); }
DenseMatrix eval_t18(CostContext& ctx, const DenseMatrix& a) { return dense(kOpT18, 0, {&a}, &ctx); }

DenseMatrix eval_ps(CostContext& ctx, const DenseMatrix& a, int degree) {
    if (degree != 2 && degree != 4 && degree != 6 && degree != 9 && degree != 16)
        throw std::invalid_argument("unsupported Paterson-Stockmeyer degree");
    return dense(kOpPs, degree, {&a}, &ctx);
}

DenseMatrix psi9(CostContext& ctx, const DenseMatrix& a) { return dense(kOpPsi9, 0, {&a}, &ctx); }

DenseMatrix eval_taylor_new(CostContext& ctx, const DenseMatrix& a, int degree) {
    if (degree != 1 && degree != 2 && degree != 4 && degree != 8 && degree != 12 && degree != 18)
        throw std::invalid_argument("unsupported degree for the new decomposition");
    return dense(kOpTaylorNew, degree, {&a}, &ctx);
}

DenseMatrix eval_taylor_ps(CostContext& ctx, const DenseMatrix& a, int degree) {
    if (degree != 1 && degree != 2 && degree != 4 && degree != 6 && degree != 9 && degree != 16)
        throw std::invalid_argument("unsupported Paterson-Stockmeyer degree");
    return dense(kOpTaylorPs, degree, {&a}, &ctx);
}

// ---- pade.hpp -----------------------------------------------------------------
PadeCoefficients pade_coeffs(int m) {
    if (m < 1 || m > 13) throw std::invalid_argument("pade order out of range");
    PadeCoefficients c;
    c.m = m;
    c.b.resize(m + 1);
    mexp_b200_pade_coefficients(m, c.b.data());
    return c;
}

DenseMatrix eval_r10(CostContext& ctx, const DenseMatrix& a) { return dense(kOpPade, 10, {&a}, &ctx); }
DenseMatrix eval_r26(CostContext& ctx, const DenseMatrix& a) { return dense(kOpPade, 26, {&a}, &ctx); }

DenseMatrix eval_pade(CostContext& ctx, const DenseMatrix& a, int order) {
    if (order < 2 || order > 26 || order % 2 != 0)
        throw std::invalid_argument("pade order must be even, 2..26");
    return dense(kOpPade, order, {&a}, &ctx);
}

}  // namespace mexp

// ---- kernels.hpp (host buffers, device arithmetic) ---------------------------
namespace mexp::kernels {

namespace {
void check(int st) {
    if (st != MEXP_OK) throw_status(st);
}
}  // namespace

void matmul(const double* a, const double* b, double* c, int n) {
    const double* in[2] = {a, b};
    check(mexp_b200_dense_call(kOpMatmul, 0, in, 2, nullptr, n, c, nullptr, nullptr, nullptr, nullptr));
}

void lincomb(const double* coeffs, const double* const* mats, int k, double* out, std::int64_t len) {
    if (k < 1 || len < 0) throw std::invalid_argument("lincomb needs equally long nonempty lists");
    if (len == 0) return;
    if (len > INT32_MAX) throw std::invalid_argument("lincomb length out of range");
    // arg 1: `n` is the flat length (the arithmetic is elementwise)
    check(mexp_b200_dense_call(kOpLincomb, 1, mats, k, coeffs, int(len), out, nullptr, nullptr, nullptr,
                               nullptr));
}

void scale(const double* a, double factor, double* out, std::int64_t len) { lincomb(&factor, &a, 1, out, len); }

double one_norm(const double* a, int n) {
    double v = 0.0;
    check(mexp_b200_dense_call(kOpOneNorm, 0, &a, 1, nullptr, n, &v, nullptr, nullptr, nullptr, nullptr));
    return v;
}

LuFactors lu_factor(const double* a, int n) {
    LuFactors f;
    f.n = n;
    f.lu.resize(std::size_t(n) * n);
    std::vector<int32_t> perm(n);
    check(mexp_b200_dense_call(kOpLuFactor, 0, &a, 1, nullptr, n, f.lu.data(), nullptr, perm.data(),
                               nullptr, nullptr));
    f.perm.assign(perm.begin(), perm.end());
    return f;
}

void lu_apply(const LuFactors& f, const double* rhs, double* x, int n) {
    if (f.n != n || f.lu.size() != std::size_t(n) * n || f.perm.size() != std::size_t(n))
        throw std::invalid_argument("dimension mismatch");
    std::vector<int32_t> perm(f.perm.begin(), f.perm.end());
    const double* in[2] = {f.lu.data(), rhs};
    check(mexp_b200_dense_call(kOpLuApply, 0, in, 2, nullptr, n, x, perm.data(), nullptr, nullptr, nullptr));
}

}  // namespace mexp::kernels
