/*
 * TEST INFRASTRUCTURE ONLY — the CPU oracle. Never linked into the product.
 *
 * Plain-C restatement of the reference's scaling-and-squaring expm for
 * Family::TaylorNew (arXiv 1710.10989, reduced-product Taylor schemes) and
 * Family::TaylorPS (Paterson-Stockmeyer Taylor, the paper's baseline) and
 * Family::PadeDiagonal (diagonal Pade r_m with a pivoted LU solve), in the
 * exact arithmetic order of the reference so results are bit-identical to it
 * when compiled with -ffp-contract=off (the reference's own flag,
 * proj/CMakeLists.txt:10-11). Pinned against the compiled reference
 * (oracle/_ref/libmexp_ref.so) and the committed fixtures in tests/golden/.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load this file's library, and only as the checker / CPU baseline.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

enum { ORC_OK = 0, ORC_NONFINITE = 1, ORC_NORM_NONFINITE = 2, ORC_INVALID = 3, ORC_SINGULAR = 7 };

/* ---- theta tables: proj/src/theta_tables.cpp:45-51 (TaylorNew rows) ---- */
static const int kDegrees[6] = {1, 2, 4, 8, 12, 18};
static const int kProducts[6] = {0, 1, 2, 3, 4, 5};
static const double kThetaDouble[6] = {2.22e-16, 2.58e-8, 3.40e-4, 4.99e-2, 2.99e-1, 1.09};
static const double kThetaSingle[6] = {1.19e-7, 5.98e-4, 5.12e-2, 5.80e-1, 1.46, 3.01};
/* TaylorPS rows: theta_tables.cpp:53-59 */
static const int kDegreesPS[6] = {1, 2, 4, 6, 9, 16};
static const int kProductsPS[6] = {0, 1, 2, 3, 4, 6};
static const double kThetaPSDouble[6] = {2.22e-16, 2.58e-8, 3.40e-4, 9.07e-3, 8.96e-2, 7.80e-1};
static const double kThetaPSSingle[6] = {1.19e-7, 5.98e-4, 5.12e-2, 2.50e-1, 7.80e-1, 2.48};
/* PadeDiagonal rows: theta_tables.cpp:61-73 */
static const int kDegreesPade[13] = {2, 4, 6, 8, 10, 12, 14, 16, 18, 20, 22, 24, 26};
static const int kProductsPade[13] = {0, 1, 2, 3, 3, 4, 4, 5, 5, 5, 6, 6, 6};
static const double kThetaPadeDouble[13] = {3.65e-8, 5.32e-4, 1.50e-2, 8.54e-2, 2.54e-1, 5.41e-1,
                                            9.50e-1, 1.47, 2.10, 2.81, 3.60, 4.46, 5.37};
static const double kThetaPadeSingle[13] = {8.46e-4, 8.09e-2, 4.26e-1, 1.05, 1.88, 2.85, 3.93,
                                            5.06, 6.25, 7.47, 8.71, 9.97, 11.2};

/* ---- scheme coefficients: proj/src/taylor_schemes.cpp:12-27,44-48,62-85 ---- */
typedef struct { double x1, x2, x3, x4, x5, x6, x7, y0, y1, y2; } t8c;

/* make_t8: closed forms in sqrt(177), x3 = 2/3, long double rounded once
 * (taylor_schemes.cpp:12-27). */
static t8c make_t8(void) {
    const long double r = sqrtl(177.0L);
    const long double x3 = 2.0L / 3.0L;
    t8c c;
    c.x1 = (double)(x3 * (1.0L + r) / 88.0L);
    c.x2 = (double)(x3 * (1.0L + r) / 352.0L);
    c.x3 = (double)x3;
    c.x4 = (double)((-271.0L + 29.0L * r) / (315.0L * x3));
    c.x5 = (double)(11.0L * (-1.0L + r) / (1260.0L * x3));
    c.x6 = (double)(11.0L * (-9.0L + r) / (5040.0L * x3));
    c.x7 = (double)((89.0L - r) / (5040.0L * x3 * x3));
    c.y0 = 1.0;
    c.y1 = 1.0;
    c.y2 = (double)((857.0L - 58.0L * r) / 630.0L);
    return c;
}

/* Printed coefficients of the 4- and 5-product schemes (paper eqs. for T12 and
 * T18; reference taylor_schemes.cpp:62-85). kT12[i][j] multiplies A^i in B_{j+1}. */
static const double kT12[4][4] = {
    {9.0198e-16, 5.31597895759871264183, 0.18188869982170434744, -2.0861320e-13},
    {0.46932117595418237389, 1.19926790417132231573, 0.05502798439925399070,
     -0.13181061013830184015},
    {-0.20099424927047284052, 0.01179296240992997031, 0.09351590770535414968,
     -0.02027855540589259079},
    {-0.04623946134063071740, 0.01108844528519167989, 0.00610700528898058230,
     -0.00675951846863086359},
};
static const double kT18A[4] = {0.0, -0.100365581030144620, -0.0080292464824115696,
                                -0.0008921384980457299};
static const double kT18B[4][5] = {
    {0.0, 0.39784974949964507614, 1.36783778460411719922, 0.49828962252538267755,
     -0.0006378981945947233},
    {-10.967639605296206259, 1.68015813878906197182, 0.05717798464788655127,
     -0.0069821012248805208, 0.00003349750170860705},
    {-0.0904316832390810561, -0.0676404519071381907, 0.06759613017704596460,
     0.02955525704293155274, -0.0000139180257516060},
    {0.0, 0.0, -0.0923364619367118592, -0.0169364939002081717, -0.0000140086798182036},
};

/* inv_factorial: 1.0 / k! with k! accumulated in double (taylor_schemes.cpp:44-48). */
static double inv_factorial(int i) {
    double f = 1.0;
    for (int k = 2; k <= i; ++k) f *= k;
    return 1.0 / f;
}

/* ---- raw kernels: proj/src/kernels.cpp ---- */

/* one_norm: column j summed rows ascending from 0.0, strict '>' max
 * (kernels.cpp:44-53). */
double oracle_one_norm(const double* a, int n) {
    double best = 0.0;
    for (int j = 0; j < n; ++j) {
        double s = 0.0;
        for (int i = 0; i < n; ++i) s += fabs(a[(size_t)i * n + j]);
        if (s > best) best = s;
    }
    return best;
}

/* matmul: memset then i-k-j accumulation, c_ij += a_ik * b_kj, no FMA
 * (kernels.cpp:16-27). */
void oracle_matmul(const double* a, const double* b, double* c, int n) {
    memset(c, 0, sizeof(double) * (size_t)n * n);
    for (int i = 0; i < n; ++i) {
        double* ci = c + (size_t)i * n;
        for (int k = 0; k < n; ++k) {
            const double aik = a[(size_t)i * n + k];
            const double* bk = b + (size_t)k * n;
            for (int j = 0; j < n; ++j) ci[j] += aik * bk[j];
        }
    }
}

/* lincomb: out = c0*m0, then += ci*mi left to right (kernels.cpp:29-37). */
static void lincomb(const double* coeffs, const double* const* mats, int k, double* out,
                    size_t len) {
    for (size_t e = 0; e < len; ++e) {
        double s = coeffs[0] * mats[0][e];
        for (int i = 1; i < k; ++i) s += coeffs[i] * mats[i][e];
        out[e] = s;
    }
}

/* add(a, b) = lincomb({1, 1}, {a, b}) (dense_matrix.cpp:94-96). */
static void add(const double* a, const double* b, double* out, size_t len) {
    const double c[2] = {1.0, 1.0};
    const double* m[2] = {a, b};
    lincomb(c, m, 2, out, len);
}

/* ---- selection: proj/src/expm.cpp:11-29; family 0 TaylorNew, 1 TaylorPS ---- */
int oracle_select_family(double norm, int accuracy, int family, int32_t* degree, int32_t* s) {
    const int ps = family == 1, pade = family == 2;
    const int ne = pade ? 13 : 6;
    const double* th = pade ? (accuracy == 0 ? kThetaPadeSingle : kThetaPadeDouble)
                     : ps ? (accuracy == 0 ? kThetaPSSingle : kThetaPSDouble)
                          : (accuracy == 0 ? kThetaSingle : kThetaDouble);
    const int* kDeg = pade ? kDegreesPade : ps ? kDegreesPS : kDegrees;
    const int* kProd = pade ? kProductsPade : ps ? kProductsPS : kProducts;
    if (!isfinite(norm) || norm < 0) return ORC_NORM_NONFINITE;
    if (norm <= th[ne - 1]) {
        int best = -1;
        for (int e = 0; e < ne; ++e) {
            if (th[e] < norm) continue; /* expm.cpp:17 */
            if (best < 0 || kProd[e] < kProd[best] ||
                (kProd[e] == kProd[best] && kDeg[e] < kDeg[best]))
                best = e;
        }
        *degree = kDeg[best];
        *s = 0;
        return ORC_OK;
    }
    int k = 0;
    while (ldexp(norm, -k) > th[ne - 1]) ++k; /* expm.cpp:27 */
    *degree = kDeg[ne - 1];
    *s = k;
    return ORC_OK;
}

int oracle_select(double norm, int accuracy, int32_t* degree, int32_t* s) {
    return oracle_select_family(norm, accuracy, 0, degree, s);
}

int oracle_products(int degree) {
    for (int e = 0; e < 6; ++e)
        if (kDegrees[e] == degree) return kProducts[e];
    return -1;
}

/* ---- schemes: proj/src/taylor_schemes.cpp ---- */

/* Scratch layout: the caller passes ws with room for 12 n*n matrices. */
static void eval_t8(const double* a, int n, double* out, double* ws) {
    static int init = 0;
    static t8c c;
    if (!init) { c = make_t8(); init = 1; }
    const size_t nn = (size_t)n * n;
    double* id = ws; double* a2 = ws + nn; double* a4 = ws + 2 * nn;
    double* t1 = ws + 3 * nn; double* t2 = ws + 4 * nn; double* a8 = ws + 5 * nn;
    memset(id, 0, sizeof(double) * nn);
    for (int i = 0; i < n; ++i) id[(size_t)i * n + i] = 1.0;
    oracle_matmul(a, a, a2, n);
    { const double k[2] = {c.x1, c.x2}; const double* m[2] = {a, a2}; lincomb(k, m, 2, t1, nn); }
    oracle_matmul(a2, t1, a4, n);
    { const double k[2] = {c.x3, 1.0}; const double* m[2] = {a2, a4}; lincomb(k, m, 2, t1, nn); }
    { const double k[4] = {c.x4, c.x5, c.x6, c.x7}; const double* m[4] = {id, a, a2, a4};
      lincomb(k, m, 4, t2, nn); }
    oracle_matmul(t1, t2, a8, n);
    { const double k[4] = {c.y0, c.y1, c.y2, 1.0}; const double* m[4] = {id, a, a2, a8};
      lincomb(k, m, 4, out, nn); } /* taylor_schemes.cpp:104-113 */
}

static void eval_t12(const double* a, int n, double* out, double* ws) {
    const size_t nn = (size_t)n * n;
    double* id = ws; double* a2 = ws + nn; double* a3 = ws + 2 * nn;
    double* b[4] = {ws + 3 * nn, ws + 4 * nn, ws + 5 * nn, ws + 6 * nn};
    double* p = ws + 7 * nn; double* a6 = ws + 8 * nn; double* t = ws + 9 * nn;
    memset(id, 0, sizeof(double) * nn);
    for (int i = 0; i < n; ++i) id[(size_t)i * n + i] = 1.0;
    oracle_matmul(a, a, a2, n);
    oracle_matmul(a2, a, a3, n);
    for (int j = 0; j < 4; ++j) {
        const double k[4] = {kT12[0][j], kT12[1][j], kT12[2][j], kT12[3][j]};
        const double* m[4] = {id, a, a2, a3};
        lincomb(k, m, 4, b[j], nn);
    }
    oracle_matmul(b[3], b[3], p, n);
    add(b[2], p, a6, nn);
    add(b[1], a6, t, nn);
    oracle_matmul(t, a6, p, n);
    add(b[0], p, out, nn); /* taylor_schemes.cpp:115-125 */
}

static void eval_t18(const double* a, int n, double* out, double* ws) {
    const size_t nn = (size_t)n * n;
    double* id = ws; double* a2 = ws + nn; double* a3 = ws + 2 * nn; double* a6 = ws + 3 * nn;
    double* b1 = ws + 4 * nn;
    double* b[4] = {ws + 5 * nn, ws + 6 * nn, ws + 7 * nn, ws + 8 * nn};
    double* p = ws + 9 * nn; double* a9 = ws + 10 * nn; double* t = ws + 11 * nn;
    memset(id, 0, sizeof(double) * nn);
    for (int i = 0; i < n; ++i) id[(size_t)i * n + i] = 1.0;
    oracle_matmul(a, a, a2, n);
    oracle_matmul(a2, a, a3, n);
    oracle_matmul(a3, a3, a6, n);
    { const double* m[4] = {id, a, a2, a3}; lincomb(kT18A, m, 4, b1, nn); }
    for (int j = 0; j < 4; ++j) {
        const double* m[5] = {id, a, a2, a3, a6};
        lincomb(kT18B[j], m, 5, b[j], nn);
    }
    oracle_matmul(b1, b[3], p, n);
    add(p, b[2], a9, nn);
    add(b[1], a9, t, nn);
    oracle_matmul(t, a9, p, n);
    add(b[0], p, out, nn); /* taylor_schemes.cpp:127-141 */
}

/* Paterson-Stockmeyer with p = 3 (degrees 6, 9) or 4 (16): chunks
 * g_i = sum_{k<p} A^k / (p i + k)!, t = g_{q-1} + A^p / m!, then
 * t = g_i + t A^p down to i = 0 (taylor_schemes.cpp:159-191). */
static void eval_ps_horner(const double* a, int n, int degree, double* out, double* ws) {
    const size_t nn = (size_t)n * n;
    const int p = degree == 16 ? 4 : 3, q = degree / p;
    double* id = ws; double* a2 = ws + nn; double* a3 = ws + 2 * nn; double* a4 = ws + 3 * nn;
    double* g[4] = {ws + 4 * nn, ws + 5 * nn, ws + 6 * nn, ws + 7 * nn};
    double* t = ws + 8 * nn; double* prod = ws + 9 * nn; double* t2 = ws + 10 * nn;
    memset(id, 0, sizeof(double) * nn);
    for (int i = 0; i < n; ++i) id[(size_t)i * n + i] = 1.0;
    oracle_matmul(a, a, a2, n);
    oracle_matmul(a2, a, a3, n);
    if (p == 4) oracle_matmul(a2, a2, a4, n);
    const double* pw[4] = {id, a, a2, a3};
    for (int i = 0; i < q; ++i) {
        double k[4];
        for (int j = 0; j < p; ++j) k[j] = inv_factorial(p * i + j);
        lincomb(k, pw, p, g[i], nn);
    }
    const double* ap = p == 4 ? a4 : a3;
    { const double k[2] = {1.0, inv_factorial(degree)}; const double* m[2] = {g[q - 1], ap};
      lincomb(k, m, 2, t, nn); }
    for (int i = q - 2; i >= 0; --i) {
        oracle_matmul(t, ap, prod, n);
        add(g[i], prod, i == 0 ? out : t2, nn);
        memcpy(t, t2, sizeof(double) * nn);
    }
}

/* eval_ps degrees 2 and 4 (taylor_schemes.cpp:146-157), 6, 9, 16 (:159-191). */
static void eval_ps(const double* a, int n, int degree, double* out, double* ws) {
    const size_t nn = (size_t)n * n;
    if (degree == 6 || degree == 9 || degree == 16) {
        eval_ps_horner(a, n, degree, out, ws);
        return;
    }
    double* id = ws; double* a2 = ws + nn; double* f0 = ws + 2 * nn; double* f1 = ws + 3 * nn;
    double* inner = ws + 4 * nn; double* p = ws + 5 * nn;
    memset(id, 0, sizeof(double) * nn);
    for (int i = 0; i < n; ++i) id[(size_t)i * n + i] = 1.0;
    oracle_matmul(a, a, a2, n);
    if (degree == 2) {
        const double k[3] = {1.0, 1.0, 0.5};
        const double* m[3] = {id, a, a2};
        lincomb(k, m, 3, out, nn);
        return;
    }
    { const double k[2] = {1.0, 1.0}; const double* m[2] = {id, a}; lincomb(k, m, 2, f0, nn); }
    { const double k[2] = {inv_factorial(2), inv_factorial(3)}; const double* m[2] = {id, a};
      lincomb(k, m, 2, f1, nn); }
    { const double k[2] = {1.0, inv_factorial(4)}; const double* m[2] = {f1, a2};
      lincomb(k, m, 2, inner, nn); }
    oracle_matmul(inner, a2, p, n);
    add(f0, p, out, nn);
}

/* eval_taylor_new degree dispatch (taylor_schemes.cpp:211-227). Returns the
 * number of products, or -1 for an unsupported degree. */
int oracle_eval_taylor_new(const double* a, int n, int degree, double* out) {
    const size_t nn = (size_t)n * n;
    double* ws = (double*)malloc(sizeof(double) * nn * 12);
    int products = -1;
    switch (degree) {
        case 1: {
            memset(ws, 0, sizeof(double) * nn);
            for (int i = 0; i < n; ++i) ws[(size_t)i * n + i] = 1.0;
            add(ws, a, out, nn);
            products = 0;
            break;
        }
        case 2: eval_ps(a, n, 2, out, ws); products = 1; break;
        case 4: eval_ps(a, n, 4, out, ws); products = 2; break;
        case 8: eval_t8(a, n, out, ws); products = 3; break;
        case 12: eval_t12(a, n, out, ws); products = 4; break;
        case 18: eval_t18(a, n, out, ws); products = 5; break;
        default: break;
    }
    free(ws);
    return products;
}

/* eval_taylor_ps (taylor_schemes.cpp:229-232): I + A, or eval_ps. */
int oracle_eval_taylor_ps(const double* a, int n, int degree, double* out) {
    const size_t nn = (size_t)n * n;
    int products = -1;
    for (int e = 0; e < 6; ++e)
        if (kDegreesPS[e] == degree) products = kProductsPS[e];
    if (products < 0) return -1;
    if (degree == 1 || degree == 2 || degree == 4) return oracle_eval_taylor_new(a, n, degree, out);
    double* ws = (double*)malloc(sizeof(double) * nn * 12);
    eval_ps(a, n, degree, out, ws);
    free(ws);
    return products;
}

/* ---- Family::PadeDiagonal: proj/src/pade.cpp, kernels.cpp:55-112 ---- */

/* pade_coeffs (pade.cpp:34-48): b_j = (2m-j)! m! / ((2m)! (m-j)! j!) as an
 * exact __int128 ratio reduced by its gcd, then long double division rounded
 * to double. */
static __int128 fact128(int n) {
    __int128 f = 1;
    for (int k = 2; k <= n; ++k) f *= k;
    return f;
}
static __int128 gcd128(__int128 a, __int128 b) {
    while (b != 0) {
        const __int128 t = a % b;
        a = b;
        b = t;
    }
    return a < 0 ? -a : a;
}
int oracle_pade_coeffs(int m, double* b) {
    if (m < 1 || m > 13) return -1;
    for (int j = 0; j <= m; ++j) {
        __int128 num = fact128(2 * m - j) * fact128(m);
        __int128 den = fact128(2 * m) * fact128(m - j) * fact128(j);
        const __int128 g = gcd128(num, den);
        num /= g;
        den /= g;
        b[j] = (double)((long double)num / (long double)den);
    }
    return m + 1;
}

/* lu_factor + lu_apply (kernels.cpp:55-112): partial pivoting with a strict
 * '>' scan, multipliers l = row[k] / piv, row[j] -= l * prow[j]; solve each
 * column of rhs gathered through perm. Returns 0, or -1 on a zero pivot. */
static int lu_solve(const double* m, const double* rhs, double* x, int n) {
    const size_t nn = (size_t)n * n;
    double* lu = (double*)malloc(sizeof(double) * nn);
    int* perm = (int*)malloc(sizeof(int) * n);
    double* y = (double*)malloc(sizeof(double) * n);
    memcpy(lu, m, sizeof(double) * nn);
    for (int i = 0; i < n; ++i) perm[i] = i;
    int st = 0;
    for (int k = 0; k < n && st == 0; ++k) {
        int p = k;
        double best = fabs(lu[(size_t)k * n + k]);
        for (int i = k + 1; i < n; ++i) {
            const double v = fabs(lu[(size_t)i * n + k]);
            if (v > best) { best = v; p = i; }
        }
        if (best == 0.0) { st = -1; break; }
        if (p != k) {
            for (int j = 0; j < n; ++j) {
                const double t = lu[(size_t)k * n + j];
                lu[(size_t)k * n + j] = lu[(size_t)p * n + j];
                lu[(size_t)p * n + j] = t;
            }
            const int t = perm[k]; perm[k] = perm[p]; perm[p] = t;
        }
        const double piv = lu[(size_t)k * n + k];
        for (int i = k + 1; i < n; ++i) {
            double* row = lu + (size_t)i * n;
            const double* prow = lu + (size_t)k * n;
            const double l = row[k] / piv;
            row[k] = l;
            for (int j = k + 1; j < n; ++j) row[j] -= l * prow[j];
        }
    }
    if (st == 0) {
        for (int col = 0; col < n; ++col) {
            for (int i = 0; i < n; ++i) y[i] = rhs[(size_t)perm[i] * n + col];
            for (int i = 1; i < n; ++i) {
                double s = y[i];
                const double* row = lu + (size_t)i * n;
                for (int j = 0; j < i; ++j) s -= row[j] * y[j];
                y[i] = s;
            }
            for (int i = n - 1; i >= 0; --i) {
                double s = y[i];
                const double* row = lu + (size_t)i * n;
                for (int j = i + 1; j < n; ++j) s -= row[j] * y[j];
                y[i] = s / row[i];
            }
            for (int i = 0; i < n; ++i) x[(size_t)i * n + col] = y[i];
        }
    }
    free(lu); free(perm); free(y);
    return st;
}

/* pade_solve (pade.cpp:26-28): (V - U)^-1 (V + U). */
static int pade_solve(const double* u, const double* v, double* out, int n) {
    const size_t nn = (size_t)n * n;
    double* p = (double*)malloc(sizeof(double) * nn);
    double* q = (double*)malloc(sizeof(double) * nn);
    { const double k[2] = {1.0, -1.0}; const double* mm[2] = {v, u}; lincomb(k, mm, 2, p, nn); }
    add(v, u, q, nn);
    const int st = lu_solve(p, q, out, n);
    free(p); free(q);
    return st;
}

/* eval_pade (pade.cpp:50-113). Returns the product count, -1 for an invalid
 * order, -2 for a singular denominator. */
int oracle_eval_pade(const double* a, int n, int order, double* out) {
    if (order < 2 || order > 26 || order % 2 != 0) return -1;
    const size_t nn = (size_t)n * n;
    const int m = order / 2;
    double b[14];
    oracle_pade_coeffs(m, b);
    double* ws = (double*)malloc(sizeof(double) * nn * 20);
    double* id = ws; double* u = ws + nn; double* v = ws + 2 * nn; double* t = ws + 3 * nn;
    double* t2 = ws + 4 * nn;
    double* pw = ws + 5 * nn; /* pw + i*nn = A^(2(i+1)), i < 6 */
    memset(id, 0, sizeof(double) * nn);
    for (int i = 0; i < n; ++i) id[(size_t)i * n + i] = 1.0;
    int products = 0;
    if (order == 10) { /* eval_r10 */
        double* a2 = pw; double* a4 = pw + nn;
        oracle_matmul(a, a, a2, n);
        oracle_matmul(a2, a2, a4, n);
        { const double k[3] = {b[5], b[3], b[1]}; const double* mm[3] = {a4, a2, id};
          lincomb(k, mm, 3, t, nn); }
        oracle_matmul(a, t, u, n);
        { const double k[3] = {b[4], b[2], b[0]}; const double* mm[3] = {a4, a2, id};
          lincomb(k, mm, 3, v, nn); }
        products = 3;
    } else if (order == 26) { /* eval_r26 */
        double* a2 = pw; double* a4 = pw + nn; double* a6 = pw + 2 * nn;
        oracle_matmul(a, a, a2, n);
        oracle_matmul(a2, a2, a4, n);
        oracle_matmul(a2, a4, a6, n);
        { const double k[3] = {b[13], b[11], b[9]}; const double* mm[3] = {a6, a4, a2};
          lincomb(k, mm, 3, t, nn); }
        oracle_matmul(a6, t, t2, n);
        { const double k[5] = {1.0, b[7], b[5], b[3], b[1]}; const double* mm[5] = {t2, a6, a4, a2, id};
          lincomb(k, mm, 5, t, nn); }
        oracle_matmul(a, t, u, n);
        { const double k[3] = {b[12], b[10], b[8]}; const double* mm[3] = {a6, a4, a2};
          lincomb(k, mm, 3, t, nn); }
        oracle_matmul(a6, t, t2, n);
        { const double k[5] = {1.0, b[6], b[4], b[2], b[0]}; const double* mm[5] = {t2, a6, a4, a2, id};
          lincomb(k, mm, 5, v, nn); }
        products = 6;
    } else { /* even-power chain */
        const int top = m - (m % 2);
        int np = 0;
        if (top >= 2) {
            oracle_matmul(a, a, pw, n);
            np = 1;
            products = 1;
            for (int e = 4; e <= top; e += 2) {
                oracle_matmul(pw, pw + (size_t)(np - 1) * nn, pw + (size_t)np * nn, n);
                ++np;
                ++products;
            }
        }
        double codd[8], ceven[8];
        const double* modd[8];
        const double* meven[8];
        int ko = 0, ke = 0;
        codd[ko] = b[1]; modd[ko++] = id;
        ceven[ke] = b[0]; meven[ke++] = id;
        for (int j = 3; j <= m; j += 2) { codd[ko] = b[j]; modd[ko++] = pw + (size_t)((j - 1) / 2 - 1) * nn; }
        for (int j = 2; j <= m; j += 2) { ceven[ke] = b[j]; meven[ke++] = pw + (size_t)(j / 2 - 1) * nn; }
        if (m >= 3) {
            lincomb(codd, modd, ko, t, nn);
            oracle_matmul(a, t, u, n);
            ++products;
        } else {
            for (size_t e = 0; e < nn; ++e) u[e] = b[1] * a[e]; /* scaled(a, b1) */
        }
        lincomb(ceven, meven, ke, v, nn);
    }
    const int st = pade_solve(u, v, out, n);
    free(ws);
    return st < 0 ? -2 : products;
}

/* expm driver (proj/src/expm.cpp:37-74): finite check, norm, select, exact
 * scaling by 2^-s, T_m, s squarings, report. */
int oracle_expm_family(const double* a, int n, int accuracy, int family, double* out,
                       int32_t* degree, int32_t* s, int64_t* cost_thirds, double* norm_in) {
    const size_t nn = (size_t)n * n;
    for (size_t e = 0; e < nn; ++e)
        if (!isfinite(a[e])) return ORC_NONFINITE; /* expm.cpp:38 */
    const double norm = oracle_one_norm(a, n);
    int32_t m = 0, k = 0;
    const int st = oracle_select_family(norm, accuracy, family, &m, &k);
    if (st != ORC_OK) return st;
    double* arg = (double*)malloc(sizeof(double) * nn);
    double* tmp = (double*)malloc(sizeof(double) * nn);
    if (k == 0) {
        memcpy(arg, a, sizeof(double) * nn);
    } else {
        const double f = ldexp(1.0, -k); /* scale: kernels.cpp:39-42 */
        for (size_t e = 0; e < nn; ++e) arg[e] = f * a[e];
    }
    const int products = family == 2 ? oracle_eval_pade(arg, n, m, out)
                       : family == 1 ? oracle_eval_taylor_ps(arg, n, m, out)
                                     : oracle_eval_taylor_new(arg, n, m, out);
    if (products == -2) { /* "singular denominator" (kernels.cpp:72) */
        free(arg);
        free(tmp);
        return ORC_SINGULAR;
    }
    for (int i = 0; i < k; ++i) { /* squarings: expm.cpp:31-35 */
        oracle_matmul(out, out, tmp, n);
        memcpy(out, tmp, sizeof(double) * nn);
    }
    free(arg);
    free(tmp);
    if (degree) *degree = m;
    if (s) *s = k;
    /* table products, + 4/3 for the Pade solve (expm.cpp:70-72) */
    if (cost_thirds) {
        int tp = products;
        if (family == 2)
            for (int e = 0; e < 13; ++e)
                if (kDegreesPade[e] == m) tp = kProductsPade[e];
        *cost_thirds = 3 * (int64_t)(tp + k) + (family == 2 ? 4 : 0);
    }
    if (norm_in) *norm_in = norm;
    return ORC_OK;
}

int oracle_expm(const double* a, int n, int accuracy, double* out, int32_t* degree,
                int32_t* s, int64_t* cost_thirds, double* norm_in) {
    return oracle_expm_family(a, n, accuracy, 0, out, degree, s, cost_thirds, norm_in);
}

/* T_m(2^-s A) squared s times with a GIVEN (m, s) instead of the selected
 * one (scale, eval_taylor_new, squarings: expm.cpp:47-61). Used to check a
 * leading block of a block-triangular matrix, whose (m, s) come from the
 * norm of the full matrix. Returns the product count or -1. */
int oracle_expm_forced(const double* a, int n, int degree, int s, double* out) {
    const size_t nn = (size_t)n * n;
    double* arg = (double*)malloc(sizeof(double) * nn);
    double* tmp = (double*)malloc(sizeof(double) * nn);
    if (s == 0) {
        memcpy(arg, a, sizeof(double) * nn);
    } else {
        const double f = ldexp(1.0, -s);
        for (size_t e = 0; e < nn; ++e) arg[e] = f * a[e];
    }
    const int products = oracle_eval_taylor_new(arg, n, degree, out);
    for (int i = 0; i < s; ++i) {
        oracle_matmul(out, out, tmp, n);
        memcpy(out, tmp, sizeof(double) * nn);
    }
    free(arg);
    free(tmp);
    return products < 0 ? -1 : products + s;
}

/* Batched driver over contiguous row-major matrices; per-matrix status. */
int oracle_expm_batch_family(const double* a, double* out, int n, int64_t batch, int accuracy,
                             int family, int32_t* degree, int32_t* s, int64_t* cost_thirds,
                             double* norm_in, int32_t* status) {
    const size_t nn = (size_t)n * n;
    int worst = ORC_OK;
    for (int64_t b = 0; b < batch; ++b) {
        const int st = oracle_expm_family(a + b * nn, n, accuracy, family, out + b * nn,
                                   degree ? degree + b : NULL, s ? s + b : NULL,
                                   cost_thirds ? cost_thirds + b : NULL,
                                   norm_in ? norm_in + b : NULL);
        if (st != ORC_OK) {
            for (size_t e = 0; e < nn; ++e) out[b * nn + e] = NAN;
            if (degree) degree[b] = 0;
            if (s) s[b] = 0;
            if (cost_thirds) cost_thirds[b] = 0;
            if (norm_in) norm_in[b] = NAN;
            if (worst == ORC_OK) worst = st;
        }
        if (status) status[b] = st;
    }
    return worst;
}

int oracle_expm_batch(const double* a, double* out, int n, int64_t batch, int accuracy,
                      int32_t* degree, int32_t* s, int64_t* cost_thirds, double* norm_in,
                      int32_t* status) {
    return oracle_expm_batch_family(a, out, n, batch, accuracy, 0, degree, s, cost_thirds,
                                    norm_in, status);
}

/* Coefficients as the oracle holds them (same order as ref_coefficients). */
void oracle_coefficients(double* t8, double* t12, double* t18a, double* t18b) {
    const t8c c = make_t8();
    const double v[10] = {c.x1, c.x2, c.x3, c.x4, c.x5, c.x6, c.x7, c.y0, c.y1, c.y2};
    memcpy(t8, v, sizeof v);
    memcpy(t12, kT12, sizeof kT12);
    memcpy(t18a, kT18A, sizeof kT18A);
    memcpy(t18b, kT18B, sizeof kT18B);
}
