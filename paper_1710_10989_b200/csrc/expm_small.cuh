// Batched small-n expm, fp64 (n in {8, 16, 32, 64}): one group of W warps per
// matrix, the whole expm (finite check, exact 1-norm, (m,s) selection, exact
// 2^-s scaling, T_m, s squarings) inside the group with the matrix held as
// register fragments and staged through shared memory only to re-lay out the
// operands of each product.
//
// Fragment layout: the n x n matrix is cut into 8x8 tiles; each warp owns a
// TR x TC block of tiles and, per tile, lane l holds the two elements
// (8*ti + (l>>2), 8*tj + 2*(l&3) + {0,1}) -- the accumulator layout of the
// FP64 tensor-core MMA m8n8k4 (DMMA). Elementwise work (the schemes' linear
// combinations with the identity, reference kernels.cpp:29-37) runs directly
// on fragments; a product C = X*Y (kernels.cpp:16-27) stores X and Y to
// padded shared memory and reads them back either as DMMA operands (FastOps)
// or as rows/columns for a k-ascending DMUL+DADD dot product (ExactOps,
// bit-identical to the reference's no-FMA i-k-j loop).
#pragma once

#include <type_traits>

#include "expm_common.cuh"

namespace mexp_b200 {

template <int N>
struct TileShape;  // tiles per warp block for the W warps of a group
template <> struct TileShape<8>  { static constexpr int W = 1, TR = 1, TC = 1, STASH = 0, MIN_BLOCKS = 4; };
template <> struct TileShape<16> { static constexpr int W = 2, TR = 1, TC = 2, STASH = 0, MIN_BLOCKS = 2; };
template <> struct TileShape<32> { static constexpr int W = 4, TR = 2, TC = 2, STASH = 0, MIN_BLOCKS = 1; };
template <> struct TileShape<64> { static constexpr int W = 8, TR = 2, TC = 4, STASH = 4, MIN_BLOCKS = 1; };

template <int N>
struct Group {
    using S = TileShape<N>;
    static constexpr int W = S::W;
    static constexpr int TR = S::TR;
    static constexpr int TC = S::TC;
    static constexpr int T = TR * TC;        // tiles per warp
    static constexpr int K = 2 * T;          // doubles per lane per matrix
    static constexpr int LD = N + 4;         // padded stride, LD = 4 (mod 16) doubles
    static constexpr int BLK_R = N / 8 / TR; // warp blocks per tile-row direction
    static_assert((N / 8) * (N / 8) == W * T, "tile cover");
    static constexpr int THREADS = 32 * W;
    static constexpr int NDIM = N;
    // shared memory per group, in doubles: two operand buffers + stash + scalars
    static constexpr int STASH_SLOT = K * THREADS;
    static constexpr int SMEM_DOUBLES = 2 * N * LD + S::STASH * STASH_SLOT + 2 * W + 2;

    struct Frag {
        using T = double;
        static constexpr int kCount = K;
        double v[K];
    };

    double* sx;
    double* sy;
    double* stash;
    double* scal;  // [0..W) per-warp partial max, [W] norm broadcast
    int lane, warp, tid, bar_id;

    __device__ __forceinline__ int row_of(int t) const {
        const int bi = warp % BLK_R;
        return 8 * (bi * TR + t / TC) + (lane >> 2);
    }
    __device__ __forceinline__ int col_of(int t) const {
        const int bj = warp / BLK_R;
        return 8 * (bj * TC + t % TC) + 2 * (lane & 3);
    }

    __device__ __forceinline__ void sync() const {
        if constexpr (W == 1) {
            __syncwarp();
        } else {
            asm volatile("bar.sync %0, %1;" ::"r"(bar_id), "n"(THREADS) : "memory");
        }
    }

    __device__ __forceinline__ Frag ident() const {
        Frag f;
#pragma unroll
        for (int t = 0; t < T; ++t) {
            const int r = row_of(t), c = col_of(t);
            f.v[2 * t] = (r == c) ? 1.0 : 0.0;
            f.v[2 * t + 1] = (r == c + 1) ? 1.0 : 0.0;
        }
        return f;
    }

    __device__ __forceinline__ Frag load_global(const double* m) const {
        Frag f;
#pragma unroll
        for (int t = 0; t < T; ++t) {
            const double2 v = ld_stream(reinterpret_cast<const double2*>(m + row_of(t) * N + col_of(t)));
            f.v[2 * t] = v.x;
            f.v[2 * t + 1] = v.y;
        }
        return f;
    }
    __device__ __forceinline__ void store_global(double* m, const Frag& f) const {
#pragma unroll
        for (int t = 0; t < T; ++t)
            st_stream(reinterpret_cast<double2*>(m + row_of(t) * N + col_of(t)),
                      make_double2(f.v[2 * t], f.v[2 * t + 1]));
    }
    __device__ __forceinline__ void store_smem(double* s, const Frag& f) const {
#pragma unroll
        for (int t = 0; t < T; ++t)
            *reinterpret_cast<double2*>(s + row_of(t) * LD + col_of(t)) =
                make_double2(f.v[2 * t], f.v[2 * t + 1]);
    }
    __device__ __forceinline__ Frag load_smem(const double* s) const {
        Frag f;
#pragma unroll
        for (int t = 0; t < T; ++t) {
            const double2 v = *reinterpret_cast<const double2*>(s + row_of(t) * LD + col_of(t));
            f.v[2 * t] = v.x;
            f.v[2 * t + 1] = v.y;
        }
        return f;
    }
    // Pade solve staging (pade_solve, pade.cpp:26-28): M = V - U -> sx,
    // R = V + U -> sy (row-major, stride LD)
    __device__ __forceinline__ double* lu_m() const { return sx; }
    __device__ __forceinline__ double* lu_r() const { return sy; }
    __device__ __forceinline__ int* lu_flag() const { return reinterpret_cast<int*>(scal + 2 * W); }
    __device__ __forceinline__ void stage_solve(const Frag& M, const Frag& R) const {
        sync();
        store_smem(sx, M);
        store_smem(sy, R);
        sync();
    }
    __device__ __forceinline__ Frag solved() const {
        sync();
        return load_smem(sy);
    }

    // Stash a fragment in a thread-private slot (conflict-free, same layout back).
    __device__ __forceinline__ void put(int slot, const Frag& f) const {
        double2* p = reinterpret_cast<double2*>(stash + slot * STASH_SLOT);
#pragma unroll
        for (int t = 0; t < T; ++t) p[t * THREADS + tid] = make_double2(f.v[2 * t], f.v[2 * t + 1]);
    }
    __device__ __forceinline__ Frag get(int slot) const {
        const double2* p = reinterpret_cast<const double2*>(stash + slot * STASH_SLOT);
        Frag f;
#pragma unroll
        for (int t = 0; t < T; ++t) {
            const double2 v = p[t * THREADS + tid];
            f.v[2 * t] = v.x;
            f.v[2 * t + 1] = v.y;
        }
        return f;
    }

    // C = X * Y (same = X and Y are the same matrix: squarings, A*A).
    template <class Ops>
    __device__ __forceinline__ Frag mm(const Frag& X, const Frag& Y, bool same) const {
        return mm_impl<Ops>(X, Y, same, nullptr);
    }
    template <class Ops>
    __device__ __forceinline__ Frag sq_first(const Frag& A) const {
        return mm_impl<Ops>(A, A, true, nullptr);
    }
    // C = X * Y + B (add(matmul(X, Y), B), dense_matrix.cpp:94-96). The fast
    // path seeds the DMMA accumulators with B; the exact path adds after the
    // product, in the reference's order.
    template <class Ops>
    __device__ __forceinline__ Frag mm_add(const Frag& X, const Frag& Y, bool same,
                                           const Frag& B) const {
        if constexpr (Ops::kExact) {
            Frag P = mm_impl<Ops>(X, Y, same, nullptr);
#pragma unroll
            for (int e = 0; e < K; ++e) P.v[e] = Ops::add(P.v[e], B.v[e]);
            return P;
        } else {
            return mm_impl<Ops>(X, Y, same, &B);
        }
    }

    template <class Ops>
    __device__ __forceinline__ Frag mm_impl(const Frag& X, const Frag& Y, bool same,
                                            const Frag* init) const {
        sync();  // previous product's readers are done with sx/sy
        store_smem(sx, X);
        if (!same) store_smem(sy, Y);
        sync();
        const double* py = same ? sx : sy;
        Frag C;
        if constexpr (Ops::kExact) {
            // c_ij = 0.0 + x_i0*y_0j + x_i1*y_1j + ... (k ascending, each
            // multiply and add rounded): reference kernels.cpp:16-27.
#pragma unroll
            for (int t = 0; t < T; ++t) {
                const int r = row_of(t), c = col_of(t);
                double c0 = 0.0, c1 = 0.0;
#pragma unroll 4
                for (int k = 0; k < N; k += 2) {
                    const double2 xa = *reinterpret_cast<const double2*>(sx + r * LD + k);
                    const double2 y0 = *reinterpret_cast<const double2*>(py + k * LD + c);
                    const double2 y1 = *reinterpret_cast<const double2*>(py + (k + 1) * LD + c);
                    c0 = ExactOps::mac(c0, xa.x, y0.x);
                    c1 = ExactOps::mac(c1, xa.x, y0.y);
                    c0 = ExactOps::mac(c0, xa.y, y1.x);
                    c1 = ExactOps::mac(c1, xa.y, y1.y);
                }
                C.v[2 * t] = c0;
                C.v[2 * t + 1] = c1;
            }
        } else {
#pragma unroll
            for (int t = 0; t < K; ++t) C.v[t] = init ? init->v[t] : 0.0;
            const int bi = warp % BLK_R, bj = warp / BLK_R;
            const int ar = lane >> 2, aq = lane & 3;
#pragma unroll 2
            for (int k = 0; k < N; k += 4) {
                double af[TR], bf[TC];
#pragma unroll
                for (int i = 0; i < TR; ++i) af[i] = sx[(8 * (bi * TR + i) + ar) * LD + k + aq];
#pragma unroll
                for (int j = 0; j < TC; ++j) bf[j] = py[(k + aq) * LD + 8 * (bj * TC + j) + ar];
#pragma unroll
                for (int i = 0; i < TR; ++i)
#pragma unroll
                    for (int j = 0; j < TC; ++j)
                        dmma_8x8x4(C.v[2 * (i * TC + j)], C.v[2 * (i * TC + j) + 1], af[i], bf[j]);
            }
        }
        return C;
    }
};

// ---- elementwise linear combinations (reference lincomb, kernels.cpp:29-37):
// out = c0*m0, then out += ci*mi left to right. With ExactOps every term is
// evaluated literally (the identity enters as a full matrix, c*0.0 included,
// as in the reference). The fast path skips zero coefficients and starts an
// identity term (ID0) from its diagonal value instead of multiplying.
__device__ __forceinline__ bool nonzero_bits(double x) { return __double_as_longlong(x) != 0; }
__device__ __forceinline__ bool nonzero_bits(float x) { return __float_as_int(x) != 0; }
// c where the identity entry id is 1, 0 where it is +0 (per component)
__device__ __forceinline__ double id_term(double id, double c) { return nonzero_bits(id) ? c : 0.0; }
__device__ __forceinline__ float id_term(float id, double c) { return nonzero_bits(id) ? float(c) : 0.f; }
__device__ __forceinline__ float2 id_term(float2 id, double c) {
    return make_float2(nonzero_bits(id.x) ? float(c) : 0.f, nonzero_bits(id.y) ? float(c) : 0.f);
}

template <class Ops, class F>
__device__ __forceinline__ void lc_rest(F&, int) {}
template <class Ops, class F, class... R>
__device__ __forceinline__ void lc_rest(F& r, int e, double c, const F& m, R... rest) {
    if (Ops::kExact || c != 0.0) r.v[e] = Ops::mac(r.v[e], c, m.v[e]);
    lc_rest<Ops>(r, e, rest...);
}
template <class Ops, bool ID0 = false, class F, class... R>
__device__ __forceinline__ F lc(double c0, const F& m0, R... rest) {
    using T = typename F::T;
    F r;
#pragma unroll
    for (int e = 0; e < F::kCount; ++e) {
        if constexpr (!Ops::kExact && ID0)  // identity entry is 1.0 or +0.0: test the
            r.v[e] = id_term(m0.v[e], c0);  // bits on the ALU, not the FP64 pipe
        else if (!Ops::kExact && c0 == 0.0)
            r.v[e] = id_term(T{}, 0.0);
        else
            r.v[e] = Ops::mul(c0, m0.v[e]);
        lc_rest<Ops>(r, e, rest...);
    }
    return r;
}
// add(a, b) = lincomb({1, 1}, {a, b}) (dense_matrix.cpp:94-96); 1.0*x is exact.
template <class Ops, class F>
__device__ __forceinline__ F addm(const F& a, const F& b) {
    F r;
#pragma unroll
    for (int e = 0; e < F::kCount; ++e) r.v[e] = Ops::add(a.v[e], b.v[e]);
    return r;
}

// A3 = A2 * A. Groups that keep the scaled A's product operand from sq_first
// in registers (kKeepsAT: the 8x8 warp group) skip restaging A.
template <class G, class = void>
struct keeps_at : std::false_type {};
template <class G>
struct keeps_at<G, std::void_t<decltype(G::kKeepsAT)>> : std::bool_constant<G::kKeepsAT> {};
template <class Ops, class G>
__device__ __forceinline__ typename G::Frag mm_by_a(const G& g, const typename G::Frag& X,
                                                    const typename G::Frag& A) {
    if constexpr (keeps_at<G>::value)
        return g.template mm_a<Ops>(X, A);
    else
        return g.template mm<Ops>(X, A, false);
}

// ---- the schemes (reference taylor_schemes.cpp:104-157, 211-227) -----------
template <class Ops, class G>
__device__ typename G::Frag eval_taylor_new(const G& g, int degree, const typename G::Frag& A) {
    using F = typename G::Frag;
    const F I = g.ident();
    switch (degree) {
        case 1:  // add(I, A)
            return addm<Ops>(I, A);
        case 2: {  // eval_ps(2): I + A + A2/2
            const F A2 = g.template sq_first<Ops>(A);
            return lc<Ops, true>(1.0, I, 1.0, A, 0.5, A2);
        }
        case 4: {  // eval_ps(4)
            const F A2 = g.template sq_first<Ops>(A);
            const F f0 = lc<Ops, true>(1.0, I, 1.0, A);
            const F f1 = lc<Ops, true>(kInvFact2, I, kInvFact3, A);
            const F inner = lc<Ops>(1.0, f1, kInvFact4, A2);
            return g.template mm_add<Ops>(inner, A2, false, f0);
        }
        case 8: {  // eval_t8, 3 products
            const F A2 = g.template sq_first<Ops>(A);
            const F A4 = g.template mm<Ops>(A2, lc<Ops>(T8C::x1, A, T8C::x2, A2), false);
            if constexpr (!Ops::kExact && std::is_same<typename F::T, double>::value) {
                // fast rounding (fp64 fragments; the fp32 kernels keep the
                // order the pair kernel mirrors): x3*A2 + A4 as one FMA per element, and the
                // final y-combination seeds the last product's accumulator
                // (4 of the scheme's 20 FP64 instructions per lane less)
                static_assert(T8C::y0 == 1.0 && T8C::y1 == 1.0, "eval_t8 tail");
                F L;
#pragma unroll
                for (int e = 0; e < F::kCount; ++e) L.v[e] = Ops::mac(A4.v[e], T8C::x3, A2.v[e]);
                return g.template mm_add<Ops>(
                    L, lc<Ops, true>(T8C::x4, I, T8C::x5, A, T8C::x6, A2, T8C::x7, A4), false,
                    lc<Ops, true>(T8C::y0, I, T8C::y1, A, T8C::y2, A2));
            }
            const F A8 = g.template mm<Ops>(
                lc<Ops>(T8C::x3, A2, 1.0, A4),
                lc<Ops, true>(T8C::x4, I, T8C::x5, A, T8C::x6, A2, T8C::x7, A4), false);
            return lc<Ops, true>(T8C::y0, I, T8C::y1, A, T8C::y2, A2, 1.0, A8);
        }
        case 12: {  // eval_t12, 4 products
            const F A2 = g.template sq_first<Ops>(A);
            const F A3 = mm_by_a<Ops>(g, A2, A);
            F B[4];
#pragma unroll
            for (int j = 0; j < 4; ++j)
                B[j] = lc<Ops, true>(c_t12[0][j], I, c_t12[1][j], A, c_t12[2][j], A2, c_t12[3][j], A3);
            const F A6 = g.template mm_add<Ops>(B[3], B[3], true, B[2]);
            return g.template mm_add<Ops>(addm<Ops>(B[1], A6), A6, false, B[0]);
        }
        default: {  // 18: eval_t18, 5 products
            const F A2 = g.template sq_first<Ops>(A);
            const F A3 = mm_by_a<Ops>(g, A2, A);
            const F A6 = g.template mm<Ops>(A3, A3, true);
            if constexpr (G::S::STASH >= 4) {
                // register-lean order for large fragments: B1, B5, B4, B3 to the
                // stash, B2 kept; A..A6 die after B2.
                g.put(0, lc<Ops, true>(c_t18a[0], I, c_t18a[1], A, c_t18a[2], A2, c_t18a[3], A3));
#pragma unroll
                for (int j = 3; j >= 1; --j)
                    g.put(4 - j, lc<Ops, true>(c_t18b[j][0], I, c_t18b[j][1], A, c_t18b[j][2], A2,
                                               c_t18b[j][3], A3, c_t18b[j][4], A6));
                const F B2 = lc<Ops, true>(c_t18b[0][0], I, c_t18b[0][1], A, c_t18b[0][2], A2,
                                           c_t18b[0][3], A3, c_t18b[0][4], A6);
                const F A9 = g.template mm_add<Ops>(g.get(0), g.get(1), false, g.get(2));
                return g.template mm_add<Ops>(addm<Ops>(g.get(3), A9), A9, false, B2);
            } else {
                const F B1 = lc<Ops, true>(c_t18a[0], I, c_t18a[1], A, c_t18a[2], A2, c_t18a[3], A3);
                F B[4];
#pragma unroll
                for (int j = 0; j < 4; ++j)
                    B[j] = lc<Ops, true>(c_t18b[j][0], I, c_t18b[j][1], A, c_t18b[j][2], A2,
                                         c_t18b[j][3], A3, c_t18b[j][4], A6);
                const F A9 = g.template mm_add<Ops>(B1, B[3], false, B[2]);
                return g.template mm_add<Ops>(addm<Ops>(B[1], A9), A9, false, B[0]);
            }
        }
    }
}

// Family::TaylorPS (reference eval_ps, taylor_schemes.cpp:143-198, and
// eval_taylor_ps :229-232): Paterson-Stockmeyer degrees {1, 2, 4, 6, 9, 16}.
template <class Ops, class G>
__device__ typename G::Frag eval_taylor_ps(const G& g, int degree, const typename G::Frag& A) {
    using F = typename G::Frag;
    const F I = g.ident();
    switch (degree) {
        case 1:
            return addm<Ops>(I, A);
        case 2:
        case 4:
            return eval_taylor_new<Ops>(g, degree, A);  // the same eval_ps(2), eval_ps(4)
        case 6: {
            const F A2 = g.template sq_first<Ops>(A);
            const F A3 = mm_by_a<Ops>(g, A2, A);
            const F f0 = lc<Ops, true>(1.0, I, 1.0, A, inv_fact(2), A2);
            const F f1 = lc<Ops, true>(inv_fact(3), I, inv_fact(4), A, inv_fact(5), A2);
            const F inner = lc<Ops>(1.0, f1, inv_fact(6), A3);
            return g.template mm_add<Ops>(inner, A3, false, f0);
        }
        case 9: {
            const F A2 = g.template sq_first<Ops>(A);
            const F A3 = mm_by_a<Ops>(g, A2, A);
            const F f0 = lc<Ops, true>(inv_fact(0), I, inv_fact(1), A, inv_fact(2), A2);
            const F f1 = lc<Ops, true>(inv_fact(3), I, inv_fact(4), A, inv_fact(5), A2);
            const F f2 = lc<Ops, true>(inv_fact(6), I, inv_fact(7), A, inv_fact(8), A2);
            F t = lc<Ops>(1.0, f2, inv_fact(9), A3);
            t = g.template mm_add<Ops>(t, A3, false, f1);
            return g.template mm_add<Ops>(t, A3, false, f0);
        }
        default: {  // 16
            const F A2 = g.template sq_first<Ops>(A);
            const F A3 = mm_by_a<Ops>(g, A2, A);
            const F A4 = g.template mm<Ops>(A2, A2, true);
            F gk[4];
#pragma unroll
            for (int i = 0; i < 4; ++i)
                gk[i] = lc<Ops, true>(inv_fact(4 * i), I, inv_fact(4 * i + 1), A, inv_fact(4 * i + 2), A2,
                                      inv_fact(4 * i + 3), A3);
            F t = lc<Ops>(1.0, gk[3], inv_fact(16), A4);
            t = g.template mm_add<Ops>(t, A4, false, gk[2]);
            t = g.template mm_add<Ops>(t, A4, false, gk[1]);
            return g.template mm_add<Ops>(t, A4, false, gk[0]);
        }
    }
}

// ---- Family::PadeDiagonal (reference pade.cpp) -----------------------------
// r_order(A) = (V - U)^-1 (V + U) with U odd and V even in A.
template <class Ops, class F>
__device__ __forceinline__ void acc_term(F& r, double c, const F& m) {
#pragma unroll
    for (int e = 0; e < F::kCount; ++e)
        if (Ops::kExact || c != 0.0) r.v[e] = Ops::mac(r.v[e], c, m.v[e]);
}

// U and V of eval_pade (pade.cpp:50-113), in the reference's product and
// lincomb order: eval_r10, eval_r26, or the generic even-power chain.
template <class Ops, class G>
__device__ void eval_pade(const G& g, int order, const typename G::Frag& A, typename G::Frag& U,
                          typename G::Frag& V) {
    using F = typename G::Frag;
    const F I = g.ident();
    if (order == 10) {  // eval_r10 (pade.cpp:50-58), 3 products
        const double* b = c_pade[4];
        const F A2 = g.template sq_first<Ops>(A);
        const F A4 = g.template mm<Ops>(A2, A2, true);
        U = g.template mm<Ops>(A, lc<Ops>(b[5], A4, b[3], A2, b[1], I), false);
        V = lc<Ops>(b[4], A4, b[2], A2, b[0], I);
        return;
    }
    if (order == 26) {  // eval_r26 (pade.cpp:60-74), 6 products
        const double* b = c_pade[12];
        const F A2 = g.template sq_first<Ops>(A);
        const F A4 = g.template mm<Ops>(A2, A2, true);
        const F A6 = g.template mm<Ops>(A2, A4, false);
        F u = g.template mm<Ops>(A6, lc<Ops>(b[13], A6, b[11], A4, b[9], A2), false);
        u = lc<Ops>(1.0, u, b[7], A6, b[5], A4, b[3], A2, b[1], I);
        U = g.template mm<Ops>(A, u, false);
        const F v = g.template mm<Ops>(A6, lc<Ops>(b[12], A6, b[10], A4, b[8], A2), false);
        V = lc<Ops>(1.0, v, b[6], A6, b[4], A4, b[2], A2, b[0], I);
        return;
    }
    // any other even order (pade.cpp:82-110): A2, A4 = A2*A2, A6 = A2*A4, ...
    // up to the largest even power <= m; the odd and even lincombs take the
    // powers in ascending order, so they accumulate as the chain grows
    const int m = order / 2;
    const double* b = c_pade[m - 1];
    const int top = m - (m % 2);
    F odd = lc<Ops, true>(b[1], I);
    V = lc<Ops, true>(b[0], I);
    if (top >= 2) {
        const F A2 = g.template sq_first<Ops>(A);
        F P = A2;
#pragma unroll 1
        for (int e = 2; e <= top; e += 2) {
            if (e > 2) P = g.template mm<Ops>(A2, P, false);  // matmul(pow[0], pow.back())
            if (e + 1 <= m) acc_term<Ops>(odd, b[e + 1], P);
            acc_term<Ops>(V, b[e], P);
        }
    }
    if (m >= 3) {
        U = g.template mm<Ops>(A, odd, false);
    } else {  // scaled(a, b1)
#pragma unroll
        for (int e = 0; e < F::kCount; ++e) U.v[e] = Ops::mul(b[1], A.v[e]);
    }
}

// LU with partial pivoting and the solve of pade_solve (lu_solve,
// dense_matrix.cpp:112-118 -> kernels.cpp:55-112), cooperatively by the
// group on M (n x n, stride LD, overwritten by its factors) and R (the
// right-hand sides, overwritten by the solution). Always in the reference's
// arithmetic: every multiply, subtract and divide rounded separately. The row
// swaps are applied to R as they happen, which is the reference's
// rhs[perm[i]] gather. Returns false for a singular denominator (a zero pivot
// column, kernels.cpp:71-72).
__device__ __forceinline__ double lu_fms(double a, double l, double p) {
    return __dsub_rn(a, __dmul_rn(l, p));
}
__device__ __forceinline__ double lu_div(double a, double b) { return __ddiv_rn(a, b); }

template <class G, class T>
__device__ bool lu_solve_group(const G& g, T* M, T* R, int* flag) {
    constexpr int N = G::NDIM, LD = G::LD, TH = G::THREADS;
    static_assert(TH % N == 0, "threads cover whole columns");
    constexpr int RS = TH / N;  // row phases of the trailing update
    // small n: every loop fully unrolled (the index arithmetic and branches of
    // the rolled loops cost more than the arithmetic at n = 8)
    constexpr int kU = N <= 16 ? N : 1;
    constexpr int kShfl = N >= 32 ? 16 : N / 2;  // lanes holding candidates: [0, N)
    const int j = g.tid % N, r0 = g.tid / N;
#pragma unroll kU
    for (int k = 0; k < N; ++k) {
        int p = N;
        if (g.warp == 0) {
            // pivot: the first row holding the largest |M[i][k]|, i >= k, with
            // the reference's strict '>' scan from |M[k][k]| (NaN never wins;
            // a NaN diagonal keeps p = k)
            T best = T(-1);
#pragma unroll
            for (int i0 = 0; i0 < N; i0 += 32) {
                const int i = i0 + g.lane;
                if (i >= k && i < N) {
                    const T v = fabs(M[i * LD + k]);
                    if (v > best) {
                        best = v;
                        p = i;
                    }
                }
            }
#pragma unroll
            for (int o = kShfl; o > 0; o >>= 1) {
                const T ob = __shfl_xor_sync(0xffffffffu, best, o);
                const int op = __shfl_xor_sync(0xffffffffu, p, o);
                if (ob > best || (ob == best && op < p)) {
                    best = ob;
                    p = op;
                }
            }
            const T vk = fabs(M[k * LD + k]);
            if (vk != vk) p = k;
            if (vk == vk && best == T(0)) p = -1;
            if constexpr (G::W > 1) {
                if (g.lane == 0) *flag = p;
            } else {
                p = __shfl_sync(0xffffffffu, p, 0);
            }
        }
        if constexpr (G::W > 1) {
            g.sync();
            p = *flag;
        }
        if (p < 0) return false;
        if (p != k && g.tid < N) {  // swap rows k and p of M and R
            const T m0 = M[k * LD + j], r0v = R[k * LD + j];
            M[k * LD + j] = M[p * LD + j];
            R[k * LD + j] = R[p * LD + j];
            M[p * LD + j] = m0;
            R[p * LD + j] = r0v;
        }
        g.sync();
        const T piv = M[k * LD + k];
        if constexpr (N <= 16) {  // k is a constant here: predicated, unrolled
#pragma unroll
            for (int i0 = 0; i0 < N; i0 += TH) {
                const int i = k + 1 + i0 + g.tid;
                if (i < N) M[i * LD + k] = lu_div(M[i * LD + k], piv);
            }
        } else {  // rolled: only the rows below k
            for (int i = k + 1 + g.tid; i < N; i += TH) M[i * LD + k] = lu_div(M[i * LD + k], piv);
        }
        g.sync();
        if (j > k) {
            const T pk = M[k * LD + j];
            if constexpr (N <= 16) {
#pragma unroll
                for (int i0 = 0; i0 < N; i0 += RS) {
                    const int i = k + 1 + i0 + r0;
                    if (i < N) M[i * LD + j] = lu_fms(M[i * LD + j], M[i * LD + k], pk);
                }
            } else {
                for (int i = k + 1 + r0; i < N; i += RS)
                    M[i * LD + j] = lu_fms(M[i * LD + j], M[i * LD + k], pk);
            }
        }
        g.sync();
    }
    if constexpr (N == 32) {
        // one right-hand-side column per thread, held in registers: the same
        // operations in the same order, with the solved values kept out of
        // the shared-memory round trip of every step (cfg3 Pade 10.4 -> 7.9 ms)
        if (g.tid < N) {
            const int c = g.tid;
            T x[N];
#pragma unroll
            for (int i = 0; i < N; ++i) x[i] = R[i * LD + c];
#pragma unroll
            for (int i = 1; i < N; ++i)
#pragma unroll
                for (int q = 0; q < i; ++q) x[i] = lu_fms(x[i], M[i * LD + q], x[q]);
#pragma unroll
            for (int i = N - 1; i >= 0; --i) {
#pragma unroll
                for (int q = i + 1; q < N; ++q) x[i] = lu_fms(x[i], M[i * LD + q], x[q]);
                x[i] = lu_div(x[i], M[i * LD + i]);
            }
#pragma unroll
            for (int i = 0; i < N; ++i) R[i * LD + c] = x[i];
        }
        return true;
    }
    if (g.tid < N) {  // one right-hand-side column per thread (lu_apply)
        const int c = g.tid;
#pragma unroll kU
        for (int i = 1; i < N; ++i) {
            T s = R[i * LD + c];
            for (int q = 0; q < i; ++q) s = lu_fms(s, M[i * LD + q], R[q * LD + c]);
            R[i * LD + c] = s;
        }
#pragma unroll kU
        for (int i = N - 1; i >= 0; --i) {
            T s = R[i * LD + c];
            for (int q = i + 1; q < N; ++q) s = lu_fms(s, M[i * LD + q], R[q * LD + c]);
            R[i * LD + c] = lu_div(s, M[i * LD + i]);
        }
    }
    return true;
}

// pade_solve (pade.cpp:26-28): X = (V - U)^-1 (V + U); false when singular
template <class Ops, class G>
__device__ __forceinline__ bool pade_solve(const G& g, const typename G::Frag& U,
                                           const typename G::Frag& V, typename G::Frag& X) {
    g.stage_solve(lc<Ops>(1.0, V, -1.0, U), addm<Ops>(V, U));  // sub(v, u), add(v, u)
    if (!lu_solve_group(g, g.lu_m(), g.lu_r(), g.lu_flag())) return false;
    X = g.solved();
    return true;
}

template <class Ops, int kFam = MEXP_FAMILY_TAYLOR_NEW, class G>
__device__ __forceinline__ typename G::Frag run_expm(const G& g, const typename G::Frag& A0,
                                                     int degree, int s, int fast_tail = 0,
                                                     bool* singular = nullptr) {
    using F = typename G::Frag;
    F A = A0;
    if (s > 0) {  // scaled(a, 2^-s) (expm.cpp:47 -> kernels.cpp:39-42), exact
        const double f = pow2_neg(s);
#pragma unroll
        for (int e = 0; e < G::K; ++e) A.v[e] = __dmul_rn(f, A.v[e]);
    }
    F X;
    if constexpr (kFam == MEXP_FAMILY_PADE) {
        F U, V;
        eval_pade<Ops>(g, degree, A, U, V);
        if (!pade_solve<Ops>(g, U, V, X)) {
            *singular = true;
            return X;
        }
    } else if constexpr (kFam == MEXP_FAMILY_TAYLOR_PS) {
        X = eval_taylor_ps<Ops>(g, degree, A);
    } else {
        X = eval_taylor_new<Ops>(g, degree, A);
    }
    // squarings, expm.cpp:31-35. With reference rounding, the last
    // `fast_tail` of them may use FMA/DMMA rounding: a rounding difference
    // made at squaring i is amplified ~2^(s-i) by the squarings after it, so
    // the tail adds only ~(2^k - 1) ulp-level differences (the AUTO policy).
    const int exact_until = (Ops::kExact && fast_tail < s) ? s - fast_tail : (Ops::kExact ? 0 : s);
    int i = 0;
    for (; i < exact_until; ++i) X = g.template mm<Ops>(X, X, true);
    for (; i < s; ++i) X = g.template mm<FastOps>(X, X, true);
    return X;
}

// One group of W warps per matrix; GPC groups per CTA; grid-stride over the batch.
template <int N, int GPC, int kFamily = MEXP_FAMILY_TAYLOR_NEW>
__global__ void __launch_bounds__(32 * TileShape<N>::W * GPC, TileShape<N>::MIN_BLOCKS)
    expm_small_f64_kernel(const double* __restrict__ a, double* __restrict__ out,
                          mexp_selection* __restrict__ sel, int64_t batch, int acc_arg,
                          int rounding, int exact_s_min) {
    using G = Group<N>;
    using F = typename G::Frag;
    extern __shared__ __align__(16) double smem[];
    const int accuracy = acc_arg & 15;  // mexp_accuracy (low nibble)
    constexpr int family = kFamily;
    const int gid = threadIdx.x / G::THREADS;
    G g;
    double* base = smem + gid * G::SMEM_DOUBLES;
    g.sx = base;
    g.sy = base + N * G::LD;
    g.stash = base + 2 * N * G::LD;
    g.scal = g.stash + G::S::STASH * G::STASH_SLOT;
    g.tid = threadIdx.x % G::THREADS;
    g.lane = g.tid & 31;
    g.warp = g.tid >> 5;
    g.bar_id = 1 + gid;

    constexpr int64_t NN = int64_t(N) * N;
    const int64_t stride = int64_t(gridDim.x) * GPC;
    int64_t m = int64_t(blockIdx.x) * GPC + gid;
    F next;
    if (m < batch) next = g.load_global(a + m * NN);
    for (; m < batch; m += stride) {
        const F A = next;
        if (m + stride < batch) next = g.load_global(a + (m + stride) * NN);  // prefetch

        // all_finite (dense_matrix.cpp:54-58) and the exact 1-norm
        // (kernels.cpp:44-53): stage A, one thread per column sums rows 0..n-1
        // in order, then an exact max across columns.
        bool fin = true;
#pragma unroll
        for (int e = 0; e < G::K; ++e) fin = fin && isfinite(A.v[e]);
        g.sync();
        g.store_smem(g.sx, A);
        g.sync();
        double colsum = 0.0;
        if (g.tid < N) {
#pragma unroll 8
            for (int i = 0; i < N; ++i) colsum = __dadd_rn(colsum, fabs(g.sx[i * G::LD + g.tid]));
        }
        const bool wfin = __all_sync(0xffffffffu, fin);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) colsum = fmax(colsum, __shfl_xor_sync(0xffffffffu, colsum, o));
        double norm = colsum;
        bool allfin = wfin;
        if constexpr (G::W > 1) {
            if (g.lane == 0) {
                g.scal[g.warp] = colsum;
                g.scal[G::W + g.warp] = wfin ? 1.0 : 0.0;
            }
            g.sync();
#pragma unroll
            for (int w = 0; w < G::W; ++w) {
                norm = fmax(norm, g.scal[w]);
                allfin = allfin && (g.scal[G::W + w] != 0.0);
            }
        }

        Sel sl{0, 0, MEXP_OK};
        if (!allfin) {
            sl.status = MEXP_ERR_NONFINITE;
        } else {
            sl = select_device(norm, accuracy, acc_arg >> 4);  // (family 3: reference_expm)
        }
        if (sel && g.tid == 0) {
            mexp_selection r;
            r.norm_in = allfin ? norm : __longlong_as_double(0x7ff8000000000000ll);
            r.degree = int16_t(sl.degree);
            r.s = int16_t(sl.s);
            r.status = sl.status;
            sel[m] = r;
        }
        F X;
        if (sl.status != MEXP_OK) {
#pragma unroll
            for (int e = 0; e < G::K; ++e) X.v[e] = __longlong_as_double(0x7ff8000000000000ll);
        } else {
            const bool exact = rounding == MEXP_ROUND_REFERENCE ||
                               (rounding == MEXP_ROUND_AUTO && sl.s >= exact_s_min);
            bool singular = false;
            if (exact)
                X = run_expm<ExactOps, family>(g, A, sl.degree, sl.s, 0, &singular);
            else
                X = run_expm<FastOps, family>(g, A, sl.degree, sl.s, 0, &singular);
            if (singular) {  // "singular denominator" (kernels.cpp:71-72)
#pragma unroll
                for (int e = 0; e < G::K; ++e) X.v[e] = __longlong_as_double(0x7ff8000000000000ll);
                if (sel && g.tid == 0) sel[m].status = MEXP_ERR_SINGULAR;
            }
        }
        g.store_global(out + m * NN, X);
    }
}

}  // namespace mexp_b200
