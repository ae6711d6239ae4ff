// Batched 8x8 fp64 expm with the diagonal Pade family (reference pade.cpp):
// the 8x8 warp kernel's layout (expm_n8.cuh), four matrices per warp round.
//
//   1. prologue for the 4 matrices at once (loads, finite votes, exact
//      1-norm, selection) -- as expm8_f64_kernel;
//   2. per matrix: U, V by eval_pade on the register fragments, then
//      M = V - U and R = V + U written row-major into the matrix's 1 KB tile;
//   3. the pivoted LU and both triangular solves for all 4 matrices at once:
//      lane l works on column l & 7 of matrix l >> 3, so all 32 lanes are
//      busy (a one-matrix warp leaves 24 idle in the solves); operations and
//      their order are the reference's (lu_solve_group in expm_small.cuh);
//   4. per matrix: X = R from the tile, the s squarings, the store.
#pragma once

#include "expm_n8.cuh"

namespace mexp_b200 {

template <int kMinBlocks = 8>
__global__ void __launch_bounds__(32 * kN8WarpsPerBlock, kMinBlocks)
    expm8_pade_kernel(const double* __restrict__ a, double* __restrict__ out,
                      mexp_selection* __restrict__ sel, int64_t batch, int acc_arg, int rounding,
                      int exact_s_min, unsigned long long* __restrict__ ticket) {
    using Group8 = Group8T<false>;
    using F = Group8::Frag;
    __shared__ __align__(16) char tiles[kN8WarpsPerBlock][kN8Mpw][1024];
    const int accuracy = acc_arg & 15, family = acc_arg >> 4;  // Pade, or reference_expm's rule
    const int lane = threadIdx.x & 31;
    const int wib = threadIdx.x >> 5;
    Group8 g;
    g.init(tiles[wib][0], lane);
    char* const wt = tiles[wib][0];

    const int jm = lane >> 3, c8 = lane & 7, cp = c8 >> 1;
    const uint32_t half = uint32_t(c8 & 1) << 3;
    const char* nb0 = wt + jm * 1024 + ((((cp >> 1)) << 5) | ((cp & 1) << 4)) + half;
    const char* nb1 = wt + jm * 1024 + (((1 ^ (cp >> 1)) << 5) | ((cp & 1) << 4)) + half;

    const int64_t rounds = (batch + kN8Mpw - 1) / kN8Mpw;
    const int64_t rstride = int64_t(gridDim.x) * kN8WarpsPerBlock;
    int64_t rd = int64_t(blockIdx.x) * kN8WarpsPerBlock + wib;
    for (; rd < rounds;) {
        const int64_t m0 = rd * kN8Mpw;
        double2 cur[kN8Mpw];
#pragma unroll
        for (int j = 0; j < kN8Mpw; ++j)
            cur[j] = (m0 + j < batch) ? ld_stream(reinterpret_cast<const double2*>(a + (m0 + j) * 64) + lane)
                                      : make_double2(0.0, 0.0);
        uint32_t finbits = 0;
#pragma unroll
        for (int j = 0; j < kN8Mpw; ++j)
            if (__all_sync(0xffffffffu, isfinite(cur[j].x) && isfinite(cur[j].y))) finbits |= 1u << j;
        __syncwarp();
#pragma unroll
        for (int j = 0; j < kN8Mpw; ++j) *reinterpret_cast<double2*>(wt + j * 1024 + g.st) = cur[j];
        __syncwarp();
        double colsum = 0.0;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const char* p = (((i >> 1) & 1) ? nb1 : nb0) + (unit8(i, 0) & ~0x20u);
            colsum = __dadd_rn(colsum, fabs(*reinterpret_cast<const double*>(p)));
        }
        unsigned long long nb = __double_as_longlong(colsum);
#pragma unroll
        for (int o = 1; o < 8; o <<= 1) {
            const unsigned long long w = __shfl_xor_sync(0xffffffffu, nb, o);
            nb = w > nb ? w : nb;
        }
        const double norm = __longlong_as_double(nb);
        const bool allfin = (finbits >> jm) & 1u;
        Sel sl{0, 0, MEXP_OK};
        if (!allfin)
            sl.status = MEXP_ERR_NONFINITE;
        else
            sl = select_device(norm, accuracy, family);
        if (sel && c8 == 0 && m0 + jm < batch) {
            mexp_selection rec;
            rec.norm_in = allfin ? norm : __longlong_as_double(0x7ff8000000000000ll);
            rec.degree = int16_t(sl.degree);
            rec.s = int16_t(sl.s);
            rec.status = sl.status;
            sel[m0 + jm] = rec;
        }
        const int info = sl.degree | (sl.s << 5) | (sl.status << 20);

        // ---- 2. U, V -> M = V - U, R = V + U, row-major in tile j ----
#pragma unroll 1
        for (int j = 0; j < kN8Mpw; ++j) {
            if (m0 + j >= batch) break;
            const int inf = __shfl_sync(0xffffffffu, info, 8 * j);
            const int degree = inf & 31, s = (inf >> 5) & 0x7fff, status = inf >> 20;
            if (status != MEXP_OK) continue;
            g.tile = wt + j * 1024;
            g.fscale = pow2_neg(s);
            const double2 v = *reinterpret_cast<const double2*>(g.tile + g.st);
            F A;
            const double f = pow2_neg(s);  // scaled(a, 2^-s), exact
            A.v[0] = __dmul_rn(f, v.x);
            A.v[1] = __dmul_rn(f, v.y);
            const bool exact = rounding == MEXP_ROUND_REFERENCE ||
                               (rounding == MEXP_ROUND_AUTO && s >= exact_s_min);
            F P, Q;
            if (exact) {
                F U, V;
                eval_pade<ExactOps>(g, degree, A, U, V);
                P = lc<ExactOps>(1.0, V, -1.0, U);  // sub(v, u)
                Q = addm<ExactOps>(V, U);          // add(v, u)
            } else {
                F U, V;
                eval_pade<FastOps>(g, degree, A, U, V);
                P = lc<FastOps>(1.0, V, -1.0, U);
                Q = addm<FastOps>(V, U);
            }
            __syncwarp();  // the products are done with the tile
            double* const t = reinterpret_cast<double*>(g.tile);
            *reinterpret_cast<double2*>(t + 8 * g.r + 2 * g.q) = make_double2(P.v[0], P.v[1]);
            *reinterpret_cast<double2*>(t + 64 + 8 * g.r + 2 * g.q) = make_double2(Q.v[0], Q.v[1]);
        }
        __syncwarp();

        // ---- 3. LU with partial pivoting + solves, 4 matrices at once ----
        // lane: matrix jm = lane >> 3, column c8 = lane & 7
        const bool act = (m0 + jm < batch) && sl.status == MEXP_OK;
        double* const M = reinterpret_cast<double*>(wt + jm * 1024);
        double* const R = M + 64;
        bool singular = false;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            // pivot (kernels.cpp:62-73): first row of the largest |M[i][k]|,
            // i >= k, strict '>' from |M[k][k]|; NaN never wins, a NaN
            // diagonal keeps k
            double best = -1.0;
            int p = 8;
            if (act && c8 >= k) {
                best = fabs(M[8 * c8 + k]);
                p = c8;
                if (best != best) best = -1.0, p = 8;
            }
#pragma unroll
            for (int o = 4; o > 0; o >>= 1) {  // within the matrix's 8 lanes
                const double ob = __shfl_xor_sync(0xffffffffu, best, o);
                const int op = __shfl_xor_sync(0xffffffffu, p, o);
                if (ob > best || (ob == best && op < p)) {
                    best = ob;
                    p = op;
                }
            }
            const double vk = fabs(M[8 * k + k]);
            if (vk != vk) p = k;
            if (act && vk == vk && best == 0.0) singular = true;
            if (singular) p = k;
            if (act && p != k) {
                const double mk = M[8 * k + c8], rk = R[8 * k + c8];
                M[8 * k + c8] = M[8 * p + c8];
                R[8 * k + c8] = R[8 * p + c8];
                M[8 * p + c8] = mk;
                R[8 * p + c8] = rk;
            }
            __syncwarp();
            if (act && c8 > k) M[8 * c8 + k] = lu_div(M[8 * c8 + k], M[8 * k + k]);
            __syncwarp();
            if (act && c8 > k) {
                const double pk = M[8 * k + c8];
#pragma unroll
                for (int i = k + 1; i < 8; ++i) M[8 * i + c8] = lu_fms(M[8 * i + c8], M[8 * i + k], pk);
            }
            __syncwarp();
        }
        if (act && !singular) {  // lu_apply: one right-hand-side column per lane
#pragma unroll
            for (int i = 1; i < 8; ++i) {
                double s = R[8 * i + c8];
#pragma unroll
                for (int q = 0; q < i; ++q) s = lu_fms(s, M[8 * i + q], R[8 * q + c8]);
                R[8 * i + c8] = s;
            }
#pragma unroll
            for (int i = 7; i >= 0; --i) {
                double s = R[8 * i + c8];
#pragma unroll
                for (int q = i + 1; q < 8; ++q) s = lu_fms(s, M[8 * i + q], R[8 * q + c8]);
                R[8 * i + c8] = lu_div(s, M[8 * i + i]);
            }
        }
        if (singular && c8 == 0 && sel) sel[m0 + jm].status = MEXP_ERR_SINGULAR;
        const uint32_t singbits = __ballot_sync(0xffffffffu, singular && c8 == 0);
        __syncwarp();

        // ---- 4. squarings (expm.cpp:31-35) and the store ----
#pragma unroll 1
        for (int j = 0; j < kN8Mpw; ++j) {
            const int64_t m = m0 + j;
            if (m >= batch) break;
            const int inf = __shfl_sync(0xffffffffu, info, 8 * j);
            const int s = (inf >> 5) & 0x7fff, status = inf >> 20;
            g.tile = wt + j * 1024;
            F X;
            if (status != MEXP_OK || ((singbits >> (8 * j)) & 1u)) {
                X.v[0] = X.v[1] = __longlong_as_double(0x7ff8000000000000ll);
            } else {
                const double2 v =
                    *reinterpret_cast<const double2*>(reinterpret_cast<double*>(g.tile) + 64 + 8 * g.r + 2 * g.q);
                X.v[0] = v.x;
                X.v[1] = v.y;
                const bool exact = rounding == MEXP_ROUND_REFERENCE ||
                                   (rounding == MEXP_ROUND_AUTO && s >= exact_s_min);
                if (exact)
                    for (int i = 0; i < s; ++i) X = g.template mm<ExactOps>(X, X, true);
                else
                    for (int i = 0; i < s; ++i) X = g.template mm<FastOps>(X, X, true);
            }
            st_stream(reinterpret_cast<double2*>(out + m * 64) + lane, make_double2(X.v[0], X.v[1]));
        }
        unsigned long long t = 0;
        if (lane == 0) t = atomicAdd(ticket, 1ull);
        rd = rstride + int64_t(__shfl_sync(0xffffffffu, t, 0));
    }
    release_ticket(ticket);
}

}  // namespace mexp_b200
