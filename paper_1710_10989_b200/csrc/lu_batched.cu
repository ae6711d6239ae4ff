// Batched LU with partial pivoting and the Pade solve X = (V - U)^-1 (V + U)
// for the large-n path (n > 64), on all listed matrices at once
// (reference lu_solve: dense_matrix.cpp:112-118 -> kernels.cpp:55-112).
//
// Right-looking blocked LU, panel width NB = 64, per panel:
//   lu_col_kernel, once per panel column c (+1 finishing step): every CTA
//     owns 64 rows of the panel; it scales column c-1 by its pivot, applies
//     that column's rank-1 update to the panel columns right of it, and finds
//     its rows' largest |M[r][c]|; the matrix's last CTA to finish (atomic
//     ticket) picks the pivot (largest value, ties to the lower row, NaN
//     never wins -- the reference's strict '>' scan) and swaps the two rows
//     across the panel;
//   laswp_kernel: the panel's row swaps on the columns outside it and on R;
//   trsm_kernel<lower, unit>: U12 = L11^-1 A12;
//   gemm_sub_kernel: A22 -= L21 U12 on the FP64 tensor cores (DMMA).
// Then the solves, blocked the same way: R_j = L_jj^-1 R_j, R_>j -= L_>j,j R_j
// forward, R_j = U_jj^-1 R_j, R_<j -= U_<j,j R_j backward.
// Pivot order and multipliers follow the reference; the trailing updates use
// FMA/DMMA rounding (the large-n path is FAST-only).
#include <algorithm>
#include <cstdlib>
#include <string>

#include <cooperative_groups.h>

#include "async_buffer.hpp"
#include "device_once.hpp"
#include "expm_common.cuh"
#include "lu_batched.cuh"

namespace mexp_b200 {

namespace {

constexpr int NB = 64;         // panel width
constexpr int COL_ROWS = 64;   // rows per CTA in the column step
constexpr int COL_THREADS = 256;
constexpr int TRSM_THREADS = 128;
constexpr int GBM = 128, GBN = 64;  // gemm_sub tile: 8 warps of 32 x 32, two CTAs per SM
constexpr int GLDX = NB + 4;   // X tile row stride (doubles), 4 (mod 16)
constexpr int GLDY = GBN + 4;  // Y tile row stride
constexpr size_t GEMM_SUB_SMEM = (size_t(GBM) * GLDX + size_t(NB) * GLDY) * sizeof(double);

thread_local std::string g_lu_err;

#define LUCUDA(call)                                                             \
    do {                                                                         \
        cudaError_t e_ = (call);                                                 \
        if (e_ != cudaSuccess) {                                                 \
            g_lu_err = std::string(#call) + ": " + cudaGetErrorString(e_);       \
            return MEXP_ERR_CUDA;                                                \
        }                                                                        \
    } while (0)

__device__ __forceinline__ bool better(double v, int r, double bv, int br) {
    return v > bv || (v == bv && r < br);  // NaN never wins; ties to the lower row
}

// Column step c of the panel [c0, c0 + NB). finish = (c == c0 + NB): only the
// scaling of the panel's last column.
__global__ void __launch_bounds__(COL_THREADS) lu_col_kernel(
    double* __restrict__ Mb, int np, const int32_t* __restrict__ list, int c0, int c,
    double* __restrict__ part_v, int* __restrict__ part_r, unsigned* __restrict__ counter,
    int* __restrict__ piv, mexp_selection* __restrict__ sel) {
    const int64_t m = list[blockIdx.y];
    double* M = Mb + m * int64_t(np) * np;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const bool upd = c > c0, search = c < c0 + NB;
    const int jm = c - 1 - c0;  // panel column being eliminated
    double u0 = 0.0, u1 = 0.0, pv = 1.0;
    if (upd) {
        const double* urow = M + int64_t(c - 1) * np + c0;
        u0 = urow[lane];
        u1 = urow[32 + lane];
        pv = M[int64_t(c - 1) * np + (c - 1)];
    }
    const int js = c - c0;  // panel column searched
    double best = -1.0;
    int brow = np;
    const int rbeg = c + blockIdx.x * COL_ROWS;
    // the warp's rows are all loaded before the first store (one memory
    // round trip per CTA rather than one per row)
    constexpr int RPW = COL_ROWS / (COL_THREADS / 32);
    double w0[RPW], w1[RPW];
#pragma unroll
    for (int t = 0; t < RPW; ++t) {
        const int r = rbeg + warp + t * (COL_THREADS / 32);
        w0[t] = w1[t] = 0.0;
        if (r < np) {
            const double* row = M + int64_t(r) * np + c0;
            w0[t] = row[lane];
            w1[t] = row[32 + lane];
        }
    }
#pragma unroll
    for (int t = 0; t < RPW; ++t) {
        const int i = warp + t * (COL_THREADS / 32);
        const int r = rbeg + i;
        if (r >= np) break;
        double* row = M + int64_t(r) * np + c0;
        double v0 = w0[t], v1 = w1[t];
        if (upd) {
            const double mine = jm < 32 ? v0 : v1;
            const double l = __shfl_sync(0xffffffffu, mine, jm & 31) / pv;  // row[k] / piv
            if (jm < 32) {
                if (lane == jm) v0 = l;
                if (lane > jm) v0 = fma(-l, u0, v0);
                v1 = fma(-l, u1, v1);
            } else {
                if (lane == (jm & 31)) v1 = l;
                if (lane > (jm & 31)) v1 = fma(-l, u1, v1);
            }
            row[lane] = v0;
            row[32 + lane] = v1;
        }
        if (search) {
            const double cv = fabs(__shfl_sync(0xffffffffu, js < 32 ? v0 : v1, js & 31));
            if (better(cv, r, best, brow)) {
                best = cv;
                brow = r;
            }
        }
    }
    if (!search) return;
    __shared__ double sb[COL_THREADS / 32];
    __shared__ int sr[COL_THREADS / 32];
    __shared__ bool last;
    if (lane == 0) {
        sb[warp] = best;
        sr[warp] = brow;
    }
    __syncthreads();
    const int G = gridDim.x, maxg = np / COL_ROWS;
    if (threadIdx.x == 0) {
        for (int w = 1; w < COL_THREADS / 32; ++w)
            if (better(sb[w], sr[w], best, brow)) {
                best = sb[w];
                brow = sr[w];
            }
        part_v[m * maxg + blockIdx.x] = best;
        part_r[m * maxg + blockIdx.x] = brow;
        __threadfence();
        last = atomicAdd(counter + m, 1u) == unsigned(G - 1);
    }
    __syncthreads();
    if (!last) return;
    __shared__ int sp;
    if (threadIdx.x == 0) {
        __threadfence();
        double bv = -1.0;
        int br = np;
        for (int b = 0; b < G; ++b) {
            const double v = __ldcg(part_v + m * maxg + b);
            const int r = __ldcg(part_r + m * maxg + b);
            if (better(v, r, bv, br)) {
                bv = v;
                br = r;
            }
        }
        const double dk = fabs(__ldcg(M + int64_t(c) * np + c));
        int p = br;
        if (dk != dk) p = c;  // a NaN diagonal: the reference's scan never moves
        else if (bv == 0.0) {  // "singular denominator" (kernels.cpp:71-72)
            p = c;
            sel[m].status = MEXP_ERR_SINGULAR;
        }
        piv[m * int64_t(np) + c] = p;
        counter[m] = 0u;
        sp = p;
    }
    __syncthreads();
    const int p = sp;
    if (p != c && threadIdx.x < NB) {  // swap rows c and p across the panel
        double* rc = M + int64_t(c) * np + c0 + threadIdx.x;
        double* rp = M + int64_t(p) * np + c0 + threadIdx.x;
        const double a = __ldcg(rc), b = __ldcg(rp);
        *rc = b;
        *rp = a;
    }
}

// Whole-panel factorisation for np - c0 <= 512: one cluster of G = ceil((np -
// c0) / 64) CTAs per matrix, CTA b holding rows [c0 + 64b, c0 + 64b + 64) of
// the panel in registers (4 warps; warp w, slot t: row c0 + 64b + w + 4t; lane: columns
// lane and 32 + lane), so the panel is read and written once instead of once
// per column. Per column, each CTA posts in its shared memory its best
// candidate (value, row and row data; CTA 0 also |diagonal| and row c),
// double-buffered by column parity -> one cluster barrier -> warp 0 of every
// CTA reduces the G posts (DSMEM) to the same pivot and copies the pivot row
// (and, at the pivot's owner, old row c) into local shared memory -> swap and
// eliminate. The arithmetic, the pivot rule and the swaps are lu_col_kernel's,
// so the factors are bit-equal.
constexpr int PANEL_MAX_CTAS = 8;
// a value select that keeps both arrays in registers (a ternary on two array
// elements can become a select of the array addresses, i.e. local memory)
__device__ __forceinline__ double pick(bool hi, double a, double b) {
    const long long mask = -static_cast<long long>(hi);
    return __longlong_as_double((__double_as_longlong(b) & mask) | (__double_as_longlong(a) & ~mask));
}
// v[idx] for a runtime idx without indexing the register array (an indexed
// access would move the array to local memory)
template <int R>
__device__ __forceinline__ double slot(const double (&v)[R], int idx) {
    long long acc = 0;
#pragma unroll
    for (int t = 0; t < R; ++t) acc |= __double_as_longlong(v[t]) & -static_cast<long long>(t == idx);
    return __longlong_as_double(acc);
}
#ifndef MEXP_PANEL_WARPS
#define MEXP_PANEL_WARPS 4
#endif
#ifndef MEXP_PANEL_MINB
#define MEXP_PANEL_MINB 4
#endif
constexpr int PANEL_THREADS = 32 * MEXP_PANEL_WARPS;
template <int G>
__global__ void __cluster_dims__(G, 1, 1) __launch_bounds__(PANEL_THREADS, MEXP_PANEL_MINB)
    lu_panel_cluster_kernel(double* __restrict__ Mb, int np, const int32_t* __restrict__ list, int c0,
                            int* __restrict__ piv, mexp_selection* __restrict__ sel) {
    namespace cg = cooperative_groups;
    cg::cluster_group cluster = cg::this_cluster();
    const int b = int(cluster.block_rank());
    const int64_t m = list[blockIdx.y];
    double* M = Mb + m * int64_t(np) * np;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    constexpr int W = PANEL_THREADS / 32, RPW = COL_ROWS / W;
    __shared__ double wv[W];
    __shared__ int wr[W];
    __shared__ __align__(16) double prow[NB];  // the pivot row (new row c), copied from its post
    __shared__ __align__(16) double crow[NB];  // old row c, at the pivot's owner
    __shared__ int s_p;
    const int rb = c0 + COL_ROWS * b;  // first row of this CTA
    double v0[RPW], v1[RPW];
#pragma unroll
    for (int t = 0; t < RPW; ++t) {
        const int r = rb + warp + W * t;
        v0[t] = v1[t] = 0.0;
        if (r < np) {
            const double* row = M + int64_t(r) * np + c0;
            v0[t] = row[lane];
            v1[t] = row[32 + lane];
        }
    }
    // posts, double-buffered by column parity: this CTA's best candidate
    // (value, row, row data) and, in CTA 0, |diagonal| and row c
    __shared__ double post_v[2], post_d[2];
    __shared__ int post_r[2];
    __shared__ __align__(16) double post_row[2][NB];
    __shared__ __align__(16) double post_crow[2][NB];
    __shared__ int s_w, s_t, s_q;
    for (int j = 0; j < NB; ++j) {
        const int c = c0 + j, par = j & 1;
        const bool hi = j >= 32;  // column j is in v1 (lanes hold columns lane, 32 + lane)
        const bool own_c = b == 0 && warp == (j & (W - 1));
        if (lane == (j & 31)) {
            double best = -1.0;
            int brow = np;
#pragma unroll
            for (int t = 0; t < RPW; ++t) {
                const int r = rb + warp + W * t;
                if (r >= c && r < np) {
                    const double cv = fabs(pick(hi, v0[t], v1[t]));
                    if (better(cv, r, best, brow)) {
                        best = cv;
                        brow = r;
                    }
                }
            }
            wv[warp] = best;
            wr[warp] = brow;
            if (own_c) post_d[par] = fabs(pick(hi, slot(v0, j / W), slot(v1, j / W)));
        }
        if (own_c) {
            post_crow[par][lane] = slot(v0, j / W);
            post_crow[par][32 + lane] = slot(v1, j / W);
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            double best = wv[0];
            int brow = wr[0];
            for (int w = 1; w < W; ++w)
                if (better(wv[w], wr[w], best, brow)) {
                    best = wv[w];
                    brow = wr[w];
                }
            post_v[par] = best;
            post_r[par] = brow;
            s_w = brow < np ? (brow - rb) & (W - 1) : -1;
            s_t = brow < np ? (brow - rb) / W : 0;
        }
        __syncthreads();
        if (warp == s_w) {
            post_row[par][lane] = slot(v0, s_t);
            post_row[par][32 + lane] = slot(v1, s_t);
        }
        cluster.sync();
        // warp 0: the pivot from the G posts (lane q reads CTA q's), then the
        // pivot row and, at the pivot's owner, old row c into local memory
        if (warp == 0) {
            double bv = -1.0;
            int br = np, bq = 0;
            if (lane < G) {
                bv = *cluster.map_shared_rank(&post_v[par], lane);
                br = *cluster.map_shared_rank(&post_r[par], lane);
                bq = lane;
            }
#pragma unroll
            for (int o = 1; o < 8; o <<= 1) {
                const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
                const int orow = __shfl_xor_sync(0xffffffffu, br, o);
                const int oq = __shfl_xor_sync(0xffffffffu, bq, o);
                if (better(ov, orow, bv, br)) {
                    bv = ov;
                    br = orow;
                    bq = oq;
                }
            }
            const double dk = *cluster.map_shared_rank(&post_d[par], 0);
            int p = br;
            if (dk != dk || bv == 0.0) {  // NaN diagonal / "singular denominator"
                p = c;
                bq = 0;
            }
            if (b == 0 && lane == 0) {
                piv[m * int64_t(np) + c] = p;
                if (dk == dk && bv == 0.0) sel[m].status = MEXP_ERR_SINGULAR;
            }
            const double* src = p == c ? cluster.map_shared_rank(post_crow[par], 0)
                                       : cluster.map_shared_rank(post_row[par], bq);
            prow[lane] = src[lane];
            prow[32 + lane] = src[32 + lane];
            if (p != c && b == bq) {
                const double* cr = cluster.map_shared_rank(post_crow[par], 0);
                crow[lane] = cr[lane];
                crow[32 + lane] = cr[32 + lane];
            }
            if (lane == 0) s_p = p;
        }
        __syncthreads();
        const int p = s_p;
        const double u0 = prow[lane], u1 = prow[32 + lane];
        if (p != c) {
            const int pb = (p - c0) / COL_ROWS, pw = (p - rb) & (W - 1), pt = ((p - c0) % COL_ROWS) / W;
            const bool own_p = b == pb && warp == pw;
            const double cr0 = crow[lane], cr1 = crow[32 + lane];
#pragma unroll
            for (int t = 0; t < RPW; ++t) {
                const bool tc = own_c && t == (j / W), tp = own_p && t == pt;
                v0[t] = pick(tc, pick(tp, v0[t], cr0), u0);
                v1[t] = pick(tc, pick(tp, v1[t], cr1), u1);
            }
        }
        const double pv = prow[j];
#pragma unroll
        for (int t = 0; t < RPW; ++t) {
            const int r = rb + warp + W * t;
            if (r <= c || r >= np) continue;
            const double mine = pick(hi, v0[t], v1[t]);
            const double l = __shfl_sync(0xffffffffu, mine, j & 31) / pv;  // row[k] / piv
            if (j < 32) {
                if (lane == j) v0[t] = l;
                if (lane > j) v0[t] = fma(-l, u0, v0[t]);
                v1[t] = fma(-l, u1, v1[t]);
            } else {
                if (lane == (j & 31)) v1[t] = l;
                if (lane > (j & 31)) v1[t] = fma(-l, u1, v1[t]);
            }
        }
        __syncthreads();  // prow / crow / s_p are rewritten in the next column
    }
#pragma unroll
    for (int t = 0; t < RPW; ++t) {
        const int r = rb + warp + W * t;
        if (r < np) {
            double* row = M + int64_t(r) * np + c0;
            row[lane] = v0[t];
            row[32 + lane] = v1[t];
        }
    }
    cluster.sync();  // no CTA exits while a peer may still write its shared memory
}

// The panel's row swaps (in order) on M's columns outside [c0, c0 + NB)
// (blockIdx.z = 0) and on every column of R (blockIdx.z = 1).
__global__ void laswp_kernel(double* __restrict__ Mb, double* __restrict__ Rb, int np,
                             const int32_t* __restrict__ list, int c0,
                             const int* __restrict__ piv) {
    const int64_t m = list[blockIdx.y];
    const int col = blockIdx.x * blockDim.x + threadIdx.x;
    if (col >= np) return;
    double* X = (blockIdx.z == 0 ? Mb : Rb) + m * int64_t(np) * np;
    if (blockIdx.z == 0 && col >= c0 && col < c0 + NB) return;
    const int* pv = piv + m * int64_t(np);
    for (int c = c0; c < c0 + NB; ++c) {
        const int p = pv[c];
        if (p != c) {
            const double a = X[int64_t(c) * np + col];
            X[int64_t(c) * np + col] = X[int64_t(p) * np + col];
            X[int64_t(p) * np + col] = a;
        }
    }
}

// 16-byte cp.async, zero-filled when !ok
__device__ __forceinline__ void cp_async16_z(double* smem, const double* gmem, bool ok) {
    const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(d), "l"(gmem), "r"(ok ? 16 : 0)
                 : "memory");
}

// X[r0 .. r0 + NB) x [cb, cb + ncols) <- T^-1 X with T the NB x NB diagonal
// block of M at (r0, r0): unit lower (kLower) or upper. One column per thread.
template <bool kLower>
__global__ void __launch_bounds__(TRSM_THREADS) trsm_kernel(const double* __restrict__ Mb,
                                                            double* __restrict__ Xb, int np,
                                                            const int32_t* __restrict__ list,
                                                            int r0, int cb, int ncols) {
    const int64_t m = list[blockIdx.y];
    const double* M = Mb + m * int64_t(np) * np;
    double* X = Xb + m * int64_t(np) * np;
    // the diagonal block by cp.async: all of it in flight at once (a load ->
    // shared store loop waits one memory round trip per iteration)
    __shared__ __align__(16) double T[NB][NB + 2];
    for (int e = threadIdx.x; e < NB * NB / 2; e += TRSM_THREADS) {
        const int i = e / (NB / 2), k = (e % (NB / 2)) * 2;
        cp_async16_z(&T[i][k], M + int64_t(r0 + i) * np + r0 + k, true);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    __syncthreads();
    const int col = cb + blockIdx.x * TRSM_THREADS + threadIdx.x;
    if (col >= cb + ncols) return;
    double x[NB];
#pragma unroll
    for (int i = 0; i < NB; ++i) x[i] = X[int64_t(r0 + i) * np + col];
    if constexpr (kLower) {
#pragma unroll
        for (int i = 1; i < NB; ++i)
#pragma unroll
            for (int q = 0; q < i; ++q) x[i] = fma(-T[i][q], x[q], x[i]);
    } else {
#pragma unroll
        for (int i = NB - 1; i >= 0; --i) {
#pragma unroll
            for (int q = i + 1; q < NB; ++q) x[i] = fma(-T[i][q], x[q], x[i]);
            x[i] = x[i] / T[i][i];
        }
    }
#pragma unroll
    for (int i = 0; i < NB; ++i) X[int64_t(r0 + i) * np + col] = x[i];
}

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

// C[rc .. rc + rows) x [cc .. cc + cols) -= X[rc.., kc .. kc + NB) * Y[kc.., cc..]
// (C may alias X's or Y's matrix, never the same elements)
// (all of one matrix, row stride np); 128 x 64 tiles, 8 warps of 32 x 32.
struct SubArgs {
    double* C;
    const double* X;
    const double* Y;
    int rc, cc, kc, rows, cols, np;
    const int32_t* list;
};

__global__ void __launch_bounds__(256, 2) gemm_sub_kernel(SubArgs a) {
    extern __shared__ __align__(16) double sm[];
    double* sx = sm;                 // GBM x GLDX
    double* sy = sm + GBM * GLDX;    // NB x GLDY
    const int64_t m = a.list[blockIdx.z];
    const int64_t base = m * int64_t(a.np) * a.np;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int wm = warp >> 1, wn = warp & 1;
    const int r = lane >> 2, q = lane & 3;
    const int tr = blockIdx.y * GBM, tc = blockIdx.x * GBN;  // tile origin within the block
    // The operand tiles stream into shared memory by cp.async (no registers,
    // no ordering against the shared stores), and the accumulators start as
    // -C (D = X Y + (-C) on DMMA, so the tile result is -D = C - X Y exactly,
    // rounding being sign-symmetric): every load of the tile is in flight at
    // once, one memory round trip per tile.
    for (int e = tid; e < GBM * NB / 2; e += 256) {
        const int i = e / (NB / 2), k = (e % (NB / 2)) * 2;
        const bool ok = tr + i < a.rows;
        cp_async16_z(sx + i * GLDX + k, a.X + base + int64_t(a.rc + (ok ? tr + i : 0)) * a.np + a.kc + k, ok);
    }
    for (int e = tid; e < NB * GBN / 2; e += 256) {
        const int k = e / (GBN / 2), j = (e % (GBN / 2)) * 2;
        const bool ok = tc + j < a.cols;
        cp_async16_z(sy + k * GLDY + j, a.Y + base + int64_t(a.kc + k) * a.np + a.cc + (ok ? tc + j : 0), ok);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
    double acc[4][4][2];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int row = tr + wm * 32 + i * 8 + r;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int col = tc + wn * 32 + j * 8 + 2 * q;
            double2 v = make_double2(0.0, 0.0);
            if (row < a.rows && col < a.cols)
                v = *reinterpret_cast<const double2*>(a.C + base + int64_t(a.rc + row) * a.np + a.cc + col);
            acc[i][j][0] = -v.x;
            acc[i][j][1] = -v.y;
        }
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    __syncthreads();
    const double* px = sx + (wm * 32 + r) * GLDX + q;
    const double* py = sy + q * GLDY + wn * 32 + r;
#pragma unroll 4
    for (int k = 0; k < NB; k += 4) {
        double af[4], bf[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) af[i] = px[i * 8 * GLDX + k];
#pragma unroll
        for (int j = 0; j < 4; ++j) bf[j] = py[k * GLDY + j * 8];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) dmma(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int row = tr + wm * 32 + i * 8 + r;
        if (row >= a.rows) continue;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int col = tc + wn * 32 + j * 8 + 2 * q;
            if (col >= a.cols) continue;
            *reinterpret_cast<double2*>(a.C + base + int64_t(a.rc + row) * a.np + a.cc + col) =
                make_double2(-acc[i][j][0], -acc[i][j][1]);
        }
    }
}

int sub(double* C, const double* X, const double* Y, int rc, int cc, int kc, int rows, int cols,
        int np, const int32_t* list, int count, cudaStream_t st, std::atomic<uint64_t>* launches) {
    if (rows <= 0 || cols <= 0 || count == 0) return MEXP_OK;
    static PerDevice attr_once;
    attr_once([] {
        cudaFuncSetAttribute(gemm_sub_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             int(GEMM_SUB_SMEM));
    });
    SubArgs a{C, X, Y, rc, cc, kc, rows, cols, np, list};
    for (int z0 = 0; z0 < count; z0 += 65535) {
        a.list = list + z0;
        const dim3 grid((cols + GBN - 1) / GBN, (rows + GBM - 1) / GBM, std::min(count - z0, 65535));
        gemm_sub_kernel<<<grid, 256, GEMM_SUB_SMEM, st>>>(a);
        launches->fetch_add(1, std::memory_order_relaxed);
    }
    return MEXP_OK;
}

template <int G>
void launch_panel(double* M, int np, const int32_t* list, int count, int c0, int* piv,
                  mexp_selection* sel, cudaStream_t st) {
    lu_panel_cluster_kernel<G><<<dim3(G, count), PANEL_THREADS, 0, st>>>(M, np, list, c0, piv, sel);
}

int panel_cluster(double* M, int np, const int32_t* list, int count, int c0, int G, int* piv,
                  mexp_selection* sel, cudaStream_t st, std::atomic<uint64_t>* launches) {
    switch (G) {
        case 1: launch_panel<1>(M, np, list, count, c0, piv, sel, st); break;
        case 2: launch_panel<2>(M, np, list, count, c0, piv, sel, st); break;
        case 3: launch_panel<3>(M, np, list, count, c0, piv, sel, st); break;
        case 4: launch_panel<4>(M, np, list, count, c0, piv, sel, st); break;
        case 5: launch_panel<5>(M, np, list, count, c0, piv, sel, st); break;
        case 6: launch_panel<6>(M, np, list, count, c0, piv, sel, st); break;
        case 7: launch_panel<7>(M, np, list, count, c0, piv, sel, st); break;
        case 8: launch_panel<8>(M, np, list, count, c0, piv, sel, st); break;
        default: return MEXP_ERR_UNSUPPORTED;
    }
    launches->fetch_add(1, std::memory_order_relaxed);
    LUCUDA(cudaGetLastError());
    return MEXP_OK;
}

// T^-1 for the NB x NB diagonal block T of M at (r0, r0) (unit lower or
// upper), one column per thread by substitution on e_j, into W (list
// position z: W + z NB^2, row-major).
template <bool kLower>
__global__ void __launch_bounds__(NB) tri_inv_kernel(const double* __restrict__ Mb, int np,
                                                     const int32_t* __restrict__ list, int r0,
                                                     double* __restrict__ Wb) {
    const int64_t m = list[blockIdx.y];
    const double* M = Mb + m * int64_t(np) * np;
    double* W = Wb + int64_t(blockIdx.y) * NB * NB;
    __shared__ __align__(16) double T[NB][NB + 2];
    for (int e = threadIdx.x; e < NB * NB / 2; e += NB) {
        const int i = e / (NB / 2), k = (e % (NB / 2)) * 2;
        cp_async16_z(&T[i][k], M + int64_t(r0 + i) * np + r0 + k, true);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    __syncthreads();
    const int j = threadIdx.x;
    double x[NB];
#pragma unroll
    for (int i = 0; i < NB; ++i) x[i] = i == j ? 1.0 : 0.0;
    if constexpr (kLower) {
#pragma unroll
        for (int i = 1; i < NB; ++i)
#pragma unroll
            for (int q = 0; q < i; ++q) x[i] = fma(-T[i][q], x[q], x[i]);
    } else {
#pragma unroll
        for (int i = NB - 1; i >= 0; --i) {
#pragma unroll
            for (int q = i + 1; q < NB; ++q) x[i] = fma(-T[i][q], x[q], x[i]);
            x[i] = x[i] / T[i][i];
        }
    }
#pragma unroll
    for (int i = 0; i < NB; ++i) W[i * NB + j] = x[i];
}

// X[r0 .. r0 + NB) x [cb + 64 bx, ..+64) <- W_z X (in place: a CTA loads its
// whole 64-column tile before it stores) on DMMA; 8 warps of 16 x 32.
constexpr int TM_LD = NB + 4;
constexpr size_t TRI_MM_SMEM = size_t(2) * NB * TM_LD * sizeof(double);
__global__ void __launch_bounds__(256) tri_mm_kernel(const double* __restrict__ Wb, double* __restrict__ Xb,
                                                     int np, const int32_t* __restrict__ list, int r0,
                                                     int cb) {
    extern __shared__ __align__(16) double tsm[];
    double* sw = tsm;               // NB x TM_LD
    double* sxt = tsm + NB * TM_LD;  // NB x TM_LD
    const int64_t m = list[blockIdx.y];
    double* X = Xb + m * int64_t(np) * np;
    const double* W = Wb + int64_t(blockIdx.y) * NB * NB;
    const int c0 = cb + 64 * blockIdx.x;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int e = tid; e < NB * NB / 2; e += 256) {
        const int i = e / (NB / 2), k = (e % (NB / 2)) * 2;
        cp_async16_z(sw + i * TM_LD + k, W + i * NB + k, true);
        cp_async16_z(sxt + i * TM_LD + k, X + int64_t(r0 + i) * np + c0 + k, true);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    __syncthreads();
    const int wm = warp >> 1, wn = warp & 1;  // 4 x 2 warps of 16 x 32
    const int r = lane >> 2, q = lane & 3;
    double acc[2][4][2];
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    const double* pa = sw + (16 * wm + r) * TM_LD + q;
    const double* pb = sxt + q * TM_LD + 32 * wn + r;
#pragma unroll 4
    for (int k = 0; k < NB; k += 4) {
        double af[2], bf[4];
#pragma unroll
        for (int i = 0; i < 2; ++i) af[i] = pa[8 * i * TM_LD + k];
#pragma unroll
        for (int j = 0; j < 4; ++j) bf[j] = pb[k * TM_LD + 8 * j];
#pragma unroll
        for (int i = 0; i < 2; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) dmma(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
    __syncthreads();  // every warp is done reading the tile before it is overwritten
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j)
            *reinterpret_cast<double2*>(X + int64_t(r0 + 16 * wm + 8 * i + r) * np + c0 + 32 * wn + 8 * j + 2 * q) =
                make_double2(acc[i][j][0], acc[i][j][1]);
}

template <bool kLower>
int trsm(const double* M, double* X, int np, const int32_t* list, int count, int r0, int cb,
         int ncols, cudaStream_t st, std::atomic<uint64_t>* launches, double* W = nullptr) {
    if (ncols <= 0) return MEXP_OK;
    // DMMA path (MEXP_TRSM_DMMA=0: per-column substitution): T^-1 by
    // substitution on the identity, then X <- T^-1 X on the tensor pipe
    static const bool dmma_path = [] {
        const char* e = std::getenv("MEXP_TRSM_DMMA");
        return !(e && std::atoi(e) == 0);
    }();
    if (dmma_path && W && ncols % 64 == 0) {
        static PerDevice attr_once;
        attr_once([] {
            cudaFuncSetAttribute(tri_mm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(TRI_MM_SMEM));
        });
        for (int z0 = 0; z0 < count; z0 += 65535) {
            const int zc = std::min(count - z0, 65535);
            tri_inv_kernel<kLower><<<dim3(1, zc), NB, 0, st>>>(M, np, list + z0, r0, W);
            tri_mm_kernel<<<dim3(ncols / 64, zc), 256, TRI_MM_SMEM, st>>>(W, X, np, list + z0, r0, cb);
            launches->fetch_add(2, std::memory_order_relaxed);
        }
        return MEXP_OK;
    }
    for (int z0 = 0; z0 < count; z0 += 65535) {
        const dim3 grid((ncols + TRSM_THREADS - 1) / TRSM_THREADS, std::min(count - z0, 65535));
        trsm_kernel<kLower><<<grid, TRSM_THREADS, 0, st>>>(M, X, np, list + z0, r0, cb, ncols);
        launches->fetch_add(1, std::memory_order_relaxed);
    }
    return MEXP_OK;
}

}  // namespace

const char* lu_last_error() { return g_lu_err.c_str(); }

int lu_solve_batched(double* M, double* R, int np, int64_t batch, const int32_t* d_list, int count,
                     mexp_selection* d_sel, cudaStream_t st, std::atomic<uint64_t>* launches) {
    if (count == 0) return MEXP_OK;
    if (np % NB != 0 || count > 65535) return MEXP_ERR_UNSUPPORTED;
    const int maxg = np / COL_ROWS;
    // scratch: pivots (batch x np), per-CTA partial maxima, per-matrix tickets
    const size_t piv_b = sizeof(int) * size_t(batch) * np;
    const size_t pv_b = sizeof(double) * size_t(batch) * maxg;
    const size_t pr_b = sizeof(int) * size_t(batch) * maxg;
    const size_t ct_b = sizeof(unsigned) * size_t(batch);
    AsyncBuffer scratch_buf(st);
    LUCUDA(scratch_buf.alloc(piv_b + pv_b + pr_b + ct_b + 64));
    // the diagonal blocks' inverses for the DMMA triangular solves
    AsyncBuffer tinv_buf(st);
    LUCUDA(tinv_buf.alloc(sizeof(double) * size_t(count) * NB * NB));
    double* tinv = tinv_buf.get<double>();
    char* scratch = scratch_buf.get<char>();
    double* part_v = reinterpret_cast<double*>(scratch);
    int* piv = reinterpret_cast<int*>(scratch + pv_b);
    int* part_r = reinterpret_cast<int*>(scratch + pv_b + piv_b);
    unsigned* counter = reinterpret_cast<unsigned*>(scratch + pv_b + piv_b + pr_b);
    LUCUDA(cudaMemsetAsync(counter, 0, ct_b, st));
    int r;
    // panels of at most 512 rows: one cluster kernel per panel (MEXP_LU_PANEL=0
    // forces the per-column kernels)
    static const bool panel_ok = [] {
        const char* e = std::getenv("MEXP_LU_PANEL");
        return !(e && std::atoi(e) == 0);
    }();
    for (int c0 = 0; c0 < np; c0 += NB) {
        const int G = (np - c0 + COL_ROWS - 1) / COL_ROWS;
        if (panel_ok && G <= PANEL_MAX_CTAS) {
            if ((r = panel_cluster(M, np, d_list, count, c0, G, piv, d_sel, st, launches))) return r;
        } else
        for (int c = c0; c <= c0 + NB; ++c) {
            if (c >= np) break;
            const dim3 grid((np - c + COL_ROWS - 1) / COL_ROWS, count);
            lu_col_kernel<<<grid, COL_THREADS, 0, st>>>(M, np, d_list, c0, c, part_v, part_r,
                                                         counter, piv, d_sel);
            launches->fetch_add(1, std::memory_order_relaxed);
        }
        laswp_kernel<<<dim3((np + 255) / 256, count, 2), 256, 0, st>>>(M, R, np, d_list, c0, piv);
        launches->fetch_add(1, std::memory_order_relaxed);
        const int rest = np - c0 - NB;
        if (rest > 0) {
            if ((r = trsm<true>(M, M, np, d_list, count, c0, c0 + NB, rest, st, launches, tinv))) return r;
            if ((r = sub(M, M, M, c0 + NB, c0 + NB, c0, rest, rest, np, d_list, count, st, launches)))
                return r;
        }
    }
    // forward: L Y = P R
    for (int j = 0; j < np; j += NB) {
        if ((r = trsm<true>(M, R, np, d_list, count, j, 0, np, st, launches, tinv))) return r;
        if ((r = sub(R, M, R, j + NB, 0, j, np - j - NB, np, np, d_list, count, st, launches))) return r;
    }
    // backward: U X = Y
    for (int j = np - NB; j >= 0; j -= NB) {
        if ((r = trsm<false>(M, R, np, d_list, count, j, 0, np, st, launches, tinv))) return r;
        if ((r = sub(R, M, R, 0, 0, j, j, np, np, d_list, count, st, launches))) return r;
    }
    LUCUDA(cudaGetLastError());
    return MEXP_OK;
}

}  // namespace mexp_b200
