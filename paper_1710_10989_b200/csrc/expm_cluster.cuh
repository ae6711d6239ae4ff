// Latency path for few fp64 matrices of n in (32, 64] (cfg1: ONE 64x64
// matrix): a thread-block cluster of 4 CTAs on 4 SMs computes one expm.
//
// CTA c of the cluster owns rows [16c, 16c + 16) of every matrix variable as
// DMMA-accumulator fragments (4 warps, each a 16 x 16 block). A product
// C = X * Y needs all of Y: each CTA writes its 16 rows of Y into the Y tile
// of all four CTAs through distributed shared memory (st to mapa'd
// addresses), one cluster barrier (release/acquire) publishes them, and each
// CTA computes its 16 rows of C locally -- DMMA for FastOps, the reference's
// k-ordered DMUL+DADD for ExactOps. X and Y tiles are double-buffered by
// product parity, so one cluster barrier per product suffices: a buffer is
// rewritten two products after its last read, and every CTA has passed the
// intervening barrier only after finishing that read.
//
// The group exposes the interface of Group<N> (expm_small.cuh), so the same
// eval_taylor_new / eval_taylor_ps / run_expm code runs on it unchanged.
#pragma once

#include <cooperative_groups.h>

#include "expm_small.cuh"

namespace mexp_b200 {

#ifdef MEXP_CLUSTER_TRACE
__device__ __forceinline__ unsigned long long gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
__device__ unsigned long long g_trace_t[64];
__device__ const char* g_trace_tag[64];
__device__ int g_trace_n;
#define CTRACE(tag)                                                           \
    do {                                                                      \
        if (threadIdx.x == 0 && blockIdx.x == 0 && g_trace_n < 64) {          \
            g_trace_t[g_trace_n] = gtime();                                   \
            g_trace_tag[g_trace_n++] = tag;                                   \
        }                                                                     \
    } while (0)
#define CTRACE_DUMP()                                                         \
    do {                                                                      \
        if (threadIdx.x == 0 && blockIdx.x == 0) {                            \
            for (int i = 0; i < g_trace_n; ++i)                               \
                printf("trace %s %llu\n", g_trace_tag[i], g_trace_t[i]);     \
            g_trace_n = 0;                                                    \
        }                                                                     \
    } while (0)
#else
#define CTRACE(tag) \
    do {            \
    } while (0)
#define CTRACE_DUMP() \
    do {              \
    } while (0)
#endif

constexpr int kClusterCtas = 4;
constexpr int kClusterWarps = 4;  // warps per CTA

struct ClusterShape {
    static constexpr int STASH = 0;
};

struct ClusterGroup64 {
    using S = ClusterShape;
    static constexpr int N = 64;
    static constexpr int ROWS = N / kClusterCtas;  // 16 rows per CTA
    static constexpr int TR = ROWS / 8;             // 2 tile rows
    static constexpr int TC = 2;                    // 2 tile columns per warp
    static constexpr int T = TR * TC;
    static constexpr int K = 2 * T;                 // doubles per lane per matrix
    static constexpr int LD = N + 4;                // padded stride, 4 (mod 16)
    static constexpr int THREADS = 32 * kClusterWarps;
    // shared memory: X tiles [2][ROWS][LD], Y tiles [2][N][LD], scalars
    static constexpr int SMEM_DOUBLES = 2 * ROWS * LD + 2 * N * LD + 2 * kClusterWarps + 2;
    static_assert(kClusterWarps * TC * 8 == N, "warps cover the columns");

    struct Frag {
        using T = double;
        static constexpr int kCount = K;
        double v[K];
    };

    double* sx;  // local rows of X, two buffers of ROWS x LD
    double* sy;  // all rows of Y, two buffers of N x LD
    double* sy_peer[kClusterCtas];  // buffer 0 of the Y tile of every CTA of the cluster
    double* scal;
    int rank, lane, warp, tid;
    mutable int buf;

    __device__ __forceinline__ int lrow_of(int t) const { return 8 * (t / TC) + (lane >> 2); }
    __device__ __forceinline__ int row_of(int t) const { return ROWS * rank + lrow_of(t); }
    __device__ __forceinline__ int col_of(int t) const { return 16 * warp + 8 * (t % TC) + 2 * (lane & 3); }

    __device__ __forceinline__ void sync() const { __syncthreads(); }
    __device__ __forceinline__ static void cluster_sync() {
        asm volatile("barrier.cluster.arrive.release.aligned;\n"
                     "barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
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

    // this CTA's rows of a row-major n x n matrix
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

    __device__ __forceinline__ void put(int, const Frag&) const {}
    __device__ __forceinline__ Frag get(int) const { return Frag{}; }

    template <class Ops>
    __device__ __forceinline__ Frag mm(const Frag& X, const Frag& Y, bool same) const {
        return mm_impl<Ops>(X, Y, same, nullptr);
    }
    template <class Ops>
    __device__ __forceinline__ Frag sq_first(const Frag& A) const {
        return mm_impl<Ops>(A, A, true, nullptr);
    }
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
        const int b = buf;
        buf ^= 1;
        double* const xs = sx + b * (ROWS * LD);
        // publish this CTA's rows of Y to every CTA (own tile included)
#pragma unroll
        for (int t = 0; t < T; ++t) {
            const int off = row_of(t) * LD + col_of(t);
            const double2 v = make_double2(Y.v[2 * t], Y.v[2 * t + 1]);
#pragma unroll
            for (int p = 0; p < kClusterCtas; ++p)
                *reinterpret_cast<double2*>(sy_peer[p] + b * (N * LD) + off) = v;
            if (!same)
                *reinterpret_cast<double2*>(xs + lrow_of(t) * LD + col_of(t)) =
                    make_double2(X.v[2 * t], X.v[2 * t + 1]);
        }
        CTRACE("mm_pub");
        cluster_sync();
        CTRACE("mm_sync");
        const double* const ys = sy + b * (N * LD);
        // X rows: the local tile, or (X == Y) this CTA's rows of the Y tile
        const double* const px = same ? ys + ROWS * rank * LD : xs;
        Frag C;
        if constexpr (Ops::kExact) {
#pragma unroll
            for (int t = 0; t < T; ++t) {
                const int r = lrow_of(t), c = col_of(t);
                double c0 = 0.0, c1 = 0.0;
#pragma unroll 4
                for (int k = 0; k < N; k += 2) {
                    const double2 xa = *reinterpret_cast<const double2*>(px + r * LD + k);
                    const double2 y0 = *reinterpret_cast<const double2*>(ys + k * LD + c);
                    const double2 y1 = *reinterpret_cast<const double2*>(ys + (k + 1) * LD + c);
                    c0 = ExactOps::mac(c0, xa.x, y0.x);
                    c1 = ExactOps::mac(c1, xa.x, y0.y);
                    c0 = ExactOps::mac(c0, xa.y, y1.x);
                    c1 = ExactOps::mac(c1, xa.y, y1.y);
                }
                C.v[2 * t] = c0;
                C.v[2 * t + 1] = c1;
            }
        } else {
            // two accumulators per tile (k-steps alternate): the dependent
            // DMMA chain per tile is 8 long instead of 16
            Frag D;
#pragma unroll
            for (int e = 0; e < K; ++e) {
                C.v[e] = init ? init->v[e] : 0.0;
                D.v[e] = 0.0;
            }
            const int ar = lane >> 2, aq = lane & 3;
#pragma unroll 4
            for (int k = 0; k < N; k += 8) {
                double af[2][TR], bf[2][TC];
#pragma unroll
                for (int h = 0; h < 2; ++h) {
#pragma unroll
                    for (int i = 0; i < TR; ++i) af[h][i] = px[(8 * i + ar) * LD + k + 4 * h + aq];
#pragma unroll
                    for (int j = 0; j < TC; ++j) bf[h][j] = ys[(k + 4 * h + aq) * LD + 16 * warp + 8 * j + ar];
                }
#pragma unroll
                for (int i = 0; i < TR; ++i)
#pragma unroll
                    for (int j = 0; j < TC; ++j) {
                        const int t = i * TC + j;
                        dmma_8x8x4(C.v[2 * t], C.v[2 * t + 1], af[0][i], bf[0][j]);
                        dmma_8x8x4(D.v[2 * t], D.v[2 * t + 1], af[1][i], bf[1][j]);
                    }
            }
#pragma unroll
            for (int e = 0; e < K; ++e) C.v[e] += D.v[e];
            CTRACE("mm_done");
        }
        return C;
    }
};

// One cluster of kClusterCtas CTAs per matrix; clusters stride over the batch.
__global__ void __cluster_dims__(kClusterCtas, 1, 1) __launch_bounds__(ClusterGroup64::THREADS, 1)
    expm64_cluster_kernel(const double* __restrict__ a, double* __restrict__ out,
                          mexp_selection* __restrict__ sel, int64_t batch, int acc_arg,
                          int rounding, int exact_s_min) {
    namespace cg = cooperative_groups;
    using G = ClusterGroup64;
    using F = G::Frag;
    constexpr int N = G::N, LD = G::LD;
    extern __shared__ __align__(16) double smem[];
    cg::cluster_group cluster = cg::this_cluster();
    const int accuracy = acc_arg & 15, family = acc_arg >> 4;
    G g;
    g.rank = int(cluster.block_rank());
    g.tid = threadIdx.x;
    g.lane = threadIdx.x & 31;
    g.warp = threadIdx.x >> 5;
    g.buf = 0;
    g.sx = smem;
    g.sy = smem + 2 * G::ROWS * LD;
    g.scal = g.sy + 2 * N * LD;
    for (int p = 0; p < kClusterCtas; ++p) g.sy_peer[p] = cluster.map_shared_rank(g.sy, p);

    const int64_t nclusters = gridDim.x / kClusterCtas;
    for (int64_t m = blockIdx.x / kClusterCtas; m < batch; m += nclusters) {
        const double* am = a + m * int64_t(N) * N;
        CTRACE("start");
        // all_finite and the exact 1-norm (kernels.cpp:44-53) over the whole
        // matrix, redundantly in every CTA (same order, same result): stage A
        // in the local Y tile, one thread per column sums rows 0..63 in order
        double* const ys = g.sy + g.buf * (N * LD);
        __syncthreads();
        bool fin = true;
        {
            // all 16 loads of a thread in flight at once (the latency of one
            // L2/HBM round trip, not sixteen)
            constexpr int kPer = N * N / 2 / G::THREADS;
            double2 v[kPer];
#pragma unroll
            for (int i = 0; i < kPer; ++i)
                v[i] = ld_stream(reinterpret_cast<const double2*>(am) + threadIdx.x + i * G::THREADS);
#pragma unroll
            for (int i = 0; i < kPer; ++i) {
                const int e = threadIdx.x + i * G::THREADS;
                fin = fin && isfinite(v[i].x) && isfinite(v[i].y);
                *reinterpret_cast<double2*>(ys + (2 * e / N) * LD + (2 * e) % N) = v[i];
            }
        }
        const int allfin = __syncthreads_and(fin);
        double colsum = 0.0;
        if (threadIdx.x < N) {
#pragma unroll 8
            for (int i = 0; i < N; ++i) colsum = __dadd_rn(colsum, fabs(ys[i * LD + threadIdx.x]));
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) colsum = fmax(colsum, __shfl_xor_sync(0xffffffffu, colsum, o));
        if (g.lane == 0) g.scal[g.warp] = colsum;
        __syncthreads();
        double norm = g.scal[0];
#pragma unroll
        for (int w = 1; w < kClusterWarps; ++w) norm = fmax(norm, g.scal[w]);
        Sel sl{0, 0, MEXP_OK};
        if (!allfin)
            sl.status = MEXP_ERR_NONFINITE;
        else
            sl = select_device(norm, accuracy, family);
        if (sel && g.rank == 0 && threadIdx.x == 0) {
            mexp_selection r;
            r.norm_in = allfin ? norm : __longlong_as_double(0x7ff8000000000000ll);
            r.degree = int16_t(sl.degree);
            r.s = int16_t(sl.s);
            r.status = sl.status;
            sel[m] = r;
        }
        F A;
#pragma unroll
        for (int t = 0; t < G::T; ++t) {  // this CTA's rows, from the staged tile
            const double2 v = *reinterpret_cast<const double2*>(ys + g.row_of(t) * LD + g.col_of(t));
            A.v[2 * t] = v.x;
            A.v[2 * t + 1] = v.y;
        }
        // every CTA has read the staged A before any CTA writes Y tiles
        CTRACE("prologue");
        G::cluster_sync();
        CTRACE("prologue_sync");
        F X;
        if (sl.status != MEXP_OK) {
#pragma unroll
            for (int e = 0; e < G::K; ++e) X.v[e] = __longlong_as_double(0x7ff8000000000000ll);
        } else {
            const bool exact = rounding == MEXP_ROUND_REFERENCE ||
                               (rounding == MEXP_ROUND_AUTO && sl.s >= exact_s_min);
            if (family == MEXP_FAMILY_TAYLOR_PS) {
                X = exact ? run_expm<ExactOps, MEXP_FAMILY_TAYLOR_PS>(g, A, sl.degree, sl.s)
                          : run_expm<FastOps, MEXP_FAMILY_TAYLOR_PS>(g, A, sl.degree, sl.s);
            } else {
                X = exact ? run_expm<ExactOps>(g, A, sl.degree, sl.s)
                          : run_expm<FastOps>(g, A, sl.degree, sl.s);
            }
        }
        CTRACE("expm_done");
        g.store_global(out + m * int64_t(N) * N, X);
        // the next matrix's staging reuses the Y tiles peers may still read
        G::cluster_sync();
    }
    CTRACE_DUMP();
}

}  // namespace mexp_b200
