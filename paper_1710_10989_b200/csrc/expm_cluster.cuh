// Latency path for few fp64 matrices of n in (32, 64] (cfg1: ONE 64x64
// matrix): a thread-block cluster of 4 CTAs on 4 SMs computes one expm.
//
// The 64 x 64 variables are split 2 x 2: CTA r = 2 bi + bj owns block
// (bi, bj) as DMMA-accumulator fragments. A product exchanges blocks through
// distributed shared memory with st.async (bytes counted on the receiver's
// mbarrier), so the only waits in the product chain are each CTA's wait for
// its own two panels; see ClusterGroup64. The exact 1-norm (sequential over
// all rows, as the reference sums) is computed redundantly by every CTA from
// the whole matrix.
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

__device__ __forceinline__ uint32_t cta_smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
// the same shared-memory offset in CTA `rank` of the cluster
__device__ __forceinline__ uint32_t peer_addr(uint32_t local, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(local), "r"(rank));
    return r;
}
// 16 bytes into a peer CTA's shared memory; completes as transaction bytes
// on the peer's mbarrier (measured faster here than row-wise bulk copies)
__device__ __forceinline__ void st_async2(uint32_t addr, double a, double b, uint32_t mbar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];" ::"r"(
                     addr),
                 "d"(a), "d"(b), "r"(mbar)
                 : "memory");
}

// 2 x 2 block decomposition: CTA rank r = 2 bi + bj owns block (bi, bj) of
// every matrix variable (32 x 32; 4 warps, each a 16 x 16 quarter). C = X Y
// needs X's row panel bi and Y's column panel bj: each CTA writes its X and
// Y blocks into its own panels and, with st.async, into the row neighbour's
// (r ^ 1) row panel and the column neighbour's (r ^ 2) column panel; the
// bytes complete on the receiver's mbarrier -- 16 KB each way per product.
// A CTA waits for its 16 KB (and __syncthreads for its own blocks) and
// computes its block locally. No cluster-wide barrier in the product loop.
// Panels are double-buffered by product parity; a CTA writes a buffer only
// after both neighbours have sent it the previous product's data, i.e.
// after they finished reading it.
struct ClusterGroup64 {
    using S = ClusterShape;
    static constexpr int N = 64;
    static constexpr int B = N / 2;       // block size
    static constexpr int TR = 2, TC = 2;  // tiles per warp
    static constexpr int T = TR * TC;
    static constexpr int K = 2 * T;       // doubles per lane per matrix
    static constexpr int LDX = N + 4;     // row panel [B][LDX]
    static constexpr int LDY = B + 4;     // column panel [N][LDY]
    static constexpr int LD = N;          // the prologue's staging tile (64 x 64)
    static constexpr int THREADS = 32 * kClusterWarps;
    static constexpr int X_DOUBLES = B * LDX, Y_DOUBLES = N * LDY;
    // two row panels, two column panels, the staging tile, scalars, mbarriers
    static constexpr int SMEM_DOUBLES = 2 * X_DOUBLES + 2 * Y_DOUBLES + N * N + 2 * kClusterWarps + 2 + 2;
    static constexpr unsigned kPeerBytes = 2u * B * B * sizeof(double);  // the two incoming blocks

    struct Frag {
        using T = double;
        static constexpr int kCount = K;
        double v[K];
    };

    double* sx;     // 2 row panels
    double* sy;     // 2 column panels
    double* stage;  // A, whole, for the 1-norm (no peer ever writes it)
    double* scal;
    uint64_t* mbar; // 2 mbarriers (one per panel buffer)
    uint32_t sx_row, sy_col, mbar_row, mbar_col;  // neighbours' addresses (buffer 0)
    uint32_t mbar_me;
    int rank, bi, bj, lane, warp, tid;
    mutable int buf;
    mutable unsigned phase;  // bit b: parity of mbarrier b

    __device__ __forceinline__ int lrow(int t) const { return 16 * (warp >> 1) + 8 * (t / TC) + (lane >> 2); }
    __device__ __forceinline__ int lcol(int t) const { return 16 * (warp & 1) + 8 * (t % TC) + 2 * (lane & 3); }
    __device__ __forceinline__ int row_of(int t) const { return B * bi + lrow(t); }
    __device__ __forceinline__ int col_of(int t) const { return B * bj + lcol(t); }

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
                                           const Frag& Bm) const {
        if constexpr (Ops::kExact) {
            Frag P = mm_impl<Ops>(X, Y, same, nullptr);
#pragma unroll
            for (int e = 0; e < K; ++e) P.v[e] = Ops::add(P.v[e], Bm.v[e]);
            return P;
        } else {
            return mm_impl<Ops>(X, Y, same, &Bm);
        }
    }

    template <class Ops>
    __device__ __forceinline__ Frag mm_impl(const Frag& X, const Frag& Y, bool,
                                            const Frag* init) const {
        const int b = buf;
        buf ^= 1;
        const uint32_t xo = uint32_t(b * X_DOUBLES * sizeof(double));
        const uint32_t yo = uint32_t(b * Y_DOUBLES * sizeof(double));
        const uint32_t mo = uint32_t(b * sizeof(uint64_t));
        if (tid == 0)
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mbar_me + mo),
                         "r"(kPeerBytes)
                         : "memory");
        // X block -> row panels (row neighbour's, own) at columns [B bj, B bj + B);
        // Y block -> column panels (column neighbour's, own) at rows [B bi, B bi + B)
        double* const pxb = sx + b * X_DOUBLES;
        double* const pyb = sy + b * Y_DOUBLES;
#pragma unroll
        for (int t = 0; t < T; ++t) {
            const int xi = lrow(t) * LDX + B * bj + lcol(t);
            const int yi = (B * bi + lrow(t)) * LDY + lcol(t);
            st_async2(sx_row + xo + uint32_t(xi * sizeof(double)), X.v[2 * t], X.v[2 * t + 1], mbar_row + mo);
            st_async2(sy_col + yo + uint32_t(yi * sizeof(double)), Y.v[2 * t], Y.v[2 * t + 1], mbar_col + mo);
            *reinterpret_cast<double2*>(pxb + xi) = make_double2(X.v[2 * t], X.v[2 * t + 1]);
            *reinterpret_cast<double2*>(pyb + yi) = make_double2(Y.v[2 * t], Y.v[2 * t + 1]);
        }
        __syncthreads();  // own blocks
        CTRACE("mm_sent");
        // both panels complete (all 32 KB landed)
        const unsigned par = (phase >> b) & 1u;
        asm volatile(
            "{\n"
            ".reg .pred P1;\n"
            "WAIT:\n"
            "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P1, [%0], %1;\n"
            "@!P1 bra WAIT;\n"
            "}\n" ::"r"(mbar_me + mo),
            "r"(par)
            : "memory");
        phase ^= 1u << b;
        CTRACE("mm_landed");
        const double* const px = sx + b * X_DOUBLES;
        const double* const py = sy + b * Y_DOUBLES;
        Frag C;
        if constexpr (Ops::kExact) {
#pragma unroll
            for (int t = 0; t < T; ++t) {
                const int r = lrow(t), c = lcol(t);
                double c0 = 0.0, c1 = 0.0;
#pragma unroll 4
                for (int k = 0; k < N; k += 2) {
                    const double2 xa = *reinterpret_cast<const double2*>(px + r * LDX + k);
                    const double2 y0 = *reinterpret_cast<const double2*>(py + k * LDY + c);
                    const double2 y1 = *reinterpret_cast<const double2*>(py + (k + 1) * LDY + c);
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
            for (int e = 0; e < K; ++e) C.v[e] = init ? init->v[e] : 0.0;
            const int ar = lane >> 2, aq = lane & 3;
            const double* const pxw = px + (16 * (warp >> 1) + ar) * LDX + aq;
            const double* const pyw = py + aq * LDY + 16 * (warp & 1) + ar;
#pragma unroll 4
            for (int k = 0; k < N; k += 4) {
                double af[TR], bf[TC];
#pragma unroll
                for (int i = 0; i < TR; ++i) af[i] = pxw[8 * i * LDX + k];
#pragma unroll
                for (int j = 0; j < TC; ++j) bf[j] = pyw[k * LDY + 8 * j];
#pragma unroll
                for (int i = 0; i < TR; ++i)
#pragma unroll
                    for (int j = 0; j < TC; ++j)
                        dmma_8x8x4(C.v[2 * (i * TC + j)], C.v[2 * (i * TC + j) + 1], af[i], bf[j]);
            }
            CTRACE("mm_done");
        }
        return C;
    }
};

// One cluster of kClusterCtas CTAs per matrix; clusters stride over the batch.
// one instantiation per family: a smaller kernel image (its first launch after
// an L2 flush fetches every instruction line from HBM)
template <int kFamily>
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
    const int accuracy = acc_arg & 15;
    constexpr int family = kFamily;
    G g;
    g.rank = int(cluster.block_rank());
    g.bi = g.rank >> 1;
    g.bj = g.rank & 1;
    g.tid = threadIdx.x;
    g.lane = threadIdx.x & 31;
    g.warp = threadIdx.x >> 5;
    g.buf = 0;
    g.phase = 0;
    g.sx = smem;
    g.sy = smem + 2 * G::X_DOUBLES;
    g.stage = g.sy + 2 * G::Y_DOUBLES;
    g.scal = g.stage + N * N;
    g.mbar = reinterpret_cast<uint64_t*>(g.scal + 2 * kClusterWarps + 2);
    g.mbar_me = cta_smem_u32(g.mbar);
    g.sx_row = peer_addr(cta_smem_u32(g.sx), unsigned(g.rank ^ 1));
    g.mbar_row = peer_addr(g.mbar_me, unsigned(g.rank ^ 1));
    g.sy_col = peer_addr(cta_smem_u32(g.sy), unsigned(g.rank ^ 2));
    g.mbar_col = peer_addr(g.mbar_me, unsigned(g.rank ^ 2));
    if (threadIdx.x == 0) {
        for (int i = 0; i < 2; ++i)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(g.mbar_me + 8u * i) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    // the mbarriers are initialised before any peer signals them; after this
    // one barrier the CTAs only wait on their own mbarriers
    G::cluster_sync();

    const int64_t nclusters = gridDim.x / kClusterCtas;
    for (int64_t m = blockIdx.x / kClusterCtas; m < batch; m += nclusters) {
        const double* am = a + m * int64_t(N) * N;
        CTRACE("start");
        // all_finite and the exact 1-norm (kernels.cpp:44-53) over the whole
        // matrix, redundantly in every CTA (same order, same result): stage A
        // in the local Y tile, one thread per column sums rows 0..63 in order
        double* const ys = g.stage;
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
        // (no barrier: peers write only the panels, never the staging tile;
        // a panel is written only after its owner sent that panel buffer's
        // previous data, see ClusterGroup64)
        CTRACE("prologue");
        F X;
        if (sl.status != MEXP_OK) {
#pragma unroll
            for (int e = 0; e < G::K; ++e) X.v[e] = __longlong_as_double(0x7ff8000000000000ll);
        } else {
            const bool exact = rounding == MEXP_ROUND_REFERENCE ||
                               (rounding == MEXP_ROUND_AUTO && sl.s >= exact_s_min);
            X = exact ? run_expm<ExactOps, family>(g, A, sl.degree, sl.s)
                      : run_expm<FastOps, family>(g, A, sl.degree, sl.s);
        }
        CTRACE("expm_done");
        g.store_global(out + m * int64_t(N) * N, X);
        // no cluster barrier here: every byte a peer sent this CTA has been
        // waited for, and the next matrix's staging starts with __syncthreads
    }
    CTRACE_DUMP();
}

}  // namespace mexp_b200
