// Batched small-n expm in fp32 storage and arithmetic (BASELINE cfg3: 32x32).
//
// Products are FP32 FMAs on the SIMT pipes (never TF32: the tolerance is
// 50*n*2^-24 and TF32 rounds operands to 10 bits), issued as packed FFMA2
// (fma.rn.f32x2, sm_100): two correctly rounded fp32 FMAs per instruction,
// the same FMA rate as scalar FFMA (measured 71 TF either way) with half the
// instructions, which is what this kernel is short of (issue slots and
// instruction cache). One group of W warps per matrix; each lane owns a
// TR x TC register tile of every matrix variable, kept as TC/2 column pairs.
// A product C = X*Y streams X^T and Y rows out of shared memory (X stored
// transposed so a lane's TR rows of column k are one vector load; Y's TC
// columns of row k are TC/4 float4 loads shared by the lanes of a tile
// column). The exact 1-norm and the (m, s) selection run in fp64 on the fp32
// values promoted to double, i.e. exactly the reference's norm of the same
// data (kernels.cpp:44-53), so (m, s) match bit for bit.
#include "device_once.hpp"
#include "expm_small.cuh"
#include "expm_small_f32.cuh"
#include "expm_pairs32.cuh"

namespace mexp_b200 {

struct F32Ops {  // on packed pairs; coefficients rounded once to fp32
    static constexpr bool kExact = false;
    __device__ __forceinline__ static float2 mul(double c, float2 m) {
        const float cf = float(c);
        return __fmul2_rn(make_float2(cf, cf), m);
    }
    __device__ __forceinline__ static float2 add(float2 a, float2 b) { return __fadd2_rn(a, b); }
    __device__ __forceinline__ static float2 mac(float2 acc, double c, float2 m) {
        const float cf = float(c);
        return __ffma2_rn(make_float2(cf, cf), m, acc);
    }
};

template <int N> struct ShapeF32;
//                                   warps  tile rows  tile cols  stash slots
template <> struct ShapeF32<8>  { static constexpr int W = 1, TR = 1, TC = 2, STASH = 4; };
template <> struct ShapeF32<16> { static constexpr int W = 1, TR = 2, TC = 4, STASH = 4; };
// 32x32: one warp per matrix, 4x8 lane tiles (measured: 2 warps of 4x4 tiles
// is shared-memory bound, 824 vs 799 us for cfg3)
template <> struct ShapeF32<32> { static constexpr int W = 1, TR = 4, TC = 8, STASH = 4; };
template <> struct ShapeF32<64> { static constexpr int W = 4, TR = 4, TC = 8, STASH = 4; };

template <int N>
struct GroupF32 {
    using S = ShapeF32<N>;
    static constexpr int W = S::W, TR = S::TR, TC = S::TC, TP = TC / 2;
    static constexpr int THREADS = 32 * W;
    static constexpr int GC = N / TC;          // tile columns
    static constexpr int K = TR * TP;          // column pairs per lane per matrix
    static_assert((N / TR) * GC == THREADS, "tile cover");
    static constexpr int LD = N + 4;           // padded row stride (floats)
    static constexpr int STASH_SLOT = 2 * K * THREADS;
    static constexpr int SMEM_FLOATS = 2 * N * LD + S::STASH * STASH_SLOT + 4 * W + 4;

    struct Frag {
        using T = float2;
        static constexpr int kCount = K;
        float2 v[K];
    };

    float* sxt;  // X transposed: sxt[k * LD + i] = X[i][k]
    float* sy;   // Y row-major
    float* stash;
    double* scal;  // per-warp partial results (8-byte aligned)
    int lane, warp, tid, bar_id, ti, tj;

    // pair p = r * TP + cp of the lane's tile -> row, first column
    __device__ __forceinline__ int row_of(int r) const { return ti * TR + r; }
    __device__ __forceinline__ int col_of(int c) const {
        if constexpr (TC >= 4)
            return 4 * tj + (c & 3) + (c >> 2) * (4 * GC);
        else
            return TC * tj + c;
    }

    __device__ __forceinline__ void sync() const {
        if constexpr (W == 1)
            __syncwarp();
        else
            asm volatile("bar.sync %0, %1;" ::"r"(bar_id), "n"(THREADS) : "memory");
    }

    __device__ __forceinline__ Frag ident() const {
        Frag f;
#pragma unroll
        for (int r = 0; r < TR; ++r)
#pragma unroll
            for (int cp = 0; cp < TP; ++cp) {
                const int c = col_of(2 * cp);
                f.v[r * TP + cp] = make_float2(row_of(r) == c ? 1.f : 0.f, row_of(r) == c + 1 ? 1.f : 0.f);
            }
        return f;
    }

    __device__ __forceinline__ Frag load_global(const float* m) const {
        Frag f;
#pragma unroll
        for (int r = 0; r < TR; ++r) {
            if constexpr (TC >= 4) {
#pragma unroll
                for (int h = 0; h < TC / 4; ++h) {
                    const float4 v = ld_stream(reinterpret_cast<const float4*>(m + row_of(r) * N + col_of(4 * h)));
                    f.v[r * TP + 2 * h] = make_float2(v.x, v.y);
                    f.v[r * TP + 2 * h + 1] = make_float2(v.z, v.w);
                }
            } else {
#pragma unroll
                for (int cp = 0; cp < TP; ++cp)
                    f.v[r * TP + cp] = __ldcs(reinterpret_cast<const float2*>(m + row_of(r) * N + col_of(2 * cp)));
            }
        }
        return f;
    }
    __device__ __forceinline__ void store_global(float* m, const Frag& f) const {
#pragma unroll
        for (int r = 0; r < TR; ++r) {
            if constexpr (TC >= 4) {
#pragma unroll
                for (int h = 0; h < TC / 4; ++h) {
                    const float2 a = f.v[r * TP + 2 * h], b = f.v[r * TP + 2 * h + 1];
                    st_stream(reinterpret_cast<float4*>(m + row_of(r) * N + col_of(4 * h)),
                              make_float4(a.x, a.y, b.x, b.y));
                }
            } else {
#pragma unroll
                for (int cp = 0; cp < TP; ++cp)
                    __stcs(reinterpret_cast<float2*>(m + row_of(r) * N + col_of(2 * cp)), f.v[r * TP + cp]);
            }
        }
    }
    // Operand buffers. TC == 8 shapes (n = 32, 64): both operands row-major,
    // unpadded, with the 16-byte chunk c of row i stored at chunk
    // c ^ swz(i) (swz below); a lane's 8 columns are chunks tj and tj + GC.
    // Per product the lane reads X[its 4 rows][4 k] as four float4 and Y[k][its
    // 8 columns] as two float4 per k: the same vector loads as a transposed X,
    // but no transposing scalar stores, and a squaring (X == Y) stores once.
    // The swizzle makes all three access patterns bank-conflict-free: the X
    // chunk loads (rows 4ti + r over the warp's ti), the Y row loads and the
    // fragment stores (8 lanes per phase over 8 distinct bank quads).
#ifndef MEXP_F32_SWZ
#define MEXP_F32_SWZ 1
#endif
#ifndef MEXP_F32_UNROLL
#define MEXP_F32_UNROLL 4
#endif
    static constexpr int kUnrollQ = MEXP_F32_UNROLL;
    static constexpr bool kSwz = MEXP_F32_SWZ && (TC == 8 && TR == 4);
    __device__ __forceinline__ static int swz(int i) {
        const int t = (i >> 2) & 7;  // 8 row quads -> chunk xor {0,4,1,5,2,6,3,7}
        return ((t & 1) << 2) | (t >> 1);
    }
    __device__ __forceinline__ static int at(int i, int j) {  // element (i, j) of a buffer
        if constexpr (kSwz)
            return i * N + 4 * ((j >> 2) ^ swz(i)) + (j & 3);
        else
            return i * LD + j;
    }

    __device__ __forceinline__ void store_rows(float* s, const Frag& f) const {
        if constexpr (kSwz) {
#pragma unroll
            for (int r = 0; r < TR; ++r) {
                const int i = row_of(r);
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const float2 a = f.v[r * TP + 2 * h], b = f.v[r * TP + 2 * h + 1];
                    *reinterpret_cast<float4*>(s + i * N + 4 * ((tj + h * GC) ^ swz(i))) =
                        make_float4(a.x, a.y, b.x, b.y);
                }
            }
        } else {
#pragma unroll
            for (int r = 0; r < TR; ++r)
#pragma unroll
                for (int cp = 0; cp < TP; ++cp)
                    *reinterpret_cast<float2*>(s + row_of(r) * LD + col_of(2 * cp)) = f.v[r * TP + cp];
        }
    }
    __device__ __forceinline__ void store_cols(float* s, const Frag& f) const {
#pragma unroll
        for (int cp = 0; cp < TP; ++cp)
#pragma unroll
            for (int r = 0; r < TR; ++r) {
                s[col_of(2 * cp) * LD + row_of(r)] = f.v[r * TP + cp].x;
                s[(col_of(2 * cp) + 1) * LD + row_of(r)] = f.v[r * TP + cp].y;
            }
    }

    __device__ __forceinline__ void put(int slot, const Frag& f) const {
        float2* p = reinterpret_cast<float2*>(stash + slot * STASH_SLOT);
#pragma unroll
        for (int e = 0; e < K; ++e) p[e * THREADS + tid] = f.v[e];
    }
    __device__ __forceinline__ Frag get(int slot) const {
        const float2* p = reinterpret_cast<const float2*>(stash + slot * STASH_SLOT);
        Frag f;
#pragma unroll
        for (int e = 0; e < K; ++e) f.v[e] = p[e * THREADS + tid];
        return f;
    }

    template <class Ops>
    __device__ __forceinline__ Frag mm(const Frag& X, const Frag& Y, bool same) const {
        return mm_impl(X, Y, nullptr, same);
    }
    template <class Ops>
    __device__ __forceinline__ Frag mm_add(const Frag& X, const Frag& Y, bool same,
                                           const Frag& B) const {
        return mm_impl(X, Y, &B, same);
    }
    template <class Ops>
    __device__ __forceinline__ Frag sq_first(const Frag& A) const {
        return mm_impl(A, A, nullptr, true);
    }
#ifndef MEXP_F32_NOINLINE
#define MEXP_F32_NOINLINE 1
#endif
#if MEXP_F32_NOINLINE
#define MEXP_F32_KLOOP_ATTR __noinline__
#else
#define MEXP_F32_KLOOP_ATTR __forceinline__
#endif
    // C += X * Y over the swizzled buffers: pxl = the lane's first X row,
    // sxl = its chunk xor. One out-of-line copy serves every product of the
    // schemes and squarings (inlined copies overflow the instruction cache).
    __device__ MEXP_F32_KLOOP_ATTR static Frag kloop(const float* pxl, const float* sy, int sxl, int tj,
                                                     Frag C) {
            // software-pipelined k loop: the next k-chunk of X and the next row
            // of Y are loaded while the current ones feed the FFMA2s. All
            // swizzles are per chunk q (Y) or per lane (X): addresses are a
            // base pointer plus immediates.
            constexpr int C1 = 4 * GC;           // offset of the lane's 2nd column chunk
            float4 xc[TR], yc[2];
#pragma unroll
            for (int r = 0; r < TR; ++r) xc[r] = *reinterpret_cast<const float4*>(pxl + r * N + 4 * sxl);
            int c0 = 4 * tj;  // chunk 0's swizzle is 0
            yc[0] = *reinterpret_cast<const float4*>(sy + c0);
            yc[1] = *reinterpret_cast<const float4*>(sy + (c0 ^ C1));
#pragma unroll kUnrollQ
            for (int q = 0; q < N / 4; ++q) {
                const int qn = (q + 1) & (N / 4 - 1);
                const float* xq = pxl + 4 * (qn ^ sxl);
                float4 xn[TR];
#pragma unroll
                for (int r = 0; r < TR; ++r) xn[r] = *reinterpret_cast<const float4*>(xq + r * N);
                const float* yq = sy + 4 * q * N + c0;
                const int c0n = 4 * (tj ^ swz(4 * qn));
                const float* yqn = sy + 4 * qn * N;
#pragma unroll
                for (int kk = 0; kk < 4; ++kk) {
                    float4 yn[2];
                    if (kk < 3) {
                        yn[0] = *reinterpret_cast<const float4*>(yq + (kk + 1) * N);
                        yn[1] = *reinterpret_cast<const float4*>(yq + (kk + 1) * N + ((c0 ^ C1) - c0));
                    } else {
                        yn[0] = *reinterpret_cast<const float4*>(yqn + c0n);
                        yn[1] = *reinterpret_cast<const float4*>(yqn + (c0n ^ C1));
                    }
#pragma unroll
                    for (int r = 0; r < TR; ++r) {
                        const float a = kk == 0 ? xc[r].x : kk == 1 ? xc[r].y : kk == 2 ? xc[r].z : xc[r].w;
#pragma unroll
                        for (int h = 0; h < 2; ++h) {
                            C.v[r * TP + 2 * h] = __ffma2_rn(make_float2(a, a), make_float2(yc[h].x, yc[h].y),
                                                             C.v[r * TP + 2 * h]);
                            C.v[r * TP + 2 * h + 1] = __ffma2_rn(make_float2(a, a), make_float2(yc[h].z, yc[h].w),
                                                                 C.v[r * TP + 2 * h + 1]);
                        }
                    }
#pragma unroll
                    for (int h = 0; h < 2; ++h) yc[h] = yn[h];
                }
#pragma unroll
                for (int r = 0; r < TR; ++r) xc[r] = xn[r];
                c0 = c0n;
            }
        return C;
    }

    __device__ __forceinline__ Frag mm_impl(const Frag& X, const Frag& Y, const Frag* init,
                                            bool same) const {
        Frag C;
#pragma unroll
        for (int e = 0; e < K; ++e) C.v[e] = init ? init->v[e] : make_float2(0.f, 0.f);
        if constexpr (kSwz) {
            sync();
            store_rows(sy, Y);
            if (!same) store_rows(sxt, X);
            sync();
            const float* px = same ? sy : sxt;
            C = kloop(px + 4 * ti * N, sy, swz(4 * ti), tj, C);
        } else {
            sync();
            store_cols(sxt, X);
            store_rows(sy, Y);
            sync();
#pragma unroll 2
            for (int k = 0; k < N; ++k) {
                float a[TR];
                float2 b[TP];
                const float* xa = sxt + k * LD + ti * TR;
#pragma unroll
                for (int r = 0; r < TR; ++r) a[r] = xa[r];
                const float* yb = sy + k * LD;
#pragma unroll
                for (int cp = 0; cp < TP; ++cp) b[cp] = *reinterpret_cast<const float2*>(yb + col_of(2 * cp));
#pragma unroll
                for (int r = 0; r < TR; ++r)
#pragma unroll
                    for (int cp = 0; cp < TP; ++cp)
                        C.v[r * TP + cp] = __ffma2_rn(make_float2(a[r], a[r]), b[cp], C.v[r * TP + cp]);
            }
        }
        return C;
    }
};

template <int N, int GPC, int kFamily = MEXP_FAMILY_TAYLOR_NEW>
__global__ void __launch_bounds__(32 * ShapeF32<N>::W * GPC)
    expm_small_f32_kernel(const float* __restrict__ a, float* __restrict__ out,
                          mexp_selection* __restrict__ sel, int64_t batch, int acc_arg) {
    const int accuracy = acc_arg & 15;  // mexp_accuracy (low nibble)
    constexpr int family = kFamily;
    using G = GroupF32<N>;
    using F = typename G::Frag;
    extern __shared__ __align__(16) float smemf[];
    const int gid = threadIdx.x / G::THREADS;
    G g;
    float* base = smemf + gid * G::SMEM_FLOATS;
    g.sxt = base;
    g.sy = base + N * G::LD;
    g.stash = base + 2 * N * G::LD;
    g.scal = reinterpret_cast<double*>(g.stash + G::S::STASH * G::STASH_SLOT);
    g.tid = threadIdx.x % G::THREADS;
    g.lane = g.tid & 31;
    g.warp = g.tid >> 5;
    g.bar_id = 1 + gid;
    g.ti = g.tid / G::GC;
    g.tj = g.tid % G::GC;
    if constexpr (N == 32) {
        // An aligned quad of lanes owns a 2x2 block of lane tiles (bit 8 of
        // acc_arg; MEXP_F32_LANES=0 keeps lane = 4 ti + tj). The shared-memory
        // pipe merges identical addresses only inside an aligned lane quad and
        // serves 8 (quad, address) requests per LDS.128 wavefront
        // (tools/lds_patterns.cu): the Y row loads (address by tj) then cost 2
        // wavefronts instead of 4, the X loads (address by ti) 2 as before --
        // 24 instead of 40 wavefronts per 4 k. Lanes move only inside their
        // group of 8, so every per-phase bank-conflict property of the swizzle
        // holds; same arithmetic per element, so the same bits.
        if (acc_arg & 0x100) {
            const int l = g.lane;
            g.ti = ((l >> 3) << 1) | ((l >> 1) & 1);
            g.tj = (((l >> 2) & 1) << 1) | (l & 1);
        }
    }

    constexpr int64_t NN = int64_t(N) * N;
    const int64_t stride = int64_t(gridDim.x) * GPC;
    for (int64_t m = int64_t(blockIdx.x) * GPC + gid; m < batch; m += stride) {
        F A = g.load_global(a + m * NN);
        bool fin = true;
#pragma unroll
        for (int e = 0; e < G::K; ++e) fin = fin && isfinite(A.v[e].x) && isfinite(A.v[e].y);
        g.sync();
        g.store_rows(g.sy, A);
        g.sync();
        // exact 1-norm of the promoted values, rows ascending (kernels.cpp:44-53)
        double colsum = 0.0;
        for (int j = g.tid; j < N; j += G::THREADS) {
            double s = 0.0;
            for (int i = 0; i < N; ++i) s = __dadd_rn(s, fabs(double(g.sy[G::at(i, j)])));
            colsum = fmax(colsum, s);
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
        if (!allfin)
            sl.status = MEXP_ERR_NONFINITE;
        else
            sl = select_device(norm, accuracy, family);
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
            const float nan = __int_as_float(0x7fc00000);
#pragma unroll
            for (int e = 0; e < G::K; ++e) X.v[e] = make_float2(nan, nan);
        } else {
            if (sl.s > 0) {  // exact scaling by 2^-s, rounded once to float
                const double f = pow2_neg(sl.s);
#pragma unroll
                for (int e = 0; e < G::K; ++e)
                    A.v[e] = make_float2(float(f * double(A.v[e].x)), float(f * double(A.v[e].y)));
            }
            // (the Pade family in fp32 storage runs on the fp64 engine, capi.cu)
            if constexpr (family == MEXP_FAMILY_TAYLOR_PS)
                X = eval_taylor_ps<F32Ops>(g, sl.degree, A);
            else
                X = eval_taylor_new<F32Ops>(g, sl.degree, A);
            for (int i = 0; i < sl.s; ++i) X = g.template mm<F32Ops>(X, X, true);
        }
        g.store_global(out + m * NN, X);
    }
}

namespace {
int sm_count() {
    static int v = [] {
        int dev = 0, s = 148;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&s, cudaDevAttrMultiProcessorCount, dev);
        return s;
    }();
    return v;
}

template <int N, int GPC, int kFamily>
int launch_f32(const float* a, float* out, mexp_selection* sel, int64_t batch, int accuracy,
               cudaStream_t st, std::atomic<uint64_t>* launches) {
    using G = GroupF32<N>;
    auto kern = expm_small_f32_kernel<N, GPC, kFamily>;
    const size_t smem = size_t(G::SMEM_FLOATS) * GPC * sizeof(float);
    static PerDevice attr_once;
    attr_once([&] { cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)); });
    static int bps = [&] {
        int b = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, kern, G::THREADS * GPC, smem);
        return b > 0 ? b : 1;
    }();
    const int64_t want = (batch + GPC - 1) / GPC;
    const int64_t cap = int64_t(bps) * sm_count();
    const int grid = int(want < cap ? want : cap);
    if (grid == 0) return MEXP_OK;
    static const int quad_lanes = [] {
        const char* e = std::getenv("MEXP_F32_LANES");
        return (e ? std::atoi(e) : 1) ? 0x100 : 0;
    }();
    kern<<<grid, G::THREADS * GPC, smem, st>>>(a, out, sel, batch, accuracy | quad_lanes);
    launches->fetch_add(1, std::memory_order_relaxed);
    return cudaGetLastError() == cudaSuccess ? MEXP_OK : MEXP_ERR_CUDA;
}
}  // namespace

template <int kFamily>
int run_small_f32_family(const float* d_a, float* d_out, mexp_selection* d_sel, int np,
                         int64_t batch, int acc_arg, cudaStream_t st,
                         std::atomic<uint64_t>* launches) {
    switch (np) {
        case 8: return launch_f32<8, 8, kFamily>(d_a, d_out, d_sel, batch, acc_arg, st, launches);
        case 16: return launch_f32<16, 4, kFamily>(d_a, d_out, d_sel, batch, acc_arg, st, launches);
        case 32:
            if (kFamily == MEXP_FAMILY_TAYLOR_NEW && pairs32_enabled(batch))
                return run_pairs32_f32(d_a, d_out, d_sel, batch, acc_arg, st, launches);
            return launch_f32<32, 2, kFamily>(d_a, d_out, d_sel, batch, acc_arg, st, launches);
        case 64: return launch_f32<64, 1, kFamily>(d_a, d_out, d_sel, batch, acc_arg, st, launches);
    }
    return MEXP_ERR_UNSUPPORTED;
}

// acc_arg = mexp_accuracy | mexp_family << 4; one kernel instantiation per family
int run_small_f32(const float* d_a, float* d_out, mexp_selection* d_sel, int np, int64_t batch,
                  int acc_arg, cudaStream_t st, std::atomic<uint64_t>* launches) {
    if ((acc_arg >> 4) == MEXP_FAMILY_TAYLOR_PS)
        return run_small_f32_family<MEXP_FAMILY_TAYLOR_PS>(d_a, d_out, d_sel, np, batch, acc_arg,
                                                           st, launches);
    return run_small_f32_family<MEXP_FAMILY_TAYLOR_NEW>(d_a, d_out, d_sel, np, batch, acc_arg, st,
                                                        launches);
}

}  // namespace mexp_b200
