// Batched 8x8 fp64 expm (BASELINE cfg2): one warp per matrix, no tile of the
// matrix ever leaves the warp except one 512-byte shared-memory transpose per
// product.
//
// Lane l = 4r + q holds M[r][2q], M[r][2q+1] of every matrix variable M --
// the accumulator layout of the FP64 tensor-core MMA m8n8k4 (DMMA), and the
// layout a coalesced 16-byte load of a row-major 8x8 block gives directly.
//
// Product C = X*Y as two DMMAs with the summation index permuted: DMMA #1
// sums k in {0,2,4,6}, DMMA #2 k in {1,3,5,7}. Then the A operand lane l
// needs is X[r][2q] (#1) and X[r][2q+1] (#2) -- its own registers -- and the
// B operand is Y[2q][r], Y[2q+1][r]: Y transposed, obtained by one 16-byte
// store and two 8-byte loads per lane through a 512-byte tile whose 16-byte
// unit (i, c) (row i, column pair c) sits at slot 8c + (i ^ c). That swizzle
// makes the store (4 wavefronts), the transposed loads (2 + 2), the row
// loads of the exact path and the column reads of the 1-norm conflict-free.
//
// Reference-exact rounding (ExactOps) computes c_rj = 0.0 + x_r0*y_0j + ... +
// x_r7*y_7j with separately rounded DMUL/DADD in k order, as the reference's
// i-k-j loop does (kernels.cpp:16-27), from the same tile.
#pragma once

#include "expm_small.cuh"

namespace mexp_b200 {

#ifdef MEXP_N8_NOSYNC_EXPERIMENT  // measurement only: compiler barrier instead of the warp barrier
#define MEXP_N8_SYNC() asm volatile("" ::: "memory")
#else
#define MEXP_N8_SYNC() __syncwarp()
#endif

// Byte offset of the 16-byte unit (i, c) = (M[i][2c], M[i][2c+1]) in a
// warp's 512-byte tile. The slot
//   8*(i>>1) | 4*((i&1) ^ (i>>2)) | 2*(((c>>1) ^ (i>>1)) & 1) | (c&1)
// is a bijection onto 32 slots that is bank-conflict-free per access phase
// (8 lanes for 16-byte, 16 lanes for 8-byte accesses) for: the lane stores
// (r, q); the transposed 8-byte loads (2q, r) and (2q+1, r); the row loads
// (r, c) and column-pair loads (k, q) of the exact product; and the column
// reads of the 1-norm (verified exhaustively in tests/test_layouts.py).
// Note unit8(i, c) == unit8(i, 0) ^ (c << 4).
__host__ __device__ __forceinline__ constexpr uint32_t unit8(int i, int c) {
    return uint32_t(((i >> 1) << 3) | (((i & 1) ^ (i >> 2)) << 2) |
                    ((((c >> 1) ^ (i >> 1)) & 1) << 1) | (c & 1))
           << 4;
}

// kSharedY: the reference-rounded product's Y operand goes through a warp-wide
// scratch tile (ytile) instead of the second half of the matrix's own 1 KB tile.
template <bool kSplit, bool kSharedY = false>
struct Group8T {
    struct S {
        static constexpr int STASH = 0;
    };
    static constexpr int K = 2;
    struct Frag {
        using T = double;
        static constexpr int kCount = 2;
        double v[2];
    };

    char* tile;      // this warp's tiles: [0, 512) X / fast, [512, 1024) Y (exact)
    char* ytile;     // kSharedY: the Y (exact) scratch tile
    __device__ __forceinline__ char* ybase() const { return kSharedY ? ytile : tile + 512; }
    uint32_t st;     // unit (r, q)
    uint32_t ld0;    // element (2q,   r)
    uint32_t ld1;    // element (2q+1, r)
    uint32_t rowb;   // unit (r, 0)
    uint32_t qx;     // q << 4: unit (k, q) = unit8(k, 0) ^ qx
    int r, q;
    double fscale;   // 2^-s, applied to the staged (unscaled) A by sq_first
    bool scaled;     // s > 0
    // the scaled A's transposed DMMA operand, kept from sq_first for A3 = A2 A
    static constexpr bool kKeepsAT = true;
    mutable double bt0, bt1;

    __device__ __forceinline__ void init(char* warp_tile, int lane) {
        tile = warp_tile;
        set_lanes(lane, false);
        fscale = 1.0;
        scaled = true;
    }
    // Which unit (r, q) = (M[r][2q], M[r][2q+1]) a lane owns.
    //   DMMA mapping (quads = false): lane = 4r + q, the m8n8k4 accumulator layout.
    //   Quad mapping (quads = true; reference-rounded products only): an aligned
    //   quad of lanes owns a 2x2 block of units, r = 2(l>>3) + ((l>>1)&1),
    //   q = 2((l>>2)&1) + (l&1). The shared-memory pipe merges identical addresses
    //   only inside an aligned lane quad and serves 8 (quad, address) requests
    //   per LDS.128 wavefront, never fewer than 2 wavefronts per LDS.128
    //   (tools/lds_patterns.cu), so the X-row loads (address by r) and the Y
    //   column-pair loads (address by q) cost 2 wavefronts each, against 2
    //   and 4 with lane = 4r + q: 28 instead of 44
    //   wavefronts per product, which is what bounds the reference-rounded
    //   product (profiles/cfg2_variants_r2.txt). Same arithmetic per element,
    //   so the same bits; the owner of unit (r, q) loads and stores it at
    //   row-major position 4r + q either way.
    __device__ __forceinline__ void set_lanes(int lane, bool quads) {
        r = quads ? ((lane >> 3) << 1) | ((lane >> 1) & 1) : lane >> 2;
        q = quads ? (((lane >> 2) & 1) << 1) | (lane & 1) : lane & 3;
        st = unit8(r, q);
        ld0 = unit8(2 * q, r >> 1) + ((r & 1) << 3);
        ld1 = unit8(2 * q + 1, r >> 1) + ((r & 1) << 3);
        rowb = unit8(r, 0);
        qx = uint32_t(q) << 4;
    }
    __device__ __forceinline__ int unit_index() const { return 4 * r + q; }

    // The diagonal test goes through an opaque (volatile) move, re-evaluated
    // per matrix: otherwise the compiler hoists every identity term
    // (diag ? c : 0, one per scheme coefficient) out of the batch loop as
    // loop-invariant values, keeps them in ~30 registers and spills them.
    __device__ __forceinline__ Frag ident() const {
        int d;
        asm volatile("sub.s32 %0, %1, %2;" : "=r"(d) : "r"(r), "r"(2 * q));
        Frag f;
        f.v[0] = d == 0 ? 1.0 : 0.0;
        f.v[1] = d == 1 ? 1.0 : 0.0;
        return f;
    }

    template <class Ops>
    __device__ __forceinline__ Frag mm(const Frag& X, const Frag& Y, bool same) const {
        return mm_impl<Ops>(X, Y, same, nullptr);
    }
    template <class Ops>
    __device__ __forceinline__ Frag mm_add(const Frag& X, const Frag& Y, bool same,
                                           const Frag& B) const {
        if constexpr (Ops::kExact) {
            Frag P = mm_impl<Ops>(X, Y, same, nullptr);
            P.v[0] = Ops::add(P.v[0], B.v[0]);
            P.v[1] = Ops::add(P.v[1], B.v[1]);
            return P;
        } else {
            return mm_impl<Ops>(X, Y, same, &B);
        }
    }
    // A2 = A*A for the scaled A, right after the 1-norm staged the UNSCALED A
    // in the tile (fast path): the transposed operand is read from there and
    // scaled on load (exact: a power of two).
    template <class Ops>
    __device__ __forceinline__ Frag sq_first(const Frag& A) const {
        if constexpr (Ops::kExact) {
            return mm_impl<Ops>(A, A, true, nullptr);
        } else {
            double y0 = *reinterpret_cast<const double*>(tile + ld0);
            double y1 = *reinterpret_cast<const double*>(tile + ld1);
            if (scaled) {  // s > 0 (predicated: no FP64-pipe slot when s = 0)
                y0 *= fscale;
                y1 *= fscale;
            }
            bt0 = y0;
            bt1 = y1;
            Frag C;
            C.v[0] = C.v[1] = 0.0;
            if constexpr (kSplit) {
                double e0 = 0.0, e1 = 0.0;
                dmma_8x8x4(C.v[0], C.v[1], A.v[0], y0);
                dmma_8x8x4(e0, e1, A.v[1], y1);
                C.v[0] += e0;
                C.v[1] += e1;
            } else {
                dmma_8x8x4(C.v[0], C.v[1], A.v[0], y0);
                dmma_8x8x4(C.v[0], C.v[1], A.v[1], y1);
            }
            return C;
        }
    }

    // X * A with the operand sq_first left in registers (no staging round
    // trip; the same DMMA operand values, so the same bits)
    template <class Ops>
    __device__ __forceinline__ Frag mm_a(const Frag& X, const Frag& A) const {
        if constexpr (Ops::kExact) {
            return mm_impl<Ops>(X, A, false, nullptr);
        } else {
            Frag C;
            C.v[0] = C.v[1] = 0.0;
            dmma_8x8x4(C.v[0], C.v[1], X.v[0], bt0);
            dmma_8x8x4(C.v[0], C.v[1], X.v[1], bt1);
            return C;
        }
    }

    template <class Ops>
    __device__ __forceinline__ Frag mm_impl(const Frag& X, const Frag& Y, bool same,
                                            const Frag* init) const {
        Frag C;
        MEXP_N8_SYNC();  // readers of the previous product are done with the tile
        if constexpr (Ops::kExact) {
            *reinterpret_cast<double2*>(tile + st) = make_double2(X.v[0], X.v[1]);
            if (!same) *reinterpret_cast<double2*>(ybase() + st) = make_double2(Y.v[0], Y.v[1]);
            MEXP_N8_SYNC();
            const char* ty = same ? tile : ybase();
            double c0 = 0.0, c1 = 0.0;
            // row r of X in two halves (k ascending): 8 registers live, not 16
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                double x[4];
#pragma unroll
                for (int c = 0; c < 2; ++c) {
                    const double2 v = *reinterpret_cast<const double2*>(tile + (rowb ^ ((2 * h + c) << 4)));
                    x[2 * c] = v.x;
                    x[2 * c + 1] = v.y;
                }
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const double2 y = *reinterpret_cast<const double2*>(ty + (unit8(4 * h + k, 0) ^ qx));
                    c0 = ExactOps::mac(c0, x[k], y.x);
                    c1 = ExactOps::mac(c1, x[k], y.y);
                }
            }
            C.v[0] = c0;
            C.v[1] = c1;
        } else {
            *reinterpret_cast<double2*>(tile + st) = make_double2(Y.v[0], Y.v[1]);
            MEXP_N8_SYNC();
            const double y0 = *reinterpret_cast<const double*>(tile + ld0);
            const double y1 = *reinterpret_cast<const double*>(tile + ld1);
            C.v[0] = init ? init->v[0] : 0.0;
            C.v[1] = init ? init->v[1] : 0.0;
            if constexpr (kSplit) {
                // two independent half-products (even / odd k) summed after:
                // latency DMMA + DADD instead of two chained DMMAs (26 cycles
                // each), at the price of 2 DADDs on the shared FP64 pipe
                double e0 = 0.0, e1 = 0.0;
                dmma_8x8x4(C.v[0], C.v[1], X.v[0], y0);
                dmma_8x8x4(e0, e1, X.v[1], y1);
                C.v[0] += e0;
                C.v[1] += e1;
            } else {
                dmma_8x8x4(C.v[0], C.v[1], X.v[0], y0);
                dmma_8x8x4(C.v[0], C.v[1], X.v[1], y1);
            }
        }
        return C;
    }
};

// The work ticket {round counter, finished CTAs}: the last CTA to finish
// zeroes both, so the slot is ready for the next launch -- including the
// replay of a CUDA graph that captured this one.
__device__ __forceinline__ void release_ticket(unsigned long long* ticket) {
    __syncwarp();
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        if (atomicAdd(ticket + 1, 1ull) == gridDim.x - 1ull) {
            ticket[0] = 0ull;
            ticket[1] = 0ull;
            __threadfence();
        }
    }
}

constexpr int kN8WarpsPerBlock = 4;  // 128-thread blocks
constexpr int kN8Mpw = 4;            // matrices per warp per round

// One round = 4 consecutive matrices per warp. The prologue (load, finite
// check, exact 1-norm, selection, selection record) runs for the 4 at once so
// all 32 lanes work: lane l sums column l&7 of matrix l>>3. Then the schemes
// run one matrix at a time, each on its own 1 KB tile (which still holds its
// unscaled A for sq_first).
// kExact: 0 = exact-rounded matrices inline; 1 = fast kernel that defers the
// matrices needing reference rounding to a worklist (expm8_exact_kernel).
// kFamily (mexp_family) is a template parameter: the TaylorNew kernel carries
// no Paterson-Stockmeyer code.
template <bool kSplit, int kDefer, int kMinBlocks = 8, int kFamily = MEXP_FAMILY_TAYLOR_NEW>
__global__ void __launch_bounds__(32 * kN8WarpsPerBlock, kMinBlocks)
    expm8_f64_kernel(const double* __restrict__ a, double* __restrict__ out,
                     mexp_selection* __restrict__ sel, int64_t batch, int acc_arg, int rounding_arg,
                     int exact_s_min, int32_t* __restrict__ worklist, int32_t* __restrict__ wcount,
                     unsigned long long* __restrict__ ticket) {
    using Group8 = Group8T<kSplit>;
    using F = typename Group8::Frag;
    __shared__ __align__(16) char tiles[kN8WarpsPerBlock][kN8Mpw][1024];
    const int rounding = rounding_arg & 0xff;  // mexp_rounding
    // accuracy in the low 4 bits (mexp_accuracy); the family is kFamily
    const int accuracy = acc_arg & 15;
    constexpr int family = kFamily;
    const int lane = threadIdx.x & 31;
    const int wib = threadIdx.x >> 5;
    Group8 g;
    g.init(tiles[wib][0], lane);
    char* const wt = tiles[wib][0];

    // 1-norm column reads of lane l: matrix jm = l >> 3, column c8 = l & 7;
    // element (i, c8) at unit8(i, 0) & ~0x20 plus one of two lane bases
    const int jm = lane >> 3, c8 = lane & 7, cp = c8 >> 1;
    const uint32_t half = uint32_t(c8 & 1) << 3;
    const char* nb0 = wt + jm * 1024 + ((((cp >> 1)) << 5) | ((cp & 1) << 4)) + half;
    const char* nb1 = wt + jm * 1024 + (((1 ^ (cp >> 1)) << 5) | ((cp & 1) << 4)) + half;

    const int64_t rounds = (batch + kN8Mpw - 1) / kN8Mpw;
    const int64_t rstride = int64_t(gridDim.x) * kN8WarpsPerBlock;
    int64_t rd = int64_t(blockIdx.x) * kN8WarpsPerBlock + wib;

    // rounds are handed out dynamically after the first: per-matrix cost varies
    // ~5x (degree, s, reference rounding), so a static stride leaves a long tail
    for (; rd < rounds;) {
        const int64_t m0 = rd * kN8Mpw;
        // 4 coalesced 16-byte loads per lane (2 KB per warp) in flight at once;
        // with ~8 warps per scheduler the loads of one warp overlap the
        // schemes of the others
        double2 cur[kN8Mpw];
#pragma unroll
        for (int j = 0; j < kN8Mpw; ++j)
            cur[j] = (m0 + j < batch) ? ld_stream(reinterpret_cast<const double2*>(a + (m0 + j) * 64) + lane)
                                      : make_double2(0.0, 0.0);

        // all_finite (dense_matrix.cpp:54-58), one ballot per matrix
        uint32_t finbits = 0;
#pragma unroll
        for (int j = 0; j < kN8Mpw; ++j)
            if (__all_sync(0xffffffffu, isfinite(cur[j].x) && isfinite(cur[j].y))) finbits |= 1u << j;

        // stage the 4 (unscaled) matrices, one tile each
        __syncwarp();
#pragma unroll
        for (int j = 0; j < kN8Mpw; ++j) *reinterpret_cast<double2*>(wt + j * 1024 + g.st) = cur[j];
        __syncwarp();

        // exact 1-norm (kernels.cpp:44-53): column sum over rows 0..7 in order
        double colsum = 0.0;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const char* p = (((i >> 1) & 1) ? nb1 : nb0) + (unit8(i, 0) & ~0x20u);
            colsum = __dadd_rn(colsum, fabs(*reinterpret_cast<const double*>(p)));
        }
        // max over the 8 columns: non-negative doubles order like their bits
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

#pragma unroll 1
        for (int j = 0; j < kN8Mpw; ++j) {
            const int64_t m = m0 + j;
            if (m >= batch) break;
            const int inf = __shfl_sync(0xffffffffu, info, 8 * j);
            const int degree = inf & 31, s = (inf >> 5) & 0x7fff, status = inf >> 20;
            g.tile = wt + j * 1024;
            const bool exact = status == MEXP_OK &&
                               (rounding == MEXP_ROUND_REFERENCE ||
                                (rounding == MEXP_ROUND_AUTO && s >= exact_s_min));
            if constexpr (kDefer) {
                if (exact) {
                    if (lane == 0) worklist[atomicAdd(wcount, 1)] = int32_t(m);
                    continue;
                }
            } else {
                if (exact) {
                    // reference rounding on the quad lane mapping (set_lanes)
                    g.set_lanes(lane, true);
                    const double2 v = *reinterpret_cast<const double2*>(g.tile + g.st);
                    F A;
                    A.v[0] = v.x;
                    A.v[1] = v.y;
                    g.fscale = pow2_neg(s);
                    g.scaled = s > 0;
                    const F X = run_expm<ExactOps, family>(g, A, degree, s, 0);
                    st_stream(reinterpret_cast<double2*>(out + m * 64) + g.unit_index(),
                              make_double2(X.v[0], X.v[1]));
                    g.set_lanes(lane, false);
                    continue;
                }
            }
            F A;  // back from the staged tile (keeps 16 registers free)
            const double2 v = *reinterpret_cast<const double2*>(g.tile + g.st);
            A.v[0] = v.x;
            A.v[1] = v.y;
            F X;
            if (status != MEXP_OK) {
                X.v[0] = X.v[1] = __longlong_as_double(0x7ff8000000000000ll);
            } else {
                g.fscale = pow2_neg(s);
                g.scaled = s > 0;
                X = run_expm<FastOps, family>(g, A, degree, s, 0);
            }
            st_stream(reinterpret_cast<double2*>(out + m * 64) + lane, make_double2(X.v[0], X.v[1]));
        }
        unsigned long long t = 0;
        if (lane == 0) t = atomicAdd(ticket, 1ull);
        rd = rstride + int64_t(__shfl_sync(0xffffffffu, t, 0));
    }
    release_ticket(ticket);
}

// Reference-rounded 8x8 expm for the matrices listed in worklist[0, *wcount)
// (or, with worklist == nullptr, for all of [0, batch)): one warp per matrix,
// its own prologue (the selection records were written by the fast kernel).
template <int kFamily = MEXP_FAMILY_TAYLOR_NEW>
__global__ void __launch_bounds__(32 * kN8WarpsPerBlock, 8)
    expm8_exact_kernel(const double* __restrict__ a, double* __restrict__ out,
                       mexp_selection* __restrict__ sel, int64_t batch, int acc_arg,
                       const int32_t* __restrict__ worklist, const int32_t* __restrict__ wcount) {
    using Group8 = Group8T<false>;
    using F = Group8::Frag;
    __shared__ __align__(16) char tiles[kN8WarpsPerBlock][1024];
    const int accuracy = acc_arg & 15;
    constexpr int family = kFamily;
    const int lane = threadIdx.x & 31;
    const int wib = threadIdx.x >> 5;
    Group8 g;
    g.init(tiles[wib], lane);
    const int64_t count = worklist ? int64_t(*wcount) : batch;
    const int64_t stride = int64_t(gridDim.x) * kN8WarpsPerBlock;
    for (int64_t w = int64_t(blockIdx.x) * kN8WarpsPerBlock + wib; w < count; w += stride) {
        const int64_t m = worklist ? int64_t(worklist[w]) : w;
        F A;
        const double2 v = ld_stream(reinterpret_cast<const double2*>(a + m * 64) + lane);
        A.v[0] = v.x;
        A.v[1] = v.y;
        const bool allfin = __all_sync(0xffffffffu, isfinite(v.x) && isfinite(v.y));
        __syncwarp();
        *reinterpret_cast<double2*>(g.tile + g.st) = v;
        __syncwarp();
        double colsum = 0.0;
        if (lane < 8) {
            const uint32_t half = (lane & 1) << 3;
#pragma unroll
            for (int i = 0; i < 8; ++i)
                colsum = __dadd_rn(colsum, fabs(*reinterpret_cast<const double*>(
                                               g.tile + unit8(i, lane >> 1) + half)));
        }
        unsigned long long nb = __double_as_longlong(colsum);
#pragma unroll
        for (int o = 1; o < 8; o <<= 1) {
            const unsigned long long x = __shfl_xor_sync(0xffffffffu, nb, o);
            nb = x > nb ? x : nb;
        }
        const double norm = __longlong_as_double(__shfl_sync(0xffffffffu, nb, 0));
        Sel sl{0, 0, MEXP_OK};
        if (!allfin)
            sl.status = MEXP_ERR_NONFINITE;
        else
            sl = select_device(norm, accuracy, family);
        if (!worklist && sel && lane == 0) {
            mexp_selection rec;
            rec.norm_in = allfin ? norm : __longlong_as_double(0x7ff8000000000000ll);
            rec.degree = int16_t(sl.degree);
            rec.s = int16_t(sl.s);
            rec.status = sl.status;
            sel[m] = rec;
        }
        F X;
        if (sl.status != MEXP_OK) {
            X.v[0] = X.v[1] = __longlong_as_double(0x7ff8000000000000ll);
        } else {
            g.fscale = pow2_neg(sl.s);
            g.scaled = sl.s > 0;
            X = run_expm<ExactOps, family>(g, A, sl.degree, sl.s, 0);
        }
        st_stream(reinterpret_cast<double2*>(out + m * 64) + lane, make_double2(X.v[0], X.v[1]));
    }
}

// ---------------------------------------------------------------------------
// The pipelined 8x8 kernel (default for TaylorNew / TaylorPS): the same round
// structure and the same arithmetic as expm8_f64_kernel (bit-identical
// results), with the global-memory and work-ticket latencies taken off the
// warps' critical path:
//   * A round's four matrices arrive by cp.async straight into their swizzled
//     staging tiles (two alternating sets per warp), issued while the previous
//     round is still computing; the prologue never waits on DRAM.
//   * The next round is claimed (atomicAdd on the work ticket) before matrix
//     kClaimAt of the current round and its copy is issued before matrix kPF,
//     so neither the L2 atomic round trip nor the DRAM latency stalls a warp.
//   * all_finite rides on the 1-norm: a column sum of |a_ij| is Inf/NaN iff
//     the column holds a non-finite entry or the sum overflows, so the per-
//     entry test (and the two error statuses it separates) runs only for a
//     round whose norm is non-finite.
//   * theta_m come in as kernel parameters (constant-bank operands), the
//     2^-s scale and the rounding decision are made once per round in the
//     4-wide prologue and handed to the per-matrix loop by shuffle.
// ---------------------------------------------------------------------------
struct N8Params {
    double theta[6];   // theta_entry(family, accuracy, 0..5)
    int accuracy;      // mexp_accuracy (the rare non-finite path's select_device)
    int exact_from_s;  // matrices with s >= this run reference rounding
                       // (0: all, REFERENCE; INT_MAX: none, FAST)
    uint32_t static_rounds;  // rounds [0, static_rounds) are dealt round-robin (a multiple
                             // of the warp count), the rest by the work ticket
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async16_zfill(uint32_t dst, const void* src, uint32_t bytes) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
    asm volatile("cp.async.wait_all;" ::: "memory");
}

// scaled(a, 2^-s), the scheme, the squarings (run_expm without its own 2^-s:
// g.fscale holds it)
template <class Ops, int kFam, class G>
__device__ __forceinline__ typename G::Frag run_expm8(const G& g, typename G::Frag A, int degree,
                                                      int s) {
    using F = typename G::Frag;
    if (s > 0) {
        A.v[0] = __dmul_rn(g.fscale, A.v[0]);
        A.v[1] = __dmul_rn(g.fscale, A.v[1]);
    }
    F X;
    if constexpr (kFam == MEXP_FAMILY_TAYLOR_PS)
        X = eval_taylor_ps<Ops>(g, degree, A);
    else
        X = eval_taylor_new<Ops>(g, degree, A);
    for (int i = 0; i < s; ++i) X = g.template mm<Ops>(X, X, true);
    return X;
}

constexpr int kN8InfoBad = 1 << 30;   // status != MEXP_OK: the result is NaN
constexpr int kN8InfoSkip = 1 << 29;  // past the end of the batch

template <int kFamily = MEXP_FAMILY_TAYLOR_NEW, int kClaimAt = 1, int kPF = 3, int kMinBlocks = 8>
__global__ void __launch_bounds__(32 * kN8WarpsPerBlock, kMinBlocks)
    expm8_pipe_kernel(const double* __restrict__ a, double* __restrict__ out,
                      mexp_selection* __restrict__ sel, int64_t batch, const N8Params prm,
                      unsigned long long* __restrict__ ticket) {
    // kClaimAt < 0: static round-robin rounds (no work ticket; experiments)
    static_assert(kClaimAt < kPF && kPF < kN8Mpw, "claim before the copy, inside the round");
    using Group8 = Group8T<false, true>;
    using F = typename Group8::Frag;
    // per warp: two sets of four 512-byte staging tiles + the exact path's Y scratch
    __shared__ __align__(16) char tiles[kN8WarpsPerBlock][2][kN8Mpw][512];
    __shared__ __align__(16) char yscratch[kN8WarpsPerBlock][512];
    __shared__ int infos[kN8WarpsPerBlock][kN8Mpw];
    constexpr int family = kFamily;
    constexpr bool ps = kFamily == MEXP_FAMILY_TAYLOR_PS;
    constexpr uint32_t kSet = kN8Mpw * 512;
    const int lane = threadIdx.x & 31;
    const int wib = threadIdx.x >> 5;
    Group8 g;
    g.init(tiles[wib][0][0], lane);
    g.ytile = yscratch[wib];
    char* const wbase = tiles[wib][0][0];
    const uint32_t wbase_s = smem_u32(wbase);

    // 1-norm column reads of lane l: matrix jm = l >> 3, column c8 = l & 7
    const int jm = lane >> 3, c8 = lane & 7, cp = c8 >> 1;
    const uint32_t half = uint32_t(c8 & 1) << 3;
    const uint32_t n0 = jm * 512 + ((((cp >> 1)) << 5) | ((cp & 1) << 4)) + half;
    const uint32_t n1 = jm * 512 + (((1 ^ (cp >> 1)) << 5) | ((cp & 1) << 4)) + half;

    const uint32_t rounds = uint32_t((batch + kN8Mpw - 1) / kN8Mpw);  // < 2^32: checked by the host
    const uint32_t rstride = gridDim.x * kN8WarpsPerBlock;
    uint32_t rd = blockIdx.x * kN8WarpsPerBlock + wib;
    uint32_t cur = 0;  // byte offset of the current set

    auto copy_round = [&](uint32_t r, uint32_t setoff) {
        const int64_t mb = int64_t(r) * kN8Mpw;
        const double* src = a + mb * 64 + lane * 2;
        const uint32_t dst = wbase_s + setoff + g.st;
        if (mb + kN8Mpw <= batch) {
#pragma unroll
            for (int j = 0; j < kN8Mpw; ++j) cp_async16(dst + j * 512, src + j * 64);
        } else {  // the last, partial round: zero-filled tiles past the batch
#pragma unroll
            for (int j = 0; j < kN8Mpw; ++j) {
                const bool ok = mb + j < batch;
                cp_async16_zfill(dst + j * 512, ok ? src + j * 64 : a, ok ? 16u : 0u);
            }
        }
    };
    if (rd < rounds) copy_round(rd, 0);

    while (rd < rounds) {
        const int64_t m0 = int64_t(rd) * kN8Mpw;
        cp_async_wait_all();
        __syncwarp();
        char* const set = wbase + cur;

        // exact 1-norm (kernels.cpp:44-53): column sum over rows 0..7 in order
        double colsum = 0.0;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const char* p = set + (((i >> 1) & 1) ? n1 : n0) + (unit8(i, 0) & ~0x20u);
            colsum = __dadd_rn(colsum, fabs(*reinterpret_cast<const double*>(p)));
        }
        // max over the 8 columns: non-negative doubles order like their bits,
        // and a NaN or Inf sum orders above every finite one
        unsigned long long nb = __double_as_longlong(colsum) & 0x7fffffffffffffffull;
#pragma unroll
        for (int o = 1; o < 8; o <<= 1) {
            const unsigned long long w = __shfl_xor_sync(0xffffffffu, nb, o);
            nb = w > nb ? w : nb;
        }
        const double norm = __longlong_as_double(nb);
        int degree = 0, s = 0, status = MEXP_OK;
        bool allfin = true;
        if (__any_sync(0xffffffffu, uint32_t(nb >> 32) >= 0x7ff00000u)) {
            // a non-finite entry (dense_matrix.cpp:54-58) or an overflowing
            // norm somewhere in the round: the per-entry test decides
            uint32_t finbits = 0;
#pragma unroll
            for (int j = 0; j < kN8Mpw; ++j) {
                const double2 v = *reinterpret_cast<const double2*>(set + j * 512 + g.st);
                if (__all_sync(0xffffffffu, isfinite(v.x) && isfinite(v.y))) finbits |= 1u << j;
            }
            allfin = (finbits >> jm) & 1u;
            if (!allfin) {
                status = MEXP_ERR_NONFINITE;
            } else {
                // the norm of matrix jm alone (its own columns' max is what nb holds)
                const Sel sl = select_device(norm, prm.accuracy, family);
                degree = sl.degree;
                s = sl.s;
                status = sl.status;
            }
        } else if (norm <= prm.theta[5]) {
            // select_device's table walk with the thetas from the parameters
            const int e = int(prm.theta[0] < norm) + int(prm.theta[1] < norm) +
                          int(prm.theta[2] < norm) + int(prm.theta[3] < norm) +
                          int(prm.theta[4] < norm);
            degree = ps ? ps_degree_of(e) : (e < 4 ? (1 << e) : (e == 4 ? 12 : 18));
        } else {
            const long long tb = __double_as_longlong(prm.theta[5]);
            const int k = int(nb >> 52) - int(tb >> 52);
            const double t = __longlong_as_double(tb + (static_cast<long long>(k) << 52));
            degree = ps ? 16 : 18;
            s = k + int(norm > t);
        }
        if (sel && c8 == 0 && m0 + jm < batch) {
            mexp_selection rec;
            rec.norm_in = allfin ? norm : __longlong_as_double(0x7ff8000000000000ll);
            rec.degree = int16_t(degree);
            rec.s = int16_t(s);
            rec.status = status;
            sel[m0 + jm] = rec;
        }
        // (degree, s, flags) per matrix through shared memory: the per-matrix
        // loop reads them back by broadcast, no register lives across it
        if (c8 == 0)
            infos[wib][jm] = degree | (s << 5) | (status != MEXP_OK ? kN8InfoBad : 0) |
                             (m0 + jm >= batch ? kN8InfoSkip : 0) |
                             (s >= prm.exact_from_s ? int(0x80000000u) : 0);
        __syncwarp();

        uint32_t t = 0, nrd = 0;
#pragma unroll 1
        for (int j = 0; j < kN8Mpw; ++j) {
            // plain atom (inline asm): the compiler's warp-aggregated form
            // shuffles the result at once and would wait for the round trip here
            // the next round: round-robin while it lies in the static part,
            // else claimed from the ticket
            const bool dyn = kClaimAt >= 0 && rd + rstride >= prm.static_rounds;
            if (j == kClaimAt && dyn && lane == 0)
                asm volatile("atom.global.add.u32 %0, [%1], 1;" : "=r"(t) : "l"(ticket) : "memory");
            if (j == kPF) {
                nrd = dyn ? prm.static_rounds + __shfl_sync(0xffffffffu, t, 0) : rd + rstride;
                if (nrd < rounds) copy_round(nrd, cur ^ kSet);
            }
            const int inf = infos[wib][j];
            if (inf & kN8InfoSkip) continue;
            g.tile = set + j * 512;
            const int deg = inf & 31, sj = (inf >> 5) & 0x7fff;
            // 2^-s from its high word (the low word is 0: s <= 1025 for any finite norm)
            g.fscale = __hiloint2double(
                int(sj <= 1022 ? uint32_t(1023 - sj) << 20 : 1u << ((1042 - sj) & 31)), 0);
            g.scaled = sj > 0;
            if (inf < 0 && !(inf & kN8InfoBad)) {
                // reference rounding on the quad lane mapping (set_lanes)
                g.set_lanes(lane, true);
                const double2 v = *reinterpret_cast<const double2*>(g.tile + g.st);
                F A;
                A.v[0] = v.x;
                A.v[1] = v.y;
                const F X = run_expm8<ExactOps, family>(g, A, deg, sj);
                st_stream(reinterpret_cast<double2*>(out + (m0 + j) * 64) + g.unit_index(),
                          make_double2(X.v[0], X.v[1]));
                g.set_lanes(lane, false);
                continue;
            }
            const double2 v = *reinterpret_cast<const double2*>(g.tile + g.st);
            F A;
            A.v[0] = v.x;
            A.v[1] = v.y;
            F X;
            if (inf & kN8InfoBad)
                X.v[0] = X.v[1] = __longlong_as_double(0x7ff8000000000000ll);
            else
                X = run_expm8<FastOps, family>(g, A, deg, sj);
            st_stream(reinterpret_cast<double2*>(out + (m0 + j) * 64) + lane, make_double2(X.v[0], X.v[1]));
        }
        rd = nrd;
        cur ^= kSet;
    }
    release_ticket(ticket);
}

}  // namespace mexp_b200
