// Batched 32x32 fp32 expm, Family::TaylorNew (BASELINE cfg3): two matrices
// of the same (degree, s) class per warp, 8x8 register tiles, the scheme's
// intermediates parked in tensor memory.
//
// Why this shape. A product C = X*Y on FFMA streams X columns and Y rows out
// of shared memory; a lane owning a TR x TC output tile loads TR + TC floats
// per TR*TC FMAs. With one warp per 32x32 matrix the tile is 4x8 (12 floats
// per 32 FMAs): shared memory saturates at 2/3 of the FFMA rate
// (profiles/ncu_cfg3_auto_r2.txt). A half warp per matrix gives every lane an
// 8x8 tile (16 floats per 64 FMAs), which balances the two pipes. But each
// live matrix then costs 64 registers per lane, and T18 keeps A, A2, A3, A6
// alive while it forms B1..B5: those go to TMEM (tcgen05.st / tcgen05.ld,
// each lane its own TMEM row), and registers hold only the accumulator tile
// and the k-loop operands.
//
// Both halves of a warp run one instruction stream (tcgen05.ld/st are
// warp-collective), so the two matrices must share (degree, s). A pre-pass
// (select32_kernel: finite check, exact fp64 1-norm, selection record --
// kernels.cpp:44-53, expm.cpp:11-29) computes each matrix's class, and a
// counting sort (scatter32_kernel) lists the matrices by class,
// most expensive first; the main kernel takes consecutive pairs of that list.
// A pair whose classes differ (at most one per class boundary) runs as two
// passes with both halves on one matrix.
//
// Arithmetic: every operation of eval_taylor_new / the squarings in the same
// order as the one-warp kernel (expm_small_f32.cu, F32Ops): products are
// k-ascending FFMA chains from the accumulator's initial value, the linear
// combinations start from the identity entry (or +0) and add c*M terms with
// FFMA in the reference's term order (taylor_schemes.cpp:104-141, 146-157,
// 211-227). The two kernels produce the same bits.
#include <atomic>
#include <cstdint>
#include <cstdlib>

#include "async_buffer.hpp"
#include "device_once.hpp"
#include "expm_common.cuh"
#include "expm_pairs32.cuh"

namespace mexp_b200 {
namespace {

constexpr int N = 32;
constexpr int NN = N * N;
constexpr int kWarps = 4;                    // one per TMEM lane quadrant
constexpr int kTmemCols = 128;               // 2 slots x 64 columns per lane
#ifndef MEXP_PAIRS_CTAS
#define MEXP_PAIRS_CTAS 2
#endif
constexpr int kCtasPerSm = MEXP_PAIRS_CTAS;  // CTAs of 4 warps per SM (TMEM: 128 columns each)
constexpr int kBufFloats = NN + N;           // a 32x32 operand buffer + one pad row
#ifndef MEXP_PAIRS_PREFETCH
#define MEXP_PAIRS_PREFETCH 1
#endif
constexpr bool kPrefetch = MEXP_PAIRS_PREFETCH;
// X, Y, and the next pair's matrix (prefetch), plus 64 bytes: the second
// half's buffers sit half a bank row from the first half's, so the X loads of
// the two halves (one LDS.64 wavefront for the warp) hit different banks
#ifndef MEXP_PAIRS_SKEW
#define MEXP_PAIRS_SKEW 16
#endif
constexpr int kHalfFloats = 2 * kBufFloats + (kPrefetch ? NN : 0) + MEXP_PAIRS_SKEW;
constexpr int kSmemBytes = kWarps * 2 * kHalfFloats * 4 + 16;
static_assert(kCtasPerSm * kSmemBytes <= 227 * 1024, "smem");
static_assert(kCtasPerSm * kTmemCols <= 512, "tmem");
constexpr int kNumKeys = 64 * 8 + 1;
constexpr int kScatterChunk = 512;  // matrices per scatter block (>= the SM count of blocks for cfg3)

// class key, ascending = most products first (the main kernel's pairs are
// handed out in key order, so the expensive ones start first)
__device__ __forceinline__ int class_key(int degree, int s, int status) {
    if (status != MEXP_OK) return kNumKeys - 1;
    const int e = degree == 1 ? 0 : degree == 2 ? 1 : degree == 4 ? 2 : degree == 8 ? 3 : degree == 12 ? 4 : 5;
    const int sc = s < 63 ? s : 63;
    return (63 - sc) * 8 + (5 - e);
}

// (degree, s, status) in one word: degree < 32, 0 <= s < 2^16, status < 16
__device__ __forceinline__ uint32_t pack_info(int degree, int s, int status) {
    return uint32_t(degree) | (uint32_t(s) << 5) | (uint32_t(status) << 21);
}
__device__ __forceinline__ int info_degree(uint32_t i) { return int(i & 31u); }
__device__ __forceinline__ int info_s(uint32_t i) { return int((i >> 5) & 0xffffu); }
__device__ __forceinline__ int info_status(uint32_t i) { return int(i >> 21); }
__device__ __forceinline__ int info_key(uint32_t i) {
    return class_key(info_degree(i), info_s(i), info_status(i));
}

// ---- pre-pass: selection records, class keys and their histogram ----------
__global__ void __launch_bounds__(256) select32_kernel(const float* __restrict__ a,
                                                      mexp_selection* __restrict__ sel,
                                                      uint32_t* __restrict__ info,
                                                      int* __restrict__ hist, int64_t batch,
                                                      int accuracy) {
    __shared__ int sh[kNumKeys];
    for (int i = threadIdx.x; i < kNumKeys; i += blockDim.x) sh[i] = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int wpb = blockDim.x >> 5;
    for (int64_t m = int64_t(blockIdx.x) * wpb + w; m < batch; m += int64_t(gridDim.x) * wpb) {
        // lane j sums column j over rows 0..31 in order, in fp64 on the
        // promoted values (kernels.cpp:44-53): the reference's norm of this data
        const float* p = a + m * NN + lane;
        float v[N];
#pragma unroll
        for (int i = 0; i < N; ++i) v[i] = __ldcs(p + i * N);
        bool fin = true;
        double cs = 0.0;
#pragma unroll
        for (int i = 0; i < N; ++i) {
            fin = fin && isfinite(v[i]);
            cs = __dadd_rn(cs, fabs(double(v[i])));
        }
        const bool allfin = __all_sync(0xffffffffu, fin);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) cs = fmax(cs, __shfl_xor_sync(0xffffffffu, cs, o));
        Sel sl{0, 0, MEXP_OK};
        if (!allfin)
            sl.status = MEXP_ERR_NONFINITE;
        else
            sl = select_device(cs, accuracy, MEXP_FAMILY_TAYLOR_NEW);
        if (lane == 0) {
            mexp_selection r;
            r.norm_in = allfin ? cs : __longlong_as_double(0x7ff8000000000000ll);
            r.degree = int16_t(sl.degree);
            r.s = int16_t(sl.s);
            r.status = sl.status;
            sel[m] = r;
            info[m] = pack_info(sl.degree, sl.s, sl.status);
            atomicAdd(&sh[class_key(sl.degree, sl.s, sl.status)], 1);
        }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < kNumKeys; i += blockDim.x)
        if (sh[i]) atomicAdd(&hist[i], sh[i]);
}

// List position of every matrix. Each block scans the class histogram itself
// (513 counts: cheaper than a separate launch), reserves one range per class
// for its chunk from the running per-class counters, then places its
// matrices in it (order inside a class is irrelevant: every matrix's
// arithmetic is independent of its partner's).
__global__ void __launch_bounds__(1024) scatter32_kernel(const uint32_t* __restrict__ info,
                                                         const int* __restrict__ hist,
                                                         int* __restrict__ running,
                                                         int2* __restrict__ list, int64_t batch) {
    __shared__ int start[1024], lh[kNumKeys], base[kNumKeys];
    __shared__ int rank[kScatterChunk];
    const int t = threadIdx.x;
    const int v = t < kNumKeys ? hist[t] : 0;
    start[t] = v;
    if (t < kNumKeys) lh[t] = 0;
    __syncthreads();
    for (int off = 1; off < 1024; off <<= 1) {  // inclusive scan
        const int x = t >= off ? start[t - off] : 0;
        __syncthreads();
        start[t] += x;
        __syncthreads();
    }
    const int64_t m0 = int64_t(blockIdx.x) * kScatterChunk;
    const int cnt = int(batch - m0 < kScatterChunk ? batch - m0 : kScatterChunk);
    for (int i = t; i < cnt; i += blockDim.x) rank[i] = atomicAdd(&lh[info_key(info[m0 + i])], 1);
    __syncthreads();
    for (int k = t; k < kNumKeys; k += blockDim.x)
        if (lh[k]) base[k] = start[k] - hist[k] + atomicAdd(&running[k], lh[k]);
    __syncthreads();
    for (int i = t; i < cnt; i += blockDim.x) {
        const uint32_t w = info[m0 + i];
        list[base[info_key(w)] + rank[i]] = make_int2(int(m0 + i), int(w));
    }
}

// ---- tensor memory ----------------------------------------------------------
// 32x32b shape: thread t of the warp reads / writes TMEM lane (quadrant base +
// t), consecutive 32-bit columns. Slot k of a lane's matrix = columns
// [64k, 64k + 64), row r of the lane's 8x8 tile at 64k + 8r.
// (no "memory" clobbers: TMEM is not generic memory, the tcgen05 asm
// statements keep their order among themselves as volatile asm, and the
// compiler stays free to hoist the next row's shared-memory loads above them)
__device__ __forceinline__ void tm_st8(uint32_t addr, const float (&v)[8]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"r"(addr),
        "f"(v[0]), "f"(v[1]), "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7]));
}
__device__ __forceinline__ void tm_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;"); }
__device__ __forceinline__ void tm_ld8(uint32_t addr, float (&v)[8]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                 : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]), "=f"(v[4]), "=f"(v[5]),
                   "=f"(v[6]), "=f"(v[7])
                 : "r"(addr));
}
// completes every outstanding tcgen05.ld of the thread; the operands tie the
// loaded registers to the wait so no use is scheduled above it
__device__ __forceinline__ void tm_wait_ld(float (&v)[8], float (&w)[8]) {
    asm volatile("tcgen05.wait::ld.sync.aligned;"
                 : "+f"(v[0]), "+f"(v[1]), "+f"(v[2]), "+f"(v[3]), "+f"(v[4]), "+f"(v[5]),
                   "+f"(v[6]), "+f"(v[7]), "+f"(w[0]), "+f"(w[1]), "+f"(w[2]), "+f"(w[3]),
                   "+f"(w[4]), "+f"(w[5]), "+f"(w[6]), "+f"(w[7]));
}

using Acc = float2[32];  // the lane's 8x8 tile: row r = pairs 4r .. 4r+3

struct Lane {
    int ti, tj;      // tile (8ti.., 8tj..) of the half's matrix
    bool diag;       // ti == tj: the tile holds the diagonal entries (r, r)
    float* xbuf;     // this half's X operand buffer
    float* ybuf;     // this half's Y operand buffer
    uint32_t tm;     // TMEM address of the lane's row, column 0
};

// Operand buffers: row-major 32x32 with the 16-byte chunk c of row i at chunk
// c ^ ((i >> 3) & 3). Conflict-free for the tile-row stores and loads (one
// 8-lane phase = rows 8ti + r of ti in {0,1} or {2,3}, chunks 2tj + {0,1}),
// the X loads (one 16-lane phase = rows 8ti + r of the four ti, one chunk)
// and the Y loads (row k, chunks 2tj + {0,1}).
__device__ __forceinline__ int swz(int i) { return (i >> 3) & 3; }
__device__ __forceinline__ float* row_chunk(float* buf, int i, int c) {
    return buf + i * N + 4 * (c ^ swz(i));
}
__device__ __forceinline__ void store_row(const Lane& L, float* buf, int r, const float (&o)[8]) {
    const int i = 8 * L.ti + r;
    *reinterpret_cast<float4*>(row_chunk(buf, i, 2 * L.tj)) = make_float4(o[0], o[1], o[2], o[3]);
    *reinterpret_cast<float4*>(row_chunk(buf, i, 2 * L.tj + 1)) = make_float4(o[4], o[5], o[6], o[7]);
}
__device__ __forceinline__ void load_row(const Lane& L, float* buf, int r, float (&o)[8]) {
    const int i = 8 * L.ti + r;
    const float4 u = *reinterpret_cast<const float4*>(row_chunk(buf, i, 2 * L.tj));
    const float4 v = *reinterpret_cast<const float4*>(row_chunk(buf, i, 2 * L.tj + 1));
    o[0] = u.x, o[1] = u.y, o[2] = u.z, o[3] = u.w, o[4] = v.x, o[5] = v.y, o[6] = v.z, o[7] = v.w;
}
__device__ __forceinline__ void acc_row(const Acc& C, int r, float (&o)[8]) {
#pragma unroll
    for (int p = 0; p < 4; ++p) {
        o[2 * p] = C[4 * r + p].x;
        o[2 * p + 1] = C[4 * r + p].y;
    }
}
__device__ __forceinline__ void set_acc_row(Acc& C, int r, const float (&o)[8]) {
#pragma unroll
    for (int p = 0; p < 4; ++p) C[4 * r + p] = make_float2(o[2 * p], o[2 * p + 1]);
}
__device__ __forceinline__ void store_buf(const Lane& L, float* buf, const Acc& C) {
#pragma unroll
    for (int r = 0; r < 8; ++r) {
        float o[8];
        acc_row(C, r, o);
        store_row(L, buf, r, o);
    }
}
__device__ __forceinline__ void tm_store(const Lane& L, int slot, const Acc& C) {
#pragma unroll
    for (int r = 0; r < 8; ++r) {
        float o[8];
        acc_row(C, r, o);
        tm_st8(L.tm + 64 * slot + 8 * r, o);
    }
    tm_wait_st();
}
// rows r of slots 0 and 1
__device__ __forceinline__ void tm_rows(const Lane& L, int r, float (&s0)[8], float (&s1)[8]) {
    tm_ld8(L.tm + 8 * r, s0);
    tm_ld8(L.tm + 64 + 8 * r, s1);
    tm_wait_ld(s0, s1);
}
// (plain zero stores compile to UMOV + MOV pairs through uniform registers;
// a 64-bit move of zero is one CS2R per pair)
__device__ __forceinline__ void zero_acc(Acc& C) {
#pragma unroll
    for (int e = 0; e < 32; ++e) {
        unsigned long long z;
        asm("mov.b64 %0, 0;" : "=l"(z));
        C[e] = *reinterpret_cast<const float2*>(&z);
    }
}

// ---- one row of a linear combination (F32Ops of expm_small_f32.cu) ---------
// identity start: c0 on the diagonal entry (r, r) of a diagonal tile, +0 elsewhere
__device__ __forceinline__ void id_start(float (&o)[8], int r, bool diag, double c0) {
#pragma unroll
    for (int c = 0; c < 8; ++c) o[c] = 0.f;
    o[r] = diag ? float(c0) : 0.f;
}
__device__ __forceinline__ void mac_row(float (&o)[8], double c, const float (&m)[8]) {
    if (c != 0.0) {
        const float cf = float(c);
#pragma unroll
        for (int p = 0; p < 4; ++p) {
            const float2 t = __ffma2_rn(make_float2(cf, cf), make_float2(m[2 * p], m[2 * p + 1]),
                                        make_float2(o[2 * p], o[2 * p + 1]));
            o[2 * p] = t.x;
            o[2 * p + 1] = t.y;
        }
    }
}
__device__ __forceinline__ void mul_row(float (&o)[8], double c, const float (&m)[8]) {
    const float cf = float(c);
#pragma unroll
    for (int p = 0; p < 4; ++p) {
        const float2 t = __fmul2_rn(make_float2(cf, cf), make_float2(m[2 * p], m[2 * p + 1]));
        o[2 * p] = t.x;
        o[2 * p + 1] = t.y;
    }
}
__device__ __forceinline__ void add_row(float (&o)[8], const float (&a)[8], const float (&b)[8]) {
#pragma unroll
    for (int p = 0; p < 4; ++p) {
        const float2 t = __fadd2_rn(make_float2(a[2 * p], a[2 * p + 1]), make_float2(b[2 * p], b[2 * p + 1]));
        o[2 * p] = t.x;
        o[2 * p + 1] = t.y;
    }
}
// the T18 / T12 combinations of {I, A, A2, A3(, A6)} with coefficient column j
__device__ __forceinline__ void t18_b(float (&o)[8], int j, int r, bool diag, const float (&a)[8],
                                      const float (&a2)[8], const float (&a3)[8], const float (&a6)[8]) {
    id_start(o, r, diag, c_t18b[j][0]);
    mac_row(o, c_t18b[j][1], a);
    mac_row(o, c_t18b[j][2], a2);
    mac_row(o, c_t18b[j][3], a3);
    mac_row(o, c_t18b[j][4], a6);
}
__device__ __forceinline__ void t12_b(float (&o)[8], int j, int r, bool diag, const float (&a)[8],
                                      const float (&a2)[8], const float (&a3)[8]) {
    id_start(o, r, diag, c_t12[0][j]);
    mac_row(o, c_t12[1][j], a);
    mac_row(o, c_t12[2][j], a2);
    mac_row(o, c_t12[3][j], a3);
}

// ---- the product: C += X * Y, k ascending ----------------------------------
// Lane tile rows 8ti..8ti+7 of X (one float2 = 2 k per row), row k of Y at
// the tile's 8 columns (two float4). Per 4 k: 16 LDS.64 + 8 LDS.128 for 128
// FFMA2 (the X and Y operands of the next k are loaded while the current ones
// feed the FFMAs). One call site: the pair kernel's step loop.
__device__ __forceinline__ float4 lds4(const float* p) { return *reinterpret_cast<const float4*>(p); }
__device__ __forceinline__ float2 lds2(const float* p) { return *reinterpret_cast<const float2*>(p); }

__device__ __forceinline__ void fma_k(Acc& C, const float2 (&x)[8], int odd, const float4& y0,
                                      const float4& y1) {
#pragma unroll
    for (int r = 0; r < 8; ++r) {
        const float a = odd ? x[r].y : x[r].x;
        const float2 aa = make_float2(a, a);
        C[4 * r + 0] = __ffma2_rn(aa, make_float2(y0.x, y0.y), C[4 * r + 0]);
        C[4 * r + 1] = __ffma2_rn(aa, make_float2(y0.z, y0.w), C[4 * r + 1]);
        C[4 * r + 2] = __ffma2_rn(aa, make_float2(y1.x, y1.y), C[4 * r + 2]);
        C[4 * r + 3] = __ffma2_rn(aa, make_float2(y1.z, y1.w), C[4 * r + 3]);
    }
}

__device__ __forceinline__ void kloop(const Lane& L, const float* px, const float* py, Acc& C) {
    // X: row 8ti + r, chunk q at physical chunk q ^ ti (bits 0-1) -> base
    // xb[q & 3] = row + 4 * ((q & 3) ^ ti), plus 16 * (q >> 2)
    const float* xr = px + 8 * L.ti * N;
    const float* xb0 = xr + 4 * (0 ^ L.ti);
    const float* xb1 = xr + 4 * (1 ^ L.ti);
    const float* xb2 = xr + 4 * (2 ^ L.ti);
    const float* xb3 = xr + 4 * (3 ^ L.ti);
    // Y: row k, chunks 2tj + c at physical (2tj + c) ^ f, f = (k >> 3) & 3:
    // 8 * (tj ^ (f >> 1)) + 4 * (c ^ (f & 1))
    const float* yb0 = py + 8 * L.tj;
    const float* yb1 = py + 8 * (L.tj ^ 1);
    float2 xa[8], xn[8];
#pragma unroll
    for (int r = 0; r < 8; ++r) xa[r] = lds2(xb0 + r * N);
    float4 y0 = lds4(yb0), y1 = lds4(yb0 + 4);
#pragma unroll 1
    for (int j = 0; j < 2; ++j) {  // k in [16j, 16j + 16)
        const int jo = 16 * j;
        // f >> 1 == (j + (kn >> 4)) & 1 for the rows 16j + kn, kn in [1, 16]
        const float* ybj = j ? yb1 : yb0;
        const float* ybn = j ? yb0 : yb1;
#pragma unroll
        for (int hq = 0; hq < 8; ++hq) {  // k pair 2hq, 2hq + 1 (relative to 16j)
            // next k pair's X (past k = 31: the pad row, unused)
            const int hn = hq + 1;
            const int qn = hn >> 1;  // its chunk (relative)
            const float* xq = (qn & 3) == 0 ? xb0 : (qn & 3) == 1 ? xb1 : (qn & 3) == 2 ? xb2 : xb3;
#pragma unroll
            for (int r = 0; r < 8; ++r) xn[r] = lds2(xq + jo + 16 * (qn >> 2) + 2 * (hn & 1) + r * N);
#pragma unroll
            for (int kk = 0; kk < 2; ++kk) {
                const int kn = 2 * hq + kk + 1;  // next Y row, relative to 16j
                const int lo = (kn >> 3) & 1;  // f & 1
                const float* yr = ((kn >> 4) ? ybn : ybj) + (jo + kn) * N;
                const float4 yn0 = lds4(yr + 4 * lo), yn1 = lds4(yr + 4 - 4 * lo);
                fma_k(C, xa, kk, y0, y1);
                y0 = yn0;
                y1 = yn1;
            }
#pragma unroll
            for (int r = 0; r < 8; ++r) xa[r] = xn[r];
        }
    }
}

// ---- the steps of eval_taylor_new + squarings -------------------------------
// step < P (the degree's product count): prepare the operand buffers and the
// accumulator start of product #step, which then runs with X = the returned
// buffer and Y = py. At step == P, finish() applies a trailing linear
// combination (T8, degree 2, degree 1); the steps after are the s squarings.
// Returns nullptr when done.
//
// Where the scheme's matrices live (a lane's tile rows are read and rewritten
// in place, each lane touching only its own chunks, so no extra buffers):
//   T18: A in Y until B5 replaces it, A2 in TMEM slot 1, A3 in X until B1
//        replaces it; B3 and B2 are formed in the same pass as B1, B5, B4
//        (while A..A6 are at hand) and parked in slots 0 and 1.
//   T12: A in Y until B[3] replaces it, A2 in X; B[1], B[0] parked in slots.
//   T8:  A in slot 0, A2 in slot 1. PS4, degree 2: A in Y.
__device__ __forceinline__ const float* stage(const Lane& L, int degree, int step, int s, Acc& C,
                                              const float*& py) {
    const int P = products_of_degree(degree);
    py = L.ybuf;
    if (step < P) {
        __syncwarp();  // the previous product's readers are done with the buffers
        if (step == 0) {  // A2 = A * A
            if (degree == 8) tm_store(L, 0, C);
            store_buf(L, L.ybuf, C);
            zero_acc(C);
            __syncwarp();
            return L.ybuf;
        }
        if (degree == 18) {
            if (step == 1) {  // A3 = A2 * A
                tm_store(L, 1, C);
                store_buf(L, L.xbuf, C);
                zero_acc(C);
            } else if (step == 2) {  // A6 = A3 * A3
                store_buf(L, L.xbuf, C);
                zero_acc(C);
                py = L.xbuf;
            } else if (step == 3) {  // A9 = B1 * B5 + B4 (B5 = B[3], B4 = B[2]); park B3, B2
#pragma unroll
                for (int r = 0; r < 8; ++r) {
                    float a[8], a2[8], a3[8], a6[8], o[8], unused[8];
                    tm_ld8(L.tm + 64 + 8 * r, a2);
                    load_row(L, L.ybuf, r, a);
                    load_row(L, L.xbuf, r, a3);
                    acc_row(C, r, a6);
                    tm_wait_ld(a2, unused);
                    id_start(o, r, L.diag, c_t18a[0]);
                    mac_row(o, c_t18a[1], a);
                    mac_row(o, c_t18a[2], a2);
                    mac_row(o, c_t18a[3], a3);
                    store_row(L, L.xbuf, r, o);
                    t18_b(o, 3, r, L.diag, a, a2, a3, a6);
                    store_row(L, L.ybuf, r, o);
                    t18_b(o, 1, r, L.diag, a, a2, a3, a6);
                    tm_st8(L.tm + 8 * r, o);
                    t18_b(o, 0, r, L.diag, a, a2, a3, a6);
                    tm_st8(L.tm + 64 + 8 * r, o);
                    t18_b(o, 2, r, L.diag, a, a2, a3, a6);
                    set_acc_row(C, r, o);
                }
                tm_wait_st();
            } else {  // step 4: T = (B3 + A9) * A9 + B2
#pragma unroll
                for (int r = 0; r < 8; ++r) {
                    float b3[8], b2[8], a9[8], o[8];
                    tm_rows(L, r, b3, b2);
                    acc_row(C, r, a9);
                    add_row(o, b3, a9);
                    store_row(L, L.xbuf, r, o);
                    store_row(L, L.ybuf, r, a9);
                    set_acc_row(C, r, b2);
                }
            }
        } else if (degree == 12) {
            if (step == 1) {  // A3 = A2 * A
                store_buf(L, L.xbuf, C);
                zero_acc(C);
            } else if (step == 2) {  // A6 = B[3] * B[3] + B[2]; park B[1], B[0]
#pragma unroll
                for (int r = 0; r < 8; ++r) {
                    float a[8], a2[8], a3[8], o[8];
                    load_row(L, L.ybuf, r, a);
                    load_row(L, L.xbuf, r, a2);
                    acc_row(C, r, a3);
                    t12_b(o, 3, r, L.diag, a, a2, a3);
                    store_row(L, L.ybuf, r, o);
                    t12_b(o, 1, r, L.diag, a, a2, a3);
                    tm_st8(L.tm + 8 * r, o);
                    t12_b(o, 0, r, L.diag, a, a2, a3);
                    tm_st8(L.tm + 64 + 8 * r, o);
                    t12_b(o, 2, r, L.diag, a, a2, a3);
                    set_acc_row(C, r, o);
                }
                tm_wait_st();
                __syncwarp();
                return L.ybuf;
            } else {  // step 3: T = (B[1] + A6) * A6 + B[0]
#pragma unroll
                for (int r = 0; r < 8; ++r) {
                    float b1[8], b0[8], a6[8], o[8];
                    tm_rows(L, r, b1, b0);
                    acc_row(C, r, a6);
                    add_row(o, b1, a6);
                    store_row(L, L.xbuf, r, o);
                    store_row(L, L.ybuf, r, a6);
                    set_acc_row(C, r, b0);
                }
            }
        } else if (degree == 8) {
            if (step == 1) {  // A4 = A2 * (x1 A + x2 A2)
                tm_store(L, 1, C);
#pragma unroll
                for (int r = 0; r < 8; ++r) {
                    float a[8], a2[8], o[8];
                    load_row(L, L.ybuf, r, a);
                    acc_row(C, r, a2);
                    store_row(L, L.xbuf, r, a2);
                    mul_row(o, T8C::x1, a);
                    mac_row(o, T8C::x2, a2);
                    store_row(L, L.ybuf, r, o);
                }
                zero_acc(C);
            } else {  // step 2: A8 = (x3 A2 + A4) * (x4 I + x5 A + x6 A2 + x7 A4)
#pragma unroll
                for (int r = 0; r < 8; ++r) {
                    float a[8], a2[8], a4[8], o[8];
                    tm_rows(L, r, a, a2);
                    acc_row(C, r, a4);
                    mul_row(o, T8C::x3, a2);
                    mac_row(o, 1.0, a4);
                    store_row(L, L.xbuf, r, o);
                    id_start(o, r, L.diag, T8C::x4);
                    mac_row(o, T8C::x5, a);
                    mac_row(o, T8C::x6, a2);
                    mac_row(o, T8C::x7, a4);
                    store_row(L, L.ybuf, r, o);
                }
                zero_acc(C);
            }
        } else {  // degree 4, step 1: T = (f1 + A2/24) * A2 + f0 (eval_ps(4))
#pragma unroll
            for (int r = 0; r < 8; ++r) {
                float a[8], a2[8], f0[8], f1[8], o[8];
                load_row(L, L.ybuf, r, a);
                acc_row(C, r, a2);
                id_start(f0, r, L.diag, 1.0);
                mac_row(f0, 1.0, a);
                id_start(f1, r, L.diag, kInvFact2);
                mac_row(f1, kInvFact3, a);
                mul_row(o, 1.0, f1);
                mac_row(o, kInvFact4, a2);
                store_row(L, L.xbuf, r, o);
                store_row(L, L.ybuf, r, a2);
                set_acc_row(C, r, f0);
            }
        }
        __syncwarp();
        return L.xbuf;
    }
    if (step == P) {  // trailing linear combinations
        if (degree == 8) {  // y0 I + y1 A + y2 A2 + A8
#pragma unroll
            for (int r = 0; r < 8; ++r) {
                float a[8], a2[8], a8[8], o[8];
                tm_rows(L, r, a, a2);
                acc_row(C, r, a8);
                id_start(o, r, L.diag, T8C::y0);
                mac_row(o, T8C::y1, a);
                mac_row(o, T8C::y2, a2);
                mac_row(o, 1.0, a8);
                set_acc_row(C, r, o);
            }
        } else if (degree == 2) {  // I + A + A2/2 (A still in Y: the product only read it)
#pragma unroll
            for (int r = 0; r < 8; ++r) {
                float a[8], a2[8], o[8];
                load_row(L, L.ybuf, r, a);
                acc_row(C, r, a2);
                id_start(o, r, L.diag, 1.0);
                mac_row(o, 1.0, a);
                mac_row(o, 0.5, a2);
                set_acc_row(C, r, o);
            }
        } else if (degree == 1) {  // add(I, A)
#pragma unroll
            for (int r = 0; r < 8; ++r) {
                float a[8], id[8], o[8];
                acc_row(C, r, a);
                id_start(id, r, L.diag, 1.0);
                add_row(o, id, a);
                set_acc_row(C, r, o);
            }
        }
    }
    if (step - P < s) {  // a squaring
        __syncwarp();
        store_buf(L, L.ybuf, C);
        __syncwarp();
        zero_acc(C);
        return L.ybuf;
    }
    return nullptr;
}

__device__ __forceinline__ void load_tile(const Lane& L, const float* m, Acc& C) {
#pragma unroll
    for (int r = 0; r < 8; ++r) {
        const float* p = m + (8 * L.ti + r) * N + 8 * L.tj;
        const float4 u = ld_stream(reinterpret_cast<const float4*>(p));
        const float4 v = ld_stream(reinterpret_cast<const float4*>(p + 4));
        C[4 * r + 0] = make_float2(u.x, u.y);
        C[4 * r + 1] = make_float2(u.z, u.w);
        C[4 * r + 2] = make_float2(v.x, v.y);
        C[4 * r + 3] = make_float2(v.z, v.w);
    }
}
__device__ __forceinline__ void store_tile(const Lane& L, float* m, const Acc& C) {
#pragma unroll
    for (int r = 0; r < 8; ++r) {
        float* p = m + (8 * L.ti + r) * N + 8 * L.tj;
        st_stream(reinterpret_cast<float4*>(p), make_float4(C[4 * r].x, C[4 * r].y, C[4 * r + 1].x, C[4 * r + 1].y));
        st_stream(reinterpret_cast<float4*>(p + 4),
                  make_float4(C[4 * r + 2].x, C[4 * r + 2].y, C[4 * r + 3].x, C[4 * r + 3].y));
    }
}

// the next pair's matrix of this half, one 16-byte cp.async per tile chunk,
// into the operand buffers' swizzled layout (each lane later reads back only
// the chunks it copied itself)
__device__ __forceinline__ void prefetch_tile(const Lane& L, float* pbuf, const float* m) {
    if constexpr (!kPrefetch) return;
#pragma unroll
    for (int r = 0; r < 8; ++r) {
        const int i = 8 * L.ti + r;
#pragma unroll
        for (int c = 0; c < 2; ++c)
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(
                             uint32_t(__cvta_generic_to_shared(row_chunk(pbuf, i, 2 * L.tj + c)))),
                         "l"(m + i * N + 8 * L.tj + 4 * c)
                         : "memory");
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
}
__device__ __forceinline__ void load_tile_smem(const Lane& L, float* pbuf, Acc& C) {
#pragma unroll
    for (int r = 0; r < 8; ++r) {
        float o[8];
        load_row(L, pbuf, r, o);
        set_acc_row(C, r, o);
    }
}

// pair q of the class-sorted list: {m_a, info_a, m_b, info_b} (a single
// matrix at an odd batch's end is paired with itself)
__device__ __forceinline__ int4 pair_at(const int2* __restrict__ list, int64_t q, int64_t batch) {
    if (2 * q + 1 < batch) return *reinterpret_cast<const int4*>(list + 2 * q);
    const int2 x = list[2 * q];
    return make_int4(x.x, x.y, x.x, x.y);
}

__global__ void __launch_bounds__(32 * kWarps, kCtasPerSm)
    expm32_pairs_kernel(const float* __restrict__ a, float* __restrict__ out,
                        const int2* __restrict__ list, int64_t batch, int quad_lanes) {
    extern __shared__ __align__(16) float smem[];
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + kWarps * 2 * kHalfFloats);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         uint32_t(__cvta_generic_to_shared(tmem_slot))),
                     "n"(kTmemCols)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = *tmem_slot;

    const int h = lane >> 4, hl = lane & 15;
    Lane L;
    // An aligned quad of lanes owns a 2x2 block of tiles. The shared-memory
    // pipe merges identical addresses only inside an aligned lane quad and
    // serves 16 (quad, address) requests per 64-bit wavefront, 8 per 128-bit
    // one (tools/lds_patterns.cu): with two ti and two tj per quad an X load
    // (address by ti, LDS.64) is 1 wavefront and a Y load (address by tj,
    // LDS.128) 2, against 1-2 and 4 with (ti, tj) = (hl >> 2, hl & 3) --
    // 16 instead of 24-32 wavefronts per two k of the product loop.
    // (quad_lanes = 0, MEXP_PAIRS_LANES=0: the row-major lane order, for A/B runs)
    L.ti = quad_lanes ? ((hl >> 3) << 1) | ((hl >> 1) & 1) : hl >> 2;
    L.tj = quad_lanes ? (((hl >> 2) & 1) << 1) | (hl & 1) : hl & 3;
    L.diag = L.ti == L.tj;
    L.xbuf = smem + (warp * 2 + h) * kHalfFloats;
    L.ybuf = L.xbuf + kBufFloats;
    L.tm = tmem + (uint32_t(32 * warp) << 16);
    float* const pbuf = L.ybuf + kBufFloats;

    // Pairs p, p + stride, ...: the next pair's matrices are copied into pbuf
    // by cp.async while the current pair computes (issued once the current
    // pair's first step has consumed pbuf), and the list entry of the pair
    // after next is loaded one pair ahead.
    const int64_t npairs = (batch + 1) / 2;
    const int64_t stride = int64_t(gridDim.x) * kWarps;
    const int64_t first = int64_t(blockIdx.x) * kWarps + warp;
    const int64_t count = first < npairs ? (npairs - first + stride - 1) / stride : 0;
    auto pair_index = [&](int64_t k) { return first + k * stride; };
    int4 cur = make_int4(0, 0, 0, 0), nxt = cur;
    if (count > 0) {
        cur = pair_at(list, pair_index(0), batch);
        prefetch_tile(L, pbuf, a + int64_t(h ? cur.z : cur.x) * NN);
        nxt = count > 1 ? pair_at(list, pair_index(1), batch) : cur;
    }
    for (int64_t k = 0; k < count; ++k) {
        bool pending = k + 1 < count;
        asm volatile("cp.async.wait_all;" ::: "memory");
        const bool joint = cur.y == cur.w;
#pragma unroll 1
        for (int rep = 0; rep < (joint ? 1 : 2); ++rep) {
            const int64_t m = joint ? (h ? cur.z : cur.x) : (rep ? cur.z : cur.x);
            const bool write = joint || h == rep;
            const uint32_t info = uint32_t(rep ? cur.w : cur.y);
            const int degree = info_degree(info), s = info_s(info);
            Acc C;
            if (info_status(info) != MEXP_OK) {
                const float nan = __int_as_float(0x7fc00000);
#pragma unroll
                for (int e = 0; e < 32; ++e) C[e] = make_float2(nan, nan);
            } else {
                if (joint && kPrefetch)
                    load_tile_smem(L, pbuf, C);
                else
                    load_tile(L, a + m * NN, C);
                if (s > 0) {  // exact scaling by 2^-s, rounded once to float
                    if (s <= 126) {
                        const float f = __int_as_float((127 - s) << 23);
#pragma unroll
                        for (int e = 0; e < 32; ++e) C[e] = __fmul2_rn(make_float2(f, f), C[e]);
                    } else {
                        const double f = pow2_neg(s);
#pragma unroll
                        for (int e = 0; e < 32; ++e)
                            C[e] = make_float2(float(f * double(C[e].x)), float(f * double(C[e].y)));
                    }
                }
#pragma unroll 1
                for (int step = 0;; ++step) {
                    const float* py;
                    const float* px = stage(L, degree, step, s, C, py);
                    if (pending) {  // step 0 has consumed the values read from pbuf
                        prefetch_tile(L, pbuf, a + int64_t(h ? nxt.z : nxt.x) * NN);
                        pending = false;
                    }
                    if (!px) break;
                    kloop(L, px, py, C);
                }
            }
            if (write) store_tile(L, out + m * NN, C);
        }
        if (pending) prefetch_tile(L, pbuf, a + int64_t(h ? nxt.z : nxt.x) * NN);
        cur = nxt;
        if (k + 2 < count) nxt = pair_at(list, pair_index(k + 2), batch);
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(kTmemCols)
                     : "memory");
}

int sm_count_pairs() {
    int dev = 0, v = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    return v;
}

}  // namespace

// MEXP_F32_PAIRS: 0 = the one-warp kernel, 1 = the pair kernel at any batch,
// unset = the pair kernel from 8192 matrices up (below that its pre-pass and
// part-filled grid cost more than they save: the host pipeline's 16 MiB
// chunks of 4096 matrices measured e2e 9.6e6 vs 1.0e7 expm/s). Read per call
// (a getenv), so tests can compare both kernels in one process.
bool pairs32_enabled(int64_t batch) {
    if (batch > (int64_t(1) << 31) - 2) return false;  // the class list holds int32 indices
    const char* e = std::getenv("MEXP_F32_PAIRS");
    if (e) return std::atoi(e) != 0;
    return batch >= 8192;
}

// Pre-pass (selection records, class list) and the pair kernel, in stream
// order on `st`. (Chunking the batch so that chunk c + 1's pre-pass runs next
// to chunk c's pair kernel on a side stream was measured slower: 630 vs 550 us
// for cfg3 -- each chunk's pair kernel pays its own tail, and the pre-pass
// blocks that fit beside two pair CTAs per SM are latency-bound.)
int run_pairs32_f32(const float* d_a, float* d_out, mexp_selection* d_sel, int64_t batch,
                    int accuracy, cudaStream_t st, std::atomic<uint64_t>* launches) {
    if (batch <= 0) return MEXP_OK;
    if (batch > (int64_t(1) << 31) - 2) return MEXP_ERR_UNSUPPORTED;  // int32 list
    static PerDevice attr_once;
    attr_once([] {
        cudaFuncSetAttribute(expm32_pairs_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes);
    });
    // workspace: [hist | running] ints, packed (degree, s, status) per matrix,
    // the class-sorted list {m, info}, and selection records when the caller
    // passes none (the pair kernel reads (m, s) from the list)
    const size_t hist_bytes = 2 * 1024 * sizeof(int);
    const size_t info_bytes = ((size_t(batch) * sizeof(uint32_t)) + 255) & ~size_t(255);
    const size_t list_bytes = ((size_t(batch) * sizeof(int2)) + 255) & ~size_t(255);
    const size_t sel_bytes = d_sel ? 0 : size_t(batch) * sizeof(mexp_selection);
    AsyncBuffer ws(st);
    if (ws.alloc(hist_bytes + info_bytes + list_bytes + sel_bytes) != cudaSuccess) return MEXP_ERR_CUDA;
    char* w = ws.get<char>();
    int* hist = reinterpret_cast<int*>(w);
    int* running = hist + 1024;
    uint32_t* info = reinterpret_cast<uint32_t*>(w + hist_bytes);
    int2* list = reinterpret_cast<int2*>(w + hist_bytes + info_bytes);
    mexp_selection* sel = d_sel ? d_sel
                                : reinterpret_cast<mexp_selection*>(w + hist_bytes + info_bytes + list_bytes);
    if (cudaMemsetAsync(hist, 0, 2 * 1024 * sizeof(int), st) != cudaSuccess) return MEXP_ERR_CUDA;
    const int sms = sm_count_pairs();
    const int64_t sblocks = (batch + 7) / 8;
    const int sgrid = int(sblocks < 8 * sms ? sblocks : 8 * sms);
    select32_kernel<<<sgrid, 256, 0, st>>>(d_a, sel, info, hist, batch, accuracy & 15);
    const int cgrid = int((batch + kScatterChunk - 1) / kScatterChunk);
    scatter32_kernel<<<cgrid, 1024, 0, st>>>(info, hist, running, list, batch);
    const int64_t npairs = (batch + 1) / 2;
    const int64_t want = (npairs + kWarps - 1) / kWarps;
    const int grid = int(want < kCtasPerSm * sms ? want : kCtasPerSm * sms);
    static const int quad_lanes = [] {
        const char* e = std::getenv("MEXP_PAIRS_LANES");
        return e ? std::atoi(e) : 1;
    }();
    expm32_pairs_kernel<<<grid, 32 * kWarps, kSmemBytes, st>>>(d_a, d_out, list, batch, quad_lanes);
    launches->fetch_add(3, std::memory_order_relaxed);
    return cudaGetLastError() == cudaSuccess ? MEXP_OK : MEXP_ERR_CUDA;
}

}  // namespace mexp_b200
