// reduce.cu -- inner product and Frobenius norm on sm_100a.
//
// Reference: inner_product_tensors -> inner_product_flat(a, b, 0)
// (contraction.py:457-459, elementwise.py:411-433) folds a[i] * b[i] over
// the shared multi-index; frobenius_norm = sqrt(inner(a, a))
// (contraction.py:462-464).  A whole-tensor fold cannot stay sequential on
// a GPU, so these kernels are the one place where results are not
// bit-identical to the reference: every product is formed exactly
// (TwoProd via FMA for float64; float32 products are exact in binary64)
// and summed in double-double (TwoSum) per thread, per warp, per CTA and
// across CTAs in a fixed order -- accurate to ~1 ulp of the true sum and
// deterministic run to run.  The reference's own sequential fold carries
// rounding error of order N eps sum|a b|; parity is therefore checked
// against |delta| <= rtol * sum|a_i b_i| (tests/).
//
// Kernels (all HBM-bound, persistent grid = a multiple of the SM count):
//   dot_rows   -- a and b share their fastest dimension: rows of
//                 contiguous elements (a flat same-layout buffer is one
//                 row); 128-bit streaming loads.
//   dot_tiled  -- a's and b's fastest dimensions differ (e.g. first-order
//                 x last-order): 32x32 tiles, b staged through padded
//                 shared memory so both operands are read coalesced.
// The last CTA to finish (atomic ticket) combines the per-CTA partials and
// resets the ticket, so the workspace stays zeroed for graph replay.
#include <cstdio>
#include <cstdlib>
#include <numeric>
#include <type_traits>
#include <vector>

#include "plan.h"
#include "tl_common.cuh"

namespace tl {

constexpr int kMaxPartials = 148 * 8;
// longest FMA chain per binary64 partial of a sum of squares: relative error
// <= (kFmaChain + log2(partials)) * 2^-53 < 5e-13
constexpr int64_t kFmaChain = 4096;

struct DD {  // double-double accumulator
    double hi, lo;
};

__device__ __forceinline__ void two_sum_add(DD &acc, double x) {
    const double s = acc.hi + x;
    const double bp = s - acc.hi;
    const double err = (acc.hi - (s - bp)) + (x - bp);
    acc.hi = s;
    acc.lo += err;
}
__device__ __forceinline__ void dd_add_prod(DD &acc, double a, double b) {
    const double p = a * b;
    const double e = fma(a, b, -p);  // exact product error
    two_sum_add(acc, p);
    acc.lo += e;
}
__device__ __forceinline__ DD dd_merge(DD x, DD y) {
    DD r = x;
    two_sum_add(r, y.hi);
    r.lo += y.lo;
    return r;
}

struct Acc64 {  // exact int64 accumulator (mod 2^64)
    int64_t v;
};

template <class T> struct RedAcc { using type = DD; };
template <> struct RedAcc<int64_t> { using type = Acc64; };

__device__ __forceinline__ void acc_zero(DD &a) { a.hi = 0.0; a.lo = 0.0; }
__device__ __forceinline__ void acc_zero(Acc64 &a) { a.v = 0; }
__device__ __forceinline__ void acc_prod(DD &a, double x, double y) { dd_add_prod(a, x, y); }
__device__ __forceinline__ void acc_prod(Acc64 &a, int64_t x, int64_t y) {
    a.v = (int64_t)((uint64_t)a.v + (uint64_t)x * (uint64_t)y);
}
__device__ __forceinline__ DD acc_merge(DD x, DD y) { return dd_merge(x, y); }
__device__ __forceinline__ Acc64 acc_merge(Acc64 x, Acc64 y) {
    return Acc64{(int64_t)((uint64_t)x.v + (uint64_t)y.v)};
}
__device__ __forceinline__ DD shfl_down(DD a, int d) {
    DD r;
    r.hi = __shfl_down_sync(0xffffffffu, a.hi, d);
    r.lo = __shfl_down_sync(0xffffffffu, a.lo, d);
    return r;
}
__device__ __forceinline__ Acc64 shfl_down(Acc64 a, int d) {
    return Acc64{(int64_t)__shfl_down_sync(0xffffffffu, (long long)a.v, d)};
}

struct ReduceParams {
    const void *a;
    const void *b;
    void *result;  // double* (float operands) or int64_t* (int64 operands)
    double *partials;
    unsigned int *ticket;
    int32_t sqrt_result;
    double init_f;    // inner_product_flat's init (elementwise.py:411): the fold's starting value
    int64_t init_i;
    int64_t n_rows, row_len;  // dot_rows
    DigitMap rows_a, rows_b;  // row index -> element offsets
    int32_t row_vec;          // rows are whole, aligned 16-byte vectors in both operands
    FastDiv rowv_div;         // vectors per row
    // dot_tiled
    int64_t nX, nY, n_rest;
    int64_t a_sY, b_sX;  // a's stride along Y, b's stride along X
    DigitMap rest_a, rest_b;
    int64_t tiles_x, tiles_y;
    // past 2^32 rows / tiles: a's memory order e -> b's offset
    int64_t n_elem;
    DigitMap64 b64;
};

// Block-level reduction of one accumulator per thread; returns the CTA sum
// in thread 0.
template <class Acc> __device__ Acc block_reduce(Acc v) {
    __shared__ Acc warp_part[32];
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) v = acc_merge(v, shfl_down(v, d));
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (lane == 0) warp_part[wid] = v;
    __syncthreads();
    Acc r;
    acc_zero(r);
    if (wid == 0) {
        const int nw = blockDim.x >> 5;
        if (lane < nw) r = warp_part[lane];
#pragma unroll
        for (int d = 16; d > 0; d >>= 1) r = acc_merge(r, shfl_down(r, d));
    }
    return r;
}

__device__ __forceinline__ void store_partial(double *partials, int idx, DD v) {
    partials[2 * idx] = v.hi;
    partials[2 * idx + 1] = v.lo;
}
__device__ __forceinline__ void store_partial(double *partials, int idx, Acc64 v) {
    ((int64_t *)partials)[2 * idx] = v.v;
}
__device__ __forceinline__ DD load_partial(const double *partials, int idx, DD *) {
    return DD{__ldcg(partials + 2 * idx), __ldcg(partials + 2 * idx + 1)};
}
__device__ __forceinline__ Acc64 load_partial(const double *partials, int idx, Acc64 *) {
    return Acc64{(int64_t)__ldcg((const long long *)partials + 2 * idx)};
}
__device__ __forceinline__ void write_result(const ReduceParams &P, DD v) {
    two_sum_add(v, P.init_f);  // init enters the compensated sum before its single final rounding
    double r = v.hi + v.lo;
    if (P.sqrt_result) r = sqrt(r);
    *(double *)P.result = r;
}
__device__ __forceinline__ void write_result(const ReduceParams &P, Acc64 v) {
    *(int64_t *)P.result = (int64_t)((uint64_t)v.v + (uint64_t)P.init_i);
}

// Per-CTA partial -> global; last CTA folds partials in index order.
template <class Acc> __device__ void finish(const ReduceParams &P, Acc cta) {
    __shared__ bool am_last;
    if (gridDim.x == 1) {  // one CTA: its sum is the result (no partials, no ticket)
        if (threadIdx.x == 0) write_result(P, cta);
        return;
    }
    if (threadIdx.x == 0) {
        store_partial(P.partials, blockIdx.x, cta);
        // release: the partial is visible before the ticket moves; acquire:
        // the last CTA then sees every other CTA's partial
        unsigned prev;
        asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(prev) : "l"(P.ticket) : "memory");
        am_last = (prev == gridDim.x - 1);
    }
    __syncthreads();
    if (!am_last) return;
    Acc v;
    acc_zero(v);
    for (int i = threadIdx.x; i < (int)gridDim.x; i += blockDim.x)
        v = acc_merge(v, load_partial(P.partials, i, (Acc *)nullptr));
    v = block_reduce(v);
    if (threadIdx.x == 0) {
        write_result(P, v);
        *P.ticket = 0u;  // leave the workspace zeroed
    }
}

template <class T> __device__ __forceinline__ typename std::conditional<std::is_same<T, int64_t>::value, int64_t, double>::type
as_acc(T v) {
    return v;
}

// ------------------------------------------------------------ dot_rows
// Per-thread partial sums.  float32 operands: products are exact in
// binary64, so one FMA per element (acc += a*b rounded once) into VEC
// independent accumulators -- one FP64 op per element keeps the kernel
// HBM-bound.  float64: TwoProd + TwoSum (double-double) per element.
template <class TA> struct ThreadAcc {
    DD dd[2];
    __device__ void zero() { dd[0] = DD{0.0, 0.0}; dd[1] = DD{0.0, 0.0}; }
    __device__ void add(int j, double x, double y) { dd_add_prod(dd[j & 1], x, y); }
    __device__ DD total() const { return dd_merge(dd[0], dd[1]); }
};
// FMA accumulation into 4 binary64 partials: exact products for float32;
// for float64 sums of squares (the norm) when every partial folds at most
// kFmaChain terms, so the blocked-sum bound (L + log2 P) eps stays < 1e-12.
struct FmaAcc {
    double s[4];
    __device__ void zero() { s[0] = s[1] = s[2] = s[3] = 0.0; }
    __device__ void add(int j, double x, double y) { s[j & 3] = fma(x, y, s[j & 3]); }
    __device__ DD total() const {
        DD r{s[0], 0.0};
        two_sum_add(r, s[1]);
        two_sum_add(r, s[2]);
        two_sum_add(r, s[3]);
        return r;
    }
};
template <> struct ThreadAcc<float> : FmaAcc {};
template <> struct ThreadAcc<int64_t> {
    Acc64 a;
    __device__ void zero() { a.v = 0; }
    __device__ void add(int, int64_t x, int64_t y) { acc_prod(a, x, y); }
    __device__ Acc64 total() const { return a; }
};

template <class T, int VEC> __device__ __forceinline__ void load_vec(const T *p, T (&x)[VEC]) {
    if constexpr (VEC * sizeof(T) == 16) {
        *(uint4 *)x = __ldcs((const uint4 *)p);
    } else {
#pragma unroll
        for (int j = 0; j < VEC; ++j) x[j] = __ldcs(p + j);
    }
}

template <class TA, class TB, int VEC, bool SAME, int U = 4, bool FMA_ACC = false, bool ROWV = false>
__global__ void __launch_bounds__(256) dot_rows_kernel(const __grid_constant__ ReduceParams P) {
    using Acc = typename RedAcc<TA>::type;
    typename std::conditional<FMA_ACC, FmaAcc, ThreadAcc<TA>>::type ta;
    ta.zero();
    const TA *a = (const TA *)P.a;
    const TB *b = (const TB *)P.b;
    const int64_t L = P.row_len;
    const int64_t nthreads = (int64_t)gridDim.x * blockDim.x;
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (P.n_rows == 1) {
        // flat: 128-bit streaming loads, U vectors in flight per thread
        const int64_t nv = L / VEC;
        int64_t v = tid;
        for (; v + (U - 1) * nthreads < nv; v += U * nthreads) {
            TA xa[U][VEC];
            TB xb[U][VEC];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                load_vec<TA, VEC>(a + (v + u * nthreads) * VEC, xa[u]);
                if constexpr (!SAME) load_vec<TB, VEC>(b + (v + u * nthreads) * VEC, xb[u]);
            }
#pragma unroll
            for (int u = 0; u < U; ++u)
#pragma unroll
                for (int j = 0; j < VEC; ++j) {
                    if constexpr (SAME)
                        ta.add(u * VEC + j, as_acc(xa[u][j]), as_acc(xa[u][j]));
                    else
                        ta.add(u * VEC + j, as_acc(xa[u][j]), as_acc(xb[u][j]));
                }
        }
        for (; v < nv; v += nthreads) {
            TA xa[VEC];
            TB xb[VEC];
            load_vec<TA, VEC>(a + v * VEC, xa);
            if constexpr (!SAME) load_vec<TB, VEC>(b + v * VEC, xb);
#pragma unroll
            for (int j = 0; j < VEC; ++j) {
                if constexpr (SAME)
                    ta.add(j, as_acc(xa[j]), as_acc(xa[j]));
                else
                    ta.add(j, as_acc(xa[j]), as_acc(xb[j]));
            }
        }
        for (int64_t e = nv * VEC + tid; e < L; e += nthreads) ta.add(0, as_acc(a[e]), as_acc(b[e]));
    } else if (ROWV && VEC > 1 && P.row_vec) {
        // rows along the shared fastest dimension, in a different order in b
        // (e.g. layouts (1,2,3,4) x (1,4,2,3)): 16-byte vectors, U in flight
        // per thread and operand, row starts through b's digit map
        const uint32_t nvr = (uint32_t)(L / VEC);
        const int64_t nv = P.n_rows * nvr;
        auto offs = [&](int64_t v, int64_t &oa, int64_t &ob) {
            uint32_t r, c;
            P.rowv_div.divmod((uint32_t)v, r, c);
            oa = (int64_t)r * L + (int64_t)c * VEC;
            ob = P.rows_b.map(r) + (int64_t)c * VEC;
        };
        int64_t v = tid;
        for (; v + (U - 1) * nthreads < nv; v += U * nthreads) {
            TA xa[U][VEC];
            TB xb[U][VEC];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                int64_t oa, ob;
                offs(v + u * nthreads, oa, ob);
                load_vec<TA, VEC>(a + oa, xa[u]);
                load_vec<TB, VEC>(b + ob, xb[u]);
            }
#pragma unroll
            for (int u = 0; u < U; ++u)
#pragma unroll
                for (int j = 0; j < VEC; ++j) ta.add(u * VEC + j, as_acc(xa[u][j]), as_acc(xb[u][j]));
        }
        for (; v < nv; v += nthreads) {
            TA xa[VEC];
            TB xb[VEC];
            int64_t oa, ob;
            offs(v, oa, ob);
            load_vec<TA, VEC>(a + oa, xa);
            load_vec<TB, VEC>(b + ob, xb);
#pragma unroll
            for (int j = 0; j < VEC; ++j) ta.add(j, as_acc(xa[j]), as_acc(xb[j]));
        }
    } else {
        const int64_t total = P.n_rows * L;
        for (int64_t e = tid; e < total; e += nthreads) {
            const int64_t r = e / L;
            const int64_t c = e - r * L;
            const int64_t oa = P.rows_a.map((uint32_t)r) + c;
            const int64_t ob = P.rows_b.map((uint32_t)r) + c;
            ta.add((int)c, as_acc(__ldcs(a + oa)), as_acc(__ldcs(b + ob)));
        }
    }
    Acc acc = block_reduce(ta.total());
    finish(P, acc);
}

// ------------------------------------------------------------ dot_tiled
template <class TA, class TB>
__global__ void __launch_bounds__(256) dot_tiled_kernel(const __grid_constant__ ReduceParams P) {
    using Acc = typename RedAcc<TA>::type;
    __shared__ TB tile[32][33];
    ThreadAcc<TA> ta;
    ta.zero();
    const TA *a = (const TA *)P.a;
    const TB *b = (const TB *)P.b;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int64_t tiles = P.tiles_x * P.tiles_y * P.n_rest;
    for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
        const int64_t rest = t / (P.tiles_x * P.tiles_y);
        const int64_t txy = t - rest * (P.tiles_x * P.tiles_y);
        const int64_t ty = txy / P.tiles_x;
        const int64_t tx = txy - ty * P.tiles_x;
        const int64_t x0 = tx * 32, y0 = ty * 32;
        const int64_t ra = P.rest_a.map((uint32_t)rest), rb = P.rest_b.map((uint32_t)rest);
        // b tile: coalesced along Y (b's fastest dimension)
        for (int xr = wid; xr < 32; xr += 8) {
            const int64_t x = x0 + xr, y = y0 + lane;
            if (x < P.nX && y < P.nY) tile[xr][lane] = __ldcs(b + rb + x * P.b_sX + y);
        }
        __syncthreads();
        // a: coalesced along X (a's fastest dimension); b from the tile
        for (int yr = wid; yr < 32; yr += 8) {
            const int64_t x = x0 + lane, y = y0 + yr;
            if (x < P.nX && y < P.nY) ta.add(yr, as_acc(__ldcs(a + ra + x + y * P.a_sY)), as_acc(tile[lane][yr]));
        }
        __syncthreads();
    }
    Acc acc = block_reduce(ta.total());
    finish(P, acc);
}

// ------------------------------------------------------------ dot_tiled (vector)
// Same contraction with 64x64 tiles and 16-byte loads: a is read along X
// (its unit-stride dimension) and b along Y, each thread keeps 4 + 4 vectors
// in flight; b's tile is transposed through shared memory so that a thread
// multiplies a 16-byte run of a with a 16-byte run of the transposed b tile.
constexpr int kT = 64;

template <class T>
__global__ void __launch_bounds__(256) dot_tiled_vec_kernel(const __grid_constant__ ReduceParams P) {
    using Acc = typename RedAcc<T>::type;
    constexpr int V = 16 / sizeof(T);     // elements per 16-byte vector
    constexpr int VR = kT / V;            // vectors per tile row
    constexpr int PITCH = kT;             // bt[y][x ^ swz(y)]: XOR swizzle in units of V
    __shared__ __align__(16) T bt[kT * PITCH];
    auto swz = [](int y) { return ((y / V) & 7) * V; };
    ThreadAcc<T> ta;
    ta.zero();
    const T *a = (const T *)P.a;
    const T *b = (const T *)P.b;
    const int64_t per_rest = P.tiles_x * P.tiles_y;
    const int64_t tiles = per_rest * P.n_rest;
    constexpr int NV = kT * VR / 256;  // vectors per thread per operand tile
    for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
        const int64_t rest = t / per_rest;
        const int64_t txy = t - rest * per_rest;
        const int64_t ty = txy / P.tiles_x;
        const int64_t tx = txy - ty * P.tiles_x;
        const int64_t x0 = tx * kT, y0 = ty * kT;
        const int64_t ra = P.rest_a.map((uint32_t)rest), rb = P.rest_b.map((uint32_t)rest);
        T av[NV][V], bv[NV][V];
#pragma unroll
        for (int q = 0; q < NV; ++q) {
            const int e = threadIdx.x + q * 256;
            const int row = e / VR, vc = (e % VR) * V;
            // b: row = x (fixed), along y; a: row = y (fixed), along x
            *(uint4 *)bv[q] = __ldcs((const uint4 *)(b + rb + (x0 + row) * P.b_sX + y0 + vc));
            *(uint4 *)av[q] = __ldcs((const uint4 *)(a + ra + (y0 + row) * P.a_sY + x0 + vc));
        }
#pragma unroll
        for (int q = 0; q < NV; ++q) {
            const int e = threadIdx.x + q * 256;
            const int row = e / VR, vc = (e % VR) * V;
#pragma unroll
            for (int c = 0; c < V; ++c) bt[(vc + c) * PITCH + (row ^ swz(vc + c))] = bv[q][c];  // b(x=row, y)
        }
        __syncthreads();
#pragma unroll
        for (int q = 0; q < NV; ++q) {
            const int e = threadIdx.x + q * 256;
            const int row = e / VR, vc = (e % VR) * V;  // a's row y = row, x = vc..vc+V-1
            T bb[V];
            *(uint4 *)bb = *(const uint4 *)(bt + row * PITCH + (vc ^ swz(row)));
#pragma unroll
            for (int c = 0; c < V; ++c) ta.add(c, as_acc(av[q][c]), as_acc(bb[c]));
        }
        __syncthreads();
    }
    Acc acc = block_reduce(ta.total());
    finish(P, acc);
}

// ------------------------------------------------------------ past 2^32
// Index ranges beyond the 32-bit maps (2^33+ elements with short rows or
// tiles): a is walked in its memory order, b's offset of the same element
// comes from a 64-bit digit map; same accumulators and combine.
template <class TA, class TB>
__global__ void __launch_bounds__(256) dot_generic64_kernel(const __grid_constant__ ReduceParams P) {
    using Acc = typename RedAcc<TA>::type;
    ThreadAcc<TA> ta;
    ta.zero();
    const TA *a = (const TA *)P.a;
    const TB *b = (const TB *)P.b;
    const int64_t nth = (int64_t)gridDim.x * blockDim.x;
    int j = 0;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < P.n_elem; e += nth, ++j)
        ta.add(j, as_acc(__ldcs(a + e)), as_acc(__ldcs(b + P.b64.map((uint64_t)e))));
    Acc acc = block_reduce(ta.total());
    finish(P, acc);
}

size_t reduce_workspace_bytes();

// ------------------------------------------------------------ rank one / residual
// rank_one_compose (hopm.py:123-139): B(i) = scale * u_1(i_1) * ... * u_p(i_p),
// multiplied left to right exactly as the reference does; residual
// (hopm.py:142-147): ||A - B||_F without materialising B.  A is walked in its
// memory order along rows of its fastest dimension; each element's
// multi-index comes from a digit decode of the row index.
struct RankOneParams {
    const void *a;        // residual: A (any dense layout); compose: unused
    double *out;          // compose: first-order B
    const double *u[TL_MAX_ORDER];
    const double *scale;  // device scalar (graph-capturable)
    const int32_t *gate;  // residual inside HOPM: run only if *gate == gate_value
    int32_t gate_value;
    int32_t p;
    int32_t fast;          // dimension walked along rows
    int64_t row_len, n_rows;
    FastDiv rdiv[TL_MAX_ORDER];  // row index -> indices of the other dims (storage order)
    int32_t rdim[TL_MAX_ORDER];
    int32_t nrd;
    int64_t out_stride[TL_MAX_ORDER];  // compose: first-order strides
    // reduction plumbing (residual)
    double *result;
    double *partials;
    unsigned int *ticket;
};

__device__ __forceinline__ void rank_one_row(const RankOneParams &P, int64_t row, int32_t *idx) {
    uint32_t x = (uint32_t)row;
    for (int d = 0; d < P.nrd; ++d) {
        uint32_t q, r;
        if (d == P.nrd - 1) {
            r = x;
            q = 0;
        } else {
            P.rdiv[d].divmod(x, q, r);
        }
        idx[P.rdim[d]] = (int32_t)r;
        x = q;
    }
}

__global__ void __launch_bounds__(256) rank_one_compose_kernel(const __grid_constant__ RankOneParams P) {
    const double scale = *P.scale;
    int32_t idx[TL_MAX_ORDER];
    const int64_t total = P.n_rows * P.row_len;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t row = e / P.row_len, c = e - row * P.row_len;
        rank_one_row(P, row, idx);
        idx[P.fast] = (int32_t)c;
        double v = scale;
        int64_t off = 0;
        for (int r = 0; r < P.p; ++r) {
            v = __dmul_rn(v, P.u[r][idx[r]]);
            off += (int64_t)idx[r] * P.out_stride[r];
        }
        P.out[off] = v;
    }
}

template <class TA>
__global__ void __launch_bounds__(256) residual_kernel(const __grid_constant__ RankOneParams P) {
    if (P.gate != nullptr && *(volatile const int32_t *)P.gate != P.gate_value) return;
    const double scale = *P.scale;
    const TA *a = (const TA *)P.a;
    DD acc{0.0, 0.0};
    int32_t idx[TL_MAX_ORDER];
    const int64_t total = P.n_rows * P.row_len;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t row = e / P.row_len, c = e - row * P.row_len;
        rank_one_row(P, row, idx);
        idx[P.fast] = (int32_t)c;
        double v = scale;
        for (int r = 0; r < P.p; ++r) v = __dmul_rn(v, P.u[r][idx[r]]);
        const double d = __dsub_rn((double)a[e], v);  // A's memory order == e
        dd_add_prod(acc, d, d);
    }
    ReduceParams R{};
    R.result = P.result;
    R.partials = P.partials;
    R.ticket = P.ticket;
    R.sqrt_result = 1;
    finish(R, block_reduce(acc));
}

static bool rank_one_plan(const tl_desc &a, RankOneParams &P) {
    std::vector<int> dims;
    if (!dense_order(a, dims)) return false;
    P.p = a.order;
    if (dims.empty()) {  // all extents 1
        P.fast = 0;
        P.row_len = 1;
        P.n_rows = 1;
        P.nrd = 0;
        return true;
    }
    P.fast = dims[0];
    P.row_len = a.extent[dims[0]];
    P.n_rows = volume(a) / P.row_len;
    if (P.n_rows > 0xffffffffll) return false;
    P.nrd = 0;
    for (size_t d = 1; d < dims.size(); ++d) {
        P.rdiv[P.nrd].init((uint32_t)a.extent[dims[d]]);
        P.rdim[P.nrd] = dims[d];
        ++P.nrd;
    }
    return true;
}

int rank_one_enqueue(const tl_desc &shape, const double *const *u, const double *scale_dev, double *out,
                     cudaStream_t st) {
    RankOneParams P{};
    tl_desc fo = shape;  // first-order output
    int64_t run = 1;
    for (int r = 0; r < fo.order; ++r) {
        fo.stride[r] = run;
        P.out_stride[r] = run;
        run *= fo.extent[r];
    }
    if (!rank_one_plan(fo, P)) return TL_EUNSUPPORTED;
    for (int r = 0; r < fo.order; ++r) P.u[r] = u[r];
    P.scale = scale_dev;
    P.out = out;
    const int64_t total = P.n_rows * P.row_len;
    const int64_t grid = std::max<int64_t>(1, std::min<int64_t>((total + 255) / 256, (int64_t)device_info().num_sms * 8));
    rank_one_compose_kernel<<<(unsigned)grid, 256, 0, st>>>(P);
    return cuda_status(cudaGetLastError(), "rank_one_compose launch");
}

int residual_enqueue(const tl_desc &a, const void *a_ptr, const double *const *u, const double *scale_dev,
                     const int32_t *gate, int32_t gate_value, double *result, void *ws, size_t ws_bytes,
                     cudaStream_t st) {
    if (ws == nullptr || ws_bytes < reduce_workspace_bytes()) {
        set_error("residual: workspace of %zu bytes required", reduce_workspace_bytes());
        return TL_EWORKSPACE;
    }
    RankOneParams P{};
    if (!rank_one_plan(a, P)) {
        set_error("residual: A must be a dense permutation layout");
        return TL_EUNSUPPORTED;
    }
    for (int r = 0; r < a.order; ++r) P.u[r] = u[r];
    P.a = (const unsigned char *)a_ptr + a.offset * (int64_t)dtype_size(a.dtype);
    P.scale = scale_dev;
    P.gate = gate;
    P.gate_value = gate_value;
    P.result = result;
    P.partials = (double *)ws;
    P.ticket = (unsigned int *)((unsigned char *)ws + (size_t)kMaxPartials * 2 * sizeof(double));
    const int64_t total = P.n_rows * P.row_len;
    const int64_t grid =
        std::max<int64_t>(1, std::min<int64_t>((total + 255) / 256, std::min<int64_t>(device_info().num_sms * 4, kMaxPartials)));
    if (a.dtype == TL_F32)
        residual_kernel<float><<<(unsigned)grid, 256, 0, st>>>(P);
    else if (a.dtype == TL_F64)
        residual_kernel<double><<<(unsigned)grid, 256, 0, st>>>(P);
    else {
        set_error("residual requires floating elements");
        return TL_EUNSUPPORTED;
    }
    return cuda_status(cudaGetLastError(), "residual launch");
}

// ------------------------------------------------------------ planning
size_t reduce_workspace_bytes() { return (size_t)kMaxPartials * 2 * sizeof(double) + 256; }

int reduce_enqueue(const tl_desc &a, const void *a_ptr, const tl_desc &b, const void *b_ptr, void *result,
                   bool do_sqrt, void *ws, size_t ws_bytes, cudaStream_t st, const void *init) {
    if (ws == nullptr || ws_bytes < reduce_workspace_bytes()) {
        set_error("inner/norm: workspace of %zu bytes required", reduce_workspace_bytes());
        return TL_EWORKSPACE;
    }
    std::vector<int> da, db;
    if (!dense_order(a, da) || !dense_order(b, db)) {
        set_error("inner/norm: operands must be dense permutation layouts (materialise views first)");
        return TL_EUNSUPPORTED;
    }
    const DeviceInfo &di = device_info();
    ReduceParams P{};
    const size_t sa = dtype_size(a.dtype), sb = dtype_size(b.dtype);
    P.a = (const unsigned char *)a_ptr + a.offset * (int64_t)sa;
    P.b = (const unsigned char *)b_ptr + b.offset * (int64_t)sb;
    P.result = result;
    P.partials = (double *)ws;
    P.ticket = (unsigned int *)((unsigned char *)ws + (size_t)kMaxPartials * 2 * sizeof(double));
    P.sqrt_result = do_sqrt ? 1 : 0;
    if (init != nullptr) {
        if (a.dtype == TL_I64) P.init_i = *(const int64_t *)init;
        else P.init_f = *(const double *)init;
    }
    const int64_t N = volume(a);
    const bool same_fast = da.empty() || db.empty() || da[0] == db[0];
    const bool is_int = a.dtype == TL_I64;
    if (is_int != (b.dtype == TL_I64)) {
        set_error("inner: mixing integer and floating operands is not supported");
        return TL_EUNSUPPORTED;
    }
    cudaError_t e = cudaSuccess;
    const int threads = 256;
    if (N == 0) {
        set_error("inner: empty tensor");
        return TL_EINVAL;
    }
    {
        // index ranges past the 32-bit maps: the generic 64-bit walk
        DigitList dl;
        for (int r : da) dl.push_back({a.extent[r], b.stride[r]});
        DigitList col = collapse(dl);
        bool big = N > kIdx32 && col.size() > 1;
        for (auto &dg : col) big = big || dg.first > kIdx32;
        if (big) {
            P.n_elem = N;
            build_map64(col, P.b64);
            const int64_t grid = std::min<int64_t>((N + threads - 1) / threads, std::min<int64_t>((int64_t)di.num_sms * 4, kMaxPartials));
            const unsigned G = (unsigned)grid;
            if (a.dtype == TL_F32 && b.dtype == TL_F32) dot_generic64_kernel<float, float><<<G, threads, 0, st>>>(P);
            else if (a.dtype == TL_F64 && b.dtype == TL_F64) dot_generic64_kernel<double, double><<<G, threads, 0, st>>>(P);
            else if (a.dtype == TL_F32 && b.dtype == TL_F64) dot_generic64_kernel<float, double><<<G, threads, 0, st>>>(P);
            else if (a.dtype == TL_F64 && b.dtype == TL_F32) dot_generic64_kernel<double, float><<<G, threads, 0, st>>>(P);
            else dot_generic64_kernel<int64_t, int64_t><<<G, threads, 0, st>>>(P);
            return cuda_status(cudaGetLastError(), "inner/norm (64-bit index) launch");
        }
    }
    if (same_fast) {
        // digits of a's memory order with b's strides; rows along the shared fastest dim
        DigitList dl;
        for (int r : da) dl.push_back({a.extent[r], b.stride[r]});
        DigitList col = collapse(dl);
        // a's memory index -> b offset is col; split off the row (first digit)
        int64_t row_len = 1, bstep = 1;
        if (!col.empty()) {
            row_len = col[0].first;
            bstep = col[0].second;
        }
        if (bstep != 1) {
            // same fastest dim must be unit-stride in b too
            set_error("inner: internal plan error");
            return TL_EUNSUPPORTED;
        }
        // row q of a (dense, memory order) starts at q*row_len; in b its
        // offset is the mixed-radix map of q over the remaining digits
        DigitList rb(col.begin() + (col.empty() ? 0 : 1), col.end());
        P.row_len = row_len;
        P.n_rows = N / row_len;
        if (P.n_rows > 0xffffffffll) {
            set_error("inner: too many rows");
            return TL_EUNSUPPORTED;
        }
        build_map(DigitList{{P.n_rows, row_len}}, P.rows_a);
        if (!build_map(rb, P.rows_b)) return TL_EUNSUPPORTED;
        // persistent grid: 4 CTAs per SM, each thread keeps 4 x 16 B in flight
        const int64_t work = (P.n_rows == 1) ? N / 16 : N / 4;
        static const int64_t ctas_per_sm = [] {
            const char *ev = getenv("TL_REDUCE_CTAS_PER_SM");
            return (int64_t)(ev ? atoi(ev) : 4);
        }();
        int64_t grid = std::min<int64_t>((int64_t)di.num_sms * ctas_per_sm, (work + threads - 1) / threads);
        grid = std::max<int64_t>(1, std::min<int64_t>(grid, kMaxPartials));
        const uintptr_t pa = (uintptr_t)P.a, pb = (uintptr_t)P.b;
        const bool same = (P.a == P.b) && (a.dtype == b.dtype) && P.n_rows == 1;
        const bool al = (pa % 16 == 0 && pb % 16 == 0);
        if (P.n_rows > 1 && al && a.dtype == b.dtype) {
            const int64_t V = 16 / (int64_t)sa;
            bool ok = row_len % V == 0 && N / V <= 0xffffffffll;
            for (auto &dg : rb) ok = ok && dg.second % V == 0;
            if (ok) {
                P.row_vec = 1;
                P.rowv_div.init((uint32_t)(row_len / V));
            }
        }
        const unsigned G = (unsigned)grid;
        if (a.dtype == TL_F32 && b.dtype == TL_F32) {
            if (same && al) dot_rows_kernel<float, float, 4, true, 8><<<G, threads, 0, st>>>(P);  // 8 x 16 B in flight: one stream
            else if (al && P.row_vec) dot_rows_kernel<float, float, 4, false, 4, false, true><<<G, threads, 0, st>>>(P);
            else if (al) dot_rows_kernel<float, float, 4, false><<<G, threads, 0, st>>>(P);
            else dot_rows_kernel<float, float, 1, false><<<G, threads, 0, st>>>(P);
        } else if (a.dtype == TL_F64 && b.dtype == TL_F64) {
            // sum of squares: plain FMA partials when each folds <= kFmaChain terms
            const bool fma_ok = (N + (int64_t)G * threads * 4 - 1) / ((int64_t)G * threads * 4) <= kFmaChain;
            if (same && al && fma_ok) dot_rows_kernel<double, double, 2, true, 8, true><<<G, threads, 0, st>>>(P);
            else if (same && al) dot_rows_kernel<double, double, 2, true, 8><<<G, threads, 0, st>>>(P);
            else if (al && P.row_vec) dot_rows_kernel<double, double, 2, false, 4, false, true><<<G, threads, 0, st>>>(P);
            else if (al) dot_rows_kernel<double, double, 2, false><<<G, threads, 0, st>>>(P);
            else dot_rows_kernel<double, double, 1, false><<<G, threads, 0, st>>>(P);
        } else if (a.dtype == TL_F32 && b.dtype == TL_F64) {
            dot_rows_kernel<float, double, 1, false><<<G, threads, 0, st>>>(P);
        } else if (a.dtype == TL_F64 && b.dtype == TL_F32) {
            dot_rows_kernel<double, float, 1, false><<<G, threads, 0, st>>>(P);
        } else {
            if (al && P.row_vec) dot_rows_kernel<int64_t, int64_t, 2, false, 4, false, true><<<G, threads, 0, st>>>(P);
            else if (al) dot_rows_kernel<int64_t, int64_t, 2, false><<<G, threads, 0, st>>>(P);
            else dot_rows_kernel<int64_t, int64_t, 1, false><<<G, threads, 0, st>>>(P);
        }
        e = cudaGetLastError();
    } else {
        const int X = da[0], Y = db[0];
        P.nX = a.extent[X];
        P.nY = a.extent[Y];
        P.a_sY = a.stride[Y];
        P.b_sX = b.stride[X];
        DigitList ra, rb;
        for (int r : da) {
            if (r == X || r == Y) continue;
            ra.push_back({a.extent[r], a.stride[r]});
            rb.push_back({a.extent[r], b.stride[r]});
        }
        // merge digits contiguous in both a and b
        DigitList ma, mb;
        for (size_t d = 0; d < ra.size(); ++d) {
            if (!ma.empty() && ma.back().first * ma.back().second == ra[d].second &&
                mb.back().first * mb.back().second == rb[d].second) {
                ma.back().first *= ra[d].first;
                mb.back().first *= rb[d].first;
            } else {
                ma.push_back(ra[d]);
                mb.push_back(rb[d]);
            }
        }
        P.n_rest = 1;
        for (auto &dg : ma) P.n_rest *= dg.first;
        if (!build_map(ma, P.rest_a) || !build_map(mb, P.rest_b) || P.n_rest > 0xffffffffll) return TL_EUNSUPPORTED;
        // 64x64 tiles with 16-byte vectors when every tile row is a whole,
        // aligned run of vectors in both operands
        if (a.dtype == b.dtype && (a.dtype == TL_F32 || a.dtype == TL_F64)) {
            const int64_t V = 16 / (int64_t)sa;
            bool vec = P.nX % kT == 0 && P.nY % kT == 0 && P.a_sY % V == 0 && P.b_sX % V == 0 &&
                       (uintptr_t)P.a % 16 == 0 && (uintptr_t)P.b % 16 == 0;
            for (auto &dg : ma) vec = vec && dg.second % V == 0;
            for (auto &dg : mb) vec = vec && dg.second % V == 0;
            if (vec) {
                P.tiles_x = P.nX / kT;
                P.tiles_y = P.nY / kT;
                const int64_t tiles = P.tiles_x * P.tiles_y * P.n_rest;
                const int64_t grid = std::min<int64_t>(std::min<int64_t>((int64_t)di.num_sms * 4, tiles), kMaxPartials);
                if (a.dtype == TL_F32)
                    dot_tiled_vec_kernel<float><<<(unsigned)grid, 256, 0, st>>>(P);
                else
                    dot_tiled_vec_kernel<double><<<(unsigned)grid, 256, 0, st>>>(P);
                return cuda_status(cudaGetLastError(), "inner (tiled) launch");
            }
        }
        P.tiles_x = (P.nX + 31) / 32;
        P.tiles_y = (P.nY + 31) / 32;
        const int64_t tiles = P.tiles_x * P.tiles_y * P.n_rest;
        int64_t grid = std::min<int64_t>(std::min<int64_t>((int64_t)di.num_sms * 8, tiles), kMaxPartials);
        if (a.dtype == TL_F32 && b.dtype == TL_F32) dot_tiled_kernel<float, float><<<(unsigned)grid, 256, 0, st>>>(P);
        else if (a.dtype == TL_F64 && b.dtype == TL_F64) dot_tiled_kernel<double, double><<<(unsigned)grid, 256, 0, st>>>(P);
        else if (a.dtype == TL_F32 && b.dtype == TL_F64) dot_tiled_kernel<float, double><<<(unsigned)grid, 256, 0, st>>>(P);
        else if (a.dtype == TL_F64 && b.dtype == TL_F32) dot_tiled_kernel<double, float><<<(unsigned)grid, 256, 0, st>>>(P);
        else dot_tiled_kernel<int64_t, int64_t><<<(unsigned)grid, 256, 0, st>>>(P);
        e = cudaGetLastError();
    }
    return cuda_status(e, "inner/norm launch");
}

}  // namespace tl
