// ttm_simt.cu -- ttm (contraction.py:200-298) for shapes that are not
// GEMM-shaped: few output rows J (HBM-bound, e.g. config 5's 16 x 33
// matrix), int64 and float32 operands.
//
// ttm_staged: a persistent CTA streams tiles of R consecutive [K][I] blocks
// of A (one contiguous byte range) into shared memory with a 1-D TMA bulk
// copy, keeps B in shared memory, and each thread folds one (row, i) for up
// to 16 j's at a time in registers (B reads are warp broadcasts).  The
// output tile, contiguous in first-order C when the layout allows, is
// staged in shared memory and written with coalesced stores.  Arithmetic:
// int64 exact; float32 widened to binary64 where every product is exact, so
// fma == the reference's mul-then-add and results are bit-identical;
// float64 uses fma (the DMMA semantics) within the stated 1e-12 tolerance.
//
// ttm_simt: one thread per output, the reference's fold (fallback).
#include <algorithm>
#include <cstdlib>
#include <string>
#include <type_traits>

#include "plan.h"
#include "tl_common.cuh"

namespace tl {

struct TtmSimtParams {
    const void *a;
    const void *bm;
    void *c;
    int64_t O, K, I, J;
    int64_t bs0, bs1;  // B strides (rows j, columns k)
    int64_t jstride;   // output stride of j
    int32_t ident;
    DigitMap in_map, out_map;
    // staged plan
    int32_t R;
    int64_t ntiles;
    FastDiv I_div;
    // index ranges past 2^32 (the one-thread-per-output kernel only)
    int32_t big;
    DigitMap64 in_map64, out_map64;
    // optional fused sum of squares of C (stream kernel): per-CTA partials,
    // last-CTA ticket, ssq_out = {sum C^2, sqrt(sum C^2)}
    double *ssq_out;
    double *ssq_partials;
    unsigned int *ssq_ticket;
};

template <class T, class TC>
__global__ void __launch_bounds__(256) ttm_simt_kernel(const __grid_constant__ TtmSimtParams P) {
    using Acc = typename AccOf<T>::type;
    const int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t per_o = P.J * P.I;
    if (gid >= P.O * per_o) return;
    const int64_t o = gid / per_o;
    const int64_t rem = gid - o * per_o;
    const int64_t j = rem / P.I;
    const int64_t i = rem - j * P.I;
    const T *pa = (const T *)P.a + o * P.K * P.I + i;
    const T *pb = (const T *)P.bm + j * P.bs0;
    Acc acc = Acc(0);
#pragma unroll 4
    for (int64_t k = 0; k < P.K; ++k) acc = fold_step(acc, (Acc)pa[k * P.I], (Acc)__ldg(pb + k * P.bs1));
    int64_t off;
    if (P.ident)
        off = (o * P.J + j) * P.I + i;
    else if (P.big)
        off = P.out_map64.map((uint64_t)o) + j * P.jstride + P.in_map64.map((uint64_t)i);
    else
        off = P.out_map.map((uint32_t)o) + j * P.jstride + P.in_map.map((uint32_t)i);
    ((TC *)P.c)[off] = narrow<TC>(acc);
}

// ------------------------------------------------------------ staged (small J)
constexpr int kTtmStages = 3;
// DMMA path: write fragments straight to first-order C (sector-complete per
// CTA) instead of staging the output tile in shared memory
constexpr bool kDirectStore = true;
constexpr int kJB = 16;

template <class T> __device__ __forceinline__ typename AccOf<T>::type mac(typename AccOf<T>::type acc, T a, typename AccOf<T>::type b);
template <> __device__ __forceinline__ double mac<double>(double acc, double a, double b) { return fma(a, b, acc); }
template <> __device__ __forceinline__ double mac<float>(double acc, float a, double b) { return fma((double)a, b, acc); }
template <> __device__ __forceinline__ int64_t mac<int64_t>(int64_t acc, int64_t a, int64_t b) { return fold_step(acc, a, b); }

// Shared-memory image of B.  SIMT: Bt[k][jpad] (j contiguous, jpad = J
// rounded up to 16, zero padded) so the 16 b(j, k) of one k are 8 vector
// broadcast loads.  DMMA: Bm[m][ldb] with ldb = 4 (mod 16) doubles
// (conflict-free A-fragment loads), zero padded in m and k.
__host__ __device__ __forceinline__ int64_t ttm_jpad(int64_t J) { return (J + 15) / 16 * 16; }
__host__ __device__ __forceinline__ int64_t ttm_ldb(int64_t K) {
    int64_t l = (K + 3) / 4 * 4;
    while (l % 16 != 4) l += 4;
    return l;
}

template <class T, bool DMMA> struct StagedLayout {
    size_t bbytes;
    __host__ __device__ StagedLayout(int64_t J, int64_t K) {
        const size_t n = DMMA ? (size_t)ttm_jpad(J) * ttm_ldb(K) : (size_t)K * ttm_jpad(J);
        bbytes = (n * sizeof(typename AccOf<T>::type) + 15) & ~(size_t)15;
    }
};

__device__ __forceinline__ void mma_16x8x4_s(double (&d)[4], double a0, double a1, double b) {
    asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
                 : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3])
                 : "d"(a0), "d"(a1), "d"(b));
}

// Output store for layouts whose first-order C is not the tile's contiguous
// range (kept out of line: it would otherwise be inlined per fragment value).
template <class T>
__device__ __noinline__ void store_permuted(const TtmSimtParams &P, int64_t o, uint32_t i, int64_t j, T v) {
    ((T *)P.c)[P.out_map.map((uint32_t)o) + j * P.jstride + P.in_map.map(i)] = v;
}

// MT = 0: SIMT fold; MT = 1, 2: FP64 DMMA with MT m16 tiles (J <= 16 MT)
template <class T, int MT, int NTILE = 4>
__global__ void __launch_bounds__(256) ttm_staged_kernel(const __grid_constant__ TtmSimtParams P) {
    constexpr bool DMMA = MT > 0;
    using Acc = typename AccOf<T>::type;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    __shared__ __align__(8) uint64_t full_bar[kTtmStages];
    const int64_t K = P.K, I = P.I, J = P.J;
    const int64_t KI = K * I;
    const int64_t jpad = ttm_jpad(J);
    // layout: B image | stages (R*K*I elements) | output tile (R*J*I)
    Acc *bsm = (Acc *)smem_raw;
    const size_t bbytes = StagedLayout<T, DMMA>(J, K).bbytes;
    unsigned char *stages = smem_raw + bbytes;
    const size_t stage_bytes = ((size_t)P.R * KI * sizeof(T) + 15) & ~(size_t)15;
    T *outs = (T *)(stages + kTtmStages * stage_bytes);

    if constexpr (DMMA) {
        const int64_t ldb = ttm_ldb(K);
        for (int64_t e = threadIdx.x; e < jpad * ldb; e += blockDim.x) {
            const int64_t j = e / ldb, k = e - j * ldb;
            bsm[e] = (j < J && k < K) ? (Acc)((const T *)P.bm)[j * P.bs0 + k * P.bs1] : Acc(0);
        }
    } else {
        for (int64_t e = threadIdx.x; e < K * jpad; e += blockDim.x) {
            const int64_t k = e / jpad, j = e - k * jpad;
            bsm[e] = (j < J) ? (Acc)((const T *)P.bm)[j * P.bs0 + k * P.bs1] : Acc(0);
        }
    }
    if (threadIdx.x == 0) {
        for (int s = 0; s < kTtmStages; ++s) mbar_init(&full_bar[s], 1);
        mbar_fence_init();
    }
    __syncthreads();

    const int64_t my_tiles = (P.ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x;
    auto issue = [&](int64_t q) {
        const int s = (int)(q % kTtmStages);
        const int64_t tile = (int64_t)blockIdx.x + q * gridDim.x;
        const int64_t o0 = tile * P.R;
        const int64_t rows = P.O - o0 < P.R ? P.O - o0 : P.R;
        const uint32_t bytes = (uint32_t)(rows * KI * (int64_t)sizeof(T));
        const uint32_t b16 = bytes & ~15u;
        unsigned char *dst = stages + s * stage_bytes;
        const unsigned char *src = (const unsigned char *)((const T *)P.a + o0 * KI);
        if (threadIdx.x == 0) {
            fence_proxy_async_smem();
            mbar_arrive_expect_tx(&full_bar[s], b16);
            if (b16) bulk_g2s(dst, src, b16, &full_bar[s]);
        }
        const uint32_t tail = (bytes - b16) / (uint32_t)sizeof(T);
        if (threadIdx.x < tail) cp_async<sizeof(T)>(dst + b16 + threadIdx.x * sizeof(T), src + b16 + threadIdx.x * sizeof(T));
    };
#pragma unroll
    for (int q = 0; q < kTtmStages - 1; ++q) {
        if (q < my_tiles) issue(q);
        cp_async_commit();
    }

    const uint32_t slots = (uint32_t)(P.R * I);
    for (int64_t q = 0; q < my_tiles; ++q) {
        cp_async_wait<kTtmStages - 2>();
        mbar_wait_parity(&full_bar[q % kTtmStages], (uint32_t)((q / kTtmStages) & 1));
        __syncthreads();
        if (q + kTtmStages - 1 < my_tiles) issue(q + kTtmStages - 1);
        cp_async_commit();
        const T *st = (const T *)(stages + (q % kTtmStages) * stage_bytes);
        const int64_t tile = (int64_t)blockIdx.x + q * gridDim.x;
        const int64_t o0 = tile * P.R;
        const int64_t rows = P.O - o0 < P.R ? P.O - o0 : P.R;
        auto put = [&](uint32_t r, uint32_t i, int64_t j, Acc v) {
            if (r >= rows || j >= J) return;
            if (P.ident)
                outs[((size_t)r * J + j) * I + i] = narrow<T>(v);
            else
                store_permuted<T>(P, o0 + r, i, j, narrow<T>(v));
        };
        if constexpr (DMMA) {
            // warp w takes groups of 32 positions (4 n8 tiles); all J rows
            // (jpad/16 m16 tiles); k in steps of 4 with zero padding
            const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
            const int g = lane >> 2, t = lane & 3;
            const int ldb = (int)ttm_ldb(K);
            constexpr int NT = NTILE;  // n8 tiles per warp: NT x MT independent MMA chains
            for (uint32_t p0 = warp * (8 * NT); p0 < slots; p0 += nw * (8 * NT)) {
                // this lane's B-fragment column positions (n = g) per tile
                int base[NT];
                bool okp[NT];
#pragma unroll
                for (int nt = 0; nt < NT; ++nt) {
                    uint32_t r, i;
                    const uint32_t pos = p0 + nt * 8 + g;
                    P.I_div.divmod(pos, r, i);
                    okp[nt] = pos < slots && r < rows;
                    base[nt] = okp[nt] ? (int)(r * KI + i) : 0;
                }
                double acc[MT][NT][4];
#pragma unroll
                for (int a = 0; a < MT; ++a)
#pragma unroll
                    for (int b = 0; b < NT; ++b)
#pragma unroll
                        for (int v = 0; v < 4; ++v) acc[a][b][v] = 0.0;
                const double *brow = (const double *)bsm + g * ldb + t;
                for (int k4 = 0; k4 < (int)K; k4 += 4) {
                    const int k = k4 + t;
                    const bool kok = k < (int)K;
                    double bf[NT];
#pragma unroll
                    for (int nt = 0; nt < NT; ++nt) bf[nt] = (okp[nt] && kok) ? (double)st[base[nt] + k * (int)I] : 0.0;
#pragma unroll
                    for (int mm = 0; mm < MT; ++mm) {
                        const double a0 = brow[(mm * 16) * ldb + k4], a1 = brow[(mm * 16 + 8) * ldb + k4];
#pragma unroll
                        for (int nt = 0; nt < NT; ++nt) mma_16x8x4_s(acc[mm][nt], a0, a1, bf[nt]);
                    }
                }
                // epilogue: each lane owns columns 2t, 2t+1 of every n8 tile
                const int Ji = (int)J, Ii = (int)I, rowsi = (int)rows;
#pragma unroll
                for (int nt = 0; nt < NT; ++nt) {
#pragma unroll
                    for (int v = 0; v < 2; ++v) {
                        const uint32_t pos = p0 + nt * 8 + 2 * t + v;
                        uint32_t r, i;
                        P.I_div.divmod(pos, r, i);
                        if (pos >= slots || (int)r >= rowsi) continue;
#pragma unroll
                        for (int mm = 0; mm < MT; ++mm) {
#pragma unroll
                            for (int h = 0; h < 2; ++h) {
                                const int j = mm * 16 + g + 8 * h;
                                if (j >= Ji) continue;
                                if (P.ident && kDirectStore)
                                    ((T *)P.c)[o0 * J * I + ((int)r * Ji + j) * Ii + (int)i] =
                                        narrow<T>((Acc)acc[mm][nt][2 * h + v]);
                                else if (P.ident)
                                    outs[((int)r * Ji + j) * Ii + (int)i] = narrow<T>((Acc)acc[mm][nt][2 * h + v]);
                                else
                                    put(r, i, j, (Acc)acc[mm][nt][2 * h + v]);
                            }
                        }
                    }
                }
            }
        } else {
            for (uint32_t slot = threadIdx.x; slot < slots; slot += blockDim.x) {
                uint32_t r, i;
                P.I_div.divmod(slot, r, i);
                if (r >= rows) continue;
                const T *arow = st + (size_t)r * KI + i;
                for (int64_t j0 = 0; j0 < J; j0 += kJB) {
                    Acc acc[kJB];
#pragma unroll
                    for (int jj = 0; jj < kJB; ++jj) acc[jj] = Acc(0);
                    for (int64_t k = 0; k < K; ++k) {
                        const T av = arow[k * I];
                        // 16 consecutive b(j, k) of this k: vector broadcast loads
                        const uint4 *bk = (const uint4 *)(bsm + k * jpad + j0);
                        Acc bv[kJB];
#pragma unroll
                        for (int q4 = 0; q4 < kJB * (int)sizeof(Acc) / 16; ++q4) ((uint4 *)bv)[q4] = bk[q4];
#pragma unroll
                        for (int jj = 0; jj < kJB; ++jj) acc[jj] = mac<T>(acc[jj], av, bv[jj]);
                    }
#pragma unroll
                    for (int jj = 0; jj < kJB; ++jj) put(r, i, j0 + jj, acc[jj]);
                }
            }
        }
        if (P.ident && !(DMMA && kDirectStore)) {
            __syncthreads();
            // the tile's outputs are one contiguous range of first-order C
            T *dst = (T *)P.c + o0 * J * I;
            const int n = (int)(rows * J * I);
            constexpr int VE = 16 / sizeof(T);
            if (((uintptr_t)dst & 15) == 0 && n % VE == 0) {
                const uint4 *src4 = (const uint4 *)outs;
                uint4 *dst4 = (uint4 *)dst;
                for (int e = threadIdx.x; e < n / VE; e += blockDim.x) dst4[e] = src4[e];
            } else {
                for (int e = threadIdx.x; e < n; e += blockDim.x) dst[e] = outs[e];
            }
        }
    }
    cp_async_wait<0>();
}

// float64, few rows J, output in A's order (ident): the staged DMMA tile
// with a TMA bulk epilogue.  A tile of R slabs A[o][K][I] arrives by bulk
// copy; its outputs C[o][J][I] are one contiguous range of first-order C,
// so the fragments are parked in a double-buffered shared tile and leave in
// ONE bulk store (instead of 8-byte scattered stores: 32 sectors per warp
// instruction, the LSU limit of the staged kernel).  Every warp owns a fixed
// set of 8*NT tile positions, so fragment bases and output offsets are
// computed once per kernel, not per tile.
template <int MT, int NT, int NST>
__global__ void __launch_bounds__(256) ttm_bulk_kernel(const __grid_constant__ TtmSimtParams P) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    __shared__ __align__(8) uint64_t full_bar[NST];
    const int64_t K = P.K, I = P.I, J = P.J;
    const int64_t KI = K * I;
    const int64_t jpad = ttm_jpad(J);
    const int ldb = (int)ttm_ldb(K);
    double *bsm = (double *)smem_raw;
    const size_t bbytes = StagedLayout<double, true>(J, K).bbytes;
    unsigned char *stages = smem_raw + bbytes;
    const size_t stage_bytes = ((size_t)P.R * KI * 8 + 15) & ~(size_t)15;
    const size_t otile = ((size_t)P.R * J * I * 8 + 15) & ~(size_t)15;
    double *outs = (double *)(stages + NST * stage_bytes);

    for (int64_t e = threadIdx.x; e < jpad * ldb; e += blockDim.x) {
        const int64_t j = e / ldb, k = e - j * ldb;
        bsm[e] = (j < J && k < K) ? ((const double *)P.bm)[j * P.bs0 + k * P.bs1] : 0.0;
    }
    if (threadIdx.x == 0) {
        for (int s = 0; s < NST; ++s) mbar_init(&full_bar[s], 1);
        mbar_fence_init();
    }
    __syncthreads();

    const int64_t my_tiles = (P.ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x;
    auto issue = [&](int64_t q) {
        const int s = (int)(q % NST);
        const int64_t o0 = ((int64_t)blockIdx.x + q * gridDim.x) * P.R;
        const int64_t rows = P.O - o0 < P.R ? P.O - o0 : P.R;
        const uint32_t bytes = (uint32_t)(rows * KI * 8);
        const uint32_t b16 = bytes & ~15u;
        unsigned char *dst = stages + s * stage_bytes;
        const unsigned char *src = (const unsigned char *)((const double *)P.a + o0 * KI);
        if (threadIdx.x == 0) {
            fence_proxy_async_smem();
            mbar_arrive_expect_tx(&full_bar[s], b16);
            if (b16) bulk_g2s(dst, src, b16, &full_bar[s]);
        }
        if (bytes != b16 && threadIdx.x == 0) cp_async<8>(dst + b16, src + b16);
    };
#pragma unroll
    for (int q = 0; q < NST - 1; ++q) {
        if (q < my_tiles) issue(q);
        cp_async_commit();
    }

    // fixed per-lane geometry
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int g = lane >> 2, t = lane & 3;
    const uint32_t slots = (uint32_t)(P.R * I);
    const uint32_t p0 = (uint32_t)warp * (8 * NT);
    int base[NT];     // B-fragment column (position p0 + 8 nt + g) in the stage
    bool okp[NT];
    int orow[NT][2];  // output row r of positions p0 + 8 nt + 2t + v (-1: none)
    int ooff[NT][2];  // its offset r*J*I + i in the output tile
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
        uint32_t r, i;
        const uint32_t pos = p0 + nt * 8 + g;
        P.I_div.divmod(pos, r, i);
        okp[nt] = pos < slots;
        base[nt] = okp[nt] ? (int)(r * KI + i) : 0;
#pragma unroll
        for (int v = 0; v < 2; ++v) {
            const uint32_t pv = p0 + nt * 8 + 2 * t + v;
            P.I_div.divmod(pv, r, i);
            orow[nt][v] = pv < slots ? (int)r : -1;
            ooff[nt][v] = (int)(r * J * I + i);
        }
    }
    const double *brow = bsm + g * ldb + t;
    const int Ki = (int)K, Ii = (int)I, Ji = (int)J;

    for (int64_t q = 0; q < my_tiles; ++q) {
        if (threadIdx.x == 0) bulk_wait_read<1>();  // outs[q & 1] is free (tile q-2 read out)
        cp_async_wait<NST - 2>();
        mbar_wait_parity(&full_bar[q % NST], (uint32_t)((q / NST) & 1));
        __syncthreads();
        if (q + NST - 1 < my_tiles) issue(q + NST - 1);
        cp_async_commit();
        const double *st = (const double *)(stages + (q % NST) * stage_bytes);
        const int64_t o0 = ((int64_t)blockIdx.x + q * gridDim.x) * P.R;
        const int rows = (int)(P.O - o0 < P.R ? P.O - o0 : P.R);

        double acc[MT][NT][4];
#pragma unroll
        for (int a = 0; a < MT; ++a)
#pragma unroll
            for (int b = 0; b < NT; ++b)
#pragma unroll
                for (int v = 0; v < 4; ++v) acc[a][b][v] = 0.0;
        if (p0 < slots) {
            for (int k4 = 0; k4 < Ki; k4 += 4) {
                const int k = k4 + t;
                const bool kok = k < Ki;
                double bf[NT];
#pragma unroll
                for (int nt = 0; nt < NT; ++nt) bf[nt] = (okp[nt] && kok) ? st[base[nt] + k * Ii] : 0.0;
#pragma unroll
                for (int mm = 0; mm < MT; ++mm) {
                    const double a0 = brow[(mm * 16) * ldb + k4], a1 = brow[(mm * 16 + 8) * ldb + k4];
#pragma unroll
                    for (int nt = 0; nt < NT; ++nt) mma_16x8x4_s(acc[mm][nt], a0, a1, bf[nt]);
                }
            }
            double *ot = outs + (q & 1) * (otile / 8);
#pragma unroll
            for (int nt = 0; nt < NT; ++nt)
#pragma unroll
                for (int v = 0; v < 2; ++v) {
                    if (orow[nt][v] < 0 || orow[nt][v] >= rows) continue;
#pragma unroll
                    for (int mm = 0; mm < MT; ++mm)
#pragma unroll
                        for (int h = 0; h < 2; ++h) {
                            const int j = mm * 16 + g + 8 * h;
                            if (j < Ji) ot[ooff[nt][v] + j * Ii] = acc[mm][nt][2 * h + v];
                        }
                }
        }
        fence_proxy_async_smem();
        __syncthreads();
        if (threadIdx.x == 0) {
            const uint32_t bytes = (uint32_t)(rows * J * I * 8);
            const uint32_t b16 = bytes & ~15u;
            const double *ot = outs + (q & 1) * (otile / 8);
            double *dst = (double *)P.c + o0 * J * I;
            if (b16) bulk_s2g(dst, ot, b16);
            bulk_commit();
            if (bytes != b16) dst[b16 / 8] = ot[b16 / 8];
        }
    }
    cp_async_wait<0>();
    if (threadIdx.x == 0) bulk_wait<0>();
}

// float64, few rows J, output in A's order (ident): warp-specialised stream.
// One persistent CTA per SM.  A producer thread keeps every consumer warp's
// private ring of SW tile slots filled with 1-D TMA bulk copies (full / empty
// mbarrier per slot); consumer warp w owns the CTA's local tiles w, w + NW,
// w + 2 NW, ... (its j-th tile sits in slot w*SW + j mod SW): DMMA over the
// tile's R*I positions (NT n8 tiles), fragments parked in the warp's own
// double-buffered output tile, one bulk store per tile.  No CTA-wide barrier
// in the steady state, and up to NW*SW tiles of A in flight per SM -- the
// 2-stage bulk kernel keeps one tile in flight per CTA, too few bytes for an
// HBM-bound stream of short tiles (config 5: 6 KB per tile).
// Private rings keep every barrier wait unambiguous: a slot's successive
// phases are waited on by one warp (and by the producer) strictly in order,
// so nobody waits for phase n+1 while phase n is still open -- a parity wait
// for n+1 would return at once then (it reads as the completed phase n-1).
// A shared round-robin ring allowed exactly that and hung at J = 32.
// Same per-element arithmetic as the other DMMA kernels (k-ordered FMA).
constexpr int kStreamMaxSlots = 48;
constexpr size_t kStreamSmemBudget = 220 * 1024;  // one CTA per SM (227 KB max)
// per-CTA budget with c CTAs per SM (1 KB reserved per CTA, static smem)
static size_t stream_budget(int c) { return c <= 1 ? kStreamSmemBudget : (228 * 1024) / (size_t)c - 4 * 1024; }
constexpr int kStreamMaxWarps = 8;

// Fused sum of squares of C for frobenius_norm(ttm(...)) (the config-5
// chain ttv -> ttm -> norm): lane sums (FMA, <= kSsqChain terms each) ->
// fixed-order warp tree -> warps 0..NW-1 in order (added by the CTA's last
// consumer warp to finish) -> CTA partials 0..grid-1 in a fixed order (the
// last CTA).  Every level has a fixed order, so the result is deterministic;
// relative error <= (chain + 5 + log2 NW + grid) * 2^-53 < 1e-12.
constexpr int64_t kSsqChain = 4096;
constexpr int kSsqLoadsPerLane = 8;  // grids of up to 256 CTAs combine in one round trip

struct SsqShared {
    double wpart[kStreamMaxWarps];
    unsigned int wdone;
    int cta_last;
};

__device__ __noinline__ void stream_ssq_combine(const TtmSimtParams &P, double ssq, int warp, int NW, SsqShared &sh) {
    double *wpart = sh.wpart;
    unsigned int &wdone = sh.wdone;
    int &cta_last = sh.cta_last;
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) ssq += __shfl_down_sync(0xffffffffu, ssq, d);
    int last_warp = 0;
    if (lane == 0) {
        wpart[warp] = ssq;
        __threadfence_block();
        last_warp = atomicAdd(&wdone, 1u) == (unsigned)NW - 1;
    }
    last_warp = __shfl_sync(0xffffffffu, last_warp, 0);
    if (!last_warp) return;
    __threadfence_block();
    if (lane == 0) {
        double cta = 0.0;
        for (int w = 0; w < NW; ++w) cta += *(volatile double *)&wpart[w];
        P.ssq_partials[blockIdx.x] = cta;
        unsigned prev;
        asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(prev) : "l"(P.ssq_ticket) : "memory");
        cta_last = prev == gridDim.x - 1;
    }
    __syncwarp();
    if (!*(volatile int *)&cta_last) return;
    // the last CTA: partials lane-strided in index order, then a fixed tree.
    // All of a lane's loads are issued before the first add (one L2 round
    // trip instead of one per 32 partials: the combine is the kernel's tail)
    double v = 0.0;
    const int G = (int)gridDim.x;
    if (G <= 32 * kSsqLoadsPerLane) {
        double x[kSsqLoadsPerLane];
#pragma unroll
        for (int q = 0; q < kSsqLoadsPerLane; ++q) x[q] = lane + 32 * q < G ? __ldcg(P.ssq_partials + lane + 32 * q) : 0.0;
#pragma unroll
        for (int q = 0; q < kSsqLoadsPerLane; ++q) v += x[q];  // + 0.0 past the grid: exact (v >= 0)
    } else {
        for (int i = lane; i < G; i += 32) v += __ldcg(P.ssq_partials + i);
    }
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) v += __shfl_down_sync(0xffffffffu, v, d);
    if (lane == 0) {
        P.ssq_out[0] = v;
        P.ssq_out[1] = sqrt(v);
        *P.ssq_ticket = 0u;  // leave the workspace zeroed
    }
}

template <int MT, int NT, bool SSQ = false>
__global__ void __launch_bounds__(32 * (kStreamMaxWarps + 1)) ttm_stream_kernel(const __grid_constant__ TtmSimtParams P,
                                                                              int SW) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    __shared__ __align__(8) uint64_t full_bar[kStreamMaxSlots], empty_bar[kStreamMaxSlots];
    const int64_t K = P.K, I = P.I, J = P.J;
    const int64_t KI = K * I;
    const int64_t jpad = ttm_jpad(J);
    const int ldb = (int)ttm_ldb(K);
    const int NW = (int)(blockDim.x >> 5) - 1;
    const int S = NW * SW;
    double *bsm = (double *)smem_raw;
    unsigned char *slots = smem_raw + StagedLayout<double, true>(J, K).bbytes;
    const size_t slot_bytes = ((size_t)P.R * KI * 8 + 15) & ~(size_t)15;
    const size_t otile = ((size_t)P.R * J * I * 8 + 15) & ~(size_t)15;
    unsigned char *outs = slots + (size_t)S * slot_bytes;

    __shared__ SsqShared ssq_sh;
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(&full_bar[s], 1);
            mbar_init(&empty_bar[s], 1);
        }
        mbar_fence_init();
        ssq_sh.wdone = 0u;
    }
    __syncthreads();
    // the producer starts streaming A at once; the consumer warps stage B
    // meanwhile (its global loads' latency overlaps the first tiles') and
    // meet at a named barrier of their own
    if ((int)(threadIdx.x >> 5) < NW) {
        for (int64_t e = threadIdx.x; e < jpad * ldb; e += NW * 32) {
            const int64_t j = e / ldb, k = e - j * ldb;
            bsm[e] = (j < J && k < K) ? ((const double *)P.bm)[j * P.bs0 + k * P.bs1] : 0.0;
        }
        asm volatile("bar.sync 1, %0;" ::"r"(NW * 32) : "memory");
    }

    const int64_t my_tiles = (P.ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp == NW) {
        // producer: local tile q = w + NW*j goes to slot w*SW + j mod SW once
        // that slot's previous tile (j - SW of warp w) has been released
        if (lane == 0) {
            int w = 0, js = 0;
            uint32_t jpar = 0;  // parity of fill j / SW
            bool wrapped = false;  // j >= SW: the slot has a previous tile
            // tile q starts at row o0 = (blockIdx.x + q * grid) * R: stepped, not recomputed
            const int64_t tile_bytes = (int64_t)P.R * KI * 8;
            const int64_t step_bytes = (int64_t)gridDim.x * tile_bytes;
            const unsigned char *src = (const unsigned char *)P.a + (int64_t)blockIdx.x * tile_bytes;
            int64_t o0 = (int64_t)blockIdx.x * P.R;
            const int64_t o_step = (int64_t)gridDim.x * P.R;
            for (int64_t q = 0; q < my_tiles; ++q, src += step_bytes, o0 += o_step) {
                const int s = w * SW + js;
                if (wrapped) mbar_wait_parity(&empty_bar[s], jpar ^ 1u);
                const uint32_t bytes = (P.O - o0 < P.R) ? (uint32_t)((P.O - o0) * KI * 8) : (uint32_t)tile_bytes;
                const uint32_t b16 = bytes & ~15u;
                unsigned char *dst = slots + s * slot_bytes;
                // an 8-byte tail (last tile, odd R*K*I) is copied here; the
                // arrive below releases it to the consumer
                if (bytes != b16) {
                    *(double *)(dst + b16) = *(const double *)(src + b16);
                    fence_proxy_async_smem();
                }
                mbar_arrive_expect_tx(&full_bar[s], b16);
                if (b16) bulk_g2s(dst, src, b16, &full_bar[s]);
                if (++w == NW) {
                    w = 0;
                    if (++js == SW) {
                        js = 0;
                        jpar ^= 1u;
                        wrapped = true;
                    }
                }
            }
        }
        return;
    }

    // consumer warp: fixed per-lane fragment geometry over the tile's positions
    const int g = lane >> 2, t = lane & 3;
    int base[NT], posb[NT];
    int orow[NT][2], ooff[NT][2];
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
        uint32_t r, i;
        posb[nt] = nt * 8 + g;
        P.I_div.divmod((uint32_t)posb[nt], r, i);
        // a position past the tile reads row 0 instead: its column of the
        // product is never stored (DMMA columns are independent)
        base[nt] = r < (uint32_t)P.R ? (int)(r * KI + i) : 0;
#pragma unroll
        for (int v = 0; v < 2; ++v) {
            P.I_div.divmod((uint32_t)(nt * 8 + 2 * t + v), r, i);
            orow[nt][v] = (int)r;  // >= rows for positions past the tile: skipped
            ooff[nt][v] = (int)(r * J * I + i);
        }
    }
    const double *brow = bsm + g * ldb + t;
    const int Ki = (int)K, Ii = (int)I, Ji = (int)J;
    const int Kfull = Ki & ~3;  // k-steps with all four k in range
    const bool jfull = Ji == 16 * MT;
    int parity_out = 0;
    double ssq4[4] = {0.0, 0.0, 0.0, 0.0};  // this lane's sums of squares of the outputs it stored (fused norm)
    int js = 0;         // j mod SW for this warp's j-th tile
    uint32_t jpar = 0;  // parity of fill j / SW
    for (int64_t q = warp; q < my_tiles; q += NW) {
        const int s = warp * SW + js;
        mbar_wait_parity(&full_bar[s], jpar);
        const double *st = (const double *)(slots + s * slot_bytes);
        const int64_t o0 = ((int64_t)blockIdx.x + q * gridDim.x) * P.R;
        const int rows = (int)(P.O - o0 < P.R ? P.O - o0 : P.R);

        double acc[MT][NT][4];
#pragma unroll
        for (int a = 0; a < MT; ++a)
#pragma unroll
            for (int b = 0; b < NT; ++b)
#pragma unroll
                for (int v = 0; v < 4; ++v) acc[a][b][v] = 0.0;
        // Positions past `rows` (partial last tile) fold stale slot data into
        // columns that are never stored; only k >= K must read as zero
        // (0 * stale could be NaN in a stored column).
        auto kstep = [&](int k4, bool kok) {
            const int k = k4 + t;
            double bf[NT];
#pragma unroll
            for (int nt = 0; nt < NT; ++nt) bf[nt] = kok ? st[base[nt] + k * Ii] : 0.0;
#pragma unroll
            for (int mm = 0; mm < MT; ++mm) {
                const double a0 = brow[(mm * 16) * ldb + k4], a1 = brow[(mm * 16 + 8) * ldb + k4];
#pragma unroll
                for (int nt = 0; nt < NT; ++nt) mma_16x8x4_s(acc[mm][nt], a0, a1, bf[nt]);
            }
        };
        // two m16 tiles x 4 n8 tiles keep 64 accumulator registers live:
        // unrolling 4 k-steps there spilled (148 bytes; 124 with the fused
        // norm's registers), 2 (1 with the fused norm) does not
        constexpr int KU = (MT * NT > 6) ? (SSQ ? 1 : 2) : 4;
#pragma unroll KU
        for (int k4 = 0; k4 < Kfull; k4 += 4) kstep(k4, true);
        if (Kfull < Ki) kstep(Kfull, Kfull + t < Ki);
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty_bar[s]);  // the slot is free for this warp's tile j + SW
        if (++js == SW) {
            js = 0;
            jpar ^= 1u;
        }

        double *ot = (double *)(outs + ((size_t)warp * 2 + parity_out) * otile);
        parity_out ^= 1;
        if (lane == 0) bulk_wait_read<1>();  // this buffer's previous store has been read out
        __syncwarp();
        if (rows == P.R && jfull) {
            // whole tile, J fills the m16 tiles: only positions past R*I are skipped
#pragma unroll
            for (int nt = 0; nt < NT; ++nt)
#pragma unroll
                for (int v = 0; v < 2; ++v)
#pragma unroll
                    for (int mm = 0; mm < MT; ++mm)
#pragma unroll
                        for (int h = 0; h < 2; ++h)
                            if (orow[nt][v] < P.R) {
                                const double x = acc[mm][nt][2 * h + v];
                                ot[ooff[nt][v] + (mm * 16 + g + 8 * h) * Ii] = x;
                                if (SSQ) ssq4[(2 * h + v) & 3] = fma(x, x, ssq4[(2 * h + v) & 3]);
                            }
        } else {
#pragma unroll
            for (int nt = 0; nt < NT; ++nt)
#pragma unroll
                for (int v = 0; v < 2; ++v) {
                    if (orow[nt][v] >= rows) continue;
#pragma unroll
                    for (int mm = 0; mm < MT; ++mm)
#pragma unroll
                        for (int h = 0; h < 2; ++h) {
                            const int j = mm * 16 + g + 8 * h;
                            if (j < Ji) {
                                const double x = acc[mm][nt][2 * h + v];
                                ot[ooff[nt][v] + j * Ii] = x;
                                if (SSQ) ssq4[(2 * h + v) & 3] = fma(x, x, ssq4[(2 * h + v) & 3]);
                            }
                        }
                }
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
            const uint32_t bytes = (uint32_t)(rows * J * I * 8);
            const uint32_t b16 = bytes & ~15u;
            double *dst = (double *)P.c + o0 * J * I;
            if (b16) bulk_s2g(dst, ot, b16);
            bulk_commit();
            if (bytes != b16) dst[b16 / 8] = ot[b16 / 8];
        }
    }
    if (lane == 0) bulk_wait<0>();
    if constexpr (SSQ) stream_ssq_combine(P, (ssq4[0] + ssq4[1]) + (ssq4[2] + ssq4[3]), warp, NW, ssq_sh);
}

static bool build_params(const tl_desc &a, const void *a_ptr, const tl_desc &bm, const void *b_ptr, void *c_ptr,
                         int m0, TtmSimtParams &P) {
    const int64_t J = bm.extent[0];
    Canon cn;
    if (!canon_contraction(a, m0, J, cn)) {
        set_error("ttm: operand A is not a dense permutation layout (materialise views first)");
        return false;
    }
    const size_t s = dtype_size(a.dtype);
    P.a = (const unsigned char *)a_ptr + a.offset * (int64_t)s;
    P.bm = (const unsigned char *)b_ptr + bm.offset * (int64_t)dtype_size(bm.dtype);
    P.c = c_ptr;
    P.O = cn.O;
    P.K = cn.K;
    P.I = cn.I;
    P.J = J;
    P.bs0 = bm.stride[0];
    P.bs1 = bm.stride[1];
    P.jstride = cn.jstride;
    P.ident = cn.ident ? 1 : 0;
    P.big = (cn.O > kIdx32 || cn.I > kIdx32) ? 1 : 0;
    if (P.big || !build_map(cn.inner, P.in_map) || !build_map(cn.outer, P.out_map)) {
        // past 2^32: only the one-thread-per-output kernel (64-bit maps) runs
        P.big = 1;
        build_map64(cn.inner, P.in_map64);
        build_map64(cn.outer, P.out_map64);
    }
    return true;
}

// Tuning knobs of the small-J kernels (environment, read once).
struct SmallTtmKnobs {
    int64_t stage_kb = 28, bulk_kb = 14, stream_kb = 12;
    int ntile = 4, bulk_nt = 2, bulk_st = 2, stream_nw = kStreamMaxWarps, stream_cps = 1;
    bool force_simt = false;
};
static const SmallTtmKnobs &small_ttm_knobs() {
    static const SmallTtmKnobs k = [] {
        SmallTtmKnobs v;
        auto num = [](const char *name, int64_t dflt) {
            const char *e = getenv(name);
            return e ? (int64_t)atoll(e) : dflt;
        };
        v.stage_kb = num("TL_TTM_STAGE_KB", 28);
        v.ntile = (int)num("TL_TTM_NT", 4);
        v.force_simt = getenv("TL_TTM_SIMT") != nullptr;
        v.bulk_kb = num("TL_TTM_BULK_KB", 14);
        v.bulk_nt = (int)num("TL_TTM_BULK_NT", 2);
        v.bulk_st = (int)num("TL_TTM_BULK_ST", 2);  // measured: 2 stages (more CTAs per SM) beat 3-4
        v.stream_kb = num("TL_TTM_STREAM_KB", 12);  // tile target; 0 disables the stream kernel
        v.stream_cps = (int)std::max<int64_t>(1, std::min<int64_t>(4, num("TL_TTM_STREAM_CPS", 1)));  // CTAs per SM
        v.stream_nw = (int)std::max<int64_t>(1, std::min<int64_t>(kStreamMaxWarps, num("TL_TTM_STREAM_NW", kStreamMaxWarps)));
        return v;
    }();
    return k;
}

struct StreamPlan {
    int64_t R = 0;
    int nt = 0, nw = 0, sw = 0;
    size_t smem = 0;
};
// Stream-kernel plan (host only).  R: tile positions R*I fill whole n8 tiles
// as far as possible (at most 5 per warp for J <= 16, 4 for J <= 32:
// measured best); tile <= the target; tile starts 16-byte aligned in A and C.
// Prefer tiles small enough for every consumer warp to keep two slots and
// two output tiles (measured: 5 warps with bigger tiles lose 20% at J = 32),
// then the fullest n8 tiles, then larger R.
static bool plan_stream(const TtmSimtParams &P, StreamPlan &sp) {
    const SmallTtmKnobs &kn = small_ttm_knobs();
    if (kn.stream_kb <= 0) return false;
    const int64_t KI = P.K * P.I;
    const int ntmax = P.J <= 16 ? 5 : 4;
    const size_t bb = StagedLayout<double, true>(P.J, P.K).bbytes;
    int64_t bestR = 0;
    double best_eff = 0.0;
    bool best_fit = false;
    for (int64_t R = 1; R * P.I <= 8 * ntmax && R * KI * 8 <= kn.stream_kb * 1024; ++R) {
        if ((R * KI) % 2 != 0 || (R * P.J * P.I) % 2 != 0) continue;
        const int64_t pos = R * P.I;
        const double eff = (double)pos / (double)(8 * ((pos + 7) / 8));
        const size_t per_warp = 2 * (((size_t)R * P.J * P.I * 8 + 15) & ~(size_t)15) + 2 * (((size_t)R * KI * 8 + 15) & ~(size_t)15);
        const bool fit = bb + (size_t)kn.stream_nw * per_warp <= stream_budget(kn.stream_cps);
        const bool better = (fit != best_fit) ? fit : (eff > best_eff + 1e-9 || (eff > best_eff - 1e-9 && R > bestR));
        if (bestR == 0 || better) {
            best_fit = fit;
            best_eff = eff;
            bestR = R;
        }
    }
    if (bestR == 0 || best_eff < 0.75) return false;
    const size_t slot_bytes = ((size_t)bestR * KI * 8 + 15) & ~(size_t)15;
    const size_t otile = ((size_t)bestR * P.J * P.I * 8 + 15) & ~(size_t)15;
    // NW consumer warps, each with SW >= 2 private slots and two output
    // tiles; fewer warps when the smem budget demands it
    int nw = kn.stream_nw, sw = 0;
    for (; nw >= 2; --nw) {
        const size_t budget = stream_budget(kn.stream_cps);
        if (bb + (size_t)nw * (2 * otile + 2 * slot_bytes) > budget) continue;
        sw = (int)std::min<size_t>(kStreamMaxSlots / nw, (budget - bb - (size_t)nw * 2 * otile) / ((size_t)nw * slot_bytes));
        break;
    }
    if (sw < 2) return false;
    sp.R = bestR;
    sp.nt = (int)((bestR * P.I + 7) / 8);
    sp.nw = nw;
    sp.sw = sw;
    sp.smem = bb + (size_t)nw * 2 * otile + (size_t)nw * sw * slot_bytes;
    return true;
}

struct BulkPlan {
    int64_t R = 0;
    int nt = 0, nst = 0, threads = 0;
    size_t smem = 0;
};
// Bulk-epilogue kernel plan (host only): tiles of R slabs, outputs leave by
// TMA; R*I preferably a multiple of the 8*nt positions one warp owns.
static bool plan_bulk(const TtmSimtParams &P, BulkPlan &bp) {
    const SmallTtmKnobs &kn = small_ttm_knobs();
    if (kn.bulk_kb <= 0) return false;
    const int64_t KI = P.K * P.I;
    const int nt = (kn.bulk_nt == 1 || kn.bulk_nt == 4) ? kn.bulk_nt : 2;
    const int64_t rmax = std::max<int64_t>(1, std::min<int64_t>((64 * nt) / P.I, kn.bulk_kb * 1024 / (KI * 8)));
    int64_t unit = 8 * nt;
    for (int64_t d = P.I; d > 0;) {  // unit = 8 nt / gcd(I, 8 nt)
        const int64_t r = unit % d;
        unit = d;
        d = r;
    }
    unit = 8 * nt / unit;
    int64_t R = rmax / unit * unit;
    if (R == 0 && unit * P.I <= 64 * nt && unit * KI * 8 <= 32 * 1024) R = unit;
    if (R == 0) R = rmax;
    while (R > 1 && ((R * KI * 8) % 16 != 0 || (R * P.J * P.I) % 2 != 0)) --R;
    if ((R * KI * 8) % 16 != 0 || (R * P.J * P.I) % 2 != 0) return false;
    const int threads = (int)(((R * P.I + 8 * nt - 1) / (8 * nt)) * 32);
    const size_t stage_bytes = ((size_t)R * KI * 8 + 15) & ~(size_t)15;
    const size_t otile = ((size_t)R * P.J * P.I * 8 + 15) & ~(size_t)15;
    const int nst = kn.bulk_st <= 2 ? 2 : (kn.bulk_st == 3 ? 3 : 4);
    const size_t smem = StagedLayout<double, true>(P.J, P.K).bbytes + nst * stage_bytes + 2 * otile;
    // one warp per 8*nt positions, at most the kernel's 256 threads
    if (smem > 200 * 1024 || threads > 256) return false;
    bp.R = R;
    bp.nt = nt;
    bp.nst = nst;
    bp.threads = threads;
    bp.smem = smem;
    return true;
}

// Shared gate of the small-J staged family (I <= 256, a [K][I] block <= 32 KB,
// B image <= 48 KB, 16-byte aligned A); false -> the caller uses another path.
static bool staged_family_ok(const TtmSimtParams &P, int32_t dtype) {
    const int64_t s = (int64_t)dtype_size(dtype);
    return !(P.big || P.I > 256 || P.K * P.I * s > 32 * 1024 || P.J * P.K * 8 > 48 * 1024 || (uintptr_t)P.a % 16 != 0 ||
             P.O > 0xffffffffll);
}

constexpr int kMaxSsqPartials = 148 * 8;  // the reduce workspace's partial slots

int ttm_staged_enqueue(const tl_desc &a, const void *a_ptr, const tl_desc &bm, const void *b_ptr, void *c_ptr,
                       int m0, cudaStream_t st, double *ssq_out, void *ssq_ws, int32_t *ssq_fused) {
    if (ssq_fused != nullptr) *ssq_fused = 0;
    TtmSimtParams P{};
    if (!build_params(a, a_ptr, bm, b_ptr, c_ptr, m0, P)) return TL_EUNSUPPORTED;
    if (ssq_out != nullptr && ssq_ws != nullptr) {
        P.ssq_out = ssq_out;
        P.ssq_partials = (double *)ssq_ws;
        P.ssq_ticket = (unsigned int *)((unsigned char *)ssq_ws + (size_t)kMaxSsqPartials * 2 * sizeof(double));
    }
    const int64_t s = (int64_t)dtype_size(a.dtype);
    const int64_t KI = P.K * P.I;
    if (P.O * P.I == 0) return TL_OK;
    if (!staged_family_ok(P, a.dtype)) return TL_EUNSUPPORTED;
    const SmallTtmKnobs &kn = small_ttm_knobs();
    const int64_t stage_kb = kn.stage_kb;
    const int ntile = kn.ntile;
    const bool force_simt = kn.force_simt;
    const bool dmma_ident = a.dtype == TL_F64 && P.J <= 32 && P.ident && !force_simt && (uintptr_t)c_ptr % 16 == 0;
    StreamPlan sp;
    if (dmma_ident && plan_stream(P, sp)) {
        P.R = (int32_t)sp.R;
        P.ntiles = (P.O + sp.R - 1) / sp.R;
        P.I_div.init((uint32_t)P.I);
        const DeviceInfo &di = device_info();
        const int64_t grid = std::min<int64_t>(P.ntiles, (int64_t)di.num_sms * kn.stream_cps);
        const int threads = 32 * (sp.nw + 1);
        const size_t smem = sp.smem;
        const int sw = sp.sw;
        auto go = [&](auto kern) -> int {
            cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            if (e != cudaSuccess) return cuda_status(e, "ttm stream smem");
            kern<<<(unsigned)grid, threads, smem, st>>>(P, sw);
            return cuda_status(cudaGetLastError(), "ttm stream launch");
        };
        // fused sum of squares (frobenius_norm of this output): when every
        // lane's FMA chain stays <= kSsqChain terms
        const int64_t lanes = grid * sp.nw * 32;
        const bool ssq = P.ssq_out != nullptr && (P.O * P.J * P.I + lanes - 1) / lanes <= kSsqChain &&
                         grid <= kMaxSsqPartials;
        if (!ssq) P.ssq_out = nullptr;
        if (ssq_fused != nullptr) *ssq_fused = ssq ? 1 : 0;
        if (ssq && P.J <= 16) {
            switch (sp.nt) {
                case 1: return go(ttm_stream_kernel<1, 1, true>);
                case 2: return go(ttm_stream_kernel<1, 2, true>);
                case 3: return go(ttm_stream_kernel<1, 3, true>);
                case 4: return go(ttm_stream_kernel<1, 4, true>);
                default: return go(ttm_stream_kernel<1, 5, true>);
            }
        }
        if (ssq) {
            switch (sp.nt) {
                case 1: return go(ttm_stream_kernel<2, 1, true>);
                case 2: return go(ttm_stream_kernel<2, 2, true>);
                case 3: return go(ttm_stream_kernel<2, 3, true>);
                default: return go(ttm_stream_kernel<2, 4, true>);
            }
        }
        if (P.J <= 16) {
            switch (sp.nt) {
                case 1: return go(ttm_stream_kernel<1, 1>);
                case 2: return go(ttm_stream_kernel<1, 2>);
                case 3: return go(ttm_stream_kernel<1, 3>);
                case 4: return go(ttm_stream_kernel<1, 4>);
                default: return go(ttm_stream_kernel<1, 5>);
            }
        }
        switch (sp.nt) {
            case 1: return go(ttm_stream_kernel<2, 1>);
            case 2: return go(ttm_stream_kernel<2, 2>);
            case 3: return go(ttm_stream_kernel<2, 3>);
            default: return go(ttm_stream_kernel<2, 4>);
        }
    }
    BulkPlan bp;
    if (dmma_ident && plan_bulk(P, bp)) {
        P.R = (int32_t)bp.R;
        P.ntiles = (P.O + bp.R - 1) / bp.R;
        P.I_div.init((uint32_t)P.I);
        const DeviceInfo &di = device_info();
        const int64_t per_sm = std::max<int64_t>(1, std::min<int64_t>(16, (228 * 1024) / (int64_t)(bp.smem + 2048)));
        const int64_t grid = std::min<int64_t>(P.ntiles, (int64_t)di.num_sms * per_sm);
        const int threads = bp.threads;
        const size_t smem = bp.smem;
        auto go = [&](auto kern) -> int {
            cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            if (e != cudaSuccess) return cuda_status(e, "ttm bulk smem");
            kern<<<(unsigned)grid, threads, smem, st>>>(P);
            return cuda_status(cudaGetLastError(), "ttm bulk launch");
        };
        auto pick = [&](auto mt, auto ntc) -> int {
            constexpr int MTv = decltype(mt)::value, NTv = decltype(ntc)::value;
            if (bp.nst == 2) return go(ttm_bulk_kernel<MTv, NTv, 2>);
            if (bp.nst == 3) return go(ttm_bulk_kernel<MTv, NTv, 3>);
            return go(ttm_bulk_kernel<MTv, NTv, 4>);
        };
        using I1 = std::integral_constant<int, 1>;
        using I2 = std::integral_constant<int, 2>;
        using I4 = std::integral_constant<int, 4>;
        if (bp.nt == 1) return P.J <= 16 ? pick(I1{}, I1{}) : pick(I2{}, I1{});
        if (bp.nt == 2) return P.J <= 16 ? pick(I1{}, I2{}) : pick(I2{}, I2{});
        return P.J <= 16 ? pick(I1{}, I4{}) : pick(I2{}, I4{});
    }
    const int64_t stage_target = stage_kb * 1024;
    int64_t R = std::max<int64_t>(1, std::min<int64_t>(256 / P.I, stage_target / (KI * s)));
    // keep every tile's start 16-byte aligned for the bulk copy
    while (R > 1 && (R * KI * s) % 16 != 0) --R;
    if ((R * KI * s) % 16 != 0 && P.O > R) return TL_EUNSUPPORTED;
    P.R = (int32_t)R;
    P.ntiles = (P.O + R - 1) / R;
    P.I_div.init((uint32_t)P.I);
    const bool dmma = (a.dtype == TL_F64) && P.J <= 32 && !force_simt;  // FP64 tensor cores for float64
    // SIMT: one position per thread; DMMA: 8*NT positions per warp
    const int64_t per_thread = dmma ? ntile / 4 : 1;
    const int threads =
        (int)std::min<int64_t>(256, std::max<int64_t>(32, ((R * P.I + 32 * per_thread - 1) / (32 * per_thread)) * 32));
    const size_t bbytes = dmma ? StagedLayout<double, true>(P.J, P.K).bbytes
                               : (a.dtype == TL_F32 ? StagedLayout<float, false>(P.J, P.K).bbytes
                                                    : StagedLayout<int64_t, false>(P.J, P.K).bbytes);
    const size_t stage_bytes = ((size_t)R * KI * s + 15) & ~(size_t)15;
    // the output tile is staged only for contiguous outputs of the SIMT fold
    const bool stage_out = P.ident && !(dmma && kDirectStore);
    const size_t smem = bbytes + kTtmStages * stage_bytes + (stage_out ? (size_t)R * P.J * P.I * s : 0);
    if (smem > 200 * 1024) return TL_EUNSUPPORTED;
    const DeviceInfo &di = device_info();
    const int64_t per_sm = std::max<int64_t>(1, std::min<int64_t>(8, (228 * 1024) / (int64_t)(smem + 2048)));
    const int64_t grid = std::min<int64_t>(P.ntiles, (int64_t)di.num_sms * per_sm);
    auto go = [&](auto kern) -> int {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return cuda_status(e, "ttm staged smem");
        kern<<<(unsigned)grid, threads, smem, st>>>(P);
        return cuda_status(cudaGetLastError(), "ttm staged launch");
    };
    if (dmma && ntile == 8) return P.J <= 16 ? go(ttm_staged_kernel<double, 1, 8>) : go(ttm_staged_kernel<double, 2, 8>);
    if (dmma) return P.J <= 16 ? go(ttm_staged_kernel<double, 1, 4>) : go(ttm_staged_kernel<double, 2, 4>);
    if (a.dtype == TL_F64) return go(ttm_staged_kernel<double, 0>);
    if (a.dtype == TL_F32) return go(ttm_staged_kernel<float, 0>);
    return go(ttm_staged_kernel<int64_t, 0>);
}

// Which small-J kernel a ttm with J <= 32 would use (host only; outputs are
// freshly allocated, so C is taken as 16-byte aligned).  TL_EUNSUPPORTED: the
// staged family does not apply (the caller falls back to the GETT / SIMT path).
int ttm_staged_describe(const tl_desc &a, const tl_desc &bm, int m0, std::string &out) {
    TtmSimtParams P{};
    if (!build_params(a, (const void *)0x100000, bm, (const void *)0x200000, (void *)0x300000, m0, P))
        return TL_EUNSUPPORTED;
    if (!staged_family_ok(P, a.dtype)) return TL_EUNSUPPORTED;
    const SmallTtmKnobs &kn = small_ttm_knobs();
    const bool dmma_ident = a.dtype == TL_F64 && P.J <= 32 && P.ident && !kn.force_simt;
    const std::string head = "{\"O\": " + std::to_string(P.O) + ", \"K\": " + std::to_string(P.K) + ", \"I\": " +
                             std::to_string(P.I) + ", \"J\": " + std::to_string(P.J) + ", ";
    StreamPlan sp;
    BulkPlan bp;
    if (dmma_ident && plan_stream(P, sp)) {
        out = head + "\"path\": \"stream\", \"R\": " + std::to_string(sp.R) + ", \"NT\": " + std::to_string(sp.nt) +
              ", \"warps\": " + std::to_string(sp.nw) + ", \"slots_per_warp\": " + std::to_string(sp.sw) +
              ", \"smem\": " + std::to_string(sp.smem) + "}";
    } else if (dmma_ident && plan_bulk(P, bp)) {
        out = head + "\"path\": \"bulk\", \"R\": " + std::to_string(bp.R) + ", \"threads\": " +
              std::to_string(bp.threads) + ", \"smem\": " + std::to_string(bp.smem) + "}";
    } else {
        // the staged kernel's own tile constraint (ttm_staged_enqueue)
        const int64_t s = (int64_t)dtype_size(a.dtype), KI = P.K * P.I;
        int64_t R = std::max<int64_t>(1, std::min<int64_t>(256 / P.I, kn.stage_kb * 1024 / (KI * s)));
        while (R > 1 && (R * KI * s) % 16 != 0) --R;
        if ((R * KI * s) % 16 != 0 && P.O > R) return TL_EUNSUPPORTED;
        out = head + "\"path\": \"staged\", \"R\": " + std::to_string(R) + "}";
    }
    return TL_OK;
}

// Would ttm_staged_enqueue run the stream or the bulk tile kernel?  (Outputs
// are freshly allocated, so C is taken as 16-byte aligned.)
bool ttm_tile_kernels_apply(const tl_desc &a, const tl_desc &bm, int m0) {
    TtmSimtParams P{};
    if (!build_params(a, (const void *)0x100000, bm, (const void *)0x200000, (void *)0x300000, m0, P)) return false;
    if (!staged_family_ok(P, a.dtype)) return false;
    const SmallTtmKnobs &kn = small_ttm_knobs();
    if (!(a.dtype == TL_F64 && P.J <= 32 && P.ident && !kn.force_simt)) return false;
    StreamPlan sp;
    BulkPlan bp;
    return plan_stream(P, sp) || plan_bulk(P, bp);
}

int ttm_simt_enqueue(const tl_desc &a, const void *a_ptr, const tl_desc &bm, const void *b_ptr, void *c_ptr,
                     int m0, cudaStream_t st) {
    TtmSimtParams P{};
    if (!build_params(a, a_ptr, bm, b_ptr, c_ptr, m0, P)) return TL_EUNSUPPORTED;
    const int64_t total = P.O * P.J * P.I;
    if (total == 0) return TL_OK;
    const int threads = 256;
    const int64_t grid = (total + threads - 1) / threads;
    if (grid > 0x7fffffffll) {
        set_error("ttm: %lld outputs exceed one launch", (long long)total);
        return TL_EUNSUPPORTED;
    }
    if (a.dtype == TL_F64) ttm_simt_kernel<double, double><<<(unsigned)grid, threads, 0, st>>>(P);
    else if (a.dtype == TL_F32) ttm_simt_kernel<float, float><<<(unsigned)grid, threads, 0, st>>>(P);
    else ttm_simt_kernel<int64_t, int64_t><<<(unsigned)grid, threads, 0, st>>>(P);
    return cuda_status(cudaGetLastError(), "ttm launch");
}

}  // namespace tl
