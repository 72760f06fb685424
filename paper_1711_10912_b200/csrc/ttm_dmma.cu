// ttm_dmma.cu -- float64 ttm (contraction.py:200-298) as a GETT on the FP64
// tensor cores (mma.sync f64 -> SASS DMMA.8x8x4; tcgen05 has no f64 kind).
//
// For dense A of any permutation layout (plan.h: A[O][K][I]) the product is
//     C[j, f] = sum_k B[j, k] * A'[k, f],    f = o*I + i  (free positions)
// i.e. one GEMM with M = J (rows of B), N = O*I, K = n_mode, where the
// operand A' and the first-order output are addressed through tables:
//     A'(k, f) = A + aoff[f] + k*I,     C(j, f) = C + coff[f] + j*jstride.
// The N dimension of a CTA tile is BN consecutive positions of a host-chosen
// ordering sigma of the free digits (possibly splitting digits), which makes
// the A' loads and the C stores coalesce for every layout/mode:
//   * output contiguous along j (mode 1): sigma = A's order,
//   * A contiguous along k (I == 1):       sigma = C's order,
//   * otherwise a 2-D box: 8 positions along A's fastest free digit x 16
//     along the output's fastest free digit (64-byte load runs; each CTA
//     writes whole 32-byte sectors of C).
// Default CTA tile 64 (J) x 64 (free) x 32 (k), 4 warps of 32x32, FP64
// m16n8k4 MMAs, 2-stage cp.async pipeline, three CTAs per SM (table at
// Tile1); operands in padded shared memory (pitch = 4 mod 16 doubles:
// conflict-free fragment loads), fragments double-buffered in registers; the
// epilogue stages the tile in shared memory in C order and writes whole
// warp runs of first-order C.
//
// Numerics: DMMA accumulates k in order with fused multiply-adds (measured
// on B200: DMMA.8x8x4 == 4 sequential FMAs), so results differ from the
// reference's separately rounded fold by at most ~K ulps of sum_k |A||B|;
// parity is checked at 1e-12 of that bound (tests/).
#include <algorithm>
#include <cstdlib>
#include <string>
#include <vector>
#include <type_traits>

#include "plan.h"
#include "tl_common.cuh"

namespace tl {

// CTA tile BM (J) x BN (free positions) x BK (k), NST-stage pipeline
template <int BM_, int BN_, int BK_, int NST_> struct GettTile {
    static constexpr int BM = BM_, BN = BN_, BK = BK_, NST = NST_;
    static constexpr int LDWA = BN + 4;  // pitch of the [k][n] A tile (doubles, = 4 mod 16)
    static constexpr int LDWB = BM + 4;  // pitch of the [k][m] B tile
    static constexpr int LDK = BK + 4;   // pitch of [n][k] / [m][k] tiles
    static constexpr int A_TILE = BK * LDWA > BN * LDK ? BK * LDWA : BN * LDK;  // doubles
    static constexpr int B_TILE = BK * LDWB > BM * LDK ? BK * LDWB : BM * LDK;
    static constexpr int CP = BN + 4;    // staged-epilogue row pitch
    static constexpr size_t SMEM = (size_t)NST * (A_TILE + B_TILE) * 8 + (size_t)BN * 28;
    static_assert(BM * CP <= NST * (A_TILE + B_TILE), "staged C tile must fit the operand stages");
};
// Measured on cfg3 (TFLOP/s, 6 layout/mode cases): smaller CTAs, several
// per SM, keep the DMMA pipe busier than one big CTA whose 16 warps stall
// together at every k-tile barrier (prologue/epilogue of one CTA overlap the
// main loop of the others):
//   128x128x32, 3 stages, 1 CTA/SM, 16 warps      29.3-29.7
//   128x64x32,  2 stages, 2 CTAs/SM, 8 warps       31.2-32.5
//   64x64x16,   3 stages, 3 CTAs/SM, 4 warps       31.5-32.8
//   64x64x32,   2 stages, 3 CTAs/SM, 4 warps       31.8-33.2   (default)
using Tile1 = GettTile<128, 128, 32, 3>;
using Tile4 = GettTile<128, 64, 32, 2>;
using Tile9 = GettTile<64, 64, 32, 2>;
using Tile10 = GettTile<64, 64, 16, 3>;
using Tile12 = GettTile<64, 64, 16, 2>;
// few rows (J <= 16 / <= 32, long folds): no idle MMA rows, 128 free positions per CTA
using Tile16 = GettTile<16, 128, 32, 2>;
using Tile32 = GettTile<32, 128, 32, 2>;

// warp layout: WM x WN warps, each TM m16 tiles x TN n8 tiles
template <int WM_, int WN_, int TM_, int TN_> struct GettCfg {
    static constexpr int WM = WM_, WN = WN_, TM = TM_, TN = TN_;
    static constexpr int THREADS = 32 * WM * WN;
};
using Cfg16 = GettCfg<4, 4, 2, 4>;  // Tile1: 16 warps of 32 x 32
using Cfg8x = GettCfg<4, 2, 2, 4>;  // Tile4: 8 warps of 32 x 32
using Cfg4y = GettCfg<2, 2, 2, 4>;  // Tile9/10: 4 warps of 32 x 32
using Cfg16n = GettCfg<1, 4, 1, 4>;  // Tile16: 4 warps of 16 x 32
using Cfg32n = GettCfg<1, 4, 2, 4>;  // Tile32: 4 warps of 32 x 32

struct TtmParams {
    const void *a;  // TA elements (float64, or float32 widened exactly on the fragment loads)
    const void *b;
    void *c;
    int64_t J, K, I, F;
    int64_t jstride;
    int64_t bs0, bs1;
    int32_t mtiles;
    int32_t nd;  // sigma digits (fastest first)
    int32_t box_a, box_c, box_s;  // 2-D box: store order swaps its two digits (box_s = 0: none)
    FastDiv dig[TL_MAX_DIGITS + 1];
    int64_t dig_a[TL_MAX_DIGITS + 1];
    int64_t dig_c[TL_MAX_DIGITS + 1];
};

__device__ __forceinline__ void cp_async8_zfill(void *smem_dst, const void *gmem_src, bool valid) {
    const int n = valid ? 8 : 0;
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(smem_u32(smem_dst)), "l"(gmem_src), "r"(n));
}

__device__ __forceinline__ void cp_async4_zfill(void *smem_dst, const void *gmem_src, bool valid) {
    const int n = valid ? 4 : 0;
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(smem_u32(smem_dst)), "l"(gmem_src), "r"(n));
}


__device__ __forceinline__ void cp_async16_zfill(void *smem_dst, const void *gmem_src, bool valid) {
    const int n = valid ? 16 : 0;
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(smem_dst)), "l"(gmem_src), "r"(n));
}

// one element / an adjacent pair of TA elements, zero-filled when !valid
template <class TA> __device__ __forceinline__ void cp_elem(void *d, const void *s, bool valid) {
    if constexpr (sizeof(TA) == 8) cp_async8_zfill(d, s, valid); else cp_async4_zfill(d, s, valid);
}
template <class TA> __device__ __forceinline__ void cp_pair(void *d, const void *s, bool valid) {
    if constexpr (sizeof(TA) == 8) cp_async16_zfill(d, s, valid); else cp_async8_zfill(d, s, valid);
}

__device__ __forceinline__ void mma_16x8x4(double (&d)[4], const double (&a)[2], double b) {
    asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
                 : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3])
                 : "d"(a[0]), "d"(a[1]), "d"(b));
}

template <class TA, class CFG, class TL, bool A_KMAJOR, bool B_KMAJOR, bool PAIRS, int MINB>
__global__ void __launch_bounds__(CFG::THREADS, MINB) ttm_dmma_kernel(const __grid_constant__ TtmParams P) {
    constexpr int THREADS = CFG::THREADS, TM = CFG::TM, TN = CFG::TN, WN = CFG::WN;
    constexpr int BM = TL::BM, BN = TL::BN, BK = TL::BK, NST = TL::NST;
    constexpr int LDWA = TL::LDWA, LDWB = TL::LDWB, LDK = TL::LDK, A_TILE = TL::A_TILE, B_TILE = TL::B_TILE;
    constexpr int CP = TL::CP;
    static_assert(CFG::WM * TM * 16 == BM && CFG::WN * TN * 8 == BN, "tile mismatch");
    static_assert(THREADS >= BN && THREADS >= BM, "one load column per thread");
    extern __shared__ __align__(16) unsigned char smem_raw[];
    TA *As = (TA *)smem_raw;                         // NST x A_TILE
    TA *Bs = As + NST * A_TILE;                      // NST x B_TILE
    // tables after the (double-sized) operand area, which the epilogue reuses
    int64_t *aoff = (int64_t *)(smem_raw + (size_t)NST * (A_TILE + B_TILE) * sizeof(double));  // BN
    const TA *Pa = (const TA *)P.a;
    const TA *Pb = (const TA *)P.b;
    TA *Pc = (TA *)P.c;
    int64_t *coff = aoff + BN;                       // BN  (-1: masked column)
    int64_t *coffp = coff + BN;                      // BN  C offset of store position l
    int32_t *lpos = (int32_t *)(coffp + BN);         // BN  store position of column n

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int g = lane >> 2, t = lane & 3;
    const int wm = warp / WN;
    const int wn = warp % WN;
    const int mt = blockIdx.x % P.mtiles;
    const int64_t nt = blockIdx.x / P.mtiles;
    const int64_t m0 = (int64_t)mt * BM;

    // column tables for this N tile (sigma-ordered free positions)
    auto column_offsets = [&](int64_t q, int64_t &ao, int64_t &co) {
        ao = 0;
        co = -1;
        if (q < P.F) {
            uint32_t x = (uint32_t)q;
            co = 0;
            for (int d = 0; d < P.nd; ++d) {
                uint32_t qq, r;
                if (d == P.nd - 1) {
                    r = x;
                    qq = 0;
                } else {
                    P.dig[d].divmod(x, qq, r);
                }
                ao += (int64_t)r * P.dig_a[d];
                co += (int64_t)r * P.dig_c[d];
                x = qq;
            }
        }
    };
    if (tid < BN) {
        int64_t ao, co;
        column_offsets(nt * BN + tid, ao, co);
        aoff[tid] = ao;
        coff[tid] = co;
        // store order of the staged epilogue: position l of the tile in C
        // order visits column n = perm(l) (swap the two box digits)
        int n = tid;
        if (P.box_s) {
            const int r = tid % P.box_s;
            n = tid - r + (r % P.box_c) * P.box_a + r / P.box_c;
        }
        int64_t a2, c2;
        column_offsets(nt * BN + n, a2, c2);
        coffp[tid] = c2;
        lpos[n] = tid;
    }
    __syncthreads();

    const int64_t K = P.K, I = P.I;
    const int KT = (int)((K + BK - 1) / BK);

    // Per-thread load assignment, fixed for the whole tile.  K-major
    // operands: lanes walk k (fixed k column per thread); otherwise lanes
    // walk n/m (fixed column, k rows).  Base pointers are formed once.
    constexpr int LPTA = (BK * BN) / THREADS, LPTB = (BK * BM) / THREADS;
    const int a_kk0 = A_KMAJOR ? (tid & (BK - 1)) : (tid / BN);
    const int a_nn0 = A_KMAJOR ? (tid / BK) : (tid & (BN - 1));
    const int b_kk0 = B_KMAJOR ? (tid & (BK - 1)) : (tid / BM);
    const int b_mm0 = B_KMAJOR ? (tid / BK) : (tid & (BM - 1));
    const TA *a_base_fixed = Pa + aoff[a_nn0];
    const bool a_col_ok = coff[a_nn0] >= 0;
    const TA *b_base_fixed = Pb + (m0 + b_mm0) * P.bs0;
    const bool b_row_ok = (m0 + b_mm0) < P.J;

    // 16-byte variant: pairs of elements adjacent in both global and shared
    // memory (along n / m for N-major, along k for K-major), half the LDGSTS
    constexpr int LPTA2 = LPTA / 2, LPTB2 = LPTB / 2;
    const int a_p0 = A_KMAJOR ? 2 * (tid & (BK / 2 - 1)) : 2 * (tid & (BN / 2 - 1));  // element index of pair
    const int a_q0 = A_KMAJOR ? tid / (BK / 2) : tid / (BN / 2);
    const int b_p0 = B_KMAJOR ? 2 * (tid & (BK / 2 - 1)) : 2 * (tid & (BM / 2 - 1));
    const int b_q0 = B_KMAJOR ? tid / (BK / 2) : tid / (BM / 2);

    auto load_stage = [&](int stage, int kt) {
        const int64_t k0 = (int64_t)kt * BK;
        TA *as = As + stage * A_TILE;
        TA *bs = Bs + stage * B_TILE;
        if constexpr (PAIRS) {
#pragma unroll
            for (int s = 0; s < LPTA2; ++s) {
                if constexpr (A_KMAJOR) {  // pair (k, k+1) of column nn
                    const int nn = a_q0 + s * (THREADS / (BK / 2));
                    const int64_t k = k0 + a_p0;
                    const bool ok = (k < K) && (coff[nn] >= 0);
                    cp_pair<TA>(as + nn * LDK + a_p0, Pa + (ok ? aoff[nn] + k : 0), ok);
                } else {  // pair (n, n+1) of row kk
                    const int kk = a_q0 + s * (THREADS / (BN / 2));
                    const int64_t k = k0 + kk;
                    const bool ok = (k < K) && (coff[a_p0] >= 0);
                    cp_pair<TA>(as + kk * LDWA + a_p0, Pa + (ok ? aoff[a_p0] + k * I : 0), ok);
                }
            }
#pragma unroll
            for (int s = 0; s < LPTB2; ++s) {
                if constexpr (B_KMAJOR) {
                    const int mm = b_q0 + s * (THREADS / (BK / 2));
                    const int64_t k = k0 + b_p0, j = m0 + mm;
                    const bool ok = (k < K) && (j < P.J);
                    cp_pair<TA>(bs + mm * LDK + b_p0, Pb + (ok ? j * P.bs0 + k : 0), ok);
                } else {
                    const int kk = b_q0 + s * (THREADS / (BM / 2));
                    const int64_t k = k0 + kk, j = m0 + b_p0;
                    const bool ok = (k < K) && (j < P.J);
                    cp_pair<TA>(bs + kk * LDWB + b_p0, Pb + (ok ? j + k * P.bs1 : 0), ok);
                }
            }
        } else {
#pragma unroll
            for (int s = 0; s < LPTA; ++s) {
                if constexpr (A_KMAJOR) {
                    const int nn = a_nn0 + s * (THREADS / BK);
                    const int64_t k = k0 + a_kk0;
                    const bool ok = (k < K) && (coff[nn] >= 0);
                    cp_elem<TA>(as + nn * LDK + a_kk0, Pa + (ok ? aoff[nn] + k : 0), ok);
                } else {
                    const int kk = a_kk0 + s * (THREADS / BN);
                    const int64_t k = k0 + kk;
                    const bool ok = a_col_ok && (k < K);
                    cp_elem<TA>(as + kk * LDWA + a_nn0, ok ? a_base_fixed + k * I : Pa, ok);
                }
            }
#pragma unroll
            for (int s = 0; s < LPTB; ++s) {
                if constexpr (B_KMAJOR) {
                    const int mm = b_mm0 + s * (THREADS / BK);
                    const int64_t k = k0 + b_kk0, j = m0 + mm;
                    const bool ok = (k < K) && (j < P.J);
                    cp_elem<TA>(bs + mm * LDK + b_kk0, Pb + (ok ? j * P.bs0 + k : 0), ok);
                } else {
                    const int kk = b_kk0 + s * (THREADS / BM);
                    const int64_t k = k0 + kk;
                    const bool ok = b_row_ok && (k < K);
                    cp_elem<TA>(bs + kk * LDWB + b_mm0, ok ? b_base_fixed + k * P.bs1 : Pb, ok);
                }
            }
        }
    };

    double acc[TM][TN][4];
#pragma unroll
    for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j)
#pragma unroll
            for (int v = 0; v < 4; ++v) acc[i][j][v] = 0.0;

#pragma unroll
    for (int s = 0; s < NST - 1; ++s) {
        if (s < KT) load_stage(s, s);
        cp_async_commit();
    }

    for (int kt = 0; kt < KT; ++kt) {
        cp_async_wait<NST - 2>();
        __syncthreads();
        {
            const int nk = kt + NST - 1;
            if (nk < KT) load_stage(nk % NST, nk);
            cp_async_commit();
        }
        const TA *as = As + (kt % NST) * A_TILE;
        const TA *bs = Bs + (kt % NST) * B_TILE;
        // fragments double-buffered in registers: step k4+1 is loaded from
        // shared memory while step k4's MMAs issue
        double af[2][TM][2], bf[2][TN];
        auto load_frags = [&](int buf, int k4) {
#pragma unroll
            for (int i = 0; i < TM; ++i) {
                const int m = wm * (16 * TM) + i * 16 + g;
                if constexpr (B_KMAJOR) {
                    af[buf][i][0] = bs[m * LDK + k4 + t];
                    af[buf][i][1] = bs[(m + 8) * LDK + k4 + t];
                } else {
                    af[buf][i][0] = bs[(k4 + t) * LDWB + m];
                    af[buf][i][1] = bs[(k4 + t) * LDWB + m + 8];
                }
            }
#pragma unroll
            for (int j = 0; j < TN; ++j) {
                const int n = wn * (8 * TN) + j * 8 + g;
                bf[buf][j] = A_KMAJOR ? as[n * LDK + k4 + t] : as[(k4 + t) * LDWA + n];
            }
        };
        load_frags(0, 0);
#pragma unroll
        for (int k4 = 0; k4 < BK; k4 += 4) {
            const int cur = (k4 / 4) & 1;
            if (k4 + 4 < BK) load_frags(cur ^ 1, k4 + 4);
#pragma unroll
            for (int i = 0; i < TM; ++i)
#pragma unroll
                for (int j = 0; j < TN; ++j) mma_16x8x4(acc[i][j], af[cur][i], bf[cur][j]);
        }
    }
    cp_async_wait<0>();

    // epilogue: fragments -> first-order C
    if (P.jstride == 1) {
        // C contiguous along j: fragment rows already form 64-byte runs
#pragma unroll
        for (int i = 0; i < TM; ++i) {
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int64_t j = m0 + wm * (16 * TM) + i * 16 + g + 8 * h;
                if (j >= P.J) continue;
#pragma unroll
                for (int jj = 0; jj < TN; ++jj) {
#pragma unroll
                    for (int v = 0; v < 2; ++v) {
                        const int n = wn * (8 * TN) + jj * 8 + 2 * t + v;
                        const int64_t co = coff[n];
                        if (co >= 0) Pc[co + j] = (TA)acc[i][jj][2 * h + v];
                    }
                }
            }
        }
        return;
    }
    // Otherwise stage the tile in shared memory in C order (row m, store
    // position l, skewed one double per 32 positions: 2 wavefronts per
    // access both ways) and write whole 256-byte warp runs of C.
    __syncthreads();  // every warp is done with the operand stages
    double *cs = (double *)smem_raw;
    int ln[TN][2];
#pragma unroll
    for (int jj = 0; jj < TN; ++jj)
#pragma unroll
        for (int v = 0; v < 2; ++v) {
            const int l = lpos[wn * (8 * TN) + jj * 8 + 2 * t + v];
            ln[jj][v] = l + (l >> 5);
        }
#pragma unroll
    for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int m = wm * (16 * TM) + i * 16 + g + 8 * h;
#pragma unroll
            for (int jj = 0; jj < TN; ++jj)
#pragma unroll
                for (int v = 0; v < 2; ++v) cs[m * CP + ln[jj][v]] = acc[i][jj][2 * h + v];
        }
    __syncthreads();
    {
        const int l = tid & (BN - 1);
        const int64_t co = coffp[l];
        if (co >= 0) {
            const double *src = cs + l + (l >> 5);
#pragma unroll 4
            for (int m = tid / BN; m < BM; m += THREADS / BN) {
                const int64_t j = m0 + m;
                if (j < P.J) Pc[co + j * P.jstride] = (TA)src[m * CP];
            }
        }
    }
}

// ------------------------------------------------------------------ planning
struct Digit {
    int64_t ext, as, cs;  // extent, A stride, C stride
};

static int gett_run(const tl_desc &a, const void *a_ptr, const tl_desc &bm, const void *b_ptr, void *c_ptr, int m0,
                    cudaStream_t st, std::string *describe);

int ttm_dmma_enqueue(const tl_desc &a, const void *a_ptr, const tl_desc &bm, const void *b_ptr, void *c_ptr, int m0,
                     cudaStream_t st) {
    return gett_run(a, a_ptr, bm, b_ptr, c_ptr, m0, st, nullptr);
}

// Host-only: the GETT plan (digit order sigma, operand majors, 16-byte pairs).
int ttm_dmma_describe(const tl_desc &a, const tl_desc &bm, int m0, std::string &out) {
    return gett_run(a, (const void *)0x100000, bm, (const void *)0x200000, nullptr, m0, nullptr, &out);
}

static int gett_run(const tl_desc &a, const void *a_ptr, const tl_desc &bm, const void *b_ptr, void *c_ptr, int m0,
                    cudaStream_t st, std::string *describe) {
    // CTA tile (see the table above Tile1); TL_GETT_TILE = 1, 4, 9 or 10
    static const int tile_env = [] {
        const char *e = getenv("TL_GETT_TILE");
        const int k = e ? atoi(e) : 9;
        return (k == 1 || k == 4 || k == 10 || k == 12) ? k : 9;
    }();
    static const bool few_tiles = [] {
        const char *e = getenv("TL_GETT_FEW");
        return e ? atoi(e) != 0 : true;
    }();
    const int64_t J = bm.extent[0];
    // few rows (reached for long folds, K > 128): a 16- or 32-row tile instead of 64 rows of mostly idle MMAs
    const int tile_kind = (few_tiles && a.dtype == TL_F64 && J <= 32) ? (J <= 16 ? 16 : 32) : tile_env;
    const int BM = tile_kind == 16 ? 16 : tile_kind == 32 ? 32 : tile_kind >= 9 ? 64 : 128;
    const int BN = (tile_kind == 1 || tile_kind == 16 || tile_kind == 32) ? 128 : 64;
    Canon cn;
    if (!canon_contraction(a, m0, J, cn)) {
        set_error("ttm: operand A is not a dense permutation layout (materialise views first)");
        return TL_EUNSUPPORTED;
    }
    const int64_t F = cn.O * cn.I;
    // GEMM-shaped only: few rows J (the caller tries the staged kernel
    // first for J <= 32) or tiny K / F
    if (J < 8 || cn.K < 16 || F < 64 || F > 0xffffffffll) return TL_EUNSUPPORTED;

    // free digits in A order with A strides
    std::vector<Digit> dg;
    {
        int64_t run = 1;
        for (auto &d : cn.inner) {
            dg.push_back({d.first, run, d.second});
            run *= d.first;
        }
        run = cn.K * cn.I;
        for (auto &d : cn.outer) {
            dg.push_back({d.first, run, d.second});
            run *= d.first;
        }
    }
    const bool a_kmajor = (cn.I == 1);
    std::vector<Digit> sigma;
    bool box = false;
    if (cn.jstride == 1 || dg.empty()) {
        sigma = dg;  // output contiguous along j: keep A's order
    } else if (a_kmajor) {
        sigma = dg;
        std::stable_sort(sigma.begin(), sigma.end(), [](const Digit &x, const Digit &y) { return x.cs < y.cs; });
    } else {
        // fastest free digit of A (inner, stride 1) vs of C
        size_t ic = 0;
        for (size_t d = 1; d < dg.size(); ++d)
            if (dg[d].cs < dg[ic].cs) ic = d;
        if (ic == 0) {
            sigma = dg;
        } else {
            // 2-D box: 8 along A's fastest digit (64-byte load runs) x 16
            // along C's fastest digit (whole sectors of C per CTA)
            const Digit dc = dg[ic], da = dg[0];
            box = true;
            const int64_t alo = (da.ext % 8 == 0 && da.ext > 8) ? 8 : da.ext;
            const int64_t clo = (dc.ext % 16 == 0 && dc.ext > 16) ? 16 : dc.ext;
            sigma.push_back({alo, da.as, da.cs});
            sigma.push_back({clo, dc.as, dc.cs});
            if (alo < da.ext) sigma.push_back({da.ext / alo, da.as * alo, da.cs * alo});
            if (clo < dc.ext) sigma.push_back({dc.ext / clo, dc.as * clo, dc.cs * clo});
            for (size_t d = 1; d < dg.size(); ++d)
                if (d != ic) sigma.push_back(dg[d]);
        }
    }
    if (sigma.size() > TL_MAX_DIGITS + 1) return TL_EUNSUPPORTED;
    int32_t box_a = 0, box_c = 0, box_s = 0;
    if (box) {
        // store order inside one tile: the tile holds box_a A-fast x box_c C-fast positions
        box_a = (int32_t)sigma[0].ext;
        box_c = (int32_t)std::min<int64_t>(sigma[1].ext, BN / std::max<int32_t>(1, box_a));
        box_s = box_a * box_c;
        if (box_s == 0 || BN % box_s != 0 || sigma[1].ext % box_c != 0) box_a = box_c = box_s = 0;
    }
    // float64, or float32 widened exactly on the fragment loads (binary64
    // accumulation, one rounding on store: within the float32 tolerance)
    if (a.dtype != TL_F64 && a.dtype != TL_F32) return TL_EUNSUPPORTED;
    const bool f32 = a.dtype == TL_F32;
    const int64_t es = f32 ? 4 : 8;
    if (f32 && tile_kind != 9) return TL_EUNSUPPORTED;
    TtmParams P{};
    P.a = (const char *)a_ptr + a.offset * es;
    P.b = (const char *)b_ptr + bm.offset * es;
    P.c = c_ptr;
    P.J = J;
    P.K = cn.K;
    P.I = cn.I;
    P.F = F;
    P.jstride = cn.jstride;
    P.bs0 = bm.stride[0];
    P.bs1 = bm.stride[1];
    P.mtiles = (int32_t)((J + BM - 1) / BM);
    if (sigma.empty()) sigma.push_back({1, 0, 0});
    P.nd = (int32_t)sigma.size();
    P.box_a = box_a;
    P.box_c = box_c;
    P.box_s = box_s;
    for (size_t d = 0; d < sigma.size(); ++d) {
        P.dig[d].init((uint32_t)sigma[d].ext);
        P.dig_a[d] = sigma[d].as;
        P.dig_c[d] = sigma[d].cs;
    }
    const int64_t ntiles = (F + BN - 1) / BN;
    const int64_t grid = ntiles * P.mtiles;
    if (grid > 0x7fffffffll) return TL_EUNSUPPORTED;
    const bool b_kmajor = (bm.stride[1] == 1 && bm.extent[1] > 1);
    // operand pairs (one 16-byte copy for float64, 8-byte for float32): both
    // elements adjacent in global memory, aligned, never straddling a masked column
    const uintptr_t pa = (uintptr_t)P.a, pb = (uintptr_t)P.b;
    bool pairs = (pa % (2 * es) == 0) && (pb % (2 * es) == 0);
    if (a_kmajor)
        pairs = pairs && (cn.K % 2 == 0);
    else
        pairs = pairs && sigma[0].as == 1 && sigma[0].ext % 2 == 0 && F % 2 == 0 && cn.I % 2 == 0;
    if (b_kmajor)
        pairs = pairs && (cn.K % 2 == 0) && (P.bs0 % 2 == 0);
    else
        pairs = pairs && (P.bs0 == 1) && (J % 2 == 0) && (P.bs1 % 2 == 0);
    if (describe != nullptr) {
        char buf[1024];
        int n = snprintf(buf, sizeof(buf), "{\"path\": \"gett\", \"dtype\": \"%s\", \"O\": %lld, \"K\": %lld, \"I\": %lld, \"J\": %lld, "
                         "\"jstride\": %lld, \"a_kmajor\": %d, \"b_kmajor\": %d, \"pairs\": %d, \"grid\": %lld, \"box\": %d, "
                         "\"sigma\": [",
                         f32 ? "f32" : "f64", (long long)cn.O, (long long)cn.K, (long long)cn.I, (long long)J,
                         (long long)cn.jstride,
                         a_kmajor ? 1 : 0, b_kmajor ? 1 : 0, pairs ? 1 : 0, (long long)grid, (int)box_s);
        for (size_t d = 0; d < sigma.size() && n < (int)sizeof(buf) - 64; ++d)
            n += snprintf(buf + n, sizeof(buf) - n, "%s[%lld, %lld, %lld]", d ? ", " : "", (long long)sigma[d].ext,
                          (long long)sigma[d].as, (long long)sigma[d].cs);
        snprintf(buf + n, sizeof(buf) - n, "]}");
        *describe = buf;
        return TL_OK;
    }
    auto launch = [&](auto ta, auto cfg, auto tl_, auto minb) -> int {
        using TA = decltype(ta);
        using CFG = decltype(cfg);
        using TL = decltype(tl_);
        constexpr int MINB = decltype(minb)::value;
        auto go = [&](auto kern) -> int {
            cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)TL::SMEM);
            if (e != cudaSuccess) return cuda_status(e, "ttm smem attribute");
            kern<<<(unsigned)grid, CFG::THREADS, TL::SMEM, st>>>(P);
            return cuda_status(cudaGetLastError(), "ttm dmma launch");
        };
        if (pairs) {
            if (a_kmajor)
                return b_kmajor ? go(ttm_dmma_kernel<TA, CFG, TL, true, true, true, MINB>)
                                : go(ttm_dmma_kernel<TA, CFG, TL, true, false, true, MINB>);
            return b_kmajor ? go(ttm_dmma_kernel<TA, CFG, TL, false, true, true, MINB>)
                            : go(ttm_dmma_kernel<TA, CFG, TL, false, false, true, MINB>);
        }
        if (a_kmajor)
            return b_kmajor ? go(ttm_dmma_kernel<TA, CFG, TL, true, true, false, MINB>)
                            : go(ttm_dmma_kernel<TA, CFG, TL, true, false, false, MINB>);
        return b_kmajor ? go(ttm_dmma_kernel<TA, CFG, TL, false, true, false, MINB>)
                        : go(ttm_dmma_kernel<TA, CFG, TL, false, false, false, MINB>);
    };
    if (f32) return launch(float{}, Cfg4y{}, Tile9{}, std::integral_constant<int, 3>{});
    if (tile_kind == 16) return launch(double{}, Cfg16n{}, Tile16{}, std::integral_constant<int, 2>{});
    if (tile_kind == 32) return launch(double{}, Cfg32n{}, Tile32{}, std::integral_constant<int, 2>{});
    if (tile_kind == 1) return launch(double{}, Cfg16{}, Tile1{}, std::integral_constant<int, 1>{});
    if (tile_kind == 4) return launch(double{}, Cfg8x{}, Tile4{}, std::integral_constant<int, 2>{});
    if (tile_kind == 10) return launch(double{}, Cfg4y{}, Tile10{}, std::integral_constant<int, 3>{});
    if (tile_kind == 12) return launch(double{}, Cfg4y{}, Tile12{}, std::integral_constant<int, 4>{});
    return launch(double{}, Cfg4y{}, Tile9{}, std::integral_constant<int, 3>{});
}

}  // namespace tl
