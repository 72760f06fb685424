// ttm_few.cu -- ttm (contraction.py:200-298) with few output rows (J <= 32)
// for ANY permutation layout and mode: the HBM-bound case the tile kernels of
// ttm_simt.cu only cover for first-order-compatible outputs.
//
//     C[coff(f) + j*jstride] = sum_k B[j, k] * A[aoff(f) + k*I]
//
// over the free positions f.  A CTA owns a 2-D box of positions:
//   x: `ba` consecutive values of a flattened index over the digits that come
//      FIRST in A's storage order (loads of one k-row are runs along A),
//   y: `bc` consecutive values of a flattened index over the remaining digits
//      taken in C's (first-order) order (stores are runs along C),
// with ba * bc = 128.  The box degenerates to 1-D (bc = 1) when A's and
// C's fastest free digits are the same dimension or C is contiguous along j.
// Odd extents need no divisibility: x and y are flattened over whole digit
// groups and only the last box of each group is masked.
//
// Each thread streams the column of one position (its K elements, I apart)
// through a private ring of k-rows in shared memory (cp.async.ca: when the run
// along x is shorter than a sector -- small inner blocks, contracted stride 1
// -- L1 keeps the rest of the sector for the neighbouring rows).  Two folds,
// both in k order with fused multiply-adds, so every output is the same chain
// as in the stream / bulk / GETT kernels (exact for float32, whose products
// are exact in binary64, and for int64):
//   * ttm_few_dmma_kernel (float64 / float32, K >= 9): FP64 tensor cores, a
//     warp = 4 n8 tiles of positions, persistent CTAs;
//   * ttm_few_kernel (K <= 8, int64): J accumulators per thread, b(., k)
//     broadcast from shared memory.
// Outputs are staged in shared memory and written along C (y fastest), along
// j when C is contiguous in j, or along x when x is C's fastest direction too.
#include <algorithm>
#include <cstdlib>
#include <string>
#include <type_traits>
#include <vector>

#include "plan.h"
#include "tl_common.cuh"

namespace tl {

constexpr int kFewThreads = 128;
constexpr int kFewRing = 16;  // k-rows in flight per position
enum FewStore : int32_t { kFewDirect = 0, kFewAlongY = 1, kFewAlongJ = 2 };

struct TtmFewParams {
    const void *a;
    const void *bm;
    void *c;
    int64_t I;
    int32_t K, J;
    int64_t bs0, bs1, jstride;
    int32_t ba, bc, ba_shift, bc_shift;  // box (powers of two), ba * bc = 128
    int32_t store;                       // FewStore
    int32_t pitch;                       // staged tile: elements per j row
    uint32_t X, Y;                       // extents of the flattened digit groups
    FastDiv nx_div;                      // tile -> (x box, y box), x fastest
    uint32_t ntiles;
    int32_t nxd, nyd;
    FastDiv xdiv[TL_MAX_DIGITS], ydiv[TL_MAX_DIGITS];
    int64_t xa[TL_MAX_DIGITS], xc[TL_MAX_DIGITS], ya[TL_MAX_DIGITS], yc[TL_MAX_DIGITS];
};

template <class Acc> __device__ __forceinline__ void few_ld2(const Acc *p, Acc &u, Acc &v);
template <> __device__ __forceinline__ void few_ld2<double>(const double *p, double &u, double &v) {
    const double2 t = *(const double2 *)p;
    u = t.x;
    v = t.y;
}
template <> __device__ __forceinline__ void few_ld2<int64_t>(const int64_t *p, int64_t &u, int64_t &v) {
    const longlong2 t = *(const longlong2 *)p;
    u = t.x;
    v = t.y;
}
__device__ __forceinline__ double few_mac(double acc, double a, double b) { return fma(a, b, acc); }
__device__ __forceinline__ int64_t few_mac(int64_t acc, int64_t a, int64_t b) { return fold_step(acc, a, b); }

// flattened group index -> (A offset, C offset)
__device__ __forceinline__ void few_decode(uint32_t x, int nd, const FastDiv *dv, const int64_t *sa, const int64_t *sc,
                                           int64_t &oa, int64_t &oc) {
    oa = 0;
    oc = 0;
    for (int d = 0; d < nd; ++d) {
        uint32_t q, r;
        if (d == nd - 1) {
            r = x;
            q = 0;
        } else {
            dv[d].divmod(x, q, r);
        }
        oa += (int64_t)r * sa[d];
        oc += (int64_t)r * sc[d];
        x = q;
    }
}

template <class T, int JB, int D>
__global__ void __launch_bounds__(kFewThreads) ttm_few_kernel(const __grid_constant__ TtmFewParams P) {
    using Acc = typename AccOf<T>::type;
    constexpr int BN = kFewThreads;
    constexpr int H = D / 2;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    Acc *Bs = (Acc *)smem_raw;  // [K][JB], rows j >= J zero
    const size_t bbytes = ((size_t)P.K * JB * sizeof(Acc) + 15) & ~(size_t)15;
    int64_t *tax = (int64_t *)(smem_raw + bbytes);  // [ba] A offset of x (-1: past X)
    int64_t *tcx = tax + P.ba;                      // [ba]
    int64_t *tay = tcx + P.ba;                      // [bc] (-1: past Y)
    int64_t *tcy = tay + P.bc;                      // [bc]
    int64_t *tco = tcy + P.bc;                      // [BN] C offset of position n (-1: masked)
    T *cs = (T *)(tco + BN);                        // ring [D][BN], then the staged outputs [JB][pitch]

    const int tid = threadIdx.x;
    const T *A = (const T *)P.a;
    const T *B = (const T *)P.bm;
    T *C = (T *)P.c;
    const int J = P.J, K = P.K;
    for (int idx = tid; idx < K * JB; idx += kFewThreads) {
        const int k = idx / JB, j = idx % JB;
        Bs[idx] = j < J ? (Acc)B[j * P.bs0 + k * P.bs1] : Acc(0);
    }
    uint32_t tx, ty;
    P.nx_div.divmod(blockIdx.x, ty, tx);
    if (tid < P.ba) {
        const uint64_t x = (uint64_t)tx * P.ba + tid;
        int64_t oa = -1, oc = 0;
        if (x < P.X) few_decode((uint32_t)x, P.nxd, P.xdiv, P.xa, P.xc, oa, oc);
        tax[tid] = oa;
        tcx[tid] = oc;
    }
    if (tid < P.bc) {
        const uint64_t y = (uint64_t)ty * P.bc + tid;
        int64_t oa = -1, oc = 0;
        if (y < P.Y) few_decode((uint32_t)y, P.nyd, P.ydiv, P.ya, P.yc, oa, oc);
        tay[tid] = oa;
        tcy[tid] = oc;
    }
    __syncthreads();

    const int xl = tid & (P.ba - 1), yl = tid >> P.ba_shift;
    const int64_t ax = tax[xl], ay = tay[yl];
    const bool ok = ax >= 0 && ay >= 0;
    // masked positions read (and discard) the tile's first valid column
    const T *pn = A + (ok ? ax + ay : 0);
    const int64_t I = P.I;
    Acc acc[JB];
#pragma unroll
    for (int j = 0; j < JB; ++j) acc[j] = Acc(0);

    // Each thread streams its own column of A through a private ring in
    // shared memory: two halves of H k-rows, one cp.async group per half (only
    // the issuing thread reads its slots, so cp.async.wait_group is the only
    // sync).  Up to 2H loads per position stay in flight while the
    // accumulators, not the operands, hold the registers.
    T *ring = cs + tid;
    int left = K;  // rows not yet issued
    auto issue = [&](int half) {
        T *dst = ring + half * (H * BN);
        if (left >= H) {
#pragma unroll
            for (int r = 0; r < H; ++r) {
                cp_async<sizeof(T)>(dst + r * BN, pn);
                pn += I;
            }
        } else {
            for (int r = 0; r < left; ++r) {
                cp_async<sizeof(T)>(dst + r * BN, pn);
                pn += I;
            }
        }
        left -= H;
        cp_async_commit();
    };
    issue(0);
    issue(1);
    int half = 0;
    for (int k0 = 0; k0 < K; k0 += H) {
        cp_async_wait<1>();
        const T *src = ring + half * (H * BN);
        const Acc *brow = Bs + k0 * JB;
        if (K - k0 >= H) {
            Acc x[H];
#pragma unroll
            for (int r = 0; r < H; ++r) x[r] = (Acc)src[r * BN];
            issue(half);
#pragma unroll
            for (int r = 0; r < H; ++r) {
#pragma unroll
                for (int j = 0; j < JB; j += 2) {
                    Acc b0, b1;
                    few_ld2<Acc>(brow + r * JB + j, b0, b1);
                    acc[j] = few_mac(acc[j], x[r], b0);
                    acc[j + 1] = few_mac(acc[j + 1], x[r], b1);
                }
            }
        } else {
            const int rows = K - k0;
            for (int r = 0; r < rows; ++r) {
                const Acc xr = (Acc)src[r * BN];
#pragma unroll
                for (int j = 0; j < JB; j += 2) {
                    Acc b0, b1;
                    few_ld2<Acc>(brow + r * JB + j, b0, b1);
                    acc[j] = few_mac(acc[j], xr, b0);
                    acc[j + 1] = few_mac(acc[j + 1], xr, b1);
                }
            }
        }
        half ^= 1;
    }
    cp_async_wait<0>();

    const int64_t js = P.jstride;
    if (P.store == kFewDirect) {
        // x runs along C as well: lanes write consecutive C elements per j
        if (!ok) return;
        T *pc = C + tcx[xl] + tcy[yl];
#pragma unroll
        for (int j = 0; j < JB; ++j) {
            if (j < J) *pc = narrow<T>(acc[j]);
            pc += js;
        }
        return;
    }
    const int pitch = P.pitch;
    __syncthreads();  // every thread is done with its ring slots (the staged tile aliases them)
    if (P.store == kFewAlongY) {
        {
            T *dst = cs + yl * (P.ba + 1) + xl;
#pragma unroll
            for (int j = 0; j < JB; ++j) dst[j * pitch] = narrow<T>(acc[j]);
        }
        __syncthreads();
        // y fastest: lanes write runs along C's fastest free direction; a
        // thread keeps one (x, y) of the box for every j
        const int yy = tid & (P.bc - 1), xx = tid >> P.bc_shift;
        if (tax[xx] < 0 || tay[yy] < 0) return;
        T *pc = C + tcx[xx] + tcy[yy];
        const T *src = cs + yy * (P.ba + 1) + xx;
#pragma unroll
        for (int j = 0; j < JB; ++j) {
            if (j < J) *pc = src[j * pitch];
            pc += js;
        }
        return;
    }
    // C contiguous along j: stage, then lanes write each position's J-run
    tco[tid] = ok ? tcx[xl] + tcy[yl] : -1;
#pragma unroll
    for (int j = 0; j < JB; ++j) cs[j * pitch + tid] = narrow<T>(acc[j]);
    __syncthreads();
    {
        const int j = tid % JB;
        if (j >= J) return;
        const T *src = cs + j * pitch;
#pragma unroll 4
        for (int n = tid / JB; n < BN; n += kFewThreads / JB) {
            const int64_t co = tco[n];
            if (co >= 0) C[co + j] = src[n];
        }
    }
}

// ---------------------------------------------------- float64 / float32: DMMA
// The SIMT fold above reads every b(j, k) from shared memory for every
// position (8 broadcast LDS.128 per k-row and warp: measured bound by the
// shared-memory data pipe at ~0.55 of HBM).  On the FP64 tensor cores
// (mma.sync.m16n8k4.f64 -> DMMA.8x8x4, k in order = the same FMA chain) the
// matrix fragment is 2 doubles per lane and k-step, shared by the warp's four
// n8 tiles: 6 LDS.64 per 4 k-rows instead of 36 LDS.  Each warp owns 32
// positions (4 n8 tiles) of the box; its lanes fill the ring columns of those
// 32 positions (cp.async, zero-filled past K) and read fragments across lanes
// (__syncwarp after the group wait).  float32 operands are widened on the
// fragment loads (exact products).
constexpr int kFewRingPitch = kFewThreads + 4;  // = 4 mod 16: conflict-free fragment loads

__host__ __device__ __forceinline__ int few_ldb(int K) {
    int l = (K + 3) / 4 * 4;
    while (l % 16 != 4) l += 4;
    return l;
}

__device__ __forceinline__ void few_mma(double (&d)[4], double a0, double a1, double b) {
    asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
                 : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3])
                 : "d"(a0), "d"(a1), "d"(b));
}

template <class T> __device__ __forceinline__ void few_cp_zfill(void *smem_dst, const void *gmem_src, bool valid) {
    const int n = valid ? (int)sizeof(T) : 0;
    asm volatile("cp.async.ca.shared.global [%0], [%1], %2, %3;" ::"r"(smem_u32(smem_dst)), "l"(gmem_src),
                 "n"((int)sizeof(T)), "r"(n));
}

template <class T, int MT, int D>
__global__ void __launch_bounds__(kFewThreads) ttm_few_dmma_kernel(const __grid_constant__ TtmFewParams P) {
    constexpr int BN = kFewThreads, H = D / 2, RP = kFewRingPitch, JB = 16 * MT;
    static_assert(H % 4 == 0, "whole k-steps per ring half");
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int J = P.J, K = P.K;
    const int ldb = few_ldb(K);
    double *Bm = (double *)smem_raw;  // [JB][ldb], zero padded in j and k
    // box tables, double-buffered: the next box's are built while this box's
    // outputs are written.  tab[b] = tax[ba] tcx[ba] tay[bc] tcy[bc]
    int64_t *tab0 = (int64_t *)(Bm + JB * ldb);
    const int tabn = 2 * (P.ba + P.bc);
    int64_t *tco = tab0 + 2 * tabn;       // [BN] C offset of position n (along-j stores)
    T *ringbuf = (T *)(tco + BN);         // [D][RP]
    T *cs = ringbuf + D * RP;             // [JB][pitch] staged outputs (not aliased: the next box's loads are in flight)

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int g = lane >> 2, t = lane & 3;
    const T *A = (const T *)P.a;
    const T *B = (const T *)P.bm;
    T *C = (T *)P.c;
    const int xl = tid & (P.ba - 1), yl = tid >> P.ba_shift;
    const int64_t I = P.I;
    const int pitch = P.pitch;
    const bool along_y = P.store == kFewAlongY;
    const int64_t js = P.jstride;

    // this thread's own column of a box (registers only), and its ring loads
    int64_t ax, cx, ay, cy;
    bool ok;
    const T *pn;
    int left;
    auto own_column = [&](uint32_t tile) {
        uint32_t tx, ty;
        P.nx_div.divmod(tile, ty, tx);
        ax = -1, cx = 0, ay = -1, cy = 0;
        const uint64_t x = (uint64_t)tx * P.ba + xl, y = (uint64_t)ty * P.bc + yl;
        if (x < P.X) few_decode((uint32_t)x, P.nxd, P.xdiv, P.xa, P.xc, ax, cx);
        if (y < P.Y) few_decode((uint32_t)y, P.nyd, P.ydiv, P.ya, P.yc, ay, cy);
        ok = ax >= 0 && ay >= 0;
        pn = A + (ok ? ax + ay : 0);  // masked positions read (and discard) column 0
        left = K;
    };
    T *ring = ringbuf + tid;
    auto issue = [&](int half) {
        T *dst = ring + half * (H * RP);
        if (left >= H) {
#pragma unroll
            for (int r = 0; r < H; ++r) {
                cp_async<sizeof(T)>(dst + r * RP, pn);
                pn += I;
            }
        } else if (left > 0) {
            // last rows, zero-filled up to a whole k-step
            const int upto = (left + 3) & ~3;
            for (int r = 0; r < upto; ++r) {
                few_cp_zfill<T>(dst + r * RP, r < left ? pn : A, r < left);
                if (r < left) pn += I;
            }
        }
        left -= H;
        cp_async_commit();
    };
    auto build_tables = [&](uint32_t tile, int64_t *tb) {
        // x entries are the own columns of threads 0..ba-1; y entries are decoded
        uint32_t tx, ty;
        P.nx_div.divmod(tile, ty, tx);
        if (tid < P.ba) {
            tb[tid] = ax;
            tb[P.ba + tid] = cx;
        }
        if (tid < P.bc) {
            const uint64_t y = (uint64_t)ty * P.bc + tid;
            int64_t oa = -1, oc = 0;
            if (y < P.Y) few_decode((uint32_t)y, P.nyd, P.ydiv, P.ya, P.yc, oa, oc);
            tb[2 * P.ba + tid] = oa;
            tb[2 * P.ba + P.bc + tid] = oc;
        }
    };

    uint32_t tile = blockIdx.x;
    own_column(tile);
    issue(0);
    issue(1);
    for (int m = warp; m < JB; m += kFewThreads / 32)
        for (int k = lane; k < ldb; k += 32) Bm[m * ldb + k] = (m < J && k < K) ? (double)B[m * P.bs0 + k * P.bs1] : 0.0;
    build_tables(tile, tab0);
    __syncthreads();
    int cur = 0;
    const T *frag = ringbuf + warp * 32 + g;  // + (k row) * RP + n8 tile * 8
    for (;;) {
        double acc[MT][4][4];
#pragma unroll
        for (int i = 0; i < MT; ++i)
#pragma unroll
            for (int n = 0; n < 4; ++n)
#pragma unroll
                for (int v = 0; v < 4; ++v) acc[i][n][v] = 0.0;
        int half = 0;
        for (int k0 = 0; k0 < K; k0 += H) {
            cp_async_wait<1>();
            __syncwarp();
            const T *src = frag + half * (H * RP);
            double bf[H / 4][4];
#pragma unroll
            for (int s = 0; s < H / 4; ++s)
#pragma unroll
                for (int n = 0; n < 4; ++n) bf[s][n] = (k0 + 4 * s < K) ? (double)src[(4 * s + t) * RP + n * 8] : 0.0;
            __syncwarp();  // every lane holds its fragments: the half can be refilled
            issue(half);
#pragma unroll
            for (int s = 0; s < H / 4; ++s) {
                if (k0 + 4 * s < K) {
                    const double *bm = Bm + g * ldb + k0 + 4 * s + t;
#pragma unroll
                    for (int i = 0; i < MT; ++i) {
                        const double a0 = bm[(16 * i) * ldb], a1 = bm[(16 * i + 8) * ldb];
#pragma unroll
                        for (int n = 0; n < 4; ++n) few_mma(acc[i][n], a0, a1, bf[s][n]);
                    }
                }
            }
            half ^= 1;
        }
        // this box's C offsets before the next box's column replaces them
        const int64_t my_co = ok ? cx + cy : -1;
        const int64_t *tb = tab0 + cur * tabn;
        // the ring is drained: put the next box's loads in flight before
        // this box is staged and written
        const uint32_t next = tile + gridDim.x;
        const bool more = next < P.ntiles;
        if (more) {
            own_column(next);
            issue(0);
            issue(1);
        }
        // fragments -> staged tile cs[j][pos]: row j = 16 i + g + 8 h, column n = 32 warp + 8 n8 + 2 t + v
#pragma unroll
        for (int n = 0; n < 4; ++n) {
#pragma unroll
            for (int v = 0; v < 2; ++v) {
                const int col = warp * 32 + n * 8 + 2 * t + v;
                const int pos = along_y ? (col >> P.ba_shift) * (P.ba + 1) + (col & (P.ba - 1)) : col;
#pragma unroll
                for (int i = 0; i < MT; ++i)
#pragma unroll
                    for (int h = 0; h < 2; ++h) cs[(16 * i + g + 8 * h) * pitch + pos] = (T)acc[i][n][2 * h + v];
            }
        }
        if (P.store == kFewAlongJ) tco[tid] = my_co;
        if (more) build_tables(next, tab0 + (cur ^ 1) * tabn);
        __syncthreads();
        if (P.store != kFewAlongJ) {
            // a thread keeps one position of the box for every j: lanes along y
            // (C's fastest free direction) or, for direct boxes, along x
            int xx = xl, yy = yl, pos = tid;
            if (along_y) {
                yy = tid & (P.bc - 1);
                xx = tid >> P.bc_shift;
                pos = yy * (P.ba + 1) + xx;
            }
            if (tb[xx] >= 0 && tb[2 * P.ba + yy] >= 0) {
                T *pc = C + tb[P.ba + xx] + tb[2 * P.ba + P.bc + yy];
                const T *src = cs + pos;
#pragma unroll
                for (int j = 0; j < JB; ++j) {
                    if (j < J) *pc = src[j * pitch];
                    pc += js;
                }
            }
        } else {
            // C contiguous along j: lanes write each position's J-run
            const int j = tid % JB;
            if (j < J) {
                const T *src = cs + j * pitch;
#pragma unroll 4
                for (int n = tid / JB; n < BN; n += kFewThreads / JB) {
                    const int64_t co = tco[n];
                    if (co >= 0) C[co + j] = src[n];
                }
            }
        }
        if (!more) break;
        __syncthreads();  // the staged tile and tco are free for the next box
        tile = next;
        cur ^= 1;
    }
    cp_async_wait<0>();
}

// ------------------------------------------------------------------ planning
struct FewDigit {
    int64_t ext, as, cs;
};

struct FewPlan {
    TtmFewParams P{};
    int jb = 0, mt = 1;
    bool dmma = false;
    size_t smem = 0;
    int64_t grid = 0;
};

static int ilog2(int v) {
    int s = 0;
    while ((1 << s) < v) ++s;
    return s;
}

// TL_TTM_FEW: 0 = off, 1 = where the stream / bulk tile kernels do not apply
// (default), 2 = every ttm with J <= 32
int ttm_few_mode() {
    static const int m = [] {
        const char *e = getenv("TL_TTM_FEW");
        return e ? atoi(e) : 1;
    }();
    return m;
}

static bool plan_few(const tl_desc &a, const void *a_ptr, const tl_desc &bm, const void *b_ptr, void *c_ptr, int m0,
                     FewPlan &fp) {
    const int64_t J = bm.extent[0];
    if (J < 1 || J > 32) return false;
    if (a.dtype != TL_F64 && a.dtype != TL_F32 && a.dtype != TL_I64) return false;
    Canon cn;
    if (!canon_contraction(a, m0, J, cn)) return false;
    const int64_t F = cn.O * cn.I;
    if (F < 1 || F > kIdx32 || cn.K > (1 << 20)) return false;
    const int jb = J <= 4 ? 4 : J <= 8 ? 8 : J <= 16 ? 16 : 32;
    const int BN = kFewThreads;
    // long folds: the GETT's k-tiled operands (no whole-matrix image per CTA)
    if (cn.K > 128 && J >= 8 && a.dtype != TL_I64) return false;
    // FP64 tensor cores from K = 9 (measured: below, the SIMT fold's smaller
    // fixed cost per box wins; both fold k in order with fused multiply-adds)
    const bool dmma = a.dtype != TL_I64 && cn.K > 8;
    const int mt = J <= 16 ? 1 : 2;
    const size_t bbytes = dmma ? (size_t)16 * mt * few_ldb((int)cn.K) * 8 : (((size_t)cn.K * jb * 8 + 15) & ~(size_t)15);
    if (bbytes > 96 * 1024) return false;
    // free digits in A order with A strides
    std::vector<FewDigit> dg;
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
    if (dg.empty()) dg.push_back({1, 0, 0});
    std::vector<FewDigit> gx, gy;
    int32_t store = kFewDirect, ba = BN, bc = 1;
    size_t ic = 0;
    for (size_t d = 1; d < dg.size(); ++d)
        if (dg[d].cs < dg[ic].cs) ic = d;
    if (cn.jstride == 1 || ic == 0) {
        gx = dg;
        store = cn.jstride == 1 ? kFewAlongJ : kFewDirect;
    } else {
        // x: A's fastest digits up to (not including) C's fastest digit, until
        // they span the box width with few masked lanes (an extent such as 17
        // alone would waste 41% of a width-8 box: flattening the next digit
        // into x removes the ragged edge); y: the rest in C order
        // Box width along x by the traffic mix: the output is J/K of the
        // input, so a short fold wants long runs along C (wide in y; a 32-byte
        // sector along A is enough, L1 keeps its other half for the next
        // k-rows) and a long fold long runs along A.
        const int target = cn.K >= 2 * J ? 32 : cn.K >= J ? 16 : 2 * cn.K >= J ? 8 : 4;
        auto pick = [&](int64_t X, int &b) {
            if (X <= target) {
                b = 2;
                while (b < X) b *= 2;
                return (double)b / (double)X;
            }
            b = target;
            return (double)((X + b - 1) / b * b) / (double)X;
        };
        int64_t X = 1;
        size_t r = 0;
        while (r < ic && (X < target || pick(X, ba) > 1.15)) X *= dg[r++].ext;
        pick(X, ba);
        gx.assign(dg.begin(), dg.begin() + r);
        gy.assign(dg.begin() + r, dg.end());
        std::stable_sort(gy.begin(), gy.end(), [](const FewDigit &p, const FewDigit &q) { return p.cs < q.cs; });
        bc = BN / ba;
        store = kFewAlongY;
    }
    if (gx.size() > TL_MAX_DIGITS || gy.size() > TL_MAX_DIGITS) return false;
    TtmFewParams &P = fp.P;
    const int64_t es = (int64_t)dtype_size(a.dtype);
    P.a = (const unsigned char *)a_ptr + a.offset * es;
    P.bm = (const unsigned char *)b_ptr + bm.offset * es;
    P.c = c_ptr;
    P.K = (int32_t)cn.K;
    P.I = cn.I;
    P.J = (int32_t)J;
    P.bs0 = bm.stride[0];
    P.bs1 = bm.stride[1];
    P.jstride = cn.jstride;
    P.ba = ba;
    P.bc = bc;
    P.ba_shift = ilog2(ba);
    P.bc_shift = ilog2(bc);
    P.store = store;
    int64_t X = 1, Y = 1;
    P.nxd = (int32_t)gx.size();
    for (size_t d = 0; d < gx.size(); ++d) {
        P.xdiv[d].init((uint32_t)gx[d].ext);
        P.xa[d] = gx[d].as;
        P.xc[d] = gx[d].cs;
        X *= gx[d].ext;
    }
    P.nyd = (int32_t)gy.size();
    for (size_t d = 0; d < gy.size(); ++d) {
        P.ydiv[d].init((uint32_t)gy[d].ext);
        P.ya[d] = gy[d].as;
        P.yc[d] = gy[d].cs;
        Y *= gy[d].ext;
    }
    if (gy.empty()) {
        // one y position with zero offsets
        P.nyd = 1;
        P.ydiv[0].init(1);
        P.ya[0] = P.yc[0] = 0;
    }
    P.X = (uint32_t)X;
    P.Y = (uint32_t)Y;
    const int64_t nX = (X + ba - 1) / ba, nY = (Y + bc - 1) / bc;
    if (nX * nY > 0x7fffffffll) return false;
    P.nx_div.init((uint32_t)nX);
    P.pitch = store == kFewAlongY ? bc * (ba + 1) : BN + 1;
    if (dmma) P.pitch = (P.pitch + 3) / 4 * 4 + 1;  // odd pitch: the fragment rows g, g + 8 spread over the banks
    fp.jb = jb;
    fp.dmma = dmma;
    fp.mt = mt;
    P.ntiles = (uint32_t)(nX * nY);
    fp.grid = nX * nY;
    if (dmma) {
        // persistent CTAs: ring and staged tile side by side, two table sets
        const size_t ring = (size_t)kFewRing * kFewRingPitch * es, stage = (size_t)16 * mt * P.pitch * es;
        fp.smem = bbytes + (size_t)4 * (ba + bc) * 8 + (size_t)BN * 8 + ring + stage;
        const DeviceInfo &di = device_info();
        const int64_t per_sm = std::max<int64_t>(1, std::min<int64_t>(mt == 1 ? 6 : 4, (224 * 1024) / (int64_t)(fp.smem + 1024)));
        fp.grid = std::min<int64_t>(fp.grid, (int64_t)di.num_sms * per_sm);
    } else {
        const size_t ring = (size_t)kFewRing * BN * es;
        const size_t stage = store == kFewDirect ? 0 : (size_t)jb * P.pitch * es;
        fp.smem = bbytes + (size_t)2 * (ba + bc) * 8 + (size_t)BN * 8 + std::max(ring, stage);
    }
    return fp.smem <= 150 * 1024;
}

template <class T> static int few_launch(const FewPlan &fp, cudaStream_t st) {
    auto go = [&](auto kern) -> int {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fp.smem);
        if (e != cudaSuccess) return cuda_status(e, "ttm few smem");
        kern<<<(unsigned)fp.grid, kFewThreads, fp.smem, st>>>(fp.P);
        return cuda_status(cudaGetLastError(), "ttm few launch");
    };
    if constexpr (!std::is_same<T, int64_t>::value) {
        if (fp.dmma) return fp.mt == 1 ? go(ttm_few_dmma_kernel<T, 1, kFewRing>) : go(ttm_few_dmma_kernel<T, 2, kFewRing>);
    }
    switch (fp.jb) {
        case 4: return go(ttm_few_kernel<T, 4, kFewRing>);
        case 8: return go(ttm_few_kernel<T, 8, kFewRing>);
        case 16: return go(ttm_few_kernel<T, 16, kFewRing>);
        default: return go(ttm_few_kernel<T, 32, kFewRing>);
    }
}

int ttm_few_enqueue(const tl_desc &a, const void *a_ptr, const tl_desc &bm, const void *b_ptr, void *c_ptr, int m0,
                    cudaStream_t st) {
    FewPlan fp;
    if (!plan_few(a, a_ptr, bm, b_ptr, c_ptr, m0, fp)) return TL_EUNSUPPORTED;
    if (a.dtype == TL_F64) return few_launch<double>(fp, st);
    if (a.dtype == TL_F32) return few_launch<float>(fp, st);
    return few_launch<int64_t>(fp, st);
}

int ttm_few_describe(const tl_desc &a, const tl_desc &bm, int m0, std::string &out) {
    FewPlan fp;
    if (!plan_few(a, (const void *)0x100000, bm, (const void *)0x200000, (void *)0x300000, m0, fp))
        return TL_EUNSUPPORTED;
    const TtmFewParams &P = fp.P;
    const char *st = P.store == kFewDirect ? "direct" : P.store == kFewAlongY ? "along-y" : "along-j";
    out = "{\"path\": \"few\", \"K\": " + std::to_string(P.K) + ", \"I\": " + std::to_string(P.I) + ", \"J\": " +
          std::to_string(P.J) + ", \"X\": " + std::to_string(P.X) + ", \"Y\": " + std::to_string(P.Y) + ", \"ba\": " +
          std::to_string(P.ba) + ", \"bc\": " + std::to_string(P.bc) + ", \"store\": \"" + st + "\", \"grid\": " +
          std::to_string(fp.grid) + ", \"smem\": " + std::to_string(fp.smem) + "}";
    return TL_OK;
}

}  // namespace tl
