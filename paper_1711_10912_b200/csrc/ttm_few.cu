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
// with ba * bc = 128 * NP.  The box degenerates to 1-D (bc = 1) when A's and
// C's fastest free digits are the same dimension or C is contiguous along j.
// Odd extents need no divisibility: x and y are flattened over whole digit
// groups and only the last box of each group is masked.
//
// Each thread folds NP positions for all J rows at once (J accumulators per
// position, B in shared memory as [k][j]; k in order, so every output is the
// same chain as in the other ttm kernels: fused multiply-add for float64 --
// the DMMA semantics --, exact for float32 (products are exact in binary64)
// and int64).  A is read with L1-allocating loads: when the run along x is
// shorter than a sector (small inner blocks, contracted stride 1), the rest of
// the sector is consumed by the same CTA a few k-steps later.  Outputs are
// staged in shared memory and written along C (y fastest), along j when C is
// contiguous in j, or directly when x is C's fastest direction too.
#include <algorithm>
#include <cstdlib>
#include <string>
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
    int64_t K, I, J;
    int64_t bs0, bs1, jstride;
    int32_t ba, bc, ba_shift, bc_shift;  // box (powers of two), ba * bc = 128 * NP
    int32_t store;                       // FewStore
    int32_t pitch;                       // staged tile: elements per j row
    uint32_t X, Y;                       // extents of the flattened digit groups
    FastDiv nx_div;                      // tile -> (x box, y box), x fastest
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

template <class T, int JB, int NP, int D>
__global__ void __launch_bounds__(kFewThreads) ttm_few_kernel(const __grid_constant__ TtmFewParams P) {
    using Acc = typename AccOf<T>::type;
    constexpr int BN = kFewThreads * NP;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    Acc *Bs = (Acc *)smem_raw;  // [K][JB], rows j >= J zero
    const size_t bbytes = ((size_t)P.K * JB * sizeof(Acc) + 15) & ~(size_t)15;
    int64_t *tax = (int64_t *)(smem_raw + bbytes);  // [ba] A offset of x (-1: past X)
    int64_t *tcx = tax + P.ba;                      // [ba]
    int64_t *tay = tcx + P.ba;                      // [bc] (-1: past Y)
    int64_t *tcy = tay + P.bc;                      // [bc]
    T *cs = (T *)(tcy + P.bc);                      // [JB][pitch] staged outputs

    const int tid = threadIdx.x;
    const T *A = (const T *)P.a;
    const T *B = (const T *)P.bm;
    T *C = (T *)P.c;
    for (int idx = tid; idx < (int)P.K * JB; idx += kFewThreads) {
        const int k = idx / JB, j = idx % JB;
        Bs[idx] = j < P.J ? (Acc)B[j * P.bs0 + k * P.bs1] : Acc(0);
    }
    uint32_t tx, ty;
    P.nx_div.divmod(blockIdx.x, ty, tx);
    for (int t = tid; t < P.ba; t += kFewThreads) {
        const uint64_t x = (uint64_t)tx * P.ba + t;
        int64_t oa = -1, oc = 0;
        if (x < P.X) few_decode((uint32_t)x, P.nxd, P.xdiv, P.xa, P.xc, oa, oc);
        tax[t] = oa;
        tcx[t] = oc;
    }
    for (int t = tid; t < P.bc; t += kFewThreads) {
        const uint64_t y = (uint64_t)ty * P.bc + t;
        int64_t oa = -1, oc = 0;
        if (y < P.Y) few_decode((uint32_t)y, P.nyd, P.ydiv, P.ya, P.yc, oa, oc);
        tay[t] = oa;
        tcy[t] = oc;
    }
    __syncthreads();

    Acc acc[NP][JB];
    const T *pa[NP];
    bool ok[NP];
    int xl[NP], yl[NP];
#pragma unroll
    for (int p = 0; p < NP; ++p) {
        const int n = tid + p * kFewThreads;
        xl[p] = n & (P.ba - 1);
        yl[p] = n >> P.ba_shift;
        const int64_t ax = tax[xl[p]], ay = tay[yl[p]];
        ok[p] = ax >= 0 && ay >= 0;
        pa[p] = A + (ok[p] ? ax + ay : 0);
#pragma unroll
        for (int j = 0; j < JB; ++j) acc[p][j] = Acc(0);
    }
    const int64_t K = P.K, I = P.I;
    // Each thread streams its own column(s) of A through a private ring of D
    // k-rows in shared memory (cp.async, one group per row; only the issuing
    // thread reads its slots, so cp.async.wait_group is the only sync): D
    // loads per position stay in flight while the accumulators, not the
    // operands, hold the registers.
    {
        T *ring = cs;  // [D][BN]; reused as the staged output tile afterwards
        const T *pn[NP];
#pragma unroll
        for (int p = 0; p < NP; ++p) pn[p] = pa[p];
#pragma unroll
        for (int d = 0; d < D; ++d) {
            if (d < K) {
#pragma unroll
                for (int p = 0; p < NP; ++p) {
                    if (ok[p]) cp_async<sizeof(T)>(ring + d * BN + tid + p * kFewThreads, pn[p]);
                    pn[p] += I;
                }
            }
            cp_async_commit();
        }
#pragma unroll 4
        for (int64_t k = 0; k < K; ++k) {
            cp_async_wait<D - 1>();
            const int slot = (int)(k & (D - 1));
            Acc x[NP];
#pragma unroll
            for (int p = 0; p < NP; ++p) x[p] = ok[p] ? (Acc)ring[slot * BN + tid + p * kFewThreads] : Acc(0);
            if (k + D < K) {
#pragma unroll
                for (int p = 0; p < NP; ++p) {
                    if (ok[p]) cp_async<sizeof(T)>(ring + slot * BN + tid + p * kFewThreads, pn[p]);
                    pn[p] += I;
                }
            }
            cp_async_commit();
            const Acc *brow = Bs + k * JB;
#pragma unroll
            for (int j = 0; j < JB; j += 2) {
                Acc b0, b1;
                few_ld2<Acc>(brow + j, b0, b1);
#pragma unroll
                for (int p = 0; p < NP; ++p) {
                    acc[p][j] = few_mac(acc[p][j], x[p], b0);
                    acc[p][j + 1] = few_mac(acc[p][j + 1], x[p], b1);
                }
            }
        }
        cp_async_wait<0>();
    }

    if (P.store == kFewDirect) {
        // x runs along C as well: lanes write consecutive C elements per j
#pragma unroll
        for (int p = 0; p < NP; ++p) {
            if (!ok[p]) continue;
            T *pc = C + tcx[xl[p]] + tcy[yl[p]];
#pragma unroll
            for (int j = 0; j < JB; ++j)
                if (j < P.J) pc[j * P.jstride] = narrow<T>(acc[p][j]);
        }
        return;
    }
    const int pitch = P.pitch;
    __syncthreads();  // every thread is done with its ring slots (the staged tile aliases them)
    if (P.store == kFewAlongY) {
#pragma unroll
        for (int p = 0; p < NP; ++p) {
            const int pos = yl[p] * (P.ba + 1) + xl[p];
#pragma unroll
            for (int j = 0; j < JB; ++j) cs[j * pitch + pos] = narrow<T>(acc[p][j]);
        }
        __syncthreads();
        // y fastest: lanes write runs along C's fastest free direction
        for (int idx = tid; idx < BN * JB; idx += kFewThreads) {
            const int yy = idx & (P.bc - 1);
            const int xx = (idx >> P.bc_shift) & (P.ba - 1);
            const int j = idx / BN;
            if (j >= P.J) break;
            if (tax[xx] >= 0 && tay[yy] >= 0)
                C[tcx[xx] + tcy[yy] + j * P.jstride] = cs[j * pitch + yy * (P.ba + 1) + xx];
        }
        return;
    }
    // C contiguous along j: stage, then lanes write each position's J-run
#pragma unroll
    for (int p = 0; p < NP; ++p) {
        const int n = tid + p * kFewThreads;
#pragma unroll
        for (int j = 0; j < JB; ++j) cs[j * pitch + n] = narrow<T>(acc[p][j]);
    }
    __syncthreads();
    for (int idx = tid; idx < BN * JB; idx += kFewThreads) {
        const int j = idx % JB, n = idx / JB;
        const int xx = n & (P.ba - 1), yy = n >> P.ba_shift;
        if (j < P.J && tax[xx] >= 0 && tay[yy] >= 0) C[tcx[xx] + tcy[yy] + j] = cs[j * pitch + n];
    }
}

// ------------------------------------------------------------------ planning
struct FewDigit {
    int64_t ext, as, cs;
};

struct FewPlan {
    TtmFewParams P{};
    int jb = 0, np = 0;
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
    // positions per thread (TL_TTM_FEW_NP; measured: DESIGN.md)
    static const int np_knob = [] {
        const char *e = getenv("TL_TTM_FEW_NP");
        return e ? atoi(e) : 1;
    }();
    const int np = (jb <= 16 && np_knob == 2) ? 2 : 1;
    const int BN = kFewThreads * np;
    const size_t bbytes = ((size_t)cn.K * jb * 8 + 15) & ~(size_t)15;
    if (bbytes > 64 * 1024) return false;
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
        // they span >= 16 positions; y: the rest in C order
        int64_t X = 1;
        size_t r = 0;
        while (r < ic && X < 16) X *= dg[r++].ext;
        gx.assign(dg.begin(), dg.begin() + r);
        gy.assign(dg.begin() + r, dg.end());
        std::stable_sort(gy.begin(), gy.end(), [](const FewDigit &p, const FewDigit &q) { return p.cs < q.cs; });
        // box width along x: the power of two in [2, 32] with the least masked
        // lanes in the last box (ties: 16, then wider)
        const int cand[5] = {16, 32, 8, 4, 2};
        double best = 1e30;
        for (int b : cand) {
            const double waste = (double)((X + b - 1) / b * b) / (double)X;
            if (waste < best - 1e-9) {
                best = waste;
                ba = b;
            }
        }
        bc = BN / ba;
        store = kFewAlongY;
    }
    if (gx.size() > TL_MAX_DIGITS || gy.size() > TL_MAX_DIGITS) return false;
    TtmFewParams &P = fp.P;
    const int64_t es = (int64_t)dtype_size(a.dtype);
    P.a = (const unsigned char *)a_ptr + a.offset * es;
    P.bm = (const unsigned char *)b_ptr + bm.offset * es;
    P.c = c_ptr;
    P.K = cn.K;
    P.I = cn.I;
    P.J = J;
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
    fp.jb = jb;
    fp.np = np;
    fp.grid = nX * nY;
    const size_t ring = (size_t)kFewRing * BN * es;
    const size_t stage = store == kFewDirect ? 0 : (size_t)jb * P.pitch * es;
    fp.smem = bbytes + (size_t)2 * (ba + bc) * 8 + std::max(ring, stage);
    return fp.smem <= 160 * 1024;
}

template <class T> static int few_launch(const FewPlan &fp, cudaStream_t st) {
    auto go = [&](auto kern) -> int {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fp.smem);
        if (e != cudaSuccess) return cuda_status(e, "ttm few smem");
        kern<<<(unsigned)fp.grid, kFewThreads, fp.smem, st>>>(fp.P);
        return cuda_status(cudaGetLastError(), "ttm few launch");
    };
    if (fp.np == 2) {
        switch (fp.jb) {
            case 4: return go(ttm_few_kernel<T, 4, 2, kFewRing>);
            case 8: return go(ttm_few_kernel<T, 8, 2, kFewRing>);
            default: return go(ttm_few_kernel<T, 16, 2, kFewRing>);
        }
    }
    switch (fp.jb) {
        case 4: return go(ttm_few_kernel<T, 4, 1, kFewRing>);
        case 8: return go(ttm_few_kernel<T, 8, 1, kFewRing>);
        case 16: return go(ttm_few_kernel<T, 16, 1, kFewRing>);
        default: return go(ttm_few_kernel<T, 32, 1, kFewRing>);
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
