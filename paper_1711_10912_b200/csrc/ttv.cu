// ttv.cu -- mode-m tensor-times-vector on sm_100a (contraction.py:113-194).
//
// A dense tensor of any permutation layout is A[O][K][I] (plan.h).  Every
// output C(o, i) = sum_k A[o][k][i] * b[k] is the reference's left fold in
// k order, starting from 0, with separately rounded binary64 products and
// sums -- so outputs are bit-identical to the reference for float64 and
// for float32 storage (widened exactly, rounded once on store).
//
// Two regimes, chosen by where the contracted mode sits in the layout:
//
//  * strided fibers (I >= 32, "regime B"): one thread per output vector of
//    VEC consecutive inner indices; loads are coalesced along the inner
//    block (128-bit, L1 no-allocate), k loop unrolled for memory-level
//    parallelism, b staged in shared memory.
//
//  * contiguous / short-stride fibers (I < 32, "regime S", includes the
//    contracted-stride-1 case): a persistent CTA streams tiles of R
//    consecutive [K][I] blocks through a 3-stage cp.async shared-memory
//    pipeline (k-slabs of Kc rows), with row pitch padded so the per-thread
//    sequential folds read shared memory without bank conflicts (128-bit
//    LDS along k when I == 1).  One thread owns each output fold, which is
//    what keeps the summation order identical to the reference.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <mutex>
#include <vector>
#include <cstdio>
#include <numeric>
#include <type_traits>

#include "hopm_norm.cuh"
#include "plan.h"
#include "tl_common.cuh"

namespace tl {

struct TtvParams {
    const void *a;
    const void *b;
    void *c;
    const int32_t *stop;  // optional device flag: skip all work when set (HOPM)
    FusedNorm fn;         // optional HOPM normalisation of the output (last CTA)
    int64_t b_stride;
    int32_t b_dtype;
    int32_t b_smem;  // stage b in shared memory
    int64_t O, K, I;
    int32_t ident;
    DigitMap in_map, out_map;
    // regime S plan
    int32_t R;        // [K][I] blocks (rows) per tile
    int32_t Kc;       // k-slab length
    int32_t Lp;       // smem row pitch (elements)
    int32_t nslab;    // ceil(K / Kc)
    int64_t ntiles;   // ceil(O / R)
    int32_t opt;      // outputs per thread (regime S)
    FastDiv I_div;    // divides output slot j -> (row, i)
    FastDiv pr_div;   // pieces per row, full slab
    FastDiv pr_tail;  // pieces per row, last slab
    // regime S, permuted outputs: out_map(o) = otab[o % E] + out_hi(o / E),
    // otab (int32, shared memory) holding the map of the first otab_d0 digits
    int32_t in_vec_ok;  // regime B: first inner digit's extent is a multiple of VEC
    int64_t o_mul;      // regime B: o visiting-order multiplier (1: identity)
    int32_t otab_n;   // E (0: plain digit map)
    int32_t otab_d0;
    FastDiv otab_div;
    DigitMap out_hi;
    // L2 reuse between consecutive passes over one large tensor (HOPM's two
    // passes per sweep; a ttv per mode of the same tensor): the part of A a
    // pass reads LAST is loaded with the normal L2 policy and everything
    // else evict-first, so it is still L2-resident when the next pass reads
    // it, and the next pass's streaming fills evict each other instead of it.
    // "Last" is k >= keep_k when the grid is one wave (all CTAs walk k
    // together), CTAs >= keep_cta when it is several (later CTAs start later),
    // tiles >= keep_tile for the persistent 2-D TMA rows kernel.
    // l2_stream: the policy is on (else plain loads); the output always keeps
    // the normal policy and is counted against the budget first, so a large
    // ttv output (a short fold) stays L2-resident for its consumer.
    int64_t keep_k;
    int64_t keep_cta;
    int64_t keep_tile;
    int32_t l2_stream;
};

// ------------------------------------------------------------- regime B
template <class TA, int VEC> struct VecLoad;
template <> struct VecLoad<float, 4> {
    __device__ static void ld(const float *p, double *v) {
        float4 x = ld_stream_f4(p);
        v[0] = x.x; v[1] = x.y; v[2] = x.z; v[3] = x.w;
    }
};
template <> struct VecLoad<float, 2> {
    __device__ static void ld(const float *p, double *v) {
        float2 x = ld_stream_f2(p);
        v[0] = x.x; v[1] = x.y;
    }
};
template <> struct VecLoad<float, 1> {
    __device__ static void ld(const float *p, double *v) { v[0] = ld_stream(p); }
};
template <> struct VecLoad<double, 2> {
    __device__ static void ld(const double *p, double *v) {
        double2 x = ld_stream_d2(p);
        v[0] = x.x; v[1] = x.y;
    }
};
template <> struct VecLoad<double, 1> {
    __device__ static void ld(const double *p, double *v) { v[0] = ld_stream(p); }
};
template <> struct VecLoad<int64_t, 2> {
    __device__ static void ld(const int64_t *p, int64_t *v) {
        longlong2 x = ld_stream_l2(p);
        v[0] = x.x; v[1] = x.y;
    }
};
template <> struct VecLoad<int64_t, 1> {
    __device__ static void ld(const int64_t *p, int64_t *v) { v[0] = ld_stream(p); }
};

// Raw VEC-wide streaming load kept in the storage type (float32 values are
// widened only when folded: half the registers of a widened copy, so twice
// the loads can be in flight per SM).
template <class TA, int VEC> struct RawLoad {
    __device__ static void ld(const TA *p, TA *v) {
#pragma unroll
        for (int j = 0; j < VEC; ++j) v[j] = ld_stream(p + j);
    }
    __device__ static void ld_hint(const TA *p, TA *v, uint64_t pol) {
#pragma unroll
        for (int j = 0; j < VEC; ++j) {
            if constexpr (sizeof(TA) == 8)
                asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.b64 %0, [%1], %2;"
                             : "=l"(*(uint64_t *)&v[j]) : "l"(p + j), "l"(pol));
            else
                asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.b32 %0, [%1], %2;"
                             : "=r"(*(uint32_t *)&v[j]) : "l"(p + j), "l"(pol));
        }
    }
};
template <> struct RawLoad<float, 4> {
    __device__ static void ld(const float *p, float *v) {
        const float4 x = ld_stream_f4(p);
        v[0] = x.x; v[1] = x.y; v[2] = x.z; v[3] = x.w;
    }
    __device__ static void ld_hint(const float *p, float *v, uint64_t pol) {
        asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.f32 {%0,%1,%2,%3}, [%4], %5;"
                     : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]) : "l"(p), "l"(pol));
    }
};
template <> struct RawLoad<float, 2> {
    __device__ static void ld(const float *p, float *v) {
        const float2 x = ld_stream_f2(p);
        v[0] = x.x; v[1] = x.y;
    }
    __device__ static void ld_hint(const float *p, float *v, uint64_t pol) {
        asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.f32 {%0,%1}, [%2], %3;"
                     : "=f"(v[0]), "=f"(v[1]) : "l"(p), "l"(pol));
    }
};
template <> struct RawLoad<double, 2> {
    __device__ static void ld(const double *p, double *v) {
        const double2 x = ld_stream_d2(p);
        v[0] = x.x; v[1] = x.y;
    }
    __device__ static void ld_hint(const double *p, double *v, uint64_t pol) {
        asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.f64 {%0,%1}, [%2], %3;"
                     : "=d"(v[0]), "=d"(v[1]) : "l"(p), "l"(pol));
    }
};
template <> struct RawLoad<int64_t, 2> {
    __device__ static void ld(const int64_t *p, int64_t *v) {
        const longlong2 x = ld_stream_l2(p);
        v[0] = x.x; v[1] = x.y;
    }
    __device__ static void ld_hint(const int64_t *p, int64_t *v, uint64_t pol) {
        asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.s64 {%0,%1}, [%2], %3;"
                     : "=l"(v[0]), "=l"(v[1]) : "l"(p), "l"(pol));
    }
};

template <class TC, int VEC, class Acc>
__device__ __forceinline__ void store_outputs(const TtvParams &P, int64_t o, int64_t i0, const Acc *acc) {
    TC *c = (TC *)P.c;
    if (P.ident) {
        TC *dst = c + o * P.I + i0;
        if constexpr (VEC == 4 && sizeof(TC) == 4) {
            float4 v = make_float4(narrow<TC>(acc[0]), narrow<TC>(acc[1]), narrow<TC>(acc[2]), narrow<TC>(acc[3]));
            *(float4 *)dst = v;
        } else if constexpr (VEC == 2 && std::is_same<TC, double>::value) {
            *(double2 *)dst = make_double2(acc[0], acc[1]);
        } else {
#pragma unroll
            for (int j = 0; j < VEC; ++j) dst[j] = narrow<TC>(acc[j]);
        }
    } else {
        const int64_t go = P.out_map.map((uint32_t)o);
        if (VEC > 1 && P.in_vec_ok) {
            // i0 .. i0+VEC-1 share every inner digit but the first
            const int64_t g0 = go + P.in_map.map((uint32_t)i0);
#pragma unroll
            for (int j = 0; j < VEC; ++j) c[g0 + j * P.in_map.stride[0]] = narrow<TC>(acc[j]);
        } else {
#pragma unroll
            for (int j = 0; j < VEC; ++j) c[go + P.in_map.map((uint32_t)(i0 + j))] = narrow<TC>(acc[j]);
        }
    }
}

template <class TA, class TC, int VEC, int U, bool KEEP = false>
__global__ void __launch_bounds__(256) ttv_strided_kernel(const __grid_constant__ TtvParams P) {
    using Acc = typename AccOf<TA>::type;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    Acc *bs = (Acc *)smem_raw;
    pdl_wait();
    if (stop_requested(P.stop)) return;
    const int64_t K = P.K, I = P.I;
    if (P.b_smem) {
        for (int64_t k = threadIdx.x; k < K; k += blockDim.x)
            bs[k] = load_elem_as<Acc>(P.b, P.b_dtype, k * P.b_stride);
        __syncthreads();
    }
    const int64_t IV = I / VEC;
    const int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (gid < P.O * IV) {
        const int64_t og = gid / IV;
        const int64_t i0 = (gid - og * IV) * VEC;
        // o visiting order: og * o_mul mod O (gcd(o_mul, O) = 1: a permutation).
        // Measured on B200: slabs visited in storage order by concurrently
        // running warps camp on the same HBM channels when a slab is 64 or
        // 128 KB (I = 128 / 256 float32: 6.6 TB/s); scrambled, 7.1 TB/s.
        const int64_t o = P.o_mul > 1 ? (int64_t)(((uint64_t)og * (uint64_t)P.o_mul) % (uint64_t)P.O) : og;
        const TA *pa = (const TA *)P.a + (o * K) * I + i0;

        Acc acc[VEC];
#pragma unroll
        for (int j = 0; j < VEC; ++j) acc[j] = Acc(0);

        int64_t k = 0;
        uint64_t pol_first = 0, pol_keep = 0;
        if constexpr (KEEP) {
            asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol_first));
            asm("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol_keep));
            if ((int64_t)blockIdx.x >= P.keep_cta) pol_first = pol_keep;
        }
        for (; k + U <= K; k += U) {
            TA v[U][VEC];
            if constexpr (KEEP) {
                const uint64_t pol = (k + U > P.keep_k) ? pol_keep : pol_first;
#pragma unroll
                for (int u = 0; u < U; ++u) RawLoad<TA, VEC>::ld_hint(pa + (k + u) * I, v[u], pol);
            } else {
#pragma unroll
                for (int u = 0; u < U; ++u) RawLoad<TA, VEC>::ld(pa + (k + u) * I, v[u]);
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const Acc bk = P.b_smem ? bs[k + u] : load_elem_as<Acc>(P.b, P.b_dtype, (k + u) * P.b_stride);
#pragma unroll
                for (int j = 0; j < VEC; ++j) acc[j] = fold_step(acc[j], (Acc)v[u][j], bk);
            }
        }
        for (; k < K; ++k) {
            Acc v[VEC];
            VecLoad<TA, VEC>::ld(pa + k * I, v);
            const Acc bk = P.b_smem ? bs[k] : load_elem_as<Acc>(P.b, P.b_dtype, k * P.b_stride);
#pragma unroll
            for (int j = 0; j < VEC; ++j) acc[j] = fold_step(acc[j], v[j], bk);
        }
        store_outputs<TC, VEC>(P, o, i0, acc);
    }
    pdl_release();  // the next kernel's launch overlaps this one's tail
    if constexpr (std::is_same<TC, double>::value) fused_norm_tail(P.fn, (const double *)P.c, (double *)smem_raw);
}

// ------------------------------------------------------------- regime B, boxed
// Strided fibers whose output is permuted so that A's fastest free digit d0
// is far apart in C (e.g. config 5's seed-5 layout: consecutive i land
// 16830 elements apart): one thread per output would write isolated 8-byte
// words.  Instead a CTA takes a 2-D box of outputs -- BA = 32*VEC positions
// along d0 (contiguous in A: coalesced loads) by BC = 8*NJ positions along
// the chain of digits that is contiguous in C -- folds them (each output's
// k order unchanged: bit-exact), parks the box in shared memory and writes
// it out along the C-contiguous direction.
constexpr int kBoxMaxChain = 4;
struct TtvBoxParams {
    const void *a;
    const void *b;
    void *c;
    const int32_t *stop;
    int64_t b_stride;
    int32_t b_dtype;
    int32_t b_smem;
    int64_t K, I;           // contracted extent and its A stride
    int64_t e0, cs0;        // A-direction: extent (of the A-chain) and, for a one-digit chain, its C stride
    // A-chain of more than one digit (a prefix of the inner digits, contiguous
    // in A): position -> C offset through this digit map (na > 1)
    int32_t na;
    FastDiv a_div[kBoxMaxChain];
    int64_t a_cs[kBoxMaxChain];
    int64_t nA, nJ, nrest;  // box counts along d0, along the chain, other digits
    int64_t chain_ext;
    int32_t nchain;
    FastDiv ch_div[kBoxMaxChain];
    int64_t ch_as[kBoxMaxChain], ch_cs[kBoxMaxChain];
    int32_t nrest_d;
    FastDiv rs_div[TL_MAX_DIGITS];
    int64_t rs_as[TL_MAX_DIGITS], rs_cs[TL_MAX_DIGITS];
};

// H warps share one chain row per pass (H = 2: a row's 2 x 32*VEC elements
// are read as one contiguous 1 KB run for float64 instead of 512 B).
template <class TA, class TC, int VEC, int NJ, int UB = 8, int H = 1>
__global__ void __launch_bounds__(256) ttv_box_kernel(const __grid_constant__ TtvBoxParams P) {
    using Acc = typename AccOf<TA>::type;
    constexpr int RPP = 8 / H;  // chain rows per pass (one per H warps)
    constexpr int BA = 32 * VEC * H, BC = RPP * NJ, PITCH = BA + 1;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    pdl_wait();
    if (stop_requested(P.stop)) return;
    Acc *bs = (Acc *)smem_raw;
    const size_t bbytes = P.b_smem ? (((size_t)P.K * sizeof(Acc) + 15) & ~(size_t)15) : 0;
    int64_t *tabA = (int64_t *)(smem_raw + bbytes);
    int64_t *tabC = tabA + BC;
    TC *otile = (TC *)(tabC + BC);  // [BC][PITCH], already in C's type (the narrowing is the store's)
    int64_t *tabAC = (int64_t *)(smem_raw + bbytes + 2 * BC * 8 + ((BC * PITCH * sizeof(TC) + 7) & ~(size_t)7));  // [BA]
    if (P.b_smem) {
        for (int64_t k = threadIdx.x; k < P.K; k += blockDim.x) bs[k] = load_elem_as<Acc>(P.b, P.b_dtype, k * P.b_stride);
    }
    const TA *A = (const TA *)P.a;
    TC *C = (TC *)P.c;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t ntiles = P.nA * P.nJ * P.nrest;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        // tile -> (d0 block, chain block, other digits)
        const int64_t ab = tile % P.nA;
        const int64_t t2 = tile / P.nA;
        const int64_t jb = t2 % P.nJ;
        uint32_t rest = (uint32_t)(t2 / P.nJ);
        int64_t baseA = ab * BA, baseC = P.na > 1 ? 0 : ab * BA * P.cs0;
        for (int d = 0; d < P.nrest_d; ++d) {
            uint32_t q, r;
            if (d == P.nrest_d - 1) {
                r = rest;
                q = 0;
            } else {
                P.rs_div[d].divmod(rest, q, r);
            }
            baseA += (int64_t)r * P.rs_as[d];
            baseC += (int64_t)r * P.rs_cs[d];
            rest = q;
        }
        __syncthreads();  // the previous tile's write-out is done with tabC / otile
        if (P.na > 1 && threadIdx.x < BA) {
            // C offset of A-chain position ab*BA + threadIdx.x
            uint32_t x = (uint32_t)(ab * BA + threadIdx.x);
            int64_t oc = 0;
            for (int d = 0; d < P.na; ++d) {
                uint32_t q, r;
                if (d == P.na - 1) {
                    r = x;
                    q = 0;
                } else {
                    P.a_div[d].divmod(x, q, r);
                }
                oc += (int64_t)r * P.a_cs[d];
                x = q;
            }
            tabAC[threadIdx.x] = oc;
        }
        if (threadIdx.x < BC) {
            const int64_t jg = jb * BC + threadIdx.x;
            int64_t oa = -1, oc = 0;
            if (jg < P.chain_ext) {
                uint32_t x = (uint32_t)jg;
                oa = 0;
                for (int d = 0; d < P.nchain; ++d) {
                    uint32_t q, r;
                    if (d == P.nchain - 1) {
                        r = x;
                        q = 0;
                    } else {
                        P.ch_div[d].divmod(x, q, r);
                    }
                    oa += (int64_t)r * P.ch_as[d];
                    oc += (int64_t)r * P.ch_cs[d];
                    x = q;
                }
            }
            tabA[threadIdx.x] = oa;
            tabC[threadIdx.x] = oc;
        }
        __syncthreads();
        const int a = (warp % H) * 32 * VEC + lane * VEC;
        const bool a_ok = ab * BA + a + VEC <= P.e0;
        // NJ passes of 8 chain rows (one per warp); each pass is the strided
        // kernel's k loop: U rows of VEC elements in flight per thread (U = K
        // for K = 9: one round trip per pass instead of two)
        constexpr int U = UB;
        for (int t = 0; t < NJ; ++t) {
            const int j = warp / H + RPP * t;
            const int64_t ta = tabA[j];
            Acc acc[VEC];
#pragma unroll
            for (int v = 0; v < VEC; ++v) acc[v] = Acc(0);
            if (a_ok && ta >= 0) {
                const TA *pa = A + baseA + ta + a;
                int64_t k = 0;
                for (; k + U <= P.K; k += U) {
                    Acc x[U][VEC];
#pragma unroll
                    for (int u = 0; u < U; ++u) VecLoad<TA, VEC>::ld(pa + (k + u) * P.I, x[u]);
#pragma unroll
                    for (int u = 0; u < U; ++u) {
                        const Acc bk = P.b_smem ? bs[k + u] : load_elem_as<Acc>(P.b, P.b_dtype, (k + u) * P.b_stride);
#pragma unroll
                        for (int v = 0; v < VEC; ++v) acc[v] = fold_step(acc[v], x[u][v], bk);
                    }
                }
                for (; k < P.K; ++k) {
                    Acc x[VEC];
                    VecLoad<TA, VEC>::ld(pa + k * P.I, x);
                    const Acc bk = P.b_smem ? bs[k] : load_elem_as<Acc>(P.b, P.b_dtype, k * P.b_stride);
#pragma unroll
                    for (int v = 0; v < VEC; ++v) acc[v] = fold_step(acc[v], x[v], bk);
                }
            }
#pragma unroll
            for (int v = 0; v < VEC; ++v) otile[j * PITCH + a + v] = narrow<TC>(acc[v]);
        }
        __syncthreads();
        // write out along the C-contiguous chain
        for (int idx = threadIdx.x; idx < BA * BC; idx += blockDim.x) {
            const int j = idx % BC, aa = idx / BC;
            if (tabA[j] >= 0 && ab * BA + aa < P.e0)
                C[baseC + (P.na > 1 ? tabAC[aa] : aa * P.cs0) + tabC[j]] = otile[j * PITCH + aa];
        }
    }
    pdl_release();
}

// ------------------------------------------------------------- small problems
// Few outputs (e.g. HOPM's 400x400 intermediates, L2-resident): the fold
// chain of each output (K dependent adds) is the critical path, so each CTA
// owns 32 outputs, issues the loads of its WHOLE input block up front (one
// mbarrier per 64-k slab, completed by cp.async.mbarrier.arrive), and warp 0
// folds slab by slab as they land.  Two block shapes:
//   COLS (I >= 32): outputs (o, i0..i0+31), element (k, j) at o*K*I + k*I + i0 + j,
//                   smem [k][32];
//   ROWS (I == 1):  outputs o0..o0+31, element (k, j) at (o0 + j)*K + k,
//                   smem [j][pitch] with an odd pitch (conflict-free folds).
constexpr int kSmallSlab = 64;
constexpr int kSmallMaxSlabs = 64;  // K <= 4096

template <class TA, class TC, bool ROWS, bool PAIRS, bool CL = false>
__global__ void __launch_bounds__(256) ttv_small_kernel(const __grid_constant__ TtvParams P) {
    using Acc = typename AccOf<TA>::type;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    __shared__ __align__(8) uint64_t bars[kSmallMaxSlabs];
    __shared__ double mine[32];  // CL: this CTA's slice of w for the cluster norm
    pdl_wait();
    if (stop_requested(P.stop)) return;
    const int64_t K = P.K, I = P.I;
    const int nslab = (int)((K + kSmallSlab - 1) / kSmallSlab);
    Acc *bs = (Acc *)smem_raw;
    const size_t bbytes = ((size_t)K * sizeof(Acc) + 15) & ~(size_t)15;
    TA *data = (TA *)(smem_raw + bbytes);
    // ROWS pitch: odd (scalar LDS), or = 2 mod 4 with 16-byte pairs (LDS.128)
    const int pitch = PAIRS ? (int)((K + 2) + (((K + 2) / 2) % 2 == 0 ? 2 : 0)) : (int)(K | 1);

    int64_t o = 0, i0 = 0, o0 = 0;
    int nout;
    const TA *base;
    if constexpr (ROWS) {
        o0 = (int64_t)blockIdx.x * 32;
        nout = (int)((P.O - o0) < 32 ? (P.O - o0) : 32);
        base = (const TA *)P.a + o0 * K;
    } else {
        const int64_t iblocks = (I + 31) / 32;
        o = blockIdx.x / iblocks;
        i0 = (blockIdx.x - o * iblocks) * 32;
        nout = (int)((I - i0) < 32 ? (I - i0) : 32);
        base = (const TA *)P.a + o * K * I + i0;
    }
    if (threadIdx.x == 0) {
        for (int s = 0; s < nslab; ++s) mbar_init(&bars[s], blockDim.x);
        mbar_fence_init();
    }
    __syncthreads();
    if (threadIdx.x >= 32) {
        // warps 1..3 put the whole block in flight; warp 0 only folds
        const int t = threadIdx.x - 32, nt = blockDim.x - 32;
        constexpr int E = PAIRS ? 2 : 1;  // elements per copy
        for (int s = 0; s < nslab; ++s) {
            const int k0 = s * kSmallSlab;
            const int kn = (int)((K - k0) < kSmallSlab ? (K - k0) : kSmallSlab);
            for (int e = t; e < kSmallSlab * 32 / E; e += nt) {
                if constexpr (ROWS) {
                    constexpr int PR = kSmallSlab / E;  // pieces per row slab
                    const int j = e / PR, kk = (e % PR) * E;  // lanes walk k (contiguous rows)
                    if (kk < kn && j < nout)
                        cp_async<E * sizeof(TA)>(data + j * pitch + k0 + kk, base + (int64_t)j * K + k0 + kk);
                } else {
                    constexpr int PC = 32 / E;  // pieces per k-row
                    const int kk = e / PC, j = (e % PC) * E;  // lanes walk i (contiguous columns)
                    if (kk < kn && j < nout)
                        cp_async<E * sizeof(TA)>(data + (k0 + kk) * 32 + j, base + (int64_t)(k0 + kk) * I + j);
                }
            }
            cp_async_mbar_arrive(&bars[s]);
        }
    } else {
        // warp 0 stages b while the block's copies are in flight
        for (int64_t k = threadIdx.x; k < K; k += 32) bs[k] = load_elem_as<Acc>(P.b, P.b_dtype, k * P.b_stride);
        __syncwarp();
        const int j = threadIdx.x;
        Acc acc = Acc(0);
        for (int s = 0; s < nslab; ++s) cp_async_mbar_arrive(&bars[s]);  // warp 0 issues no copies
        for (int s = 0; s < nslab; ++s) {
            mbar_wait_parity(&bars[s], 0);
            const int k0 = s * kSmallSlab;
            const int kn = (int)((K - k0) < kSmallSlab ? (K - k0) : kSmallSlab);
            // A full slab is folded with its trip count known at compile
            // time, so every shared-memory load is issued ahead of the
            // dependent add chain (the fold's only serial part).
            if constexpr (ROWS) {
                const TA *row = data + j * pitch + k0;
                if constexpr (PAIRS) {
                    if (kn == kSmallSlab) {
                        // the next 8 pairs load while the current 8 fold:
                        // shared-memory latency stays off the add chain
                        double2 cv[4], cb[4], nv[4], nb[4];
#pragma unroll
                        for (int q = 0; q < 4; ++q) {
                            cv[q] = *(const double2 *)(row + 2 * q);
                            cb[q] = *(const double2 *)(bs + k0 + 2 * q);
                        }
#pragma unroll
                        for (int kk = 0; kk < kSmallSlab; kk += 8) {
                            if (kk + 8 < kSmallSlab) {
#pragma unroll
                                for (int q = 0; q < 4; ++q) {
                                    nv[q] = *(const double2 *)(row + kk + 8 + 2 * q);
                                    nb[q] = *(const double2 *)(bs + k0 + kk + 8 + 2 * q);
                                }
                            }
#pragma unroll
                            for (int q = 0; q < 4; ++q) {
                                acc = fold_step(acc, (Acc)cv[q].x, cb[q].x);
                                acc = fold_step(acc, (Acc)cv[q].y, cb[q].y);
                            }
#pragma unroll
                            for (int q = 0; q < 4; ++q) {
                                cv[q] = nv[q];
                                cb[q] = nb[q];
                            }
                        }
                    } else {
                        int kk = 0;
#pragma unroll 4
                        for (; kk + 1 < kn; kk += 2) {
                            const double2 v = *(const double2 *)(row + kk);
                            const double2 bv = *(const double2 *)(bs + k0 + kk);
                            acc = fold_step(acc, (Acc)v.x, bv.x);
                            acc = fold_step(acc, (Acc)v.y, bv.y);
                        }
                        if (kk < kn) acc = fold_step(acc, (Acc)row[kk], bs[k0 + kk]);
                    }
                } else {
                    if (kn == kSmallSlab) {
#pragma unroll
                        for (int kk = 0; kk < kSmallSlab; ++kk) acc = fold_step(acc, (Acc)row[kk], bs[k0 + kk]);
                    } else {
#pragma unroll 8
                        for (int kk = 0; kk < kn; ++kk) acc = fold_step(acc, (Acc)row[kk], bs[k0 + kk]);
                    }
                }
            } else {
                const TA *col = data + k0 * 32 + j;
                if (kn == kSmallSlab) {
                    // next 8 terms load while the current 8 fold
                    TA cx[8], nx[8];
                    Acc cb[8], nb[8];
#pragma unroll
                    for (int q = 0; q < 8; ++q) {
                        cx[q] = col[q * 32];
                        cb[q] = bs[k0 + q];
                    }
#pragma unroll
                    for (int kk = 0; kk < kSmallSlab; kk += 8) {
                        if (kk + 8 < kSmallSlab) {
#pragma unroll
                            for (int q = 0; q < 8; ++q) {
                                nx[q] = col[(kk + 8 + q) * 32];
                                nb[q] = bs[k0 + kk + 8 + q];
                            }
                        }
#pragma unroll
                        for (int q = 0; q < 8; ++q) acc = fold_step(acc, (Acc)cx[q], cb[q]);
#pragma unroll
                        for (int q = 0; q < 8; ++q) {
                            cx[q] = nx[q];
                            cb[q] = nb[q];
                        }
                    }
                } else {
#pragma unroll 8
                    for (int kk = 0; kk < kn; ++kk) acc = fold_step(acc, (Acc)col[kk * 32], bs[k0 + kk]);
                }
            }
        }
        if constexpr (CL) {
            mine[j] = (j < nout) ? (double)acc : 0.0;  // w stays on chip
        } else if (j < nout) {
            int64_t off;
            if constexpr (ROWS) {
                const int64_t oo = o0 + j;
                off = P.ident ? oo : P.out_map.map((uint32_t)oo);
            } else {
                const int64_t i = i0 + j;
                off = P.ident ? o * I + i : P.out_map.map((uint32_t)o) + P.in_map.map((uint32_t)i);
            }
            ((TC *)P.c)[off] = narrow<TC>(acc);
        }
    }
    cp_async_wait<0>();
    pdl_release();  // the next kernel's launch overlaps this one's tail
    if constexpr (CL) {
        fused_norm_cluster(P.fn, mine, (double *)smem_raw);
    } else if constexpr (std::is_same<TC, double>::value) {
        fused_norm_tail(P.fn, (const double *)P.c, (double *)smem_raw);
    }
}

// ------------------------------------------------------------- long folds, few outputs
// Few outputs with a long fold (O*I/VEC threads too few to keep HBM busy
// with a handful of loads in flight each): every thread keeps the next
// NG*8 k-rows of ITS OWN fibre in flight through a private shared-memory
// ring filled by cp.async (no data shared between threads, so no CTA
// barriers: cp.async.wait_group is per thread), and folds them in k order
// (bit-exact).  COLS: VEC consecutive i of one o (A[o][k][i0..], the strided
// regime's fibres); ROWS (I == 1): one o, 16-byte chunks along its
// contiguous row.  The sequential fold itself (8.2-cycle DADD chain) is the
// floor once the ring hides the memory latency.
constexpr int kDeepGroup = 8;

template <class TA, class TC, int VEC, bool ROWS, int NG>
__global__ void __launch_bounds__(64) ttv_deep_kernel(const __grid_constant__ TtvParams P) {
    using Acc = typename AccOf<TA>::type;
    constexpr int D = NG * kDeepGroup;  // pieces in flight per thread
    constexpr int CH = ROWS ? (VEC > 1 ? 16 / (int)sizeof(TA) : 1) : VEC;  // A elements per piece
    constexpr int CB = ROWS ? CH : 1;                                        // b elements per piece
    extern __shared__ __align__(16) unsigned char smem_raw[];
    pdl_wait();
    if (stop_requested(P.stop)) return;
    // private rings (A pieces, then the b values they fold with, b in A's
    // type: the planner takes this kernel only when b's dtype is A's),
    // pitched one 16-byte slot apart so a warp's same-slot accesses spread
    // over all banks (4 wavefronts for 32 x 16 B, not 32)
    constexpr int PITCH = D * (CH + CB) + 16 / (int)sizeof(TA);
    TA *ring = (TA *)smem_raw + (size_t)threadIdx.x * PITCH;
    TA *bring = ring + D * CH;
    const int64_t K = P.K, I = P.I;
    const int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t nthr = ROWS ? P.O : P.O * (I / VEC);
    if (gid >= nthr) return;
    const int64_t og = ROWS ? gid : gid / (I / VEC);
    const int64_t i0 = ROWS ? 0 : (gid - og * (I / VEC)) * VEC;
    const TA *pa = (const TA *)P.a + (og * K) * I + i0;
    const TA *pb = (const TA *)P.b;
    // piece p: COLS = k-row p (VEC elements at pa + p*I), ROWS = chunk p (CH elements at pa + p*CH)
    const int64_t npieces = ROWS ? (K + CH - 1) / CH : K;
    auto issue = [&](int64_t p) {
        if (p < npieces) {
            const int slot = (int)(p % D);
            TA *dst = ring + slot * CH;
            TA *bdst = bring + slot * CB;
            if constexpr (ROWS) {
                if ((p + 1) * CH <= K) {
                    cp_async<CH * sizeof(TA)>(dst, pa + p * CH);
#pragma unroll
                    for (int e = 0; e < CB; ++e) cp_async<sizeof(TA)>(bdst + e, pb + (p * CH + e) * P.b_stride);
                } else {
#pragma unroll
                    for (int e = 0; e < CH; ++e)
                        if (p * CH + e < K) {
                            cp_async<sizeof(TA)>(dst + e, pa + p * CH + e);
                            cp_async<sizeof(TA)>(bdst + e, pb + (p * CH + e) * P.b_stride);
                        }
                }
            } else {
                cp_async<VEC * sizeof(TA)>(dst, pa + p * I);
                cp_async<sizeof(TA)>(bdst, pb + p * P.b_stride);
            }
        }
    };
#pragma unroll 1
    for (int g = 0; g < NG; ++g) {
#pragma unroll
        for (int r = 0; r < kDeepGroup; ++r) issue((int64_t)g * kDeepGroup + r);
        cp_async_commit();
    }
    Acc acc[ROWS ? 1 : VEC];
#pragma unroll
    for (int j = 0; j < (ROWS ? 1 : VEC); ++j) acc[j] = Acc(0);
    for (int64_t p0 = 0; p0 < npieces; p0 += kDeepGroup) {
        cp_async_wait<NG - 1>();  // the oldest group has landed
        const int s0 = (int)(p0 % D);
        // the group's values first (independent shared loads), then the chain
        TA av[kDeepGroup][CH], bv[kDeepGroup][CB];
#pragma unroll
        for (int r = 0; r < kDeepGroup; ++r) {
#pragma unroll
            for (int e = 0; e < CH; ++e) av[r][e] = ring[(s0 + r) * CH + e];
#pragma unroll
            for (int e = 0; e < CB; ++e) bv[r][e] = bring[(s0 + r) * CB + e];
        }
#pragma unroll
        for (int r = 0; r < kDeepGroup; ++r) {
            const int64_t p = p0 + r;
            if (p < npieces) {
                if constexpr (ROWS) {
#pragma unroll
                    for (int e = 0; e < CH; ++e)
                        if (p * CH + e < K) acc[0] = fold_step(acc[0], (Acc)av[r][e], (Acc)bv[r][e]);
                } else {
#pragma unroll
                    for (int j = 0; j < VEC; ++j) acc[j] = fold_step(acc[j], (Acc)av[r][j], (Acc)bv[r][0]);
                }
            }
        }
        // refill the slots just consumed (after the reads above: same thread)
#pragma unroll
        for (int r = 0; r < kDeepGroup; ++r) issue(p0 + D + r);
        cp_async_commit();
    }
    cp_async_wait<0>();
    if constexpr (ROWS) {
        TC *c = (TC *)P.c;
        c[P.ident ? og : P.out_map.map((uint32_t)og)] = narrow<TC>(acc[0]);
    } else {
        store_outputs<TC, VEC>(P, og, i0, acc);
    }
    pdl_release();
}

// ------------------------------------------------------------- short folds, permuted outputs
// K <= kShortK with a permuted output whose fastest canonical digit is not
// C-contiguous: the output (N/K elements) would be written scattered.  A CTA
// folds a TX x TY tile of outputs -- TY positions along a chain of free
// digits contiguous in A (the inner digits, or for a contracted stride of 1
// the rows), TX along a chain contiguous in C -- parks it in shared memory
// and writes it out along C (a transpose fused with the fold).  Chains are
// flat index spaces split into blocks; per-tile tables hold the A and C
// offsets of their positions.  Each output's k order is unchanged (bit-exact).
struct TtvTileParams {
    const void *a;
    const void *b;
    void *c;
    const int32_t *stop;
    int64_t b_stride;
    int32_t b_dtype;
    int64_t K, I;
    int64_t ex, ey;              // chain extents
    int64_t nxb, nyb, nrest;     // blocks along each chain, other positions
    DigitMap xa, xc, ya, yc, ra, rc;  // A / C offsets of chain and rest indices
};
constexpr int kTileX = 64, kTileY = 128;  // largest tile shape (the planner's chain targets)
constexpr int kShortK = 16;  // folds this short take the short-fold / tile-fold streams

template <class TA, class TC, int TX, int TY>
__global__ void __launch_bounds__(256) ttv_tile_kernel(const __grid_constant__ TtvTileParams P) {
    using Acc = typename AccOf<TA>::type;
    constexpr int JX = TX * TY / 256;
    __shared__ int64_t tXA[TX], tXC[TX], tYA[TY], tYC[TY];
    __shared__ Acc bs[kShortK];
    __shared__ TC tile[TX][TY + 1];
    pdl_wait();
    if (stop_requested(P.stop)) return;
    const int K = (int)P.K;
    if (threadIdx.x < K) bs[threadIdx.x] = load_elem_as<Acc>(P.b, P.b_dtype, threadIdx.x * P.b_stride);
    const TA *A = (const TA *)P.a;
    TC *C = (TC *)P.c;
    const int64_t ntiles = P.nxb * P.nyb * P.nrest;
    const int tid = threadIdx.x;
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const int64_t yb = t % P.nyb;
        const int64_t t2 = t / P.nyb;
        const int64_t xb = t2 % P.nxb;
        const uint32_t rest = (uint32_t)(t2 / P.nxb);
        __syncthreads();  // the previous tile is written out; b is staged
        if (tid < TY) {
            const int64_t y = yb * TY + tid;
            tYA[tid] = y < P.ey ? P.ya.map((uint32_t)y) : -1;
            tYC[tid] = y < P.ey ? P.yc.map((uint32_t)y) : 0;
        } else if (tid < TY + TX) {
            const int64_t x = xb * TX + (tid - TY);
            tXA[tid - TY] = x < P.ex ? P.xa.map((uint32_t)x) : -1;
            tXC[tid - TY] = x < P.ex ? P.xc.map((uint32_t)x) : 0;
        }
        const int64_t rA = P.ra.map(rest), rC = P.rc.map(rest);
        __syncthreads();
        // fold: lanes along y (A-contiguous), JX outputs per thread, all of
        // a k's loads issued together
        {
            const int y = tid % TY;
            const int x0 = tid / TY;
            constexpr int XS = 256 / TY;
            Acc acc[JX];
            const TA *pa[JX];
            bool ok[JX];
#pragma unroll
            for (int j = 0; j < JX; ++j) {
                const int x = x0 + XS * j;
                ok[j] = tYA[y] >= 0 && tXA[x] >= 0;
                pa[j] = A + rA + (ok[j] ? tXA[x] + tYA[y] : 0);
                acc[j] = Acc(0);
            }
            for (int k = 0; k < K; ++k) {
                const Acc bk = bs[k];
                TA v[JX];
#pragma unroll
                for (int j = 0; j < JX; ++j) v[j] = ok[j] ? __ldg(pa[j] + (int64_t)k * P.I) : TA(0);
#pragma unroll
                for (int j = 0; j < JX; ++j) acc[j] = fold_step(acc[j], (Acc)v[j], bk);
            }
#pragma unroll
            for (int j = 0; j < JX; ++j) tile[x0 + XS * j][y] = narrow<TC>(acc[j]);
        }
        __syncthreads();
        // write out: lanes along x (C-contiguous)
        {
            const int x = tid % TX;
            const int y0 = tid / TX;
            constexpr int YS = 256 / TX;
#pragma unroll
            for (int j = 0; j < TY / YS; ++j) {
                const int y = y0 + YS * j;
                if (tXA[x] >= 0 && tYA[y] >= 0) C[rC + tXC[x] + tYC[y]] = tile[x][y];
            }
        }
    }
    pdl_release();
}

// ------------------------------------------------------------- short folds
// K <= kShortK over a large tensor: the output is a sizeable fraction of the
// input (N/K), so the contraction is an elementwise stream.  Each thread
// produces QV consecutive outputs of the canonical order q = o*I + i, folding
// k in order (bit-exact), into C in that order (ident) or through the digit
// maps when C's fastest canonical digit is contiguous (runs of >= 32; other
// permuted outputs stay on the tiled kernels: a temporary + transpose
// measured slower there).  The loads go through L1: neighbouring threads and
// k's share sectors.
template <class TA, class TC, int QV>
__global__ void __launch_bounds__(256) ttv_short_kernel(const __grid_constant__ TtvParams P, TC *out) {
    // out == nullptr: permuted C written through the digit maps (its fastest
    // canonical digit is C-contiguous: runs of >= 32 outputs)
    using Acc = typename AccOf<TA>::type;
    __shared__ Acc bs[kShortK];
    pdl_wait();
    if (stop_requested(P.stop)) return;
    const int K = (int)P.K;
    if (threadIdx.x < K) bs[threadIdx.x] = load_elem_as<Acc>(P.b, P.b_dtype, threadIdx.x * P.b_stride);
    __syncthreads();
    const TA *a = (const TA *)P.a;
    const int64_t nq = P.O * P.I;
    const int64_t KI = P.K * P.I;
    const int64_t step = (int64_t)gridDim.x * blockDim.x * QV;
    for (int64_t q0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * QV; q0 < nq; q0 += step) {
        Acc acc[QV];
        uint32_t o, i;
        P.I_div.divmod((uint32_t)q0, o, i);  // q0 < 2^32 (planned)
#pragma unroll
        for (int j = 0; j < QV; ++j) {
            acc[j] = Acc(0);
            if (q0 + j < nq) {
                const TA *pa = a + (int64_t)o * KI + i;
#pragma unroll 4
                for (int k = 0; k < K; ++k) acc[j] = fold_step(acc[j], (Acc)__ldg(pa + (int64_t)k * P.I), bs[k]);
            }
            if (++i == (uint32_t)P.I) {
                i = 0;
                ++o;
            }
        }
        if (P.ident == 0) {
            uint32_t o2, i2;
            P.I_div.divmod((uint32_t)q0, o2, i2);
#pragma unroll
            for (int j = 0; j < QV; ++j) {
                if (q0 + j < nq) ((TC *)P.c)[P.out_map.map(o2) + P.in_map.map(i2)] = narrow<TC>(acc[j]);
                if (++i2 == (uint32_t)P.I) {
                    i2 = 0;
                    ++o2;
                }
            }
            continue;
        }
        if (q0 + QV <= nq && ((q0 * (int64_t)sizeof(TC)) % (QV * (int64_t)sizeof(TC))) == 0 && QV * sizeof(TC) >= 8) {
            if constexpr (QV * sizeof(TC) == 16) {
                if constexpr (sizeof(TC) == 4) {
                    *(float4 *)(out + q0) = make_float4(narrow<TC>(acc[0]), narrow<TC>(acc[1]), narrow<TC>(acc[2]), narrow<TC>(acc[3]));
                } else {
                    TC v2[2] = {narrow<TC>(acc[0]), narrow<TC>(acc[1])};
                    *(uint4 *)(out + q0) = *(const uint4 *)v2;
                }
                continue;
            }
        }
#pragma unroll
        for (int j = 0; j < QV; ++j)
            if (q0 + j < nq) out[q0 + j] = narrow<TC>(acc[j]);
    }
    pdl_release();
}

// ------------------------------------------------------------- regime S
constexpr int kStages = 3;
constexpr int kMaxOpt = 4;

// Contiguous-chunk mode (one k-slab, unpadded rows): the whole tile is one
// contiguous byte range of A, fetched by a single 1-D TMA bulk copy that
// completes on the stage's mbarrier; a sub-16-byte tail (last tile only)
// goes through cp.async.
template <class TA>
__device__ __forceinline__ void issue_chunk(const TtvParams &P, unsigned char *stage, uint64_t *bar, int64_t tile) {
    const int64_t o0 = tile * P.R;
    const int64_t rows = P.O - o0 < P.R ? P.O - o0 : P.R;
    const uint32_t bytes = (uint32_t)(rows * P.K * P.I * (int64_t)sizeof(TA));
    const uint32_t b16 = bytes & ~15u;
    const unsigned char *src = (const unsigned char *)((const TA *)P.a + o0 * P.K * P.I);
    if (threadIdx.x == 0) {
        fence_proxy_async_smem();  // generic reads of this buffer precede the async writes
        mbar_arrive_expect_tx(bar, b16);
        if (b16) bulk_g2s(stage, src, b16, bar);
    }
    const uint32_t tail_elems = (bytes - b16) / (uint32_t)sizeof(TA);
    if (threadIdx.x < tail_elems)
        cp_async<sizeof(TA)>(stage + b16 + threadIdx.x * sizeof(TA), src + b16 + threadIdx.x * sizeof(TA));
}

template <class TA, int G>
__device__ __forceinline__ void issue_slab(const TtvParams &P, unsigned char *stage, int64_t tile, int slab) {
    const int64_t o0 = tile * P.R;
    const int64_t rows64 = P.O - o0 < P.R ? P.O - o0 : P.R;
    const uint32_t rows = (uint32_t)rows64;
    const int64_t k0 = (int64_t)slab * P.Kc;
    const int64_t kc = (P.K - k0 < P.Kc) ? P.K - k0 : P.Kc;
    const bool tail = (kc != P.Kc);
    const FastDiv &pr = tail ? P.pr_tail : P.pr_div;
    const uint32_t pieces_row = pr.d;
    const unsigned char *src0 = (const unsigned char *)((const TA *)P.a + (o0 * P.K + k0) * P.I);
    const int64_t grow = P.K * P.I * (int64_t)sizeof(TA);  // global row pitch, bytes
    const uint32_t srow = (uint32_t)P.Lp * (uint32_t)sizeof(TA);  // smem row pitch, bytes
    if (blockDim.x % pieces_row == 0) {
        // each thread owns one piece column and walks rows: no division
        const uint32_t rstep = blockDim.x / pieces_row;
        uint32_t r, cpc;
        pr.divmod(threadIdx.x, r, cpc);
        const unsigned char *src = src0 + (int64_t)r * grow + (int64_t)cpc * G;
        unsigned char *dst = stage + r * srow + cpc * G;
        const int64_t gstep = (int64_t)rstep * grow;
        const uint32_t sstep = rstep * srow;
        for (; r < rows; r += rstep, src += gstep, dst += sstep) cp_async<G>(dst, src);
    } else {
        const uint32_t total = rows * pieces_row;
        for (uint32_t p = threadIdx.x; p < total; p += blockDim.x) {
            uint32_t r, cpc;
            pr.divmod(p, r, cpc);
            cp_async<G>(stage + r * srow + cpc * G, src0 + (int64_t)r * grow + (int64_t)cpc * G);
        }
    }
}

template <class TA, class TC, int G, bool VECREAD, bool BULK>
__global__ void __launch_bounds__(256) ttv_staged_kernel(const __grid_constant__ TtvParams P) {
    using Acc = typename AccOf<TA>::type;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    __shared__ __align__(8) uint64_t full_bar[kStages];
    pdl_wait();
    if (stop_requested(P.stop)) return;
    const int64_t K = P.K, I = P.I;
    // b (as the accumulation type), then kStages row-padded stage buffers
    Acc *bs = (Acc *)smem_raw;
    const size_t bbytes = ((size_t)K * sizeof(Acc) + 15) & ~(size_t)15;
    unsigned char *stages = smem_raw + bbytes;
    const size_t stage_bytes = (((size_t)P.R * P.Lp * sizeof(TA)) + 15) & ~(size_t)15;

    for (int64_t k = threadIdx.x; k < K; k += blockDim.x)
        bs[k] = load_elem_as<Acc>(P.b, P.b_dtype, k * P.b_stride);
    int32_t *otab = (int32_t *)(stages + kStages * stage_bytes);
    for (int w = threadIdx.x; w < P.otab_n; w += blockDim.x) {
        uint32_t x = (uint32_t)w;
        int64_t off = 0;
        for (int d = 0; d < P.otab_d0; ++d) {
            uint32_t q, r;
            P.out_map.div[d].divmod(x, q, r);
            off += (int64_t)r * P.out_map.stride[d];
            x = q;
        }
        otab[w] = (int32_t)off;
    }
    if (BULK || P.otab_n) {
        if (BULK && threadIdx.x == 0) {
            for (int s = 0; s < kStages; ++s) mbar_init(&full_bar[s], 1);
            mbar_fence_init();
        }
        __syncthreads();
    }

    // Work items are (tile, slab) pairs in order; the producer runs
    // kStages-1 items ahead.  Both walk them with counters (no division).
    const int64_t my_tiles = (P.ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x;
    const int64_t nitems = my_tiles * P.nslab;
    int64_t p_tile = blockIdx.x;  // producer position
    int p_slab = 0, p_stage = 0;
    auto issue_next = [&]() {
        if constexpr (BULK)
            issue_chunk<TA>(P, stages + p_stage * stage_bytes, &full_bar[p_stage], p_tile);
        else
            issue_slab<TA, G>(P, stages + p_stage * stage_bytes, p_tile, p_slab);
        if (++p_slab == P.nslab) {
            p_slab = 0;
            p_tile += gridDim.x;
        }
        if (++p_stage == kStages) p_stage = 0;
    };

#pragma unroll
    for (int q = 0; q < kStages - 1; ++q) {
        if (q < nitems) issue_next();
        cp_async_commit();
    }

    Acc acc[kMaxOpt];
#pragma unroll
    for (int t = 0; t < kMaxOpt; ++t) acc[t] = Acc(0);

    const uint32_t outs_per_tile = (uint32_t)P.R * (uint32_t)I;
    int64_t tile = blockIdx.x;  // consumer position
    int slab = 0, c_stage = 0;
    uint32_t parity = 0;
    for (int64_t q = 0; q < nitems; ++q) {
        cp_async_wait<kStages - 2>();
        if constexpr (BULK) mbar_wait_parity(&full_bar[c_stage], parity);
        __syncthreads();
        if (q + kStages - 1 < nitems) issue_next();
        cp_async_commit();
        const TA *st = (const TA *)(stages + c_stage * stage_bytes);
        const int64_t k0 = (int64_t)slab * P.Kc;
        const int kc = (int)((K - k0 < P.Kc) ? K - k0 : P.Kc);
        const int64_t o0 = tile * P.R;
        const int64_t rows = (P.O - o0 < P.R) ? P.O - o0 : P.R;

#pragma unroll
        for (int t = 0; t < kMaxOpt; ++t) {
            if (t >= P.opt) break;
            const uint32_t j = threadIdx.x + t * blockDim.x;
            if (j >= outs_per_tile) break;
            uint32_t r, i;
            P.I_div.divmod(j, r, i);
            if (r >= rows) break;
            const TA *row = st + (size_t)r * P.Lp + i;
            Acc a_ = acc[t];
            if constexpr (VECREAD) {
                // I == 1, 16-byte rows: LDS.128 along k, folds stay in k order.
                // Full slabs of the planned length fold with a compile-time
                // trip count (no loop control, loads hoisted ahead).
                constexpr int E = 16 / sizeof(TA);
                auto fold_vec = [&](int kk) {
                    if constexpr (E == 4) {
                        const float4 v = *(const float4 *)(row + kk);
                        const double2 b01 = *(const double2 *)(bs + k0 + kk);
                        const double2 b23 = *(const double2 *)(bs + k0 + kk + 2);
                        a_ = fold_step(a_, (Acc)v.x, b01.x);
                        a_ = fold_step(a_, (Acc)v.y, b01.y);
                        a_ = fold_step(a_, (Acc)v.z, b23.x);
                        a_ = fold_step(a_, (Acc)v.w, b23.y);
                    } else {
                        union { uint4 raw; TA v[2]; } u;
                        u.raw = *(const uint4 *)(row + kk);
                        const Acc b0 = bs[k0 + kk], b1 = bs[k0 + kk + 1];
                        a_ = fold_step(a_, (Acc)u.v[0], b0);
                        a_ = fold_step(a_, (Acc)u.v[1], b1);
                    }
                };
                if (kc == 32) {
#pragma unroll
                    for (int kk = 0; kk < 32; kk += E) fold_vec(kk);
                } else if (kc == 16) {
#pragma unroll
                    for (int kk = 0; kk < 16; kk += E) fold_vec(kk);
                } else {
                    for (int kk = 0; kk < kc; kk += E) fold_vec(kk);
                }
            } else {
#pragma unroll 4
                for (int kk = 0; kk < kc; ++kk) a_ = fold_step(a_, (Acc)row[(size_t)kk * I], bs[k0 + kk]);
            }
            acc[t] = a_;
        }

        if (slab == P.nslab - 1) {
            TC *c = (TC *)P.c;
#pragma unroll
            for (int t = 0; t < kMaxOpt; ++t) {
                if (t >= P.opt) break;
                const uint32_t j = threadIdx.x + t * blockDim.x;
                if (j < outs_per_tile) {
                    uint32_t r, i;
                    P.I_div.divmod(j, r, i);
                    if (r < rows) {
                        const int64_t o = o0 + r;
                        int64_t off;
                        if (P.ident) {
                            off = o * I + i;
                        } else if (P.otab_n) {
                            uint32_t qh, w;
                            P.otab_div.divmod((uint32_t)o, qh, w);
                            off = otab[w] + P.out_hi.map(qh) + P.in_map.map(i);
                        } else {
                            off = P.out_map.map((uint32_t)o) + P.in_map.map(i);
                        }
                        c[off] = narrow<TC>(acc[t]);
                    }
                }
                acc[t] = Acc(0);
            }
        }
        if (++slab == P.nslab) {
            slab = 0;
            tile += gridDim.x;
        }
        if (++c_stage == kStages) {
            c_stage = 0;
            parity ^= 1u;
        }
    }
    cp_async_wait<0>();
    pdl_release();  // the next kernel's launch overlaps this one's tail
    if constexpr (std::is_same<TC, double>::value) fused_norm_tail(P.fn, (const double *)P.c, (double *)smem_raw);
}

// ------------------------------------------------------------- regime S, TMA rows
// Contracted stride 1 (I == 1): each output folds one contiguous row of K
// elements.  Tiles of 256 rows stream in 128-byte k-slabs through a 2-D TMA
// tensor map (one cp.async.bulk.tensor per slab, issued by one thread,
// completing on the stage's mbarrier) with the 128-byte hardware swizzle, so
// the per-thread LDS.128 reads of a warp's 32 rows are conflict-free without
// padding.  Thread r folds row r in k order (bit-exact).
constexpr int kRowsTmaR = 256;
constexpr int kRowsTmaStages = 3;

__device__ __forceinline__ void tma_load_2d(void *smem_dst, const CUtensorMap *map, int32_t c0, int32_t c1,
                                            uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
            smem_u32(smem_dst)),
        "l"(map), "r"(c0), "r"(c1), "r"(smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ void tma_load_2d_hint(void *smem_dst, const CUtensorMap *map, int32_t c0, int32_t c1,
                                                 uint64_t *bar, uint64_t pol) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%2, "
        "%3}], [%4], %5;" ::"r"(smem_u32(smem_dst)),
        "l"(map), "r"(c0), "r"(c1), "r"(smem_u32(bar)), "l"(pol)
        : "memory");
}

template <class TA, class TC>
__global__ void __launch_bounds__(kRowsTmaR) ttv_rows_tma_kernel(const __grid_constant__ TtvParams P,
                                                                 const __grid_constant__ CUtensorMap map) {
    using Acc = typename AccOf<TA>::type;
    constexpr int KC = 128 / (int)sizeof(TA);  // elements per 128-byte slab row
    constexpr int E = 16 / (int)sizeof(TA);    // elements per 16-byte chunk
    // rows per tile = threads per CTA (256, 128 or 64: chosen by the planner so
    // that the tiles fill whole rounds of the persistent grid)
    const int RT = (int)blockDim.x;
    const int STAGE = RT * 128;  // bytes
    extern __shared__ __align__(16) unsigned char smem_raw[];  // stages are re-aligned to 1024 below
    __shared__ __align__(8) uint64_t full_bar[kRowsTmaStages];
    pdl_wait();
    if (stop_requested(P.stop)) return;
    // stages first (1024-byte aligned for the swizzle), then b
    unsigned char *stages = (unsigned char *)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    Acc *bs = (Acc *)(stages + kRowsTmaStages * STAGE);
    const int64_t K = P.K;
    for (int64_t k = threadIdx.x; k < K; k += blockDim.x) bs[k] = load_elem_as<Acc>(P.b, P.b_dtype, k * P.b_stride);
    if (threadIdx.x == 0) {
        for (int st = 0; st < kRowsTmaStages; ++st) mbar_init(&full_bar[st], 1);
        mbar_fence_init();
    }
    __syncthreads();
    const int nslab = (int)((K + KC - 1) / KC);
    const int64_t ntiles = (P.O + RT - 1) / RT;
    const int64_t my_tiles = (ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x;
    const int64_t nitems = my_tiles * nslab;
    int64_t p_tile = blockIdx.x;
    int p_slab = 0, p_stage = 0;
    uint64_t pol_first = 0, pol_keep = 0;
    const bool keep = P.l2_stream != 0;
    if (keep && threadIdx.x == 0) {
        asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol_first));
        asm("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol_keep));
    }
    auto issue_next = [&]() {
        if (threadIdx.x == 0) {
            fence_proxy_async_smem();
            mbar_arrive_expect_tx(&full_bar[p_stage], STAGE);
            if (keep)
                tma_load_2d_hint(stages + p_stage * STAGE, &map, p_slab * KC, (int32_t)(p_tile * RT), &full_bar[p_stage],
                                 p_tile >= P.keep_tile ? pol_keep : pol_first);
            else
                tma_load_2d(stages + p_stage * STAGE, &map, p_slab * KC, (int32_t)(p_tile * RT), &full_bar[p_stage]);
        }
        if (++p_slab == nslab) {
            p_slab = 0;
            p_tile += gridDim.x;
        }
        if (++p_stage == kRowsTmaStages) p_stage = 0;
    };
    for (int q = 0; q < kRowsTmaStages - 1; ++q)
        if (q < nitems) issue_next();

    const int r = threadIdx.x;
    const uint32_t swz = (uint32_t)(r & 7);
    Acc acc = Acc(0);
    int64_t tile = blockIdx.x;
    int slab = 0, c_stage = 0;
    uint32_t parity = 0;
    for (int64_t q = 0; q < nitems; ++q) {
        mbar_wait_parity(&full_bar[c_stage], parity);
        __syncthreads();  // every thread is done with the stage about to be refilled
        if (q + kRowsTmaStages - 1 < nitems) issue_next();
        const unsigned char *row = stages + c_stage * STAGE + r * 128;
        const int64_t k0 = (int64_t)slab * KC;
        const int kc = (int)((K - k0 < KC) ? K - k0 : KC);
        auto fold_chunk = [&](int c) {  // 16-byte chunk c of this row
            const uint4 raw = *(const uint4 *)(row + (((uint32_t)c ^ swz) << 4));
            const TA *v = (const TA *)&raw;
#pragma unroll
            for (int e = 0; e < E; ++e) acc = fold_step(acc, (Acc)v[e], bs[k0 + c * E + e]);
        };
        if (kc == KC) {
#pragma unroll
            for (int c = 0; c < 8; ++c) fold_chunk(c);
        } else {
            for (int kk = 0; kk < kc; ++kk) {
                const TA x = *(const TA *)(row + (((uint32_t)(kk / E) ^ swz) << 4) + (kk % E) * sizeof(TA));
                acc = fold_step(acc, (Acc)x, bs[k0 + kk]);
            }
        }
        if (slab == nslab - 1) {
            const int64_t o = tile * RT + r;
            if (o < P.O) {
                const int64_t off = P.ident ? o : P.out_map.map((uint32_t)o);
                ((TC *)P.c)[off] = narrow<TC>(acc);
            }
            acc = Acc(0);
        }
        if (++slab == nslab) {
            slab = 0;
            tile += gridDim.x;
        }
        if (++c_stage == kRowsTmaStages) {
            c_stage = 0;
            parity ^= 1u;
        }
    }
    pdl_release();
}

// Long folds over few column fibres (contracted stride I >= a few 16-byte
// vectors, 16-byte-aligned rows): one warp per CTA owns BI consecutive
// outputs (o, i0..i0+BI-1); slabs of BK k-rows x BI columns stream through a
// 4-stage 2-D TMA pipeline (one elected lane issues each box onto the
// stage's mbarrier; columns past I are zero-filled by the tensor map), and
// lane l folds column l in k order from shared memory (bit-exact).  b comes
// in per slab as two coalesced loads and is broadcast with shuffles.  Many
// one-warp CTAs per SM: per-thread instruction latency is hidden across them,
// the data is in flight as whole boxes (no per-element copies).
constexpr int kColsBI = 32, kColsStages = 4;
__host__ __device__ constexpr int cols_bk(int elem) { return elem == 4 ? 64 : 32; }  // 32 KB of stages either way

template <class TA, class TC>
__global__ void __launch_bounds__(32) ttv_cols_tma_kernel(const __grid_constant__ TtvParams P,
                                                          const __grid_constant__ CUtensorMap map) {
    using Acc = typename AccOf<TA>::type;
    constexpr int BI = kColsBI, BK = cols_bk((int)sizeof(TA)), NST = kColsStages;
    __shared__ __align__(128) TA st[NST][BK][BI];
    __shared__ __align__(8) uint64_t full_bar[NST];
    pdl_wait();
    if (stop_requested(P.stop)) return;
    const int lane = threadIdx.x;
    const int64_t K = P.K, I = P.I;
    const int64_t nib = (I + BI - 1) / BI;
    const int64_t o = blockIdx.x / nib;
    const int64_t i0 = (blockIdx.x - o * nib) * BI;
    const int nslab = (int)((K + BK - 1) / BK);
    if (lane == 0) {
        for (int s = 0; s < NST; ++s) mbar_init(&full_bar[s], 1);
        mbar_fence_init();
    }
    __syncwarp();
    auto issue = [&](int slab) {
        if (lane == 0 && slab < nslab) {
            const int s = slab % NST;
            fence_proxy_async_smem();
            mbar_arrive_expect_tx(&full_bar[s], (uint32_t)(BK * BI * sizeof(TA)));
            tma_load_2d(&st[s][0][0], &map, (int32_t)i0, (int32_t)(o * K + (int64_t)slab * BK), &full_bar[s]);
        }
    };
    for (int s = 0; s < NST; ++s) issue(s);
    Acc acc = Acc(0);
    uint32_t parity = 0;
    for (int slab = 0; slab < nslab; ++slab) {
        const int s = slab % NST;
        const int64_t k0 = (int64_t)slab * BK;
        // this slab's b: lane l holds b[k0 + l] and b[k0 + 32 + l]
        const Acc b0 = k0 + lane < K ? load_elem_as<Acc>(P.b, P.b_dtype, (k0 + lane) * P.b_stride) : Acc(0);
        const Acc b1 = (BK > 32 && k0 + 32 + lane < K) ? load_elem_as<Acc>(P.b, P.b_dtype, (k0 + 32 + lane) * P.b_stride) : Acc(0);
        mbar_wait_parity(&full_bar[s], parity);
        const int kn = (int)(K - k0 < BK ? K - k0 : BK);
        if (kn == BK) {
#pragma unroll 16
            for (int kk = 0; kk < BK; ++kk) {
                const Acc bk = __shfl_sync(0xffffffffu, kk < 32 ? b0 : b1, kk & 31);
                acc = fold_step(acc, (Acc)st[s][kk][lane], bk);
            }
        } else {
            for (int kk = 0; kk < kn; ++kk) {
                const Acc bk = __shfl_sync(0xffffffffu, kk < 32 ? b0 : b1, kk & 31);
                acc = fold_step(acc, (Acc)st[s][kk][lane], bk);
            }
        }
        __syncwarp();  // every lane is done with stage s
        issue(slab + NST);
        if (s == NST - 1) parity ^= 1u;
    }
    const int64_t i = i0 + lane;
    if (i < I) {
        TC *c = (TC *)P.c;
        const int64_t off = P.ident ? o * I + i : P.out_map.map((uint32_t)o) + P.in_map.map((uint32_t)i);
        c[off] = narrow<TC>(acc);
    }
    pdl_release();
}

// ------------------------------------------------------------- planning
struct TtvLaunch {
    TtvParams P;
    TtvBoxParams box;  // regime 4
    TtvTileParams tile;  // regime 7
    int regime;  // 0 = strided (B), 1 = staged (S), 2/3 = small, 4 = boxed strided
    int vec;
    int G;
    bool vecread;
    bool bulk;
    bool pdl;  // programmatic dependent launch (HOPM chains)
    int64_t keep_bytes;  // L2 reuse: bytes of A read last kept L2-resident (strided, 2-D TMA rows)
    bool small_cluster;  // small kernel + HOPM norm as one thread-block cluster
    bool rows_tma;     // regime S, I == 1, 2-D TMA tensor map
    int box_h;         // regime 4: warps per chain row (1 or 2)
    CUtensorMap tmap;
    dim3 grid, block;
    size_t smem;
};

// Regime-S plan: rows per tile, slab length, pitch, piece size.
static bool plan_staged(TtvLaunch &L, int64_t s, uintptr_t base_addr, int nsm) {
    TtvParams &P = L.P;
    const int64_t I = P.I, K = P.K, O = P.O;
    int threads = 256;
    int64_t R;
    if (I == 1) {
        R = threads;
        // rows that are not whole 16-byte vectors (K = 33 doubles = 264 bytes)
        // would be copied in 8-byte cp.async pieces (measured 0.47 of HBM);
        // with fewer rows per tile the whole tile is one contiguous, 16-byte
        // aligned range that fits a stage and streams as ONE TMA bulk copy
        // (TL_TTV_ROWS_BULK=0: off)
        static const bool rows_bulk = getenv("TL_TTV_ROWS_BULK") == nullptr || atoi(getenv("TL_TTV_ROWS_BULK")) != 0;
        if (rows_bulk && (K * s) % 16 != 0 && base_addr % 16 == 0 && K % 2 == 1 && 32 * K * s <= 32 * 1024) {
            int64_t r = std::min<int64_t>(256, (32 * 1024) / (K * s) / 32 * 32);
            while (r >= 32 && (r * K * s) % 16 != 0) r -= 32;
            if (r >= 32) R = r;
        }
        // small problems: fewer rows per tile so every SM gets a tile
        while (R > 32 && (O + R - 1) / R < nsm) R /= 2;
        threads = (int)std::max<int64_t>(32, R);
    } else {
        R = std::max<int64_t>(1, (int64_t)threads * kMaxOpt / I);
        while (R > 1 && (O + R - 1) / R < nsm && R * I > 64) R /= 2;
        threads = (int)std::min<int64_t>(256, std::max<int64_t>(32, ((R * I + 31) / 32) * 32));
    }
    // (rows of a few elements are padded to a bank-friendly pitch, e.g. 6 -> 18
    // doubles: when the padded stages overflow shared memory, halve the rows
    // per tile instead of giving the tensor to the strided kernel, whose
    // one-thread-per-fibre walk over I < 32 measured 0.08-0.17 of HBM)
    for (;; R /= 2) {
    if (I != 1) threads = (int)std::min<int64_t>(256, std::max<int64_t>(32, ((R * I + 31) / 32) * 32));
    // piece size: must divide the global row pitch and the base address
    int64_t G = 16;
    while (G > (int64_t)s && (((K * I * s) % G) != 0 || (base_addr % G) != 0)) G /= 2;
    if (((K * I * s) % G) != 0 || (base_addr % G) != 0) G = s;
    // slab length: whole [K][I] rows when a tile fits the stage budget,
    // else k-slabs whose byte offsets stay on 128-byte line boundaries
    const int64_t stage_target = 32 * 1024;  // 16-48 KB measured equal
    int64_t Kc;
    if (R * K * I * s <= stage_target) {
        Kc = K;
    } else {
        const int64_t unit = std::max<int64_t>(128 / std::gcd<int64_t>(128, I * s), G / std::gcd(G, I * s));
        Kc = stage_target / std::max<int64_t>(1, R * I * s);
        Kc = std::max<int64_t>(unit, Kc - Kc % unit);
        if (Kc >= K) Kc = K;
    }
    const int64_t L0 = Kc * I;
    int64_t Lp;
    bool vecread = false;
    if (I == 1 && G == 16) {
        vecread = true;
        Lp = L0;
        while (((Lp * s) % 16) != 0 || (((Lp * s) / 16) % 2) == 0) ++Lp;
    } else {
        const int64_t w = s / 4;            // 32-bit words per element
        const int64_t M = 32 / w;           // elements per bank cycle
        const int64_t want = (I == 1) ? 1 : (I % M);
        Lp = L0;
        if (I == 1) {
            if (Lp % 2 == 0) ++Lp;
        } else {
            while ((Lp % M) != want) ++Lp;
        }
        // keep cp.async destinations G-aligned
        while (G > s && ((Lp * s) % G) != 0) G /= 2;
    }
    const int64_t bbytes = ((K * 8) + 15) & ~15ll;
    const int64_t stage_bytes = ((R * Lp * s) + 15) & ~15ll;
    const int64_t smem = bbytes + kStages * stage_bytes;
    if (smem > 200 * 1024) {
        // (only for I <= 4, or I <= 8 with slabs of 4 KB and more, where the
        // strided kernel's per-thread streams thrash DRAM pages: K = 640, I = 6
        // 326 -> 270 us; short slabs with I = 5..6 measured better strided,
        // K = 17, I = 5: 191 vs 246 us)
        if (I != 1 && (I <= 4 || (I <= 8 && K * I * s >= 4096)) && R >= 2 && R * I > 64) continue;
        return false;
    }
    // contiguous-chunk mode: one slab, no padding -> 1-D TMA bulk copies
    L.bulk = (Kc == K) && (Lp == L0) && (base_addr % 16 == 0) && ((R * K * I * s) % 16 == 0);
    P.R = (int32_t)R;
    P.Kc = (int32_t)Kc;
    P.Lp = (int32_t)Lp;
    P.nslab = (int32_t)((K + Kc - 1) / Kc);
    P.ntiles = (O + R - 1) / R;
    P.opt = (int32_t)((R * I + threads - 1) / threads);
    if (P.opt > kMaxOpt) return false;
    P.I_div.init((uint32_t)I);
    P.pr_div.init((uint32_t)((Kc * I * s) / G));
    const int64_t ktail = K - (int64_t)(P.nslab - 1) * Kc;
    P.pr_tail.init((uint32_t)((ktail * I * s) / G));
    L.regime = 1;
    L.G = (int)G;
    L.vecread = vecread;
    L.block = dim3(threads);
    L.smem = (size_t)smem;
    // resident CTAs per SM from shared memory (228 KB/SM, 1 KB reserved per CTA)
    const int64_t per_sm = std::max<int64_t>(1, std::min<int64_t>(4, (228 * 1024) / (smem + 2048)));
    const int64_t grid = std::min<int64_t>(P.ntiles, (int64_t)nsm * per_sm);
    L.grid = dim3((unsigned)grid);
    return true;
    }
}

static bool plan_strided(TtvLaunch &L, int64_t s, uintptr_t base_addr, int nsm, int32_t a_dtype) {
    TtvParams &P = L.P;
    int vec = 1;
    if (a_dtype == TL_F32) {
        if (P.I % 4 == 0 && base_addr % 16 == 0) vec = 4;
        else if (P.I % 2 == 0 && base_addr % 8 == 0) vec = 2;
    } else {
        if (P.I % 2 == 0 && base_addr % 16 == 0) vec = 2;
    }
    const int64_t nthreads = P.O * (P.I / vec);
    static const int slab_align = [] {
        const char *e = getenv("TL_TTV_SLAB_CTA");
        return e ? atoi(e) : 1;
    }();
    int threads = 256;
    while (threads > 32 && (nthreads + threads - 1) / threads < 2 * nsm) threads /= 2;
    // one o-slab per CTA when a slab's fibers fill 128..256 threads (HOPM's
    // 400^3 mode-2 pass: 200): a slab's warps then advance through k together
    // and read each k-row as one contiguous run
    const int64_t per_slab = P.I / vec;
    if (slab_align && P.O > 1 && per_slab >= 128 && per_slab <= 256 && (P.O >= 2 * nsm)) threads = (int)per_slab;
    P.b_smem = (P.K <= 8192) ? 1 : 0;
    P.in_vec_ok = (P.in_map.n >= 1 && P.in_map.div[0].d % (uint32_t)vec == 0) ? 1 : 0;
    static const int64_t omul_env = [] {
        const char *e = getenv("TL_TTV_OMUL");
        return (int64_t)(e ? atoll(e) : 257);
    }();
    // scramble only slabs of up to 256 KB (larger ones, e.g. HOPM's 1.28 MB,
    // measure slightly better in storage order)
    // ... and not slabs of under 1 KB: consecutive threads then belong to
    // consecutive slabs, and visiting those 257 apart scatters every warp's
    // loads and stores over isolated sectors (K = 3, I = 2: 0.08 of HBM)
    int64_t m = (P.K * P.I * s <= (256 << 10) && P.K * P.I * s >= 1024) ? omul_env : 1;
    while (m > 1 && std::gcd(m, P.O) != 1) m += 2;
    P.o_mul = (P.O > 1 && m > 1) ? m % P.O : 1;
    if (P.o_mul == 0) P.o_mul = 1;
    L.regime = 0;
    L.vec = vec;
    L.block = dim3(threads);
    L.grid = dim3((unsigned)((nthreads + threads - 1) / threads));
    L.smem = P.b_smem ? (size_t)P.K * 8 : 0;
    (void)s;
    return true;
}

// <<<>>> or, for programmatic dependent launch, cudaLaunchKernelEx
template <class Kern>
static cudaError_t launch_kernel(Kern kern, const TtvLaunch &L, cudaStream_t st) {
    if (!L.pdl) {
        kern<<<L.grid, L.block, L.smem, st>>>(L.P);
        return cudaGetLastError();
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = L.grid;
    cfg.blockDim = L.block;
    cfg.dynamicSmemBytes = L.smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, L.P);
}

template <class TA, class TC>
static cudaError_t launch_box(const TtvLaunch &L, cudaStream_t st) {
    auto go = [&](auto kern) -> cudaError_t {
        if (L.smem > 48 * 1024) {
            cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L.smem);
            if (e != cudaSuccess) return e;
        }
        if (!L.pdl) {
            kern<<<L.grid, L.block, L.smem, st>>>(L.box);
            return cudaGetLastError();
        }
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = L.grid;
        cfg.blockDim = L.block;
        cfg.dynamicSmemBytes = L.smem;
        cfg.stream = st;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        return cudaLaunchKernelEx(&cfg, kern, L.box);
    };
    if constexpr (sizeof(TA) == 4) {
        if (L.vec == 4) return go(ttv_box_kernel<TA, TC, 4, 8>);
    }
    // K = 9: the whole fold in flight per pass (config 5 seed 5: 150.6 ->
    // 147.2 us at the same 64 registers; K = 10..12 would need 69-78
    // registers, one CTA per SM fewer, unmeasured)
    if (L.box_h == 2) {
        if (L.vec == 2 && L.box.K == 9) return go(ttv_box_kernel<TA, TC, 2, 8, 9, 2>);
        if (L.vec == 2) return go(ttv_box_kernel<TA, TC, 2, 8, 8, 2>);
    }
    if (L.vec == 2 && L.box.K == 9) return go(ttv_box_kernel<TA, TC, 2, 8, 9>);
    if (L.vec == 2) return go(ttv_box_kernel<TA, TC, 2, 8>);
    return go(ttv_box_kernel<TA, TC, 1, 8>);
}

// 2-D TMA tensor map for the rows kernel (driver entry point looked up once
// through the runtime, so the library needs no link-time libcuda).
static PFN_cuTensorMapEncodeTiled_v12000 tmap_encoder() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            return (PFN_cuTensorMapEncodeTiled_v12000) nullptr;
        return (PFN_cuTensorMapEncodeTiled_v12000)p;
    }();
    return fn;
}

static bool plan_rows_tma(TtvLaunch &L, const Canon &cn, int32_t dtype, int nsm) {
    static const bool off = getenv("TL_TTV_NO_TMA") != nullptr;
    const TtvParams &P = L.P;
    if (off || L.regime != 1 || cn.I != 1 || (dtype != TL_F32 && dtype != TL_F64)) return false;
    const int64_t s = dtype == TL_F32 ? 4 : 8;
    const uintptr_t base = (uintptr_t)P.a;
    if ((cn.K * s) % 16 != 0 || base % 16 != 0 || cn.O > 0x7fffffffll || cn.K > 0x7fffffffll) return false;
    if (cn.O < kRowsTmaR) return false;
    PFN_cuTensorMapEncodeTiled_v12000 enc = tmap_encoder();
    if (enc == nullptr) return false;
    // Rows per tile R (= threads per CTA) and CTAs per SM: the persistent
    // grid walks the tiles in rounds, so 625 tiles on 296 CTAs (400^3
    // float64, R = 256) take 3 rounds for 2.1 rounds of work (measured 0.835
    // of HBM).  Pick the (R, CTAs per SM) whose last round is fullest; within
    // 2% prefer the larger tile.
    const size_t bbytes = (((size_t)cn.K * 8 + 15) & ~(size_t)15);
    int bestR = kRowsTmaR, best_ps = 1;
    double best_eff = -1.0;
    static const int fixedR = [] {
        const char *e = getenv("TL_TTV_ROWS_R");  // 256 / 128 / 64: fixed rows per tile (0 = choose)
        return e ? atoi(e) : 0;
    }();
    for (int R : {256, 128, 64}) {
        if (fixedR != 0 && R != fixedR) continue;
        const size_t smem = 1024 + (size_t)kRowsTmaStages * R * 128 + bbytes;
        if (smem > 200 * 1024) continue;
        const int64_t tiles = (cn.O + R - 1) / R;
        const int max_ps = (int)std::max<int64_t>(1, std::min<int64_t>(R == 256 ? 2 : R == 128 ? 4 : 8, (228 * 1024) / ((int64_t)smem + 2048)));
        for (int ps = max_ps; ps >= 1; --ps) {
            // enough rows in flight per SM to hide the loads (one 64-thread CTA per SM measured 2x slower)
            if (R * ps < 384 && ps < max_ps) break;
            const int64_t slots = std::min<int64_t>(tiles, (int64_t)nsm * ps);
            const int64_t rounds = (tiles + slots - 1) / slots;
            const double eff = (double)tiles / (double)(rounds * slots);
            if (eff > best_eff + 0.02) {
                best_eff = eff;
                bestR = R;
                best_ps = ps;
            }
        }
    }
    if (best_eff < 0) return false;
    const cuuint64_t dims[2] = {(cuuint64_t)cn.K, (cuuint64_t)cn.O};
    const cuuint64_t strides[1] = {(cuuint64_t)(cn.K * s)};
    const cuuint32_t box[2] = {(cuuint32_t)(128 / s), (cuuint32_t)bestR};
    const cuuint32_t estr[2] = {1, 1};
    CUresult r = enc(&L.tmap, dtype == TL_F32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2,
                     (void *)P.a, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return false;
    L.rows_tma = true;
    L.block = dim3(bestR);
    L.smem = 1024 + (size_t)kRowsTmaStages * bestR * 128 + bbytes;
    const int64_t ntiles = (cn.O + bestR - 1) / bestR;
    L.grid = dim3((unsigned)std::min<int64_t>(ntiles, (int64_t)nsm * best_ps));
    return true;
}

template <class TA, class TC>
static cudaError_t launch_rows_tma(const TtvLaunch &L, cudaStream_t st) {
    auto kern = ttv_rows_tma_kernel<TA, TC>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L.smem);
    if (e != cudaSuccess) return e;
    if (!L.pdl) {
        kern<<<L.grid, L.block, L.smem, st>>>(L.P, L.tmap);
        return cudaGetLastError();
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = L.grid;
    cfg.blockDim = L.block;
    cfg.dynamicSmemBytes = L.smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, L.P, L.tmap);
}

template <class TA, class TC>
static cudaError_t launch_short(const TtvLaunch &L, void *out, cudaStream_t st) {
    if (L.vec == 4) {
        if constexpr (sizeof(TC) == 4) {
            ttv_short_kernel<TA, TC, 4><<<L.grid, L.block, 0, st>>>(L.P, (TC *)out);
            return cudaGetLastError();
        }
    }
    ttv_short_kernel<TA, TC, 2><<<L.grid, L.block, 0, st>>>(L.P, (TC *)out);
    return cudaGetLastError();
}

// Regime 5: the short-fold stream, into C in canonical order (ident) or
// through the digit maps (C's fastest canonical digit contiguous).
static int ttv_short_run(const TtvLaunch &L, int32_t a_dtype, int32_t c_dtype, void *c_ptr, cudaStream_t st) {
    cudaError_t e;
    if (a_dtype == TL_F32 && c_dtype == TL_F32) e = launch_short<float, float>(L, c_ptr, st);
    else if (a_dtype == TL_F32 && c_dtype == TL_F64) e = launch_short<float, double>(L, c_ptr, st);
    else e = launch_short<double, double>(L, c_ptr, st);
    return cuda_status(e, "ttv short-fold launch");
}

// Resident CTAs per SM of a kernel configuration (cached: no per-launch query)
static cudaError_t occupancy(const void *kern, int threads, size_t smem, int &per_sm) {
    struct Entry {
        const void *kern;
        int threads;
        size_t smem;
        int per_sm;
    };
    static std::mutex mu;
    static std::vector<Entry> cache;
    std::lock_guard<std::mutex> lk(mu);
    for (const Entry &c : cache)
        if (c.kern == kern && c.threads == threads && c.smem == smem) {
            per_sm = c.per_sm;
            return cudaSuccess;
        }
    cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, smem);
    if (e == cudaSuccess) cache.push_back({kern, threads, smem, per_sm});
    return e;
}

template <class TA, class TC>
static cudaError_t launch_typed(const TtvLaunch &L, cudaStream_t st) {
    if (L.regime == 4) return launch_box<TA, TC>(L, st);
    if (L.regime == 7) {
        if constexpr (std::is_same<TA, int64_t>::value) {
            return cudaErrorInvalidValue;
        } else {
            switch (L.G) {
                case 1: ttv_tile_kernel<TA, TC, 64, 64><<<L.grid, L.block, 0, st>>>(L.tile); break;
                case 2: ttv_tile_kernel<TA, TC, 32, 128><<<L.grid, L.block, 0, st>>>(L.tile); break;
                case 3:
                    if constexpr (sizeof(TC) == 4) {
                        ttv_tile_kernel<TA, TC, 64, 128><<<L.grid, L.block, 0, st>>>(L.tile);
                        break;
                    }
                    return cudaErrorInvalidValue;  // 64 KB of float64 tile: planned only for float32
                default: ttv_tile_kernel<TA, TC, 32, 64><<<L.grid, L.block, 0, st>>>(L.tile); break;
            }
            return cudaGetLastError();
        }
    }
    if (L.rows_tma) {
        if constexpr (std::is_same<TA, float>::value || std::is_same<TA, double>::value) return launch_rows_tma<TA, TC>(L, st);
        return cudaErrorInvalidValue;
    }
    if (L.regime == 2 || L.regime == 3) {
        auto kern = (L.regime == 3) ? ttv_small_kernel<TA, TC, true, false> : ttv_small_kernel<TA, TC, false, false>;
        if constexpr (sizeof(TA) == 8 && std::is_same<typename AccOf<TA>::type, double>::value) {
            if (L.vec == 2) kern = (L.regime == 3) ? ttv_small_kernel<TA, TC, true, true> : ttv_small_kernel<TA, TC, false, true>;
        }
        if constexpr (std::is_same<TA, double>::value && std::is_same<TC, double>::value) {
            if (L.small_cluster) {
                // HOPM fused norm over one thread-block cluster (no ticket, w via DSMEM)
                auto ck = (L.regime == 3) ? (L.vec == 2 ? ttv_small_kernel<TA, TC, true, true, true>
                                                        : ttv_small_kernel<TA, TC, true, false, true>)
                                          : (L.vec == 2 ? ttv_small_kernel<TA, TC, false, true, true>
                                                        : ttv_small_kernel<TA, TC, false, false, true>);
                cudaError_t e = cudaFuncSetAttribute(ck, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L.smem);
                if (e == cudaSuccess) e = cudaFuncSetAttribute(ck, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
                if (e != cudaSuccess) return e;
                cudaLaunchConfig_t cfg{};
                cfg.gridDim = L.grid;
                cfg.blockDim = L.block;
                cfg.dynamicSmemBytes = L.smem;
                cfg.stream = st;
                cudaLaunchAttribute attr[1];
                attr[0].id = cudaLaunchAttributeClusterDimension;
                attr[0].val.clusterDim.x = L.grid.x;
                attr[0].val.clusterDim.y = 1;
                attr[0].val.clusterDim.z = 1;
                cfg.attrs = attr;
                cfg.numAttrs = 1;
                return cudaLaunchKernelEx(&cfg, ck, L.P);
            }
        }
        if (L.smem > 48 * 1024) {
            cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L.smem);
            if (e != cudaSuccess) return e;
        }
        return launch_kernel(kern, L, st);
    }
    auto go = [&](auto kern) -> cudaError_t {
        if (L.smem > 48 * 1024) {
            cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L.smem);
            if (e != cudaSuccess) return e;
        }
        if (L.regime == 0 && L.P.l2_stream) {
            // what this pass reads last: its last k-rows (one wave) or its last CTAs
            TtvLaunch K2 = L;
            int per_sm = 0;
            cudaError_t e = occupancy((const void *)kern, (int)L.block.x, L.smem, per_sm);
            if (e != cudaSuccess) return e;
            const int64_t resident = (int64_t)per_sm * device_info().num_sms;
            const int64_t s = (int64_t)sizeof(TA);
            if ((int64_t)L.grid.x <= resident) {
                K2.P.keep_k = K2.P.K - std::min<int64_t>(K2.P.K, L.keep_bytes / (K2.P.O * K2.P.I * s));
            } else {
                const int64_t cta_bytes = (int64_t)L.block.x * L.vec * K2.P.K * s;
                K2.P.keep_cta = (int64_t)L.grid.x - std::min<int64_t>(L.grid.x, L.keep_bytes / cta_bytes);
            }
            return launch_kernel(kern, K2, st);
        }
        return launch_kernel(kern, L, st);
    };
    if (L.regime == 8) {
        if constexpr (std::is_same<TA, float>::value || std::is_same<TA, double>::value) {
            // plain stream order even in a PDL chain (griddepcontrol is then a no-op)
            ttv_cols_tma_kernel<TA, TC><<<L.grid, L.block, 0, st>>>(L.P, L.tmap);
            return cudaGetLastError();
        }
        return cudaErrorInvalidValue;
    }
    if (L.regime == 6) {
        constexpr int VF = 16 / sizeof(TA);  // full 16-byte fibre pieces
        if (L.P.I == 1) {
            // 16-byte chunks along the rows when every row starts 16-byte aligned
            if (L.vec > 1) return L.G == 16 ? go(ttv_deep_kernel<TA, TC, 2, true, 16>) : go(ttv_deep_kernel<TA, TC, 2, true, 8>);
            return L.G == 16 ? go(ttv_deep_kernel<TA, TC, 1, true, 16>) : go(ttv_deep_kernel<TA, TC, 1, true, 8>);
        }
        if (L.vec == VF) return L.G == 16 ? go(ttv_deep_kernel<TA, TC, VF, false, 16>) : go(ttv_deep_kernel<TA, TC, VF, false, 8>);
        if constexpr (VF == 4) {
            if (L.vec == 2) return L.G == 16 ? go(ttv_deep_kernel<TA, TC, 2, false, 16>) : go(ttv_deep_kernel<TA, TC, 2, false, 8>);
        }
        return L.G == 16 ? go(ttv_deep_kernel<TA, TC, 1, false, 16>) : go(ttv_deep_kernel<TA, TC, 1, false, 8>);
    }
    if (L.regime == 0) {
        constexpr int U = 8;
        const bool keep = L.P.l2_stream != 0;
        if constexpr (sizeof(TA) == 4) {
            if (L.vec == 4) return keep ? go(ttv_strided_kernel<TA, TC, 4, U, true>) : go(ttv_strided_kernel<TA, TC, 4, U>);
        }
        if (L.vec == 2) return keep ? go(ttv_strided_kernel<TA, TC, 2, U, true>) : go(ttv_strided_kernel<TA, TC, 2, U>);
        return keep ? go(ttv_strided_kernel<TA, TC, 1, U, true>) : go(ttv_strided_kernel<TA, TC, 1, U>);
    }
    if (L.bulk) {
        if (L.vecread) return go(ttv_staged_kernel<TA, TC, 16, true, true>);
        return go(ttv_staged_kernel<TA, TC, 16, false, true>);
    }
    if (L.vecread) return go(ttv_staged_kernel<TA, TC, 16, true, false>);
    switch (L.G) {
        case 16: return go(ttv_staged_kernel<TA, TC, 16, false, false>);
        case 8: return go(ttv_staged_kernel<TA, TC, 8, false, false>);
        default:
            if constexpr (sizeof(TA) == 4) return go(ttv_staged_kernel<TA, TC, 4, false, false>);
            return cudaErrorInvalidValue;
    }
}

// Canonical form + kernel choice (host only; no device access).
// Regime-B plan with a permuted output: the boxed kernel when A's fastest
// free digit d0 is not C's fastest and a C-contiguous chain of at least 16
// positions exists among the other free digits.
static bool plan_box(const Canon &cn, TtvLaunch &L, int64_t s, uintptr_t base_addr, int nsm, int64_t cs_elem) {
    static const bool off = getenv("TL_TTV_NO_BOX") != nullptr;
    if (off || cn.ident || cn.inner.empty()) return false;
    // Measured on B200: the box's 8 warps stream 8 separate A regions, which
    // costs about what scattered stores cost the plain kernel unless the fold
    // is short (K <= 32: a store per few loads, e.g. config 5's K = 9).
    if (cn.K > 32) return false;
    struct Dg {
        int64_t ext, as, cs;
    };
    std::vector<Dg> free;
    {
        int64_t run = 1;
        for (auto &d : cn.inner) {
            free.push_back({d.first, run, d.second});
            run *= d.first;
        }
        run = cn.K * cn.I;
        for (auto &d : cn.outer) {
            free.push_back({d.first, run, d.second});
            run *= d.first;
        }
    }
    const Dg d0 = free[0];
    const size_t ninner = cn.inner.size();
    // the C-fastest digit other than d0 (A's fastest), then digits continuing
    // its C run; the A-direction is then the prefix of the inner digits (all
    // contiguous in A) before the first one the C-chain uses
    int cstar = -1;
    for (size_t q = 1; q < free.size(); ++q)
        if (cstar < 0 || free[q].cs < free[cstar].cs) cstar = (int)q;
    if (cstar < 0 || free[cstar].cs > d0.cs) return false;
    std::vector<int> chain{cstar};
    int64_t cext = free[cstar].ext;
    while (cext < 64 && (int)chain.size() < kBoxMaxChain) {
        const Dg &last = free[chain.back()];
        int nxt = -1;
        for (size_t q = 1; q < free.size(); ++q) {
            if (std::find(chain.begin(), chain.end(), (int)q) != chain.end()) continue;
            if (free[q].cs == last.cs * last.ext) nxt = (int)q;
        }
        if (nxt < 0) break;
        chain.push_back(nxt);
        cext *= free[nxt].ext;
    }
    // a short or ragged C-chain (its last block of 64 mostly idle) continues
    // over the remaining digits in C order -- the chain is a flat index space
    // decoded per position, so the digits need not be C-contiguous; only
    // digits the A-chain does not need (TL_TTV_BOX_RAGGED=0: contiguous only)
    {
        static const bool fill = getenv("TL_TTV_BOX_RAGGED") == nullptr || atoi(getenv("TL_TTV_BOX_RAGGED")) != 0;
        const size_t na0 = d0.ext >= 16 ? 1 : ninner;
        auto ragged = [&](int64_t e) { return (double)((e + 63) / 64 * 64) > 1.15 * (double)e; };
        while (fill && (cext < 64 || ragged(cext)) && (int)chain.size() < kBoxMaxChain) {
            int nxt = -1;
            for (size_t q = na0; q < free.size(); ++q) {
                if (std::find(chain.begin(), chain.end(), (int)q) != chain.end()) continue;
                if (nxt < 0 || free[q].cs < free[nxt].cs) nxt = (int)q;
            }
            if (nxt < 0 || cext * free[nxt].ext > 0x7fffffffll) break;
            chain.push_back(nxt);
            cext *= free[nxt].ext;
        }
    }
    if (cext < 16 || cext > 0xffffffffll) return false;
    // A-chain: inner digits [0, na) -- d0 alone when it is long enough (the
    // tuned one-digit box), else as many inner digits as precede the C-chain
    size_t na = d0.ext >= 16 ? 1 : ninner;
    for (int q : chain)
        if ((size_t)q < na) na = (size_t)q;
    if (na == 0 || na > (size_t)kBoxMaxChain) return false;
    int64_t ea = 1;
    for (size_t q = 0; q < na; ++q) ea *= free[q].ext;
    if (ea < 16 || ea > 0xffffffffll) return false;
    TtvBoxParams &B = L.box;
    B = TtvBoxParams{};
    B.K = cn.K;
    B.I = cn.I;
    B.e0 = ea;
    B.cs0 = d0.cs;
    B.na = (int32_t)na;
    for (size_t q = 0; q < na; ++q) {
        B.a_div[q].init((uint32_t)free[q].ext);
        B.a_cs[q] = free[q].cs;
    }
    B.chain_ext = cext;
    B.nchain = (int32_t)chain.size();
    for (size_t q = 0; q < chain.size(); ++q) {
        B.ch_div[q].init((uint32_t)free[chain[q]].ext);
        B.ch_as[q] = free[chain[q]].as;
        B.ch_cs[q] = free[chain[q]].cs;
    }
    int64_t nrest = 1;
    B.nrest_d = 0;
    for (size_t q = na; q < free.size(); ++q) {
        if (std::find(chain.begin(), chain.end(), (int)q) != chain.end()) continue;
        if (free[q].ext > 0xffffffffll) return false;
        B.rs_div[B.nrest_d].init((uint32_t)free[q].ext);
        B.rs_as[B.nrest_d] = free[q].as;
        B.rs_cs[B.nrest_d] = free[q].cs;
        ++B.nrest_d;
        nrest *= free[q].ext;
    }
    if (B.nrest_d == 0) {  // keep one trivial digit so the decode loop is uniform
        B.rs_div[0].init(1);
        B.rs_as[0] = B.rs_cs[0] = 0;
        B.nrest_d = 1;
    }
    int vec = 1;
    if (s == 4 && ea % 4 == 0 && base_addr % 16 == 0 && (cn.I % 4) == 0) vec = 4;
    else if (ea % 2 == 0 && base_addr % (2 * s) == 0 && (cn.I % 2) == 0 && s <= 8) vec = 2;
    static const int box_h_env = [] {
        const char *e = getenv("TL_TTV_BOX_H");
        return e ? atoi(e) : 2;
    }();
    // two warps per chain row (1 KB runs along d0) for float64 pairs when d0 is long enough
    const int h = (box_h_env == 2 && vec == 2 && s == 8 && ea >= 128) ? 2 : 1;
    L.box_h = h;
    const int64_t BA = 32 * vec * h, BC = 64 / h;
    B.nA = (ea + BA - 1) / BA;
    B.nJ = (cext + BC - 1) / BC;
    B.nrest = nrest;
    const int64_t ntiles = B.nA * B.nJ * B.nrest;
    if (ntiles > 0x7fffffffll) return false;
    B.b_smem = (cn.K <= 8192) ? 1 : 0;
    L.regime = 4;
    L.vec = vec;
    L.block = dim3(256);
    const size_t bbytes = B.b_smem ? (((size_t)cn.K * 8 + 15) & ~(size_t)15) : 0;
    L.smem = bbytes + 2 * BC * 8 + (((size_t)BC * (BA + 1) * cs_elem + 7) & ~(size_t)7) + (size_t)BA * 8;
    const int64_t per_sm = std::max<int64_t>(1, std::min<int64_t>(8, (228 * 1024) / ((int64_t)L.smem + 2048)));
    L.grid = dim3((unsigned)std::min<int64_t>(ntiles, (int64_t)nsm * per_sm * 2));
    return true;
}

// Regime 7 plan: the fused transpose-fold for short folds with a permuted
// output.  Digits: (extent, A stride, C stride) in A order.
static bool plan_tile(const Canon &cn, TtvLaunch &L, int nsm, bool s8) {
    static const bool off = getenv("TL_TTV_NO_TILE") != nullptr;
    if (off) return false;
    struct Dg {
        int64_t ext, as, cs;
    };
    std::vector<Dg> F;
    int64_t run = 1;
    for (auto &d : cn.inner) {
        F.push_back({d.first, run, d.second});
        run *= d.first;
    }
    run = cn.K * cn.I;
    for (auto &d : cn.outer) {
        F.push_back({d.first, run, d.second});
        run *= d.first;
    }
    const size_t nf = F.size();
    if (nf < 2) return false;
    std::vector<int> used(nf, 0);
    static const int shape = getenv("TL_TTV_TILE_SHAPE") ? atoi(getenv("TL_TTV_TILE_SHAPE")) : 0;
    const int sh = (shape == 3 && s8) ? 1 : (shape & 3);  // 64 x 128 tiles only for 4-byte outputs
    const int tx = (sh & 1) ? 64 : 32, ty = (sh & 2) ? 128 : 64;
    // the C-fastest digit heads the X chain; Y: A-fastest digits before it
    // (inner, then outer when the inner block is short)
    int c0 = 0;
    for (size_t q = 1; q < nf; ++q)
        if (F[q].cs < F[c0].cs) c0 = (int)q;
    // A chain extent that leaves a ragged last block (33 in blocks of 32: half
    // the tile idle; 85 in blocks of 64: a third) is flattened together with
    // further digits -- the chains are plain mixed-radix index spaces (the
    // kernel decodes A and C offsets per position), so the digits need not be
    // contiguous: runs simply end where a digit wraps.  TL_TTV_TILE_RAGGED=0:
    // the contiguous chains only.
    static const bool fill = getenv("TL_TTV_TILE_RAGGED") == nullptr || atoi(getenv("TL_TTV_TILE_RAGGED")) != 0;
    auto ragged = [&](int64_t e, int t) { return fill && (double)((e + t - 1) / t * t) > 1.15 * (double)e; };
    std::vector<int> ych;
    int64_t ey = 1;
    for (size_t q = 0; q < nf && (ey < ty || ragged(ey, ty)); ++q) {
        if ((int)q == c0) {
            // the C-fastest digit heads the X chain; a Y chain that is still
            // short or ragged continues behind it (e.g. when it is also A's
            // fastest digit, a tiny one: longer ones took the short-fold stream)
            if (fill) continue;
            break;
        }
        // do not cross the k gap once Y is usable (unless its last block is ragged)
        if (q == cn.inner.size() && ey >= 16 && !ragged(ey, ty)) break;
        ych.push_back((int)q);
        used[q] = 1;
        ey *= F[q].ext;
    }
    // X: C-fastest remaining digit, then digits continuing its C run
    std::vector<int> xch;
    int64_t ex = 1;
    {
        int cstar = -1;
        for (size_t q = 0; q < nf; ++q)
            if (!used[q] && (cstar < 0 || F[q].cs < F[cstar].cs)) cstar = (int)q;
        if (cstar < 0) return false;
        xch.push_back(cstar);
        used[cstar] = 1;
        ex = F[cstar].ext;
        while (ex < tx) {
            const Dg &last = F[xch.back()];
            int nxt = -1;
            for (size_t q = 0; q < nf; ++q)
                if (!used[q] && F[q].cs == last.cs * last.ext) nxt = (int)q;
            if (nxt < 0) break;
            xch.push_back(nxt);
            used[nxt] = 1;
            ex *= F[nxt].ext;
        }
        // ragged or short: continue with the remaining digits in C order
        while (fill && (ex < tx || ragged(ex, tx))) {
            int nxt = -1;
            for (size_t q = 0; q < nf; ++q)
                if (!used[q] && (nxt < 0 || F[q].cs < F[nxt].cs)) nxt = (int)q;
            if (nxt < 0 || ex * F[nxt].ext > 0x7fffffffll) break;
            xch.push_back(nxt);
            used[nxt] = 1;
            ex *= F[nxt].ext;
        }
    }
    if (ex < 8 || ey < 16 || ex > 0xffffffffll || ey > 0xffffffffll) return false;
    DigitList ya, yc, xa, xc, ra, rc;
    for (int q : ych) {
        ya.push_back({F[q].ext, F[q].as});
        yc.push_back({F[q].ext, F[q].cs});
    }
    for (int q : xch) {
        xa.push_back({F[q].ext, F[q].as});
        xc.push_back({F[q].ext, F[q].cs});
    }
    int64_t nrest = 1;
    for (size_t q = 0; q < nf; ++q)
        if (!used[q]) {
            ra.push_back({F[q].ext, F[q].as});
            rc.push_back({F[q].ext, F[q].cs});
            nrest *= F[q].ext;
        }
    TtvTileParams &T = L.tile;
    T = TtvTileParams{};
    if (!build_map(ya, T.ya) || !build_map(yc, T.yc) || !build_map(xa, T.xa) || !build_map(xc, T.xc) ||
        !build_map(ra, T.ra) || !build_map(rc, T.rc) || nrest > 0xffffffffll)
        return false;
    T.K = cn.K;
    T.I = cn.I;
    T.ex = ex;
    T.ey = ey;
    L.G = sh;
    T.nxb = (ex + tx - 1) / tx;
    T.nyb = (ey + ty - 1) / ty;
    T.nrest = nrest;
    const int64_t ntiles = T.nxb * T.nyb * T.nrest;
    L.regime = 7;
    L.block = dim3(256);
    L.grid = dim3((unsigned)std::min<int64_t>(ntiles, (int64_t)nsm * 8));
    L.smem = 0;
    return true;
}

// Regime 8: few column fibres, long fold, 16-byte-aligned rows -> 2-D TMA
// boxes of kColsBK k-rows x kColsBI columns over A viewed as (K*O) x I.
static bool plan_cols_tma(TtvLaunch &L, int64_t s) {
    static const bool off = getenv("TL_TTV_NO_COLS_TMA") != nullptr;
    TtvParams &P = L.P;
    if (off || (s != 4 && s != 8)) return false;
    const uintptr_t base = (uintptr_t)P.a;
    if (base % 16 != 0 || (P.I * s) % 16 != 0 || P.I * s < 16 || P.O * P.K > 0x7fffffffll || P.I > 0x7fffffffll) return false;
    PFN_cuTensorMapEncodeTiled_v12000 enc = tmap_encoder();
    if (enc == nullptr) return false;
    const cuuint64_t dims[2] = {(cuuint64_t)P.I, (cuuint64_t)(P.O * P.K)};
    const cuuint64_t strides[1] = {(cuuint64_t)(P.I * s)};
    const cuuint32_t box[2] = {(cuuint32_t)kColsBI, (cuuint32_t)cols_bk((int)s)};
    const cuuint32_t estr[2] = {1, 1};
    CUresult r = enc(&L.tmap, s == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, (void *)P.a,
                     dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return false;
    const int64_t nib = (P.I + kColsBI - 1) / kColsBI;
    if (P.O * nib > 0x7fffffffll) return false;
    L.regime = 8;
    L.block = dim3(32);
    L.grid = dim3((unsigned)(P.O * nib));
    L.smem = 0;
    return true;
}

// Long folds over too few fibres for the strided kernel's in-register loads
// to fill HBM: the per-thread cp.async ring kernel (regime 6).  Fibres:
// O*I/VEC (columns) or O rows when the contracted stride is 1.
static void plan_deep(TtvLaunch &L, int64_t s, int nsm) {
    static const int64_t min_k = [] {
        const char *e = getenv("TL_TTV_DEEP_MIN_K");  // 0 disables the kernel
        return (int64_t)(e ? atoll(e) : 256);
    }();
    TtvParams &P = L.P;
    if (min_k <= 0 || P.K < min_k) return;
    const bool rows = P.I == 1;
    // rows: vec 2 marks 16-byte chunks (aligned rows), 1 element pieces otherwise
    const int vec = rows ? ((((uintptr_t)P.a) % 16 == 0 && (P.K * s) % 16 == 0) ? 2 : 1) : L.vec;
    const int64_t fibres = rows ? P.O : P.O * (P.I / vec);
    // below ~128 fibres per SM the strided kernel's 8 loads in flight per
    // thread cannot cover HBM latency (HOPM's 400^3 passes have 540 per SM
    // and stay on it)
    if (fibres >= (int64_t)nsm * 128) return;
    if (!rows && plan_cols_tma(L, s)) return;
    const int ng = fibres >= (int64_t)nsm * 32 ? 8 : 16;  // deeper rings for fewer fibres
    L.regime = 6;
    L.vec = vec;
    L.G = ng;
    L.block = dim3(fibres >= (int64_t)nsm * 64 ? 64 : 32);
    L.grid = dim3((unsigned)((fibres + L.block.x - 1) / L.block.x));
    L.smem = (size_t)L.block.x * (ng * kDeepGroup * (16 + 16) + 16);  // A pieces + b values (<= 16 B each) + pad
    (void)s;
}

static int ttv_make_plan(const tl_desc &a, const void *a_ptr, int m0, TtvLaunch &L, Canon &cn, bool allow_short = true,
                         bool allow_deep = true) {
    if (!canon_contraction(a, m0, 0, cn)) {
        set_error("ttv: operand A is not a dense permutation layout (materialise views first)");
        return TL_EUNSUPPORTED;
    }
    if (cn.O > 0xffffffffll || cn.I > 0xffffffffll || cn.K > 0x7fffffffll) {
        set_error("ttv: index range exceeds 32-bit digit maps");
        return TL_EUNSUPPORTED;
    }
    const DeviceInfo &di = device_info();
    TtvParams &P = L.P;
    const size_t s = dtype_size(a.dtype);
    P.a = (const unsigned char *)a_ptr + a.offset * (int64_t)s;
    P.O = cn.O;
    P.K = cn.K;
    P.I = cn.I;
    P.ident = cn.ident ? 1 : 0;
    P.otab_n = 0;
    P.otab_d0 = 0;
    if (!build_map(cn.inner, P.in_map) || !build_map(cn.outer, P.out_map)) {
        set_error("ttv: extent exceeds 32-bit digit range");
        return TL_EUNSUPPORTED;
    }
    if (P.O * P.I == 0) return TL_OK;
    const uintptr_t base = (uintptr_t)P.a;
    bool ok;
    // short folds of large tensors: an elementwise stream (+ a transpose when
    // the output is permuted)
    static const int64_t short_min = [] {
        const char *e = getenv("TL_TTV_SHORT_MB");  // smallest operand (MB) taking the short-fold path; 0 = off
        return (int64_t)(e ? atoll(e) : 64) << 20;
    }();
    // writes go straight to C when C is in canonical order (ident) or its
    // fastest canonical digit is C-contiguous for at least 32 elements
    // (whole 128-256-byte runs); other permuted outputs keep the tiled
    // kernels below (a temporary + transpose measured slower there)
    const DigitList &fast = cn.inner.empty() ? cn.outer : cn.inner;
    const bool short_direct = cn.ident || (!fast.empty() && fast[0].second == 1 && fast[0].first >= 32);
    // contracted stride 1 (rows of K): only the shortest rows -- from K ~ 8
    // the staged kernel's tiles beat the per-thread L1 loads (K = 11: 0.94 vs 0.57)
    const int64_t short_k = P.I == 1 ? 6 : kShortK;
    if (allow_short && short_min > 0 && P.K <= short_k && P.O * P.K * P.I * (int64_t)s >= short_min && P.O * P.I < 0xffffffffll &&
        a.dtype != TL_I64 && short_direct) {
        L.regime = 5;
        L.block = dim3(256);
        const int qv = (s == 4) ? 4 : 2;
        const int64_t threads = (P.O * P.I + qv - 1) / qv;
        L.grid = dim3((unsigned)std::min<int64_t>((threads + 255) / 256, (int64_t)di.num_sms * 8));
        L.vec = qv;
        P.I_div.init((uint32_t)P.I);
        L.smem = 0;
        return TL_OK;
    }
    // (K <= 4: from K ~ 9 the boxed / staged kernels do better, config 5)
    // (with the flattened chains also K <= 8 on the strided regime, I >= 32:
    //  K = 5 on the config-5 shape 275-489 -> 234-424 us, K = 6, I = 88760 of
    //  the random sweep 2167 -> 279 us; with I < 32 the staged tiles were mixed
    //  -- 405 -> 258 but 215 -> 537 and 196 -> 429 us -- and are kept; from
    //  K = 9 the boxed / strided kernels win)
    static const int64_t tile_max_k = [] {
        const char *e = getenv("TL_TTV_TILE_MAXK");
        return (int64_t)(e ? atoll(e) : 8);
    }();
    if (allow_short && short_min > 0 && (P.K <= 4 || (P.K <= tile_max_k && P.I >= 32)) && !cn.ident &&
        P.O * P.K * P.I * (int64_t)s >= short_min &&
        a.dtype != TL_I64 && plan_tile(cn, L, di.num_sms, s == 8))
        return TL_OK;
    const size_t small_bbytes = ((size_t)P.K * 8 + 15) & ~(size_t)15;
    // few outputs (<= 16384) of a small operand (<= 32 MB): latency-bound,
    // the whole-block kernels win (measured: config 1 5.6 -> 3.8 us)
    const bool small_ok = P.O * P.I * P.K * (int64_t)s <= (32ll << 20);
    const bool small_cols = small_ok && P.I >= 32 && P.O * P.I <= 16384;
    const bool small_rows = small_ok && P.I == 1 && P.O <= 16384;
    if ((small_cols || small_rows) && P.K <= kSmallSlab * kSmallMaxSlabs &&
        small_bbytes + 32 * (size_t)(P.K | 1) * s <= 200 * 1024) {
        // few outputs: whole 32-output input blocks in flight, one fold warp
        L.regime = small_rows ? 3 : 2;
        L.grid = dim3((unsigned)(small_rows ? (P.O + 31) / 32 : P.O * ((P.I + 31) / 32)));
        // 7 copy warps + the fold warp: issuing the block's 16-byte cp.async
        // copies is the fold's critical path with 3 (400^2 fold 7.3 -> 5.4 us;
        // 384/512 threads measured slower again)
        static const int small_threads = [] {
            const char *e = getenv("TL_TTV_SMALL_THREADS");
            const int v = e ? atoi(e) : 256;
            return v == 128 || v == 256 ? v : 256;
        }();
        L.block = dim3(small_threads);
        // 16-byte element pairs for float64 when every pair is aligned and in range
        const bool pairs = (a.dtype == TL_F64) && (base % 16 == 0) && (small_rows ? (P.K % 2 == 0) : (P.I % 2 == 0));
        L.vec = pairs ? 2 : 1;
        const int64_t pitch = pairs ? (P.K + 2) + (((P.K + 2) / 2) % 2 == 0 ? 2 : 0) : (P.K | 1);
        L.smem = small_bbytes + 32 * (size_t)std::max<int64_t>(pitch, P.K) * s;
        ok = true;
    } else if (P.I >= 32) {
        ok = plan_strided(L, (int64_t)s, base, di.num_sms, a.dtype);
        if (ok && allow_deep) plan_deep(L, (int64_t)s, di.num_sms);
    } else {
        ok = plan_staged(L, (int64_t)s, base, di.num_sms);
        if (ok && !P.ident && cn.outer.size() >= 3 && P.O * P.I < 0x7fffffffll) {
            // permuted output: look up the low output digits in a shared table
            int64_t E = 1;
            int d0 = 0;
            while (d0 + 1 < (int)cn.outer.size() && E * cn.outer[d0].first <= 1024) E *= cn.outer[d0++].first;
            if (d0 >= 2) {
                DigitList hi(cn.outer.begin() + d0, cn.outer.end());
                build_map(hi, P.out_hi);
                P.otab_n = (int32_t)E;
                P.otab_d0 = d0;
                P.otab_div.init((uint32_t)E);
                L.smem += (size_t)E * 4;
                const int64_t per_sm = std::max<int64_t>(1, std::min<int64_t>(4, (228 * 1024) / ((int64_t)L.smem + 2048)));
                L.grid = dim3((unsigned)std::min<int64_t>(P.ntiles, (int64_t)di.num_sms * per_sm));
            }
        }
        if (!ok) {
            ok = plan_strided(L, (int64_t)s, base, di.num_sms, a.dtype);
            if (ok && allow_deep) plan_deep(L, (int64_t)s, di.num_sms);
        }
    }
    if (!ok) {
        set_error("ttv: no launch plan");
        return TL_EUNSUPPORTED;
    }
    return TL_OK;
}

static const char *ttv_regime_name(const TtvLaunch &L) {
    switch (L.regime) {
        case 0: return "strided";
        case 1: return L.rows_tma ? "rows-tma" : (L.bulk ? "staged-bulk" : "staged");
        case 2: return "small-cols";
        case 4: return "strided-box";
        case 5: return "short-fold";
        case 6: return "deep-ring";
        case 7: return "tile-fold";
        case 8: return "cols-tma";
        default: return "small-rows";
    }
}

static bool ttv_needs64(const Canon &cn);

// Host-only description of the plan (tl_plan_describe).
int ttv_describe(const tl_desc &a, int m0, char *buf, size_t len) {
    TtvLaunch L{};
    Canon cn;
    if (canon_contraction(a, m0, 0, cn) && ttv_needs64(cn)) {
        snprintf(buf, len, "{\"O\": %lld, \"K\": %lld, \"I\": %lld, \"ident\": %d, \"regime\": \"generic64\"}",
                 (long long)cn.O, (long long)cn.K, (long long)cn.I, cn.ident ? 1 : 0);
        return TL_OK;
    }
    int rc = ttv_make_plan(a, (const void *)0x100000, m0, L, cn);
    if (rc != TL_OK) return rc;
    if (L.regime == 0) plan_box(cn, L, (int64_t)dtype_size(a.dtype), 0x100000, device_info().num_sms, (int64_t)dtype_size(a.dtype));
    if (L.regime == 1) plan_rows_tma(L, cn, a.dtype, device_info().num_sms);  // needs the driver's encoder
    snprintf(buf, len, "{\"O\": %lld, \"K\": %lld, \"I\": %lld, \"ident\": %d, \"inner_digits\": %d, "
             "\"outer_digits\": %d, \"regime\": \"%s\", \"vec\": %d, \"grid\": %u, \"block\": %u, \"smem\": %zu}",
             (long long)cn.O, (long long)cn.K, (long long)cn.I, cn.ident ? 1 : 0, (int)cn.inner.size(),
             (int)cn.outer.size(), ttv_regime_name(L), L.vec, L.grid.x, L.block.x, L.smem);
    return TL_OK;
}

// Can the small kernel's grid run as one cluster (up to 16 CTAs, non-portable
// above 8) with its shared memory?  Queried once per configuration.
static bool small_cluster_fits(const TtvLaunch &L) {
    static const bool off = getenv("TL_HOPM_NO_CLUSTER") != nullptr;
    if (off) return false;
    auto kern = (L.regime == 3) ? (L.vec == 2 ? ttv_small_kernel<double, double, true, true, true>
                                              : ttv_small_kernel<double, double, true, false, true>)
                                : (L.vec == 2 ? ttv_small_kernel<double, double, false, true, true>
                                              : ttv_small_kernel<double, double, false, false, true>);
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L.smem) != cudaSuccess ||
        cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess) {
        (void)cudaGetLastError();
        return false;
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = L.grid;
    cfg.blockDim = L.block;
    cfg.dynamicSmemBytes = L.smem;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = L.grid.x;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int clusters = 0;
    if (cudaOccupancyMaxActiveClusters(&clusters, kern, &cfg) != cudaSuccess) {
        (void)cudaGetLastError();
        return false;
    }
    return clusters >= 1;
}

// ------------------------------------------------------------- past 2^32
// Index ranges beyond the 32-bit digit maps (O or I >= 2^32, K >= 2^31, or
// a digit that large -- tensors of 2^33+ elements, which a 180 GB B200 can
// hold): one thread per output (o, i), 64-bit digit maps, the same k-ordered
// fold.  Loads coalesce along i when I > 1.  Correctness path: the tuned
// kernels above cover every tensor below that size.
struct TtvParams64 {
    const void *a;
    const void *b;
    void *c;
    const int32_t *stop;
    int64_t b_stride;
    int32_t b_dtype;
    int64_t O, K, I;
    DigitMap64 in_map, out_map;
};

template <class TA, class TC>
__global__ void __launch_bounds__(256) ttv_generic64_kernel(const __grid_constant__ TtvParams64 P) {
    using Acc = typename AccOf<TA>::type;
    if (stop_requested(P.stop)) return;
    const TA *a = (const TA *)P.a;
    const int64_t total = P.O * P.I;
    const int64_t nth = (int64_t)gridDim.x * blockDim.x;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += nth) {
        const int64_t o = t / P.I, i = t - o * P.I;
        const TA *x = a + o * P.K * P.I + i;
        Acc acc = Acc(0);
        for (int64_t k = 0; k < P.K; ++k) acc = fold_step(acc, (Acc)x[k * P.I], load_elem_as<Acc>(P.b, P.b_dtype, k * P.b_stride));
        ((TC *)P.c)[P.out_map.map((uint64_t)o) + P.in_map.map((uint64_t)i)] = narrow<TC>(acc);
    }
}

static bool ttv_needs64(const Canon &cn) {
    if (cn.O > kIdx32 || cn.I > kIdx32 || cn.K > 0x7fffffffll) return true;
    for (auto &d : cn.inner)
        if (d.first > kIdx32) return true;
    for (auto &d : cn.outer)
        if (d.first > kIdx32) return true;
    return false;
}

static int ttv_generic64_enqueue(const tl_desc &a, const void *a_ptr, const Canon &cn, const void *b_ptr,
                                 int32_t b_dtype, int64_t b_stride, int32_t c_dtype, void *c_ptr,
                                 const int32_t *stop, cudaStream_t st) {
    TtvParams64 P{};
    P.a = (const unsigned char *)a_ptr + a.offset * (int64_t)dtype_size(a.dtype);
    P.b = b_ptr;
    P.c = c_ptr;
    P.stop = stop;
    P.b_stride = b_stride;
    P.b_dtype = b_dtype;
    P.O = cn.O;
    P.K = cn.K;
    P.I = cn.I;
    build_map64(cn.inner, P.in_map);
    build_map64(cn.outer, P.out_map);
    if (P.O * P.I == 0) return TL_OK;
    const int64_t grid = std::min<int64_t>((P.O * P.I + 255) / 256, (int64_t)device_info().num_sms * 16);
    if (a.dtype == TL_F32 && c_dtype == TL_F32) ttv_generic64_kernel<float, float><<<(unsigned)grid, 256, 0, st>>>(P);
    else if (a.dtype == TL_F32 && c_dtype == TL_F64) ttv_generic64_kernel<float, double><<<(unsigned)grid, 256, 0, st>>>(P);
    else if (a.dtype == TL_F64 && c_dtype == TL_F64) ttv_generic64_kernel<double, double><<<(unsigned)grid, 256, 0, st>>>(P);
    else if (a.dtype == TL_I64 && c_dtype == TL_I64) ttv_generic64_kernel<int64_t, int64_t><<<(unsigned)grid, 256, 0, st>>>(P);
    else {
        set_error("ttv: unsupported dtype combination (a=%d, c=%d)", a.dtype, c_dtype);
        return TL_EUNSUPPORTED;
    }
    return cuda_status(cudaGetLastError(), "ttv (64-bit index) launch");
}

// Entry used by tl_ttv and by the HOPM orchestration (which passes a stop
// flag and binary64 outputs for float32 storage).
int ttv_enqueue(const tl_desc &a, const void *a_ptr, const void *b_ptr, int32_t b_dtype, int64_t b_stride,
                int32_t c_dtype, void *c_ptr, int m0, const int32_t *stop, cudaStream_t st,
                const FusedNorm *fn, bool pdl, int64_t keep_bytes) {
    TtvLaunch L{};
    Canon cn;
    if (canon_contraction(a, m0, 0, cn) && ttv_needs64(cn)) {
        if (fn != nullptr && fn->enabled) {
            set_error("hopm: index ranges past 2^32 are not supported by the fused normalisation");
            return TL_EUNSUPPORTED;
        }
        return ttv_generic64_enqueue(a, a_ptr, cn, b_ptr, b_dtype, b_stride, c_dtype, c_ptr, stop, st);
    }
    // the short-fold path (a stream + transpose) is for plain ttv calls, not
    // the HOPM chains (stop flag, fused normalisation)
    // the deep-ring kernel stages b in A's type
    int rc = ttv_make_plan(a, a_ptr, m0, L, cn, stop == nullptr && (fn == nullptr || !fn->enabled), b_dtype == a.dtype);
    if (rc != TL_OK) return rc;
    TtvParams &P = L.P;
    if (P.O * P.I == 0) return TL_OK;
    L.pdl = pdl;
    P.keep_k = P.K;  // nothing kept unless set below
    P.keep_cta = INT64_MAX;
    P.keep_tile = INT64_MAX;
    P.l2_stream = 0;
    P.b = b_ptr;
    P.c = c_ptr;
    P.stop = stop;
    P.b_stride = b_stride;
    P.b_dtype = b_dtype;
    if (fn != nullptr && fn->enabled) {
        // the last CTA stages w (= this ttv's output) and its squares in
        // its shared memory
        P.fn = *fn;
        L.smem = std::max(L.smem, 2 * (size_t)fn->n * sizeof(double));
        // few CTAs: normalise inside one thread-block cluster instead
        if ((L.regime == 2 || L.regime == 3) && a.dtype == TL_F64 && c_dtype == TL_F64 && L.grid.x <= 16 &&
            fn->n == P.O * P.I && small_cluster_fits(L))
            L.small_cluster = true;
    } else if (L.regime == 1 && plan_rows_tma(L, cn, a.dtype, device_info().num_sms)) {
        // contracted stride 1: rows through the 2-D TMA tensor map
    } else if (L.regime == 0) {
        // permuted output on the strided regime: the boxed kernel
        if (plan_box(cn, L, (int64_t)dtype_size(a.dtype), (uintptr_t)P.a, device_info().num_sms, (int64_t)dtype_size(c_dtype))) {
            TtvBoxParams &B = L.box;
            B.a = P.a;
            B.b = b_ptr;
            B.c = c_ptr;
            B.stop = stop;
            B.b_stride = b_stride;
            B.b_dtype = b_dtype;
        }
    }
    // L2 reuse only pays for tensors that stream (well past the L2 size)
    const int64_t a_bytes = P.O * P.K * P.I * (int64_t)dtype_size(a.dtype);
    if (keep_bytes > 0 && a_bytes >= 2 * (int64_t)device_info().l2_bytes && !L.small_cluster && L.regime != 4) {
        // the output (normal policy) comes out of the budget first
        const int64_t out_bytes = P.O * P.I * (int64_t)dtype_size(c_dtype);
        const int64_t in_keep = std::max<int64_t>(0, keep_bytes - out_bytes);
        const int64_t s = (int64_t)dtype_size(a.dtype);
        if (L.regime == 0) {
            P.l2_stream = 1;
            L.keep_bytes = in_keep;  // split into keep_k / keep_cta at launch (needs the occupancy)
        } else if (L.rows_tma) {
            P.l2_stream = 1;
            const int64_t rt = (int64_t)L.block.x;  // rows per tile
            const int64_t ntiles = (P.O + rt - 1) / rt;
            P.keep_tile = ntiles - std::min<int64_t>(ntiles, in_keep / (rt * P.K * s));
        }
    }
    if (L.regime == 5) return ttv_short_run(L, a.dtype, c_dtype, c_ptr, st);
    if (L.regime == 7) {
        TtvTileParams &T = L.tile;
        T.a = P.a;
        T.b = b_ptr;
        T.c = c_ptr;
        T.stop = stop;
        T.b_stride = b_stride;
        T.b_dtype = b_dtype;
    }
    cudaError_t e;
    if (a.dtype == TL_F32 && c_dtype == TL_F32) e = launch_typed<float, float>(L, st);
    else if (a.dtype == TL_F32 && c_dtype == TL_F64) e = launch_typed<float, double>(L, st);
    else if (a.dtype == TL_F64 && c_dtype == TL_F64) e = launch_typed<double, double>(L, st);
    else if (a.dtype == TL_I64 && c_dtype == TL_I64) e = launch_typed<int64_t, int64_t>(L, st);
    else {
        set_error("ttv: unsupported dtype combination (a=%d, c=%d)", a.dtype, c_dtype);
        return TL_EUNSUPPORTED;
    }
    return cuda_status(e, "ttv launch");
}

}  // namespace tl
