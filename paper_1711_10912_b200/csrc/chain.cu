// chain.cu -- times_vectors (contraction.py:481-519) as ONE cooperative launch.
//
// The reference contracts the highest mode first, one ttv at a time; each
// step's output is a fresh first-order tensor.  Here every step of the chain
// runs inside one persistent cooperative kernel, separated by grid-wide
// barriers: the pass over A (stage 0, the only large read), then the small
// folds of the shrinking intermediates (L2-resident), in the reference's
// mode order.  Each output is still the reference's left fold over k in
// order (fold_step: product and sum rounded separately), each intermediate
// is rounded to the storage type exactly as a separate ttv would store it,
// so the result is bit-identical to the p-1 separate launches.
//
// Two stage executors:
//   stream -- one thread per VEC consecutive outputs of the canonical form
//             X[O][K][I] (contracted stride I), U k-rows of 16-byte loads in
//             flight per thread, b staged in shared memory (the large pass);
//   block  -- a CTA per 32 consecutive outputs: the whole [K][32] block is put
//             in flight with cp.async (all threads), then one warp folds it
//             from shared memory (a latency-bound small fold: one L2 round
//             trip instead of K/U of them).
// Only layouts whose every step has the identity output map qualify (any
// first-order A; intermediates are first-order); others keep the separate
// launches (tl_times_vectors returns TL_EUNSUPPORTED).
#include <cooperative_groups.h>

#include <algorithm>
#include <cstdlib>
#include <mutex>
#include <vector>

#include "plan.h"
#include "tl_common.cuh"

namespace tl {

constexpr int kChainMaxStages = TL_MAX_ORDER;
constexpr int kChainThreads = 256;
constexpr int kChainU = 8;             // k-rows in flight per thread (stream stage)
constexpr int kChainMaxBSmem = 4096;   // b values staged in shared memory (stream stage)

struct ChainStage {
    const void *src;
    void *dst;
    const void *b;
    int32_t b_dtype;
    int64_t b_stride;
    int64_t O, K, I;
    int32_t block;  // executor: 1 block, 0 stream
    int32_t vec;    // stream executor: outputs per thread (1 or 16 / sizeof(T))
    int32_t kc;     // block executor: k rows staged per round
};

struct ChainParams {
    int32_t n;
    int32_t bcap;  // b values staged in shared memory
    ChainStage st[kChainMaxStages];
};

template <class T, int V> __device__ __forceinline__ void load_v(const T *p, T (&x)[V]) {
    if constexpr (V * sizeof(T) == 16) {
        *(uint4 *)x = __ldcs((const uint4 *)p);
    } else {
#pragma unroll
        for (int j = 0; j < V; ++j) x[j] = __ldcs(p + j);
    }
}

template <class T, int V>
__device__ void chain_stream(const ChainStage &S, double *bs, int bcap) {
    const int64_t K = S.K, I = S.I;
    const T *src = (const T *)S.src;
    T *dst = (T *)S.dst;
    const bool bsm = K <= bcap;
    if (bsm)
        for (int64_t k = threadIdx.x; k < K; k += blockDim.x) bs[k] = load_elem_as<double>(S.b, S.b_dtype, k * S.b_stride);
    __syncthreads();
    auto bk = [&](int64_t k) { return bsm ? bs[k] : load_elem_as<double>(S.b, S.b_dtype, k * S.b_stride); };
    const int64_t ivec = I / V;
    const int64_t total = S.O * ivec;
    const int64_t nth = (int64_t)gridDim.x * blockDim.x;
    for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < total; v += nth) {
        const int64_t o = v / ivec, i = (v - o * ivec) * V;
        const T *x = src + o * K * I + i;
        double acc[V];
#pragma unroll
        for (int j = 0; j < V; ++j) acc[j] = 0.0;
        int64_t k = 0;
        for (; k + kChainU <= K; k += kChainU) {
            T r[kChainU][V];
#pragma unroll
            for (int u = 0; u < kChainU; ++u) load_v<T, V>(x + (k + u) * I, r[u]);
#pragma unroll
            for (int u = 0; u < kChainU; ++u) {
                const double b = bk(k + u);
#pragma unroll
                for (int j = 0; j < V; ++j) acc[j] = fold_step(acc[j], (double)r[u][j], b);
            }
        }
        for (; k < K; ++k) {
            T r[V];
            load_v<T, V>(x + k * I, r);
            const double b = bk(k);
#pragma unroll
            for (int j = 0; j < V; ++j) acc[j] = fold_step(acc[j], (double)r[j], b);
        }
        T out[V];
#pragma unroll
        for (int j = 0; j < V; ++j) out[j] = narrow<T, double>(acc[j]);
        if constexpr (V * sizeof(T) == 16) {
            *(uint4 *)(dst + o * I + i) = *(const uint4 *)out;
        } else {
#pragma unroll
            for (int j = 0; j < V; ++j) dst[o * I + i + j] = out[j];
        }
    }
}

template <class T>
__device__ void chain_block(const ChainStage &S, double *bs, T *data) {
    const int64_t K = S.K, I = S.I;
    const int64_t nout = S.O * I;
    const T *src = (const T *)S.src;
    T *dst = (T *)S.dst;
    const int KC = S.kc;
    for (int64_t k = threadIdx.x; k < K; k += blockDim.x) bs[k] = load_elem_as<double>(S.b, S.b_dtype, k * S.b_stride);
    const int64_t nblk = (nout + 31) / 32;
    for (int64_t c = blockIdx.x; c < nblk; c += gridDim.x) {
        const int64_t f0 = c * 32;
        const int nf = (int)(nout - f0 < 32 ? nout - f0 : 32);
        double acc = 0.0;
        for (int64_t k0 = 0; k0 < K; k0 += KC) {
            const int kn = (int)(K - k0 < KC ? K - k0 : KC);
            __syncthreads();  // the previous round's data (and b) are consumed / staged
            // element (k, j): output f0 + j = (o, i), at src[o*K*I + k*I + i]
            for (int e = threadIdx.x; e < kn * 32; e += blockDim.x) {
                const int kk = e >> 5, j = e & 31;
                if (j < nf) {
                    const int64_t f = f0 + j;
                    const int64_t o = f / I, i = f - o * I;
                    cp_async<sizeof(T)>(data + kk * 32 + j, src + o * K * I + (k0 + kk) * I + i);
                }
            }
            cp_async_commit();
            cp_async_wait<0>();
            __syncthreads();
            if (threadIdx.x < 32) {
                const T *col = data + threadIdx.x;
                int kk = 0;
                for (; kk + 8 <= kn; kk += 8) {
                    T x[8];
                    double b[8];
#pragma unroll
                    for (int q = 0; q < 8; ++q) {
                        x[q] = col[(kk + q) * 32];
                        b[q] = bs[k0 + kk + q];
                    }
#pragma unroll
                    for (int q = 0; q < 8; ++q) acc = fold_step(acc, (double)x[q], b[q]);
                }
                for (; kk < kn; ++kk) acc = fold_step(acc, (double)col[kk * 32], bs[k0 + kk]);
            }
        }
        if (threadIdx.x < nf) dst[f0 + threadIdx.x] = narrow<T, double>(acc);
    }
}

template <class T>
__global__ void __launch_bounds__(kChainThreads) ttv_chain_kernel(const __grid_constant__ ChainParams P) {
    namespace cg = cooperative_groups;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    double *bs = (double *)smem_raw;
    T *data = (T *)(smem_raw + (((size_t)P.bcap * sizeof(double) + 15) & ~(size_t)15));
    cg::grid_group grid = cg::this_grid();
    for (int s = 0; s < P.n; ++s) {
        const ChainStage &S = P.st[s];
        if (S.block) {
            chain_block<T>(S, bs, data);
        } else if (S.vec == 16 / (int)sizeof(T)) {
            chain_stream<T, 16 / sizeof(T)>(S, bs, P.bcap);
        } else {
            chain_stream<T, 1>(S, bs, P.bcap);
        }
        if (s + 1 < P.n) grid.sync();  // stage s's outputs are complete and visible
    }
}

template <class T> static int chain_occupancy(size_t smem) {
    static std::mutex mu;
    static std::vector<std::pair<size_t, int>> cache;
    static size_t configured = 0;  // the attribute only grows: a cached smaller size stays launchable
    std::lock_guard<std::mutex> lk(mu);
    auto kern = ttv_chain_kernel<T>;
    if (smem > configured) {
        if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) return 0;
        configured = smem;
    }
    for (auto &c : cache)
        if (c.first == smem) return c.second;
    int occ = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kChainThreads, smem) != cudaSuccess) occ = 0;
    cache.push_back({smem, occ});
    return occ;
}

// stage list -> one cooperative launch.  `descs` are the successive inputs
// (descs[0] = A), `modes` zero-based per stage, outputs in `outs`.
int chain_enqueue(int n, const tl_desc *descs, const void *const *srcs, void *const *outs, const int *modes,
                  const void *const *bptrs, const int32_t *bdtypes, const int64_t *bstrides, cudaStream_t st) {
    if (n < 1 || n > kChainMaxStages) {
        set_error("times_vectors chain: %d stages (1..%d)", n, kChainMaxStages);
        return TL_EINVAL;
    }
    const int32_t dt = descs[0].dtype;
    if (dt != TL_F32 && dt != TL_F64) {
        set_error("times_vectors chain: floating tensors only");
        return TL_EUNSUPPORTED;
    }
    const size_t es = dtype_size(dt);
    const DeviceInfo &di = device_info();
    ChainParams P{};
    P.n = n;
    int64_t kmax_block = 0;
    size_t data_bytes = 0;
    // block executor budget: at most 32 x KC elements staged per round
    static const int64_t kBlockKc = [] {
        const char *ev = getenv("TL_CHAIN_KC");
        return (int64_t)(ev ? atoi(ev) : 256);
    }();
    int64_t kb = 1;
    for (int s = 0; s < n; ++s) {
        Canon cn;
        if (!canon_contraction(descs[s], modes[s], 0, cn) || !cn.ident) {
            set_error("times_vectors chain: step %d has a permuted output map", s);
            return TL_EUNSUPPORTED;
        }
        ChainStage &S = P.st[s];
        S.src = (const unsigned char *)srcs[s] + descs[s].offset * (int64_t)es;
        S.dst = outs[s];
        S.b = bptrs[s];
        S.b_dtype = bdtypes[s];
        S.b_stride = bstrides[s];
        S.O = cn.O;
        S.K = cn.K;
        S.I = cn.I;
        const int64_t nout = S.O * S.I;
        // small outputs (a few per SM), or contracted stride 1: the block executor
        S.block = (nout <= 32 * (int64_t)di.num_sms * 2 || S.I == 1) ? 1 : 0;
        const int V = (int)(16 / es);
        S.vec = (!S.block && S.I % V == 0 && (uintptr_t)S.src % 16 == 0 && (uintptr_t)S.dst % 16 == 0) ? V : 1;
        S.kc = (int)std::min<int64_t>(S.K, kBlockKc);
        if (S.K <= kChainMaxBSmem) kb = std::max<int64_t>(kb, S.K);
        if (S.block) {
            if (S.K > kChainMaxBSmem) {
                set_error("times_vectors chain: K = %lld too long for the block executor", (long long)S.K);
                return TL_EUNSUPPORTED;
            }
            kmax_block = std::max<int64_t>(kmax_block, S.kc);
        }
    }
    data_bytes = (size_t)kmax_block * 32 * es;
    P.bcap = (int32_t)kb;
    const size_t smem = (((size_t)kb * sizeof(double) + 15) & ~(size_t)15) + data_bytes;
    const int occ = (dt == TL_F64) ? chain_occupancy<double>(smem) : chain_occupancy<float>(smem);
    if (occ < 1) {
        set_error("times_vectors chain: kernel does not fit (%zu B shared memory)", smem);
        return TL_EUNSUPPORTED;
    }
    const int grid = di.num_sms * occ;
    void *args[] = {&P};
    cudaError_t e = (dt == TL_F64)
                        ? cudaLaunchCooperativeKernel((const void *)ttv_chain_kernel<double>, grid, kChainThreads, args, smem, st)
                        : cudaLaunchCooperativeKernel((const void *)ttv_chain_kernel<float>, grid, kChainThreads, args, smem, st);
    return cuda_status(e, "times_vectors chain launch");
}

}  // namespace tl
