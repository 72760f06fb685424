// norm_micro.cu -- standalone timing of float64 sum-of-squares variants at
// config 5's norm size (5,222,400 doubles, 42 MB) to find where the
// reduce kernel's fixed cost goes.  Not part of the package.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/norm_micro norm_micro.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cmath>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); exit(1); } } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

struct DD { double hi, lo; };
__device__ __forceinline__ void two_sum_add(DD &a, double x) {
    const double s = a.hi + x, bp = s - a.hi;
    a.lo += (a.hi - (s - bp)) + (x - bp);
    a.hi = s;
}
__device__ DD block_dd(DD v) {
    __shared__ DD wp[32];
    for (int d = 16; d; d >>= 1) {
        DD o{__shfl_down_sync(~0u, v.hi, d), __shfl_down_sync(~0u, v.lo, d)};
        two_sum_add(v, o.hi); v.lo += o.lo;
    }
    if ((threadIdx.x & 31) == 0) wp[threadIdx.x >> 5] = v;
    __syncthreads();
    DD r{0, 0};
    if (threadIdx.x < 32) {
        if (threadIdx.x < (blockDim.x >> 5)) r = wp[threadIdx.x];
        for (int d = 16; d; d >>= 1) {
            DD o{__shfl_down_sync(~0u, r.hi, d), __shfl_down_sync(~0u, r.lo, d)};
            two_sum_add(r, o.hi); r.lo += o.lo;
        }
    }
    return r;
}

template <bool COMBINE>
__device__ void finish(DD cta, double *partials, unsigned *ticket, double *out) {
    __shared__ bool last;
    if (threadIdx.x == 0) {
        partials[2 * blockIdx.x] = cta.hi;
        partials[2 * blockIdx.x + 1] = cta.lo;
        if (COMBINE) {
            unsigned prev;
            asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(prev) : "l"(ticket) : "memory");
            last = prev == gridDim.x - 1;
        }
    }
    if (!COMBINE) return;
    __syncthreads();
    if (!last) return;
    DD v{0, 0};
    for (int i = threadIdx.x; i < (int)gridDim.x; i += blockDim.x) {
        two_sum_add(v, __ldcg(partials + 2 * i));
        v.lo += __ldcg(partials + 2 * i + 1);
    }
    v = block_dd(v);
    if (threadIdx.x == 0) { *out = sqrt(v.hi + v.lo); *ticket = 0; }
}

// V0/V1: grid-stride, U 16-byte vectors in flight per thread
template <int U, bool COMBINE>
__global__ void __launch_bounds__(256) gs_kernel(const double *a, int64_t n, double *partials, unsigned *ticket, double *out) {
    double s[4] = {0, 0, 0, 0};
    const int64_t nv = n / 2, nt = (int64_t)gridDim.x * blockDim.x;
    int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (; v + (U - 1) * nt < nv; v += U * nt) {
        double2 x[U];
#pragma unroll
        for (int u = 0; u < U; ++u) x[u] = __ldcs((const double2 *)a + v + u * nt);
#pragma unroll
        for (int u = 0; u < U; ++u) { s[(2 * u) & 3] = fma(x[u].x, x[u].x, s[(2 * u) & 3]); s[(2 * u + 1) & 3] = fma(x[u].y, x[u].y, s[(2 * u + 1) & 3]); }
    }
    // predicated tail: the remaining < U vectors in one round trip
    {
        double2 x[U];
#pragma unroll
        for (int u = 0; u < U; ++u) x[u] = (v + u * nt < nv) ? __ldcs((const double2 *)a + v + u * nt) : make_double2(0, 0);
#pragma unroll
        for (int u = 0; u < U; ++u) { s[(2 * u) & 3] = fma(x[u].x, x[u].x, s[(2 * u) & 3]); s[(2 * u + 1) & 3] = fma(x[u].y, x[u].y, s[(2 * u + 1) & 3]); }
    }
    DD t{s[0], 0};
    two_sum_add(t, s[1]); two_sum_add(t, s[2]); two_sum_add(t, s[3]);
    finish<COMBINE>(block_dd(t), partials, ticket, out);
}


// last CTA: one warp folds the partials (no second block-wide reduction)
__device__ void finish_warp(DD cta, double *partials, unsigned *ticket, double *out) {
    __shared__ bool last;
    if (threadIdx.x == 0) {
        partials[2 * blockIdx.x] = cta.hi;
        partials[2 * blockIdx.x + 1] = cta.lo;
        unsigned prev;
        asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(prev) : "l"(ticket) : "memory");
        last = prev == gridDim.x - 1;
    }
    __syncthreads();
    if (!last || threadIdx.x >= 32) return;
    DD v{0, 0};
    for (int i = threadIdx.x; i < (int)gridDim.x; i += 32) {
        two_sum_add(v, __ldcg(partials + 2 * i));
        v.lo += __ldcg(partials + 2 * i + 1);
    }
    for (int d = 16; d; d >>= 1) {
        DD o{__shfl_down_sync(~0u, v.hi, d), __shfl_down_sync(~0u, v.lo, d)};
        two_sum_add(v, o.hi); v.lo += o.lo;
    }
    if (threadIdx.x == 0) { *out = sqrt(v.hi + v.lo); *ticket = 0; }
}

#include <cooperative_groups.h>
// clusters of CL CTAs: rank 0 gathers the cluster's CTA sums through DSMEM,
// only rank 0 writes a partial and takes a ticket
template <int U, int CL>
__global__ void __launch_bounds__(256) gs_cluster_kernel(const double *a, int64_t n, double *partials, unsigned *ticket, double *out) {
    namespace cg = cooperative_groups;
    __shared__ DD mine;
    __shared__ bool last;
    double s[4] = {0, 0, 0, 0};
    const int64_t nv = n / 2, nt = (int64_t)gridDim.x * blockDim.x;
    int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (; v + (U - 1) * nt < nv; v += U * nt) {
        double2 x[U];
#pragma unroll
        for (int u = 0; u < U; ++u) x[u] = __ldcs((const double2 *)a + v + u * nt);
#pragma unroll
        for (int u = 0; u < U; ++u) { s[(2 * u) & 3] = fma(x[u].x, x[u].x, s[(2 * u) & 3]); s[(2 * u + 1) & 3] = fma(x[u].y, x[u].y, s[(2 * u + 1) & 3]); }
    }
    {
        double2 x[U];
#pragma unroll
        for (int u = 0; u < U; ++u) x[u] = (v + u * nt < nv) ? __ldcs((const double2 *)a + v + u * nt) : make_double2(0, 0);
#pragma unroll
        for (int u = 0; u < U; ++u) { s[(2 * u) & 3] = fma(x[u].x, x[u].x, s[(2 * u) & 3]); s[(2 * u + 1) & 3] = fma(x[u].y, x[u].y, s[(2 * u + 1) & 3]); }
    }
    DD t{s[0], 0};
    two_sum_add(t, s[1]); two_sum_add(t, s[2]); two_sum_add(t, s[3]);
    t = block_dd(t);
    cg::cluster_group cl = cg::this_cluster();
    if (threadIdx.x == 0) mine = t;
    cl.sync();
    if (cl.block_rank() == 0) {
        if (threadIdx.x == 0) {
            DD c{0, 0};
            for (int r = 0; r < CL; ++r) {
                const DD *o = cl.map_shared_rank(&mine, r);
                two_sum_add(c, o->hi); c.lo += o->lo;
            }
            const int idx = blockIdx.x / CL, ncl = gridDim.x / CL;
            partials[2 * idx] = c.hi;
            partials[2 * idx + 1] = c.lo;
            unsigned prev;
            asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(prev) : "l"(ticket) : "memory");
            last = prev == ncl - 1;
        }
    }
    cl.sync();  // others keep their smem alive until rank 0 has read it
    if (cl.block_rank() != 0) return;
    __syncthreads();
    if (!last || threadIdx.x >= 32) return;
    DD w{0, 0};
    for (int i = threadIdx.x; i < (int)(gridDim.x / CL); i += 32) {
        two_sum_add(w, __ldcg(partials + 2 * i));
        w.lo += __ldcg(partials + 2 * i + 1);
    }
    for (int d = 16; d; d >>= 1) {
        DD o{__shfl_down_sync(~0u, w.hi, d), __shfl_down_sync(~0u, w.lo, d)};
        two_sum_add(w, o.hi); w.lo += o.lo;
    }
    if (threadIdx.x == 0) { *out = sqrt(w.hi + w.lo); *ticket = 0; }
}

template <int U>
__global__ void __launch_bounds__(256) gs_warpfin_kernel(const double *a, int64_t n, double *partials, unsigned *ticket, double *out) {
    double s[4] = {0, 0, 0, 0};
    const int64_t nv = n / 2, nt = (int64_t)gridDim.x * blockDim.x;
    int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (; v + (U - 1) * nt < nv; v += U * nt) {
        double2 x[U];
#pragma unroll
        for (int u = 0; u < U; ++u) x[u] = __ldcs((const double2 *)a + v + u * nt);
#pragma unroll
        for (int u = 0; u < U; ++u) { s[(2 * u) & 3] = fma(x[u].x, x[u].x, s[(2 * u) & 3]); s[(2 * u + 1) & 3] = fma(x[u].y, x[u].y, s[(2 * u + 1) & 3]); }
    }
    {
        double2 x[U];
#pragma unroll
        for (int u = 0; u < U; ++u) x[u] = (v + u * nt < nv) ? __ldcs((const double2 *)a + v + u * nt) : make_double2(0, 0);
#pragma unroll
        for (int u = 0; u < U; ++u) { s[(2 * u) & 3] = fma(x[u].x, x[u].x, s[(2 * u) & 3]); s[(2 * u + 1) & 3] = fma(x[u].y, x[u].y, s[(2 * u + 1) & 3]); }
    }
    DD t{s[0], 0};
    two_sum_add(t, s[1]); two_sum_add(t, s[2]); two_sum_add(t, s[3]);
    finish_warp(block_dd(t), partials, ticket, out);
}

// V2: contiguous chunk per CTA, all of it requested up front by TMA bulk
// copies (PIECE bytes each, one mbarrier per piece), reduced from smem.
template <int PIECE, int NP>
__global__ void __launch_bounds__(256) bulk_kernel(const double *a, int64_t n, double *partials, unsigned *ticket, double *out) {
    extern __shared__ __align__(128) unsigned char sm[];
    __shared__ __align__(8) uint64_t bar[NP];
    const int64_t per = (n + gridDim.x - 1) / gridDim.x;
    const int64_t per2 = (per + 1) & ~1ll;  // even: 16-byte aligned chunks
    const int64_t b0 = (int64_t)blockIdx.x * per2;
    const int64_t b1 = b0 + per2 < n ? b0 + per2 : n;
    const int64_t cnt = b1 > b0 ? b1 - b0 : 0;
    const int64_t bytes = cnt * 8;
    const int np = (int)((bytes + PIECE - 1) / PIECE);
    if (threadIdx.x == 0) {
        for (int p = 0; p < NP; ++p) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[p])));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        for (int p = 0; p < np; ++p) {
            const uint32_t nb = (uint32_t)((bytes - (int64_t)p * PIECE) < PIECE ? (bytes - (int64_t)p * PIECE) : PIECE);
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar[p])), "r"(nb) : "memory");
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(sm + (size_t)p * PIECE)),
                         "l"((const unsigned char *)(a + b0) + (size_t)p * PIECE), "r"(nb), "r"(smem_u32(&bar[p])) : "memory");
        }
    }
    __syncthreads();
    double s[2] = {0, 0};
    const double2 *x = (const double2 *)sm;
    for (int p = 0; p < np; ++p) {
        asm volatile("{\n\t.reg .pred q;\n\tW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 q, [%0], 0;\n\t@!q bra W_%=;\n\t}" ::"r"(smem_u32(&bar[p])) : "memory");
        const int64_t e0 = (int64_t)p * PIECE / 16, e1 = ((int64_t)p * PIECE + PIECE) / 16 < cnt / 2 ? ((int64_t)p * PIECE + PIECE) / 16 : cnt / 2;
        for (int64_t e = e0 + threadIdx.x; e < e1; e += blockDim.x) {
            const double2 v = x[e];
            s[0] = fma(v.x, v.x, s[0]);
            s[1] = fma(v.y, v.y, s[1]);
        }
    }
    if ((cnt & 1) && threadIdx.x == 0) { const double v = ((const double *)sm)[cnt - 1]; s[0] = fma(v, v, s[0]); }
    DD t{s[0], 0};
    two_sum_add(t, s[1]);
    finish<true>(block_dd(t), partials, ticket, out);
}


template <class F> float timed(cudaStream_t st, F f, double *flush, size_t flush_bytes, bool do_flush, int reps = 20) {
    // graph of reps x (optional flush + f)
    cudaGraph_t g; cudaGraphExec_t ge;
    CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeGlobal));
    for (int r = 0; r < reps; ++r) {
        if (do_flush) CK(cudaMemsetAsync(flush, r & 0xff, flush_bytes, st));
        f();
    }
    CK(cudaStreamEndCapture(st, &g));
    CK(cudaGraphInstantiate(&ge, g, 0));
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    CK(cudaGraphLaunch(ge, st));
    float best = 1e30f;
    for (int it = 0; it < 5; ++it) {
        cudaEventRecord(e0, st);
        CK(cudaGraphLaunch(ge, st));
        cudaEventRecord(e1, st);
        CK(cudaEventSynchronize(e1));
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        best = ms < best ? ms : best;
    }
    cudaGraphExecDestroy(ge); cudaGraphDestroy(g);
    return best * 1e3f / reps;
}

int main(int argc, char **argv) {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const size_t flush_bytes = 512u << 20;
    double *flush; CK(cudaMalloc(&flush, flush_bytes));
    cudaStream_t st; cudaStreamCreate(&st);
    double *parts, *out; unsigned *ticket;
    CK(cudaMalloc(&parts, 1 << 20)); CK(cudaMalloc(&out, 64)); CK(cudaMalloc(&ticket, 64));
    CK(cudaMemset(ticket, 0, 64));
    for (int64_t n : {5222400ll, 20889600ll, 134217728ll}) {
        double *a; CK(cudaMalloc(&a, n * 8));
        std::vector<double> h(n);
        for (int64_t i = 0; i < n; ++i) h[i] = (double)((i * 2654435761ull) % 1000) / 1000.0 - 0.5;
        CK(cudaMemcpy(a, h.data(), n * 8, cudaMemcpyHostToDevice));
        double ref = 0; for (auto v : h) ref += v * v; ref = sqrt(ref);
        const float tf = timed(st, [&] {}, flush, flush_bytes, true);
        auto report = [&](const char *name, auto launch) {
            const float t_hot = timed(st, launch, flush, flush_bytes, false);
            const float t_cold = timed(st, launch, flush, flush_bytes, true) - tf;
            double r; CK(cudaMemcpy(&r, out, 8, cudaMemcpyDeviceToHost));
            printf("n=%lld %-28s back-to-back %7.2f us (%6.0f GB/s)  after-flush %7.2f us (%6.0f GB/s)  relerr %.1e\n", (long long)n, name, t_hot,
                   n * 8 / (t_hot * 1e3), t_cold, n * 8 / (t_cold * 1e3), fabs(r - ref) / ref);
        };
        for (int cps : {4, 8}) {
            char nm[64];
            snprintf(nm, 64, "gs U8 %d/SM x256", cps);
            report(nm, [&] { gs_kernel<8, true><<<sms * cps / (cps == 8 ? 2 : 1), cps == 8 ? 128 : 256, 0, st>>>(a, n, parts, ticket, out); });
        }
        report("gs U16 4/SM x256", [&] { gs_kernel<16, true><<<sms * 4, 256, 0, st>>>(a, n, parts, ticket, out); });
        report("gs U8 4/SM nocombine", [&] { gs_kernel<8, false><<<sms * 4, 256, 0, st>>>(a, n, parts, ticket, out); });
        report("gs U8 4/SM warp-final", [&] { gs_warpfin_kernel<8><<<sms * 4, 256, 0, st>>>(a, n, parts, ticket, out); });
        {
            cudaLaunchConfig_t cfg{};
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeClusterDimension;
            at[0].val.clusterDim.x = 4; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
            cfg.gridDim = dim3(sms * 4); cfg.blockDim = dim3(256); cfg.stream = st; cfg.attrs = at; cfg.numAttrs = 1;
            report("gs U8 4/SM cluster4", [&] { CK(cudaLaunchKernelEx(&cfg, gs_cluster_kernel<8, 4>, (const double *)a, n, parts, ticket, out)); });
            cudaLaunchConfig_t cfg8 = cfg;
            cudaLaunchAttribute at8[1] = {at[0]};
            at8[0].val.clusterDim.x = 8; cfg8.attrs = at8;
            report("gs U8 4/SM cluster8", [&] { CK(cudaLaunchKernelEx(&cfg8, gs_cluster_kernel<8, 8>, (const double *)a, n, parts, ticket, out)); });
        }
        report("gs U4 8/SM x256", [&] { gs_kernel<4, true><<<sms * 8, 256, 0, st>>>(a, n, parts, ticket, out); });
        {
            auto k = bulk_kernel<16384, 13>;
            CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 13 * 16384));
            for (int cps : {1, 2, 4}) {
                const int64_t per = (n + sms * cps - 1) / (sms * cps) * 8;
                if (per > 13 * 16384 / cps * cps && per > 13 * 16384) continue;
                const int smem = (int)(((per + 16383) / 16384) * 16384);
                if (smem * cps > 220 * 1024 || smem > 13 * 16384) continue;
                char nm[64]; snprintf(nm, 64, "bulk %d/SM (%d KB)", cps, smem / 1024);
                report(nm, [&] { k<<<sms * cps, 256, smem, st>>>(a, n, parts, ticket, out); });
            }
        }
        CK(cudaFree(a));
    }
    return 0;
}
