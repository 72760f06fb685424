// red_probe.cu -- where a cold 42 MB float64 sum of squares spends its time.
//
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o red_probe red_probe.cu
//   ./red_probe [n_doubles]
//
// Kernels (all end with the last-CTA combine of the library's reductions
// unless noted): empty (no work, no combine), combine-only, LDG streaming
// with U 16-byte loads in flight per thread, TMA-bulk streaming with a ring
// of shared-memory slots.  Each is timed with CUDA events around a single
// launch, after a 512 MB memset that evicts L2 (cold) or back to back
// (warm), median of 21.  The bulk kernel also records %globaltimer stamps
// per CTA: start, first slot landed, last slot consumed, and the last CTA's
// end, printed as a timeline relative to the earliest start.
#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#include <vector>

#define CK(x)                                                                                 \
    do {                                                                                      \
        cudaError_t e_ = (x);                                                                 \
        if (e_ != cudaSuccess) {                                                              \
            printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
            exit(1);                                                                          \
        }                                                                                     \
    } while (0)

__device__ __forceinline__ unsigned long long gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_fence_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait_parity(uint64_t *bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *smem_dst, const void *gmem_src, uint32_t bytes, uint64_t *bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(smem_dst)),
                 "l"(gmem_src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

struct P {
    const double *x;
    int64_t n;
    double *partials;
    unsigned *ticket;
    double *result;
    unsigned long long *stamps;  // 4 per CTA
    int chunk, stages;
};

__device__ double block_sum(double v) {
    __shared__ double w[32];
    for (int d = 16; d; d >>= 1) v += __shfl_down_sync(~0u, v, d);
    if ((threadIdx.x & 31) == 0) w[threadIdx.x >> 5] = v;
    __syncthreads();
    double r = 0;
    if (threadIdx.x < 32) {
        r = threadIdx.x < blockDim.x / 32 ? w[threadIdx.x] : 0.0;
        for (int d = 16; d; d >>= 1) r += __shfl_down_sync(~0u, r, d);
    }
    return r;
}

__device__ void finish(const P &p, double cta) {
    __shared__ bool last;
    if (threadIdx.x == 0) {
        p.partials[blockIdx.x] = cta;
        unsigned prev;
        asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(prev) : "l"(p.ticket) : "memory");
        last = prev == gridDim.x - 1;
    }
    __syncthreads();
    if (!last) return;
    double v = 0;
    for (int i = threadIdx.x; i < (int)gridDim.x; i += blockDim.x) v += __ldcg(p.partials + i);
    v = block_sum(v);
    if (threadIdx.x == 0) {
        *p.result = v;
        *p.ticket = 0;
        if (p.stamps) p.stamps[4 * blockIdx.x + 3] = gtime();
    }
}

__global__ void k_empty(P p) {}
__global__ void k_combine(P p) { finish(p, 1.0); }

template <int U> __global__ void __launch_bounds__(256) k_ldg(P p) {
    const int64_t nv = p.n / 2, nt = (int64_t)gridDim.x * blockDim.x;
    double s0 = 0, s1 = 0;
    int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    for (; v + (U - 1) * nt < nv; v += U * nt) {
        double2 x[U];
#pragma unroll
        for (int u = 0; u < U; ++u) x[u] = __ldcs((const double2 *)p.x + v + u * nt);
#pragma unroll
        for (int u = 0; u < U; ++u) s0 = fma(x[u].x, x[u].x, s0), s1 = fma(x[u].y, x[u].y, s1);
    }
    for (; v < nv; v += nt) {
        double2 x = __ldcs((const double2 *)p.x + v);
        s0 = fma(x.x, x.x, s0), s1 = fma(x.y, x.y, s1);
    }
    finish(p, block_sum(s0 + s1));
}

__global__ void __launch_bounds__(256, 1) k_bulk(P p) {
    extern __shared__ __align__(128) unsigned char ring[];
    __shared__ uint64_t full[32];
    const int64_t nvec = p.n / 2;
    const int64_t per = (nvec + gridDim.x - 1) / gridDim.x;
    const int64_t v0 = blockIdx.x * per, v1 = min(nvec, v0 + per);
    const int64_t bytes = v1 > v0 ? (v1 - v0) * 16 : 0;
    const int CH = p.chunk, S = p.stages;
    const int64_t nch = (bytes + CH - 1) / CH;
    const unsigned char *g = (const unsigned char *)p.x + v0 * 16;
    if (threadIdx.x == 0) {
        p.stamps[4 * blockIdx.x] = gtime();
        for (int s = 0; s < S; ++s) mbar_init(&full[s], 1);
        mbar_fence_init();
        for (int64_t i = 0; i < min((int64_t)S, nch); ++i) {
            const uint32_t nb = (uint32_t)min((int64_t)CH, bytes - i * CH);
            mbar_arrive_expect_tx(&full[i], nb);
            bulk_g2s(ring + (size_t)i * CH, g + i * CH, nb, &full[i]);
        }
    }
    __syncthreads();
    double s0 = 0, s1 = 0;
    for (int64_t i = 0; i < nch; ++i) {
        const int s = (int)(i % S);
        mbar_wait_parity(&full[s], (uint32_t)((i / S) & 1));
        if (i == 0 && threadIdx.x == 0) p.stamps[4 * blockIdx.x + 1] = gtime();
        const int nv = (int)(min((int64_t)CH, bytes - i * CH) / 16);
        for (int q = threadIdx.x; q < nv; q += 256) {
            double2 x = *(const double2 *)(ring + (size_t)s * CH + (size_t)q * 16);
            s0 = fma(x.x, x.x, s0), s1 = fma(x.y, x.y, s1);
        }
        __syncthreads();
        if (threadIdx.x == 0 && i + S < nch) {
            const int64_t j = i + S;
            const uint32_t nb = (uint32_t)min((int64_t)CH, bytes - j * CH);
            mbar_arrive_expect_tx(&full[s], nb);
            bulk_g2s(ring + (size_t)s * CH, g + j * CH, nb, &full[s]);
        }
    }
    if (threadIdx.x == 0) p.stamps[4 * blockIdx.x + 2] = gtime();
    finish(p, block_sum(s0 + s1));
}

template <class F> float time_one(F launch, void *flush, size_t flush_bytes, bool cold) {
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    std::vector<float> ts;
    for (int it = 0; it < 23; ++it) {
        if (cold) CK(cudaMemsetAsync(flush, it & 0xff, flush_bytes));
        CK(cudaEventRecord(a));
        launch();
        CK(cudaEventRecord(b));
        CK(cudaEventSynchronize(b));
        float ms;
        CK(cudaEventElapsedTime(&ms, a, b));
        if (it >= 2) ts.push_back(ms * 1e3f);
    }
    std::sort(ts.begin(), ts.end());
    return ts[ts.size() / 2];
}

int main(int argc, char **argv) {
    const int64_t n = argc > 1 ? atoll(argv[1]) : 5222400;
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    double *x, *partials, *result;
    unsigned *ticket;
    unsigned long long *stamps;
    void *flush;
    const size_t flush_bytes = 512u << 20;
    CK(cudaMalloc(&x, n * 8));
    CK(cudaMalloc(&partials, 8192 * 8));
    CK(cudaMalloc(&result, 8));
    CK(cudaMalloc(&ticket, 4));
    CK(cudaMalloc(&stamps, 8192 * 4 * 8));
    CK(cudaMalloc(&flush, flush_bytes));
    CK(cudaMemset(x, 0, n * 8));
    CK(cudaMemset(ticket, 0, 4));
    P p{x, n, partials, ticket, result, nullptr, 16384, 12};
    printf("n = %lld doubles (%.1f MB), %d SMs; times in us (event-timed single launches, median of 21)\n",
           (long long)n, n * 8 / 1e6, sms);
    for (int cold = 1; cold >= 0; --cold) {
        const char *tag = cold ? "cold" : "warm";
        printf("[%s] empty grid=%d: %.2f\n", tag, sms * 4,
               time_one([&] { k_empty<<<sms * 4, 256>>>(p); }, flush, flush_bytes, cold));
        printf("[%s] combine-only grid=%d: %.2f\n", tag, sms,
               time_one([&] { k_combine<<<sms, 256>>>(p); }, flush, flush_bytes, cold));
        printf("[%s] combine-only grid=%d: %.2f\n", tag, sms * 4,
               time_one([&] { k_combine<<<sms * 4, 256>>>(p); }, flush, flush_bytes, cold));
        for (int cps : {4, 8}) {
            printf("[%s] ldg U=8 grid=%d: %.2f\n", tag, sms * cps,
                   time_one([&] { k_ldg<8><<<sms * cps, 256>>>(p); }, flush, flush_bytes, cold));
            printf("[%s] ldg U=4 grid=%d: %.2f\n", tag, sms * cps,
                   time_one([&] { k_ldg<4><<<sms * cps, 256>>>(p); }, flush, flush_bytes, cold));
        }
        for (int ch : {8192, 16384, 32768}) {
            for (int smem_kb : {96, 192}) {
                const int S = std::min(32, smem_kb * 1024 / ch);
                P q = p;
                q.chunk = ch;
                q.stages = S;
                q.stamps = stamps;
                CK(cudaFuncSetAttribute(k_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, S * ch));
                for (int cps : {1, 2}) {
                    if (cps * S * ch > 220 * 1024) continue;
                    const int grid = sms * cps;
                    printf("[%s] bulk chunk=%dK stages=%d grid=%d: %.2f", tag, ch / 1024, S, grid,
                           time_one([&] { k_bulk<<<grid, 256, S * ch>>>(q); }, flush, flush_bytes, cold));
                    std::vector<unsigned long long> st(grid * 4);
                    CK(cudaMemcpy(st.data(), stamps, grid * 4 * 8, cudaMemcpyDeviceToHost));
                    unsigned long long t0 = ~0ull, lastend = 0;
                    std::vector<double> first, end;
                    for (int c = 0; c < grid; ++c) {
                        t0 = std::min(t0, st[4 * c]);
                        lastend = std::max(lastend, st[4 * c + 3]);
                    }
                    for (int c = 0; c < grid; ++c) {
                        first.push_back((st[4 * c + 1] - t0) / 1e3);
                        end.push_back((st[4 * c + 2] - t0) / 1e3);
                    }
                    std::sort(first.begin(), first.end());
                    std::sort(end.begin(), end.end());
                    double maxstart = 0;
                    for (int c = 0; c < grid; ++c) maxstart = std::max(maxstart, (st[4 * c] - t0) / 1e3);
                    printf("   | last CTA start %.2f, first slot med %.2f max %.2f, stream end med %.2f max %.2f, "
                           "combine end %.2f\n",
                           maxstart, first[grid / 2], first.back(), end[grid / 2], end.back(), (lastend - t0) / 1e3);
                }
            }
        }
    }
    return 0;
}
