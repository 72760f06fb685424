// fp64_probe.cu -- FP64 pipe measurements on the B200 (sm_100a):
//   DFMA and DMMA (mma.sync f64 m8n8k4 / m16n8k4 / m16n8k8 / m16n8k16)
//   throughput, DADD dependent latency, and DMMA rounding semantics.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_probe fp64_probe.cu
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)

__global__ void dfma_tput(double *out, int iters) {
    double a[8], b = 1.0000001, c = 0.9999999;
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = threadIdx.x + i;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) a[i] = fma(a[i], b, c);
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += a[i];
    if (s == 12345.0) out[0] = s;
}

__global__ void dadd_latency(double *out, long long *cyc, int iters) {
    double x = out[1], y = out[2];
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        x = __dadd_rn(x, y);
    }
    long long t1 = clock64();
    out[0] = x;
    cyc[0] = t1 - t0;
}

template <int SHAPE>
__global__ void dmma_tput(double *out, int iters) {
    // SHAPE 0: m8n8k4, 1: m16n8k4, 2: m16n8k8, 3: m16n8k16
    double acc[8][4];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = 0.0;
    double a[8], b[4];
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = 1.0 + 1e-3 * (threadIdx.x + i);
#pragma unroll
    for (int i = 0; i < 4; ++i) b[i] = 1.0 - 1e-3 * (threadIdx.x + i);
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int t = 0; t < 8; ++t) {
            if constexpr (SHAPE == 0) {
                asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                             : "+d"(acc[t][0]), "+d"(acc[t][1]) : "d"(a[0]), "d"(b[0]));
            } else if constexpr (SHAPE == 1) {
                asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
                             : "+d"(acc[t][0]), "+d"(acc[t][1]), "+d"(acc[t][2]), "+d"(acc[t][3])
                             : "d"(a[0]), "d"(a[1]), "d"(b[0]));
            } else if constexpr (SHAPE == 2) {
                asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                             : "+d"(acc[t][0]), "+d"(acc[t][1]), "+d"(acc[t][2]), "+d"(acc[t][3])
                             : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b[0]), "d"(b[1]));
            } else {
                asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};"
                             : "+d"(acc[t][0]), "+d"(acc[t][1]), "+d"(acc[t][2]), "+d"(acc[t][3])
                             : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                               "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
            }
        }
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) s += acc[i][j];
    if (s == 12345.0) out[0] = s;
}

// one m8n8k4: D[g][2t+v] = sum_k A[g][k] B[k][2t+v] + C
__global__ void dmma_semantics(const double *A, const double *B, const double *C, double *D) {
    int lane = threadIdx.x, g = lane >> 2, t = lane & 3;
    double a = A[g * 4 + t], b = B[t * 8 + g];
    double c0 = C[g * 8 + 2 * t], c1 = C[g * 8 + 2 * t + 1];
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
    D[g * 8 + 2 * t] = c0;
    D[g * 8 + 2 * t + 1] = c1;
}

static double now_ms(cudaEvent_t a, cudaEvent_t b) { float ms; cudaEventElapsedTime(&ms, a, b); return ms; }

int main() {
    int dev = 0, nsm = 0, clk = 0;
    CK(cudaSetDevice(dev));
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
    printf("SMs %d clock(kHz) %d\n", nsm, clk);
    double *out; long long *cyc;
    CK(cudaMalloc(&out, 1 << 20));
    CK(cudaMalloc(&cyc, 64));
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    // DFMA
    {
        int iters = 20000;
        for (int w = 0; w < 2; ++w) dfma_tput<<<nsm * 4, 256>>>(out, 100);
        cudaEventRecord(e0);
        dfma_tput<<<nsm * 4, 256>>>(out, iters);
        cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
        double ms = now_ms(e0, e1);
        double flops = 2.0 * 8 * iters * (double)nsm * 4 * 256;
        printf("DFMA: %.2f TFLOP/s (%.3f ms)\n", flops / ms / 1e9, ms);
    }
    // DADD latency
    {
        double h[3] = {0, 1.0, 1e-16};
        CK(cudaMemcpy(out, h, sizeof(h), cudaMemcpyHostToDevice));
        dadd_latency<<<1, 1>>>(out, cyc, 100000);
        CK(cudaDeviceSynchronize());
        long long c; CK(cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost));
        printf("DADD dependent latency: %.2f cycles\n", c / 100000.0);
    }
    // DMMA shapes
    const char *names[4] = {"m8n8k4", "m16n8k4", "m16n8k8", "m16n8k16"};
    const double flop_per[4] = {2.0 * 8 * 8 * 4, 2.0 * 16 * 8 * 4, 2.0 * 16 * 8 * 8, 2.0 * 16 * 8 * 16};
    for (int s = 0; s < 4; ++s) {
        for (int wpb : {4, 8, 16}) {
            int iters = 4000;
            auto launch = [&](int it) {
                switch (s) {
                    case 0: dmma_tput<0><<<nsm, wpb * 32>>>(out, it); break;
                    case 1: dmma_tput<1><<<nsm, wpb * 32>>>(out, it); break;
                    case 2: dmma_tput<2><<<nsm, wpb * 32>>>(out, it); break;
                    default: dmma_tput<3><<<nsm, wpb * 32>>>(out, it); break;
                }
            };
            launch(10);
            cudaEventRecord(e0);
            launch(iters);
            cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
            double ms = now_ms(e0, e1);
            double flops = flop_per[s] * 8 * iters * (double)nsm * wpb;
            printf("DMMA %-9s warps/SM %2d: %.2f TFLOP/s\n", names[s], wpb, flops / ms / 1e9);
        }
    }
    // sustained DMMA: back-to-back launches for ~4 s (power/clock steady state)
    {
        const int wpb = 8, iters = 4000;
        double flops1 = 2.0 * 16 * 8 * 8 * 8 * iters * (double)nsm * wpb;
        cudaEventRecord(e0);
        int launches = 0;
        double ms = 0;
        while (ms < 4000.0) {
            for (int r = 0; r < 20; ++r) dmma_tput<2><<<nsm, wpb * 32>>>(out, iters);
            launches += 20;
            cudaEventRecord(e1);
            CK(cudaEventSynchronize(e1));
            ms = now_ms(e0, e1);
        }
        // last window
        cudaEventRecord(e0);
        for (int r = 0; r < 40; ++r) dmma_tput<2><<<nsm, wpb * 32>>>(out, iters);
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        double ms2 = now_ms(e0, e1);
        printf("DMMA m16n8k8 sustained (after %.1f s): %.2f TFLOP/s\n", ms / 1e3, 40 * flops1 / ms2 / 1e9);
    }
    // DMMA semantics: compare with sequential fma chain and mul+add chain
    {
        double hA[32], hB[32], hC[64], hD[64];
        srand(1);
        int n_fma = 0, n_muladd = 0, n_other = 0, n_total = 0;
        for (int trial = 0; trial < 200; ++trial) {
            for (int i = 0; i < 32; ++i) { hA[i] = (rand() / (double)RAND_MAX - 0.5) * (1 << (rand() % 20)); hB[i] = (rand() / (double)RAND_MAX - 0.5) / (1 << (rand() % 20)); }
            for (int i = 0; i < 64; ++i) hC[i] = (rand() / (double)RAND_MAX - 0.5) * (1 << (rand() % 10));
            double *dA = out + 1000, *dB = out + 2000, *dC = out + 3000, *dD = out + 4000;
            CK(cudaMemcpy(dA, hA, sizeof(hA), cudaMemcpyHostToDevice));
            CK(cudaMemcpy(dB, hB, sizeof(hB), cudaMemcpyHostToDevice));
            CK(cudaMemcpy(dC, hC, sizeof(hC), cudaMemcpyHostToDevice));
            dmma_semantics<<<1, 32>>>(dA, dB, dC, dD);
            CK(cudaMemcpy(hD, dD, sizeof(hD), cudaMemcpyDeviceToHost));
            for (int g = 0; g < 8; ++g)
                for (int j = 0; j < 8; ++j) {
                    double f = hC[g * 8 + j], m = hC[g * 8 + j];
                    for (int k = 0; k < 4; ++k) {
                        f = __builtin_fma(hA[g * 4 + k], hB[k * 8 + j], f);
                        volatile double p = hA[g * 4 + k] * hB[k * 8 + j];
                        m = m + p;
                    }
                    double d = hD[g * 8 + j];
                    ++n_total;
                    if (d == f) ++n_fma;
                    if (d == m) ++n_muladd;
                    if (d != f && d != m) ++n_other;
                }
        }
        printf("DMMA semantics over %d outputs: == seq-FMA %d, == mul+add %d, neither %d\n", n_total, n_fma, n_muladd, n_other);
    }
    return 0;
}
