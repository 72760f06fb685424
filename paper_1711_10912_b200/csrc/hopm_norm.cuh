// hopm_norm.cuh -- the per-mode normalisation step of HOPM (hopm.py:106-118)
// as a device routine, so it can run standalone (hopm_normalize_kernel) or
// fused into the tail of the ttv that produced w (last CTA to finish).
//
// Bit-exactness: the norm is the reference's sequential fold
// sqrt(0 + w0*w0 + w1*w1 + ...) done by one thread (separately rounded
// products and sums, IEEE sqrt), u = w / norm uses IEEE division.
#pragma once

#include <cooperative_groups.h>

#include "tl_common.cuh"

namespace tl {

struct HopmCtl {
    int32_t stop;
    int32_t have_prev;
    double prev;
    unsigned int ticket;  // last-CTA counter for fused normalisation
};

struct FusedNorm {
    int32_t enabled;
    int32_t r, p, sweep;
    int64_t n;
    double tol;
    double *u;
    double *l;
    double *hist;
    int32_t *info;
    HopmCtl *ctl;
};

// 0 + x[0] + x[1] + ... in order (one thread).  The next 16 values are
// loaded into registers while the current 16 are added, so the shared-memory
// latency stays off the serial add chain (~8 cycles per term, not ~24).
__device__ __forceinline__ double ordered_sum(const double *x, int64_t n) {
    double acc = 0.0;
    int64_t i = 0;
    if (n >= 16) {
        double cur[16], nxt[16];
#pragma unroll
        for (int q = 0; q < 16; ++q) cur[q] = x[q];
        for (; i + 32 <= n; i += 16) {
#pragma unroll
            for (int q = 0; q < 16; ++q) nxt[q] = x[i + 16 + q];
#pragma unroll
            for (int q = 0; q < 16; ++q) acc = __dadd_rn(acc, cur[q]);
#pragma unroll
            for (int q = 0; q < 16; ++q) cur[q] = nxt[q];
        }
#pragma unroll
        for (int q = 0; q < 16; ++q) acc = __dadd_rn(acc, cur[q]);
        i += 16;
    }
    for (; i < n; ++i) acc = __dadd_rn(acc, x[i]);
    return acc;
}

// Called by every thread of ONE block.  w: n doubles (global, written by
// this or other CTAs before a fence); stage: >= n doubles of shared memory
// or nullptr (then w is folded from global memory).
__device__ __forceinline__ void hopm_normalize_block(const double *w, const FusedNorm &f, double *stage) {
    __shared__ double nrm;
    const int64_t n = f.n;
    double *sq = stage != nullptr ? stage + n : nullptr;
    if (stage != nullptr) {
        // every thread squares its share (the products of the reference's
        // fold, rounded identically); thread 0 then only runs the add chain
        for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
            const double x = __ldcg(w + i);
            stage[i] = x;
            sq[i] = __dmul_rn(x, x);
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        double acc = 0.0;
        if (stage != nullptr) {
            acc = ordered_sum(sq, n);
        } else {
            for (int64_t i = 0; i < n; ++i) {
                const double x = __ldcg(w + i);
                acc = fold_step(acc, x, x);
            }
        }
        const double s = __dsqrt_rn(acc);
        nrm = s;
        if (s == 0.0) {
            f.info[2] = f.sweep;  // DegenerateInputError(sweep, mode), hopm.py:107-108
            f.info[3] = f.r + 1;
            f.info[0] = f.sweep - 1;
            f.ctl->stop = 1;
        } else {
            f.l[f.r] = s;
        }
    }
    __syncthreads();
    const double s = nrm;
    if (s == 0.0) return;
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x)
        f.u[i] = __ddiv_rn(stage != nullptr ? stage[i] : __ldcg(w + i), s);
    if (f.r == f.p - 1 && threadIdx.x == 0) {
        f.info[0] = f.sweep;
        f.hist[f.sweep - 1] = s;  // lambda = l[-1], hopm.py:112-113
        if (f.ctl->have_prev && fabs(s - f.ctl->prev) < f.tol) {
            f.info[1] = 1;  // converged, hopm.py:116-118
            f.ctl->stop = 1;
        }
        f.ctl->prev = s;
        f.ctl->have_prev = 1;
    }
}

// Tail of a ttv kernel: the last CTA to finish normalises w = the ttv output.
// Every thread of every CTA must call this (no early returns before it).
__device__ __forceinline__ void fused_norm_tail(const FusedNorm &f, const double *w, double *stage) {
    if (!f.enabled) return;
    __shared__ bool last;
    __syncthreads();
    if (threadIdx.x == 0) {
        // acq_rel: this CTA's outputs (ordered before by the barrier) are
        // released with the ticket; the last CTA acquires everyone's
        unsigned prev;
        asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(prev) : "l"(&f.ctl->ticket) : "memory");
        last = (prev == gridDim.x - 1);
    }
    __syncthreads();
    if (!last) return;
    hopm_normalize_block(w, f, stage);
    if (threadIdx.x == 0) f.ctl->ticket = 0u;
}

// Bookkeeping after the norm s of mode r is known (hopm.py:106-118); one
// thread.  Returns false on a zero norm (DegenerateInputError).
__device__ __forceinline__ bool hopm_record_norm(const FusedNorm &f, double s) {
    if (s == 0.0) {
        f.info[2] = f.sweep;
        f.info[3] = f.r + 1;
        f.info[0] = f.sweep - 1;
        f.ctl->stop = 1;
        return false;
    }
    f.l[f.r] = s;
    if (f.r == f.p - 1) {
        f.info[0] = f.sweep;
        f.hist[f.sweep - 1] = s;
        if (f.ctl->have_prev && fabs(s - f.ctl->prev) < f.tol) {
            f.info[1] = 1;
            f.ctl->stop = 1;
        }
        f.ctl->prev = s;
        f.ctl->have_prev = 1;
    }
    return true;
}

// Fused normalisation for a ttv launched as ONE thread-block cluster whose
// CTAs each produced <= 32 consecutive entries of w (CTA rank c owns
// w[32c .. 32c+31], held in its own shared `mine`).  No global round trip
// and no last-CTA ticket: after a cluster barrier every CTA gathers w
// through distributed shared memory, folds the same sequential norm
// (bit-identical in every CTA), and writes its own slice of u = w / s.
// `stage` is >= 2n doubles of this CTA's shared memory.
__device__ __forceinline__ void fused_norm_cluster(const FusedNorm &f, const double *mine, double *stage) {
    namespace cg = cooperative_groups;
    cg::cluster_group cl = cg::this_cluster();
    __shared__ double nrm;
    const int64_t n = f.n;
    double *sq = stage + n;
    cl.sync();  // every CTA's `mine` is complete and visible
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
        const double *src = cl.map_shared_rank(mine, (unsigned)(i / 32));
        const double x = src[i % 32];
        stage[i] = x;
        sq[i] = __dmul_rn(x, x);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        const double acc = ordered_sum(sq, n);
        const double s = __dsqrt_rn(acc);
        nrm = s;
        if (cl.block_rank() == 0) hopm_record_norm(f, s);
    }
    __syncthreads();
    const double s = nrm;
    const int64_t base = (int64_t)cl.block_rank() * 32;
    if (s != 0.0 && threadIdx.x < 32 && base + threadIdx.x < n) f.u[base + threadIdx.x] = __ddiv_rn(stage[base + threadIdx.x], s);
    cl.sync();  // no CTA leaves while others may still read its `mine`
}

}  // namespace tl
