// hopm_norm.cuh -- the per-mode normalisation step of HOPM (hopm.py:106-118)
// as a device routine, so it can run standalone (hopm_normalize_kernel) or
// fused into the tail of the ttv that produced w (last CTA to finish).
//
// Bit-exactness: the norm is the reference's sequential fold
// sqrt(0 + w0*w0 + w1*w1 + ...) done by one thread (separately rounded
// products and sums, IEEE sqrt), u = w / norm uses IEEE division.
#pragma once

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
            // blocks of 32 with a compile-time trip count: the loads issue
            // ahead of the serial add chain
            int64_t i = 0;
            for (; i + 32 <= n; i += 32) {
#pragma unroll
                for (int q = 0; q < 32; ++q) acc = __dadd_rn(acc, sq[i + q]);
            }
            for (; i < n; ++i) acc = __dadd_rn(acc, sq[i]);
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

}  // namespace tl
