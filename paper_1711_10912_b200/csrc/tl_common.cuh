// tl_common.cuh -- shared device/host building blocks for the sm_100a kernels.
//
// The reference walks tensors with a recursive MultiIterator
// (iterators.py:80-137; contraction.py:134-194).  Here that is replaced by a
// flat "digit map": a dense tensor of any permutation layout is viewed as
// A[O][K][I] (I = stride of the contracted mode, K its extent), and the
// first-order output offset of an inner index i (or outer index o) is
// sum_d digit_d(i) * ostride_d, where digit_d is a mixed-radix digit
// produced with a precomputed magic-number divider.  Everything a kernel
// needs travels by value as a __grid_constant__ parameter.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "tensorlib_b200.h"

#define TL_MAX_DIGITS TL_MAX_ORDER

// ---------------------------------------------------------------- fast divmod
// Division of a 32-bit unsigned numerator by a runtime-invariant divisor
// (Granlund-Montgomery round-up method): q = (umulhi(n, m) + n) >> s,
// evaluated in 64 bits so it is exact for every n < 2^32.
struct FastDiv {
    uint32_t d, m, s;

    __host__ __device__ FastDiv() : d(1), m(0), s(0) {}
    __host__ explicit FastDiv(uint32_t divisor) { init(divisor); }

    __host__ void init(uint32_t divisor) {
        d = divisor ? divisor : 1u;
        if (d == 1) {
            m = 0;
            s = 0;
            return;
        }
        s = 0;
        while ((1ull << s) < d) ++s;  // s = ceil(log2 d)
        m = (uint32_t)((((1ull << 32) * ((1ull << s) - d)) / d) + 1ull);
    }

    __device__ __forceinline__ uint32_t div(uint32_t n) const {
        uint64_t t = __umulhi(n, m);
        return (uint32_t)((t + n) >> s);
    }
    __device__ __forceinline__ void divmod(uint32_t n, uint32_t &q, uint32_t &r) const {
        q = div(n);
        r = n - q * d;
    }
};

// Mixed-radix digit map: offset(x) = sum_d digit_d(x) * stride[d] with
// digit 0 fastest.  The last digit needs no division (it is the quotient).
struct DigitMap {
    int32_t n;
    FastDiv div[TL_MAX_DIGITS];
    int64_t stride[TL_MAX_DIGITS];

    __device__ __forceinline__ int64_t map(uint32_t x) const {
        int64_t off = 0;
#pragma unroll 1
        for (int d = 0; d < n - 1; ++d) {
            uint32_t q, r;
            div[d].divmod(x, q, r);
            off += (int64_t)r * stride[d];
            x = q;
        }
        if (n > 0) off += (int64_t)x * stride[n - 1];
        return off;
    }
};

// The same map for index spaces past 2^32 (any digit extent, 64-bit
// numerators, native division): the generic fallback kernels for tensors
// whose O, I or volume exceed the 32-bit maps above (the reference's index
// cap is 2^63 - 1, layout.py:48).
struct DigitMap64 {
    int32_t n;
    int64_t ext[TL_MAX_DIGITS];
    int64_t stride[TL_MAX_DIGITS];

    __device__ __forceinline__ int64_t map(uint64_t x) const {
        int64_t off = 0;
#pragma unroll 1
        for (int d = 0; d < n - 1; ++d) {
            const uint64_t e = (uint64_t)ext[d];
            const uint64_t q = x / e;
            off += (int64_t)(x - q * e) * stride[d];
            x = q;
        }
        if (n > 0) off += (int64_t)x * stride[n - 1];
        return off;
    }
};

// ------------------------------------------------------------------ dtypes
template <class T> struct AccOf { using type = double; };
template <> struct AccOf<int64_t> { using type = int64_t; };

// One step of the reference's fold `acc += x * y` (contraction.py:161):
// the product is rounded to binary64, then the sum.  Explicit _rn
// intrinsics forbid FMA contraction so the result is bit-identical.
__device__ __forceinline__ double fold_step(double acc, double x, double y) {
    return __dadd_rn(acc, __dmul_rn(x, y));
}
__device__ __forceinline__ int64_t fold_step(int64_t acc, int64_t x, int64_t y) {
    return (int64_t)((uint64_t)acc + (uint64_t)x * (uint64_t)y);
}

template <class T> __device__ __forceinline__ typename AccOf<T>::type widen(T v) {
    return (typename AccOf<T>::type)v;
}

template <class TC, class Acc> __device__ __forceinline__ TC narrow(Acc v);
template <> __device__ __forceinline__ float narrow<float, double>(double v) { return __double2float_rn(v); }
template <> __device__ __forceinline__ double narrow<double, double>(double v) { return v; }
template <> __device__ __forceinline__ int64_t narrow<int64_t, int64_t>(int64_t v) { return v; }

// Read element k of a (strided, any-dtype) vector operand as the
// accumulation type.
template <class Acc>
__device__ __forceinline__ Acc load_elem_as(const void *p, int32_t dtype, int64_t idx) {
    if (dtype == TL_F32) return (Acc)(((const float *)p)[idx]);
    if (dtype == TL_F64) return (Acc)(((const double *)p)[idx]);
    return (Acc)(((const int64_t *)p)[idx]);
}

// ---------------------------------------------------------- memory helpers
// Streaming 128-bit / 64-bit loads that bypass L1 allocation (each element
// of A is read exactly once).
__device__ __forceinline__ float4 ld_stream_f4(const float *p) {
    float4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                 : "l"(p));
    return v;
}
__device__ __forceinline__ float2 ld_stream_f2(const float *p) {
    float2 v;
    asm volatile("ld.global.nc.L1::no_allocate.v2.f32 {%0,%1}, [%2];" : "=f"(v.x), "=f"(v.y) : "l"(p));
    return v;
}
__device__ __forceinline__ float ld_stream(const float *p) {
    float v;
    asm volatile("ld.global.nc.L1::no_allocate.f32 %0, [%1];" : "=f"(v) : "l"(p));
    return v;
}
__device__ __forceinline__ double2 ld_stream_d2(const double *p) {
    double2 v;
    asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0,%1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
    return v;
}
__device__ __forceinline__ double ld_stream(const double *p) {
    double v;
    asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p));
    return v;
}
__device__ __forceinline__ longlong2 ld_stream_l2(const int64_t *p) {
    longlong2 v;
    asm volatile("ld.global.nc.L1::no_allocate.v2.s64 {%0,%1}, [%2];" : "=l"(v.x), "=l"(v.y) : "l"(p));
    return v;
}
__device__ __forceinline__ int64_t ld_stream(const int64_t *p) {
    int64_t v;
    asm volatile("ld.global.nc.L1::no_allocate.s64 %0, [%1];" : "=l"(v) : "l"(p));
    return v;
}

// cp.async (LDGSTS) global -> shared, 4/8/16 bytes.
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
template <int BYTES> __device__ __forceinline__ void cp_async(void *smem_dst, const void *gmem_src) {
    if constexpr (BYTES == 16) {
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(smem_dst)), "l"(gmem_src));
    } else {
        asm volatile("cp.async.ca.shared.global [%0], [%1], %2;" ::"r"(smem_u32(smem_dst)), "l"(gmem_src),
                     "n"(BYTES));
    }
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;"); }
template <int N> __device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N));
}

// mbarrier + 1-D TMA bulk copy (cp.async.bulk -> SASS UBLKCP).
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_fence_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
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
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
// The barrier's pending count drops when all of this thread's prior cp.async
// copies have landed (counts as one arrival).
__device__ __forceinline__ void cp_async_mbar_arrive(uint64_t *bar) {
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *smem_dst, const void *gmem_src, uint32_t bytes, uint64_t *bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(smem_dst)),
                 "l"(gmem_src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
// Bulk shared -> global store (TMA engine), tracked per thread in bulk groups.
__device__ __forceinline__ void bulk_s2g(void *gmem_dst, const void *smem_src, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gmem_dst),
                 "r"(smem_u32(smem_src)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
// wait until at most N bulk groups still READ their shared source
template <int N> __device__ __forceinline__ void bulk_wait_read() {
    asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
template <int N> __device__ __forceinline__ void bulk_wait() {
    asm volatile("cp.async.bulk.wait_group %0;" ::"n"(N) : "memory");
}

// Programmatic dependent launch (no-ops for a kernel launched without the
// programmatic-serialization attribute): pdl_wait blocks until the previous
// kernel in the stream has completed and its writes are visible;
// pdl_release lets the next kernel start launching once every CTA of this
// one has called it (or exited).
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_release() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

__device__ __forceinline__ bool stop_requested(const int32_t *stop) {
    return stop != nullptr && *(volatile const int32_t *)stop != 0;
}

// ------------------------------------------------------------ host helpers
namespace tl {

struct DeviceInfo {
    int device;
    int num_sms;
    int max_smem_optin;
    int64_t l2_bytes;
};
// Cached per device on first use (no synchronisation; capture-safe after
// the first call on a device).
const DeviceInfo &device_info();

// Thread-local error string (tl_last_error).
void set_error(const char *fmt, ...);
int cuda_status(cudaError_t e, const char *what);

inline size_t dtype_size(int32_t dt) { return dt == TL_F32 ? 4 : 8; }

}  // namespace tl
