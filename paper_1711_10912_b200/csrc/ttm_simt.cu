// ttm_simt.cu -- exact-fold ttm (contraction.py:200-298) for int64 operands
// and for shapes the DMMA GETT does not tile (tiny J or K).
//
// One thread per output C(o, j, i) folds k in order from 0 with separately
// rounded binary64 products and sums -- the reference's arithmetic, so the
// result is bit-identical.  The matrix B is read through L1 (lanes of a warp
// share j or k), A is coalesced along the inner block when I >= 32.
#include "plan.h"
#include "tl_common.cuh"

namespace tl {

struct TtmSimtParams {
    const void *a;
    const void *bm;
    void *c;
    int64_t O, K, I, J;
    int64_t bs0, bs1;  // B strides (rows j, columns k)
    int64_t jstride;   // output stride of j
    int32_t ident;
    DigitMap in_map, out_map;
};

template <class T, class TC>
__global__ void __launch_bounds__(256) ttm_simt_kernel(const __grid_constant__ TtmSimtParams P) {
    using Acc = typename AccOf<T>::type;
    const int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t per_o = P.J * P.I;
    if (gid >= P.O * per_o) return;
    const int64_t o = gid / per_o;
    const int64_t rem = gid - o * per_o;
    const int64_t j = rem / P.I;
    const int64_t i = rem - j * P.I;
    const T *pa = (const T *)P.a + o * P.K * P.I + i;
    const T *pb = (const T *)P.bm + j * P.bs0;
    Acc acc = Acc(0);
#pragma unroll 4
    for (int64_t k = 0; k < P.K; ++k) acc = fold_step(acc, (Acc)pa[k * P.I], (Acc)__ldg(pb + k * P.bs1));
    int64_t off;
    if (P.ident)
        off = (o * P.J + j) * P.I + i;
    else
        off = P.out_map.map((uint32_t)o) + j * P.jstride + P.in_map.map((uint32_t)i);
    ((TC *)P.c)[off] = narrow<TC>(acc);
}

int ttm_simt_enqueue(const tl_desc &a, const void *a_ptr, const tl_desc &bm, const void *b_ptr, void *c_ptr,
                     int m0, cudaStream_t st) {
    const int64_t J = bm.extent[0];
    Canon cn;
    if (!canon_contraction(a, m0, J, cn)) {
        set_error("ttm: operand A is not a dense permutation layout (materialise views first)");
        return TL_EUNSUPPORTED;
    }
    TtmSimtParams P{};
    const size_t s = dtype_size(a.dtype);
    P.a = (const unsigned char *)a_ptr + a.offset * (int64_t)s;
    P.bm = (const unsigned char *)b_ptr + bm.offset * (int64_t)dtype_size(bm.dtype);
    P.c = c_ptr;
    P.O = cn.O;
    P.K = cn.K;
    P.I = cn.I;
    P.J = J;
    P.bs0 = bm.stride[0];
    P.bs1 = bm.stride[1];
    P.jstride = cn.jstride;
    P.ident = cn.ident ? 1 : 0;
    if (!build_map(cn.inner, P.in_map) || !build_map(cn.outer, P.out_map)) return TL_EUNSUPPORTED;
    const int64_t total = P.O * P.J * P.I;
    if (total == 0) return TL_OK;
    const int threads = 256;
    const int64_t grid = (total + threads - 1) / threads;
    if (a.dtype == TL_F64) ttm_simt_kernel<double, double><<<(unsigned)grid, threads, 0, st>>>(P);
    else if (a.dtype == TL_F32) ttm_simt_kernel<float, float><<<(unsigned)grid, threads, 0, st>>>(P);
    else ttm_simt_kernel<int64_t, int64_t><<<(unsigned)grid, threads, 0, st>>>(P);
    return cuda_status(cudaGetLastError(), "ttm launch");
}

}  // namespace tl
