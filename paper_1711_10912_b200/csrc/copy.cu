// copy.cu -- C(i) = A(i) between two layouts/stride sets of one shape.
//
// Container-layer support for the hot path: relayout (tensor.py:167-184),
// assign (tensor.py:141-165) and materialising views before a contraction
// (contraction.py:539-542).  The destination is dense; the source may be
// any strided view.  Elements are enumerated in the destination's storage
// order (stores coalesce) and the source offset comes from a digit map of
// the same index.  When the source's fastest dimension differs from the
// destination's, a 32x32 shared-memory tile transposes so that both the
// loads and the stores coalesce.
#include <algorithm>
#include <cstdlib>
#include <vector>

#include "plan.h"
#include "tl_common.cuh"

namespace tl {

struct CopyParams {
    const void *a;
    void *c;
    int64_t n;
    DigitMap amap, cmap;  // linear index (destination storage order) -> offsets
    // tiled transpose: X = destination's fastest dim, Y = source's fastest
    int64_t nX, nY, n_rest, a_sX, a_sY, c_sY, tiles_x, tiles_y;
    DigitMap rest_a, rest_c;
    DigitMap64 amap64, cmap64;  // past 2^32 elements: the generic 64-bit copy
    // rows: runs of row_len elements contiguous in both (16-byte vectors)
    int64_t row_len, n_rows, nvec;
    FastDiv vpr_div;  // vectors per row
};

template <class T> __global__ void __launch_bounds__(256) copy_kernel(const __grid_constant__ CopyParams P) {
    const T *a = (const T *)P.a;
    T *c = (T *)P.c;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < P.n; q += stride)
        c[P.cmap.map((uint32_t)q)] = a[P.amap.map((uint32_t)q)];
}

template <class T> __global__ void __launch_bounds__(256) copy64_kernel(const __grid_constant__ CopyParams P) {
    const T *a = (const T *)P.a;
    T *c = (T *)P.c;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < P.n; q += stride)
        c[P.cmap64.map((uint64_t)q)] = a[P.amap64.map((uint64_t)q)];
}

// Source and destination share their fastest (merged) digit: copy whole
// 16-byte vectors of each row; the row offsets come from the digit maps of
// the row index, evaluated once per vector (not once per element).
template <class T, int U> __global__ void __launch_bounds__(256) copy_rows_kernel(const __grid_constant__ CopyParams P) {
    constexpr int V = 16 / sizeof(T);
    const T *a = (const T *)P.a;
    T *c = (T *)P.c;
    // U vectors in flight per thread
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (; q + (U - 1) * stride < P.nvec; q += U * stride) {
        uint4 x[U];
        int64_t co[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            uint32_t row, v;
            P.vpr_div.divmod((uint32_t)(q + u * stride), row, v);
            co[u] = P.cmap.map(row) + (int64_t)v * V;
            x[u] = __ldcs((const uint4 *)(a + P.amap.map(row) + (int64_t)v * V));
        }
#pragma unroll
        for (int u = 0; u < U; ++u) *(uint4 *)(c + co[u]) = x[u];
    }
    for (; q < P.nvec; q += stride) {
        uint32_t row, v;
        P.vpr_div.divmod((uint32_t)q, row, v);
        const int64_t ao = P.amap.map(row) + (int64_t)v * V, co = P.cmap.map(row) + (int64_t)v * V;
        *(uint4 *)(c + co) = __ldcs((const uint4 *)(a + ao));
    }
}

template <class T> __global__ void __launch_bounds__(256) copy_tiled_kernel(const __grid_constant__ CopyParams P) {
    __shared__ T tile[32][33];
    const T *a = (const T *)P.a;
    T *c = (T *)P.c;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int64_t per_rest = P.tiles_x * P.tiles_y;
    const int64_t tiles = per_rest * P.n_rest;
    for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
        const int64_t rest = t / per_rest;
        const int64_t txy = t - rest * per_rest;
        const int64_t ty = txy / P.tiles_x;
        const int64_t tx = txy - ty * P.tiles_x;
        const int64_t x0 = tx * 32, y0 = ty * 32;
        const int64_t ra = P.rest_a.map((uint32_t)rest), rc = P.rest_c.map((uint32_t)rest);
        for (int xr = wid; xr < 32; xr += 8) {  // lanes along Y: source reads coalesce
            const int64_t x = x0 + xr, y = y0 + lane;
            if (x < P.nX && y < P.nY) tile[xr][lane] = a[ra + x * P.a_sX + y * P.a_sY];
        }
        __syncthreads();
        for (int yr = wid; yr < 32; yr += 8) {  // lanes along X: destination stores coalesce
            const int64_t x = x0 + lane, y = y0 + yr;
            if (x < P.nX && y < P.nY) c[rc + x + y * P.c_sY] = tile[lane][yr];
        }
        __syncthreads();
    }
}

// 64x64 tiles with 16-byte vectors on both sides: the source tile is read
// along Y (unit stride), written transposed into an XOR-swizzled shared
// tile, and stored along X (the destination's unit stride).
constexpr int kCT = 64;

template <class T> __global__ void __launch_bounds__(256) copy_tiled_vec_kernel(const __grid_constant__ CopyParams P) {
    constexpr int V = 16 / sizeof(T);
    constexpr int VR = kCT / V;
    constexpr int NV = kCT * VR / 256;
    __shared__ __align__(16) T ts[kCT * kCT];  // ts[y][x ^ swz(y)]
    auto swz = [](int y) { return ((y / V) & 7) * V; };
    const T *a = (const T *)P.a;
    T *c = (T *)P.c;
    const int64_t per_rest = P.tiles_x * P.tiles_y;
    const int64_t tiles = per_rest * P.n_rest;
    struct Origin {
        int64_t x0, y0, ra, rc;
    };
    auto origin = [&](int64_t t) {
        const int64_t rest = t / per_rest;
        const int64_t txy = t - rest * per_rest;
        const int64_t ty = txy / P.tiles_x;
        const int64_t tx = txy - ty * P.tiles_x;
        return Origin{tx * kCT, ty * kCT, P.rest_a.map((uint32_t)rest), P.rest_c.map((uint32_t)rest)};
    };
    // the next tile's loads are in flight while this tile is transposed and
    // stored (one tile of registers ahead; the loads are the long latency)
    T v[NV][V];
    auto load = [&](const Origin &o) {
#pragma unroll
        for (int q = 0; q < NV; ++q) {
            const int e = threadIdx.x + q * 256;
            const int row = e / VR, vc = (e % VR) * V;  // source row x = row, y = vc..
            *(uint4 *)v[q] = __ldcs((const uint4 *)(a + o.ra + (o.x0 + row) * P.a_sX + o.y0 + vc));
        }
    };
    int64_t t = blockIdx.x;
    if (t >= tiles) return;
    Origin cur = origin(t);
    load(cur);
    for (; t < tiles; t += gridDim.x) {
#pragma unroll
        for (int q = 0; q < NV; ++q) {
            const int e = threadIdx.x + q * 256;
            const int row = e / VR, vc = (e % VR) * V;
#pragma unroll
            for (int cc = 0; cc < V; ++cc) ts[(vc + cc) * kCT + (row ^ swz(vc + cc))] = v[q][cc];
        }
        __syncthreads();
        const int64_t tn = t + gridDim.x;
        Origin nxt = cur;
        if (tn < tiles) {
            nxt = origin(tn);
            load(nxt);
        }
#pragma unroll
        for (int q = 0; q < NV; ++q) {
            const int e = threadIdx.x + q * 256;
            const int row = e / VR, vc = (e % VR) * V;  // destination row y = row, x = vc..
            const uint4 w = *(const uint4 *)(ts + row * kCT + (vc ^ swz(row)));
            __stcs((uint4 *)(c + cur.rc + (cur.y0 + row) * P.c_sY + cur.x0 + vc), w);
        }
        __syncthreads();
        cur = nxt;
    }
}

template <class T> static cudaError_t launch_copy(const CopyParams &P, int kind, int grid, cudaStream_t st) {
    if (kind == 2)
        copy_tiled_vec_kernel<T><<<grid, 256, 0, st>>>(P);
    else if (kind == 1)
        copy_tiled_kernel<T><<<grid, 256, 0, st>>>(P);
    else if (kind == 3)
        copy64_kernel<T><<<grid, 256, 0, st>>>(P);
    else if (kind == 4) {
        static const int u = [] {
            const char *e = getenv("TL_COPY_ROWS_U");
            return e ? atoi(e) : 4;
        }();
        if (u >= 8)
            copy_rows_kernel<T, 8><<<grid, 256, 0, st>>>(P);
        else
            copy_rows_kernel<T, 4><<<grid, 256, 0, st>>>(P);
    }
    else
        copy_kernel<T><<<grid, 256, 0, st>>>(P);
    return cudaGetLastError();
}

// Load the copy kernels' code on the current device (lazy module loading
// otherwise pays ~3-12 ms on a process's first relayout / view copy).
void copy_preload() {
    cudaFuncAttributes fa;
    cudaFuncGetAttributes(&fa, copy_kernel<float>);
    cudaFuncGetAttributes(&fa, copy_kernel<double>);
    cudaFuncGetAttributes(&fa, copy_kernel<int64_t>);
    cudaFuncGetAttributes(&fa, copy_tiled_kernel<float>);
    cudaFuncGetAttributes(&fa, copy_tiled_kernel<double>);
    cudaFuncGetAttributes(&fa, copy_tiled_kernel<int64_t>);
}

int copy_enqueue(const tl_desc &a, const void *a_ptr, const tl_desc &c, void *c_ptr, cudaStream_t st) {
    std::vector<int> dc;
    if (!dense_order(c, dc)) {
        set_error("copy: destination must be dense");
        return TL_EUNSUPPORTED;
    }
    const size_t s = dtype_size(a.dtype);
    CopyParams P{};
    P.a = (const unsigned char *)a_ptr + a.offset * (int64_t)s;
    P.c = (unsigned char *)c_ptr + c.offset * (int64_t)s;
    P.n = volume(c);
    if (P.n == 0) return TL_OK;
    // source's fastest (smallest |stride|) non-trivial dimension
    int Y = -1;
    for (int r = 0; r < a.order; ++r)
        if (a.extent[r] > 1 && (Y < 0 || a.stride[r] < a.stride[Y])) Y = r;
    const int X = dc.empty() ? -1 : dc[0];
    const DeviceInfo &di = device_info();
    int kind = 0;
    int64_t grid;
    // identical dense layouts: a plain device-to-device copy
    {
        std::vector<int> da;
        bool same = dense_order(a, da) && a.order == c.order;
        for (int r = 0; same && r < a.order; ++r) same = (a.extent[r] == 1) || (a.stride[r] == c.stride[r]);
        if (same)
            return cuda_status(cudaMemcpyAsync(P.c, P.a, (size_t)P.n * s, cudaMemcpyDeviceToDevice, st), "copy");
    }
    // the tiled transposes index tiles in 64 bits and the rest digits in 32
    bool rest32 = true;
    for (int r = 0; r < c.order; ++r)
        if (r != X && r != Y && c.extent[r] > kIdx32) rest32 = false;
    if (rest32 && X >= 0 && Y >= 0) rest32 = volume(c) / (c.extent[X] * c.extent[Y]) <= kIdx32;
    if (X >= 0 && Y >= 0 && X != Y && c.extent[X] >= 8 && c.extent[Y] >= 8 && rest32) {
        kind = 1;
        P.nX = c.extent[X];
        P.nY = c.extent[Y];
        P.a_sX = a.stride[X];
        P.a_sY = a.stride[Y];
        P.c_sY = c.stride[Y];
        DigitList ra, rc;
        for (int r : dc) {
            if (r == X || r == Y) continue;
            ra.push_back({c.extent[r], a.stride[r]});
            rc.push_back({c.extent[r], c.stride[r]});
        }
        P.n_rest = 1;
        for (auto &d : rc) P.n_rest *= d.first;
        build_map(ra, P.rest_a);
        build_map(rc, P.rest_c);
        const int64_t V = 16 / (int64_t)s;
        bool vec = P.a_sY == 1 && P.nX % kCT == 0 && P.nY % kCT == 0 && P.a_sX % V == 0 && P.c_sY % V == 0 &&
                   (uintptr_t)P.a % 16 == 0 && (uintptr_t)P.c % 16 == 0;
        for (auto &d : ra) vec = vec && d.second % V == 0;
        for (auto &d : rc) vec = vec && d.second % V == 0;
        if (vec) {
            kind = 2;
            P.tiles_x = P.nX / kCT;
            P.tiles_y = P.nY / kCT;
            static const int64_t per_sm = [] {
                const char *e = getenv("TL_COPY_CTAS_PER_SM");
                return (int64_t)(e ? atoi(e) : 4);
            }();
            grid = std::min<int64_t>(P.tiles_x * P.tiles_y * P.n_rest, (int64_t)di.num_sms * per_sm);
        } else {
            P.tiles_x = (P.nX + 31) / 32;
            P.tiles_y = (P.nY + 31) / 32;
            grid = std::min<int64_t>(P.tiles_x * P.tiles_y * P.n_rest, (int64_t)di.num_sms * 16);
        }
    } else {
        DigitList la, lc;
        for (int r : dc) {
            // merge digits contiguous in both source and destination
            if (!lc.empty() && lc.back().first * lc.back().second == c.stride[r] &&
                la.back().first * la.back().second == a.stride[r]) {
                lc.back().first *= c.extent[r];
                la.back().first *= c.extent[r];
            } else {
                lc.push_back({c.extent[r], c.stride[r]});
                la.push_back({c.extent[r], a.stride[r]});
            }
        }
        grid = std::min<int64_t>((P.n + 255) / 256, (int64_t)di.num_sms * 16);
        const int64_t V = 16 / (int64_t)s;
        bool rows = P.n <= kIdx32 && !la.empty() && la[0].second == 1 && lc[0].second == 1 && la[0].first % V == 0 &&
                    (uintptr_t)P.a % 16 == 0 && (uintptr_t)P.c % 16 == 0;
        for (size_t d = 1; rows && d < la.size(); ++d) rows = la[d].second % V == 0 && lc[d].second % V == 0;
        if (rows) {
            kind = 4;  // whole 16-byte vectors along the shared fastest digit
            P.row_len = la[0].first;
            P.n_rows = P.n / P.row_len;
            P.nvec = P.n / V;
            P.vpr_div.init((uint32_t)(P.row_len / V));
            DigitList ra(la.begin() + 1, la.end()), rc(lc.begin() + 1, lc.end());
            build_map(ra, P.amap);
            build_map(rc, P.cmap);
            static const int64_t rows_per_sm = [] {
                const char *e = getenv("TL_COPY_ROWS_CTAS_PER_SM");
                return (int64_t)(e ? atoi(e) : 8);
            }();
            grid = std::min<int64_t>((P.nvec + 255) / 256, (int64_t)di.num_sms * rows_per_sm);
        } else if (P.n > kIdx32) {
            kind = 3;  // 2^32+ elements: 64-bit digit maps
            build_map64(la, P.amap64);
            build_map64(lc, P.cmap64);
        } else {
            build_map(la, P.amap);
            build_map(lc, P.cmap);
        }
    }
    cudaError_t e;
    if (s == 4) e = launch_copy<float>(P, kind, (int)grid, st);
    else e = launch_copy<double>(P, kind, (int)grid, st);  // f64 and i64 move 8-byte words
    return cuda_status(e, "copy launch");
}

}  // namespace tl
