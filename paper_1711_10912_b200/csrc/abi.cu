#include <algorithm>
// abi.cu -- extern "C" entry points of libtlb200.so (include/tensorlib_b200.h).
//
// Argument checks mirror the reference's errors (contraction.py:123-127,
// 212-222; elementwise.py:69-70; hopm.py:79-97) and return TL_EINVAL so
// the Python layer raises ValueError with the same meaning.
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <deque>
#include <initializer_list>
#include <mutex>
#include <string>
#include <vector>

#include "plan.h"
#include "tl_common.cuh"

namespace tl {

struct FusedNorm;
int ttv_enqueue(const tl_desc &a, const void *a_ptr, const void *b_ptr, int32_t b_dtype, int64_t b_stride,
                int32_t c_dtype, void *c_ptr, int m0, const int32_t *stop, cudaStream_t st,
                const FusedNorm *fn, bool pdl, int64_t keep_bytes = 0);
int ttm_simt_enqueue(const tl_desc &a, const void *a_ptr, const tl_desc &bm, const void *b_ptr, void *c_ptr,
                     int m0, cudaStream_t st);
int ttm_dmma_enqueue(const tl_desc &a, const void *a_ptr, const tl_desc &bm, const void *b_ptr, void *c_ptr,
                     int m0, cudaStream_t st);
int ttm_staged_enqueue(const tl_desc &a, const void *a_ptr, const tl_desc &bm, const void *b_ptr, void *c_ptr,
                       int m0, cudaStream_t st, double *ssq_out = nullptr, void *ssq_ws = nullptr,
                       int32_t *ssq_fused = nullptr);
size_t reduce_workspace_bytes();
int reduce_enqueue(const tl_desc &a, const void *a_ptr, const tl_desc &b, const void *b_ptr, void *result,
                   bool do_sqrt, void *ws, size_t ws_bytes, cudaStream_t st, const void *init = nullptr);
int hopm_workspace(const tl_desc &a, size_t *bytes);
int hopm_enqueue(const tl_desc &a, const void *a_ptr, const double *const *u0, double *const *u, int32_t max_sweeps,
                 double tol, double *l, double *hist, int32_t *info, double *resid, void *ws, size_t ws_bytes,
                 cudaStream_t st);
void copy_preload();
int chain_enqueue(int n, const tl_desc *descs, const void *const *srcs, void *const *outs, const int *modes,
                  const void *const *bptrs, const int32_t *bdtypes, const int64_t *bstrides, cudaStream_t st);
int copy_enqueue(const tl_desc &a, const void *a_ptr, const tl_desc &c, void *c_ptr, cudaStream_t st);
int rank_one_enqueue(const tl_desc &shape, const double *const *u, const double *scale_dev, double *out,
                     cudaStream_t st);
int residual_enqueue(const tl_desc &a, const void *a_ptr, const double *const *u, const double *scale_dev,
                     const int32_t *gate, int32_t gate_value, double *result, void *ws, size_t ws_bytes,
                     cudaStream_t st);
int ttv_describe(const tl_desc &a, int m0, char *buf, size_t len);
int ttm_dmma_describe(const tl_desc &a, const tl_desc &bm, int m0, std::string &out);
int ttm_staged_describe(const tl_desc &a, const tl_desc &bm, int m0, std::string &out);
// ttm_few.cu: J <= 32 for any layout / mode (box of positions along A x along C)
int ttm_few_enqueue(const tl_desc &a, const void *a_ptr, const tl_desc &bm, const void *b_ptr, void *c_ptr, int m0,
                    cudaStream_t st);
int ttm_few_describe(const tl_desc &a, const tl_desc &bm, int m0, std::string &out);
int ttm_few_mode();
// ttm_simt.cu: would the stream / bulk tile kernels (first-order-compatible float64 outputs) take this ttm?
bool ttm_tile_kernels_apply(const tl_desc &a, const tl_desc &bm, int m0);

static thread_local std::string g_error = "no error";

void set_error(const char *fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    g_error = buf;
}

int cuda_status(cudaError_t e, const char *what) {
    if (e == cudaSuccess) return TL_OK;
    set_error("%s: %s", what, cudaGetErrorString(e));
    return TL_ECUDA;
}

// Bytes of a large operand a ttv reads last that stay L2-resident for the
// next pass over the same tensor (TL_TTV_KEEP_MB; ttv.cu TtvParams::keep_*).
static int64_t ttv_keep_bytes() {
    static const int64_t v = [] {
        const char *e = getenv("TL_TTV_KEEP_MB");
        // measured on the config-2 step (12 ttvs of three 1 GiB tensors):
        // 0/96/128/160/200 MB -> 1976/1957/1943/1946/1950 us of ttv
        return (int64_t)(e ? atoll(e) : 128) << 20;
    }();
    return v;
}

const DeviceInfo &device_info() {
    static std::mutex mu;
    static std::deque<DeviceInfo> cache;  // stable references across push_back
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lk(mu);
    for (auto &d : cache)
        if (d.device == dev) return d;
    DeviceInfo d{};
    d.device = dev;
    cudaDeviceGetAttribute(&d.num_sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&d.max_smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    int l2 = 0;
    cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, dev);
    d.l2_bytes = l2 > 0 ? l2 : (126ll << 20);
    if (d.num_sms <= 0) d.num_sms = 148;
    cache.push_back(d);
    return cache.back();
}

static bool check_desc(const tl_desc *d, const char *what) {
    if (d == nullptr) {
        set_error("%s: null descriptor", what);
        return false;
    }
    if (d->order < 1 || d->order > TL_MAX_ORDER) {
        set_error("%s: order %d out of range 1..%d", what, d->order, TL_MAX_ORDER);
        return false;
    }
    if (d->dtype != TL_F32 && d->dtype != TL_F64 && d->dtype != TL_I64) {
        set_error("%s: unknown dtype %d", what, d->dtype);
        return false;
    }
    for (int r = 0; r < d->order; ++r) {
        if (d->extent[r] < 1) {
            set_error("%s: extents must be positive", what);
            return false;
        }
        if (d->stride[r] < 0) {
            set_error("%s: negative strides are not supported", what);
            return false;
        }
    }
    return true;
}

static bool check_ptrs(const char *what, std::initializer_list<const void *> ptrs) {
    for (const void *q : ptrs) {
        if (q == nullptr) {
            set_error("%s: null data pointer", what);
            return false;
        }
    }
    return true;
}

static bool is_first_order_dense(const tl_desc &d) {
    int64_t run = 1;
    for (int r = 0; r < d.order; ++r) {
        if (d.extent[r] > 1 && d.stride[r] != run) return false;
        run *= d.extent[r];
    }
    return true;
}

static bool is_float(int32_t dt) { return dt == TL_F32 || dt == TL_F64; }

}  // namespace tl

using namespace tl;

extern "C" {

int32_t tl_abi_version(void) { return TL_ABI_VERSION; }

int32_t tl_device_arch(void) {
#if defined(TL_ARCH)
    return TL_ARCH;
#else
    return 100;
#endif
}

const char *tl_last_error(void) { return g_error.c_str(); }

int tl_init(void) {
    // the library's runtime state, the current device's attributes and the
    // small-copy kernels, so a process's first hot-path call is not ms-slow
    cudaError_t e = cudaFree(nullptr);
    if (e != cudaSuccess) return cuda_status(e, "init");
    (void)device_info();
    copy_preload();
    return cuda_status(cudaGetLastError(), "init");
}

int tl_ttv(const tl_desc *a, const void *a_ptr, const tl_desc *b, const void *b_ptr, const tl_desc *c, void *c_ptr,
           int32_t mode, void *stream) {
    if (!check_desc(a, "ttv A") || !check_desc(b, "ttv vector") || !check_desc(c, "ttv C")) return TL_EINVAL;
    const int p = a->order;
    if (p < 2) {
        set_error("ttv requires order >= 2, got %d", p);
        return TL_EINVAL;
    }
    if (mode < 1 || mode > p) {
        set_error("mode %d out of range 1..%d", mode, p);
        return TL_EINVAL;
    }
    // vector: order 1, or an (n, 1) column (contraction.py:58-69)
    if (!(b->order == 1 || (b->order == 2 && b->extent[1] == 1))) {
        set_error("ttv vector must be a vector");
        return TL_EINVAL;
    }
    if (b->extent[0] != a->extent[mode - 1]) {
        set_error("ttv vector length %lld does not match extent %lld", (long long)b->extent[0],
                  (long long)a->extent[mode - 1]);
        return TL_EINVAL;
    }
    if (c->order != p - 1 || !is_first_order_dense(*c) || c->offset != 0) {
        set_error("ttv: output must be dense first-order of order p-1");
        return TL_EINVAL;
    }
    for (int r = 0, q = 0; r < p; ++r) {
        if (r == mode - 1) continue;
        if (c->extent[q++] != a->extent[r]) {
            set_error("ttv: output shape mismatch");
            return TL_EINVAL;
        }
    }
    if (is_float(a->dtype) != is_float(b->dtype) || is_float(a->dtype) != is_float(c->dtype)) {
        set_error("ttv: mixed integer/floating operands");
        return TL_EUNSUPPORTED;
    }
    if (!check_ptrs("ttv", {a_ptr, b_ptr, c_ptr})) return TL_EINVAL;
    const void *bp = (const unsigned char *)b_ptr + b->offset * (int64_t)dtype_size(b->dtype);
    return ttv_enqueue(*a, a_ptr, bp, b->dtype, b->stride[0], c->dtype, c_ptr, mode - 1, nullptr,
                       (cudaStream_t)stream, nullptr, false, ttv_keep_bytes());
}

static int ttm_dispatch(const tl_desc *a, const void *a_ptr, const tl_desc *bmat, const void *b_ptr, const tl_desc *c,
                        void *c_ptr, int32_t mode, void *stream, double *ssq_out, void *ssq_ws, int32_t *ssq_fused) {
    if (ssq_fused != nullptr) *ssq_fused = 0;
    if (!check_desc(a, "ttm A") || !check_desc(bmat, "ttm matrix") || !check_desc(c, "ttm C")) return TL_EINVAL;
    const int p = a->order;
    if (p < 2) {
        set_error("ttm requires order >= 2, got %d", p);
        return TL_EINVAL;
    }
    if (mode < 1 || mode > p) {
        set_error("mode %d out of range 1..%d", mode, p);
        return TL_EINVAL;
    }
    if (bmat->order != 2) {
        set_error("ttm matrix must have order 2, got %d", bmat->order);
        return TL_EINVAL;
    }
    if (bmat->extent[1] != a->extent[mode - 1]) {
        set_error("matrix columns %lld do not match extent %lld of mode %d", (long long)bmat->extent[1],
                  (long long)a->extent[mode - 1], mode);
        return TL_EINVAL;
    }
    if (c->order != p || !is_first_order_dense(*c) || c->offset != 0) {
        set_error("ttm: output must be dense first-order of order p");
        return TL_EINVAL;
    }
    for (int r = 0; r < p; ++r) {
        const int64_t want = (r == mode - 1) ? bmat->extent[0] : a->extent[r];
        if (c->extent[r] != want) {
            set_error("ttm: output shape mismatch");
            return TL_EINVAL;
        }
    }
    if (bmat->dtype != a->dtype || c->dtype != a->dtype) {
        set_error("ttm: A, B and C must share a dtype");
        return TL_EUNSUPPORTED;
    }
    if (!check_ptrs("ttm", {a_ptr, b_ptr, c_ptr})) return TL_EINVAL;
    cudaStream_t st = (cudaStream_t)stream;
    // few rows J (<= 32): the staged tile kernels (HBM-bound; DMMA for
    // float64); GEMM-shaped float64 or float32 -> DMMA GETT (float32 widened:
    // its products are exact in binary64, so the FMA chain equals the
    // reference's fold); anything else -> one thread per output
    const bool few_rows = bmat->extent[0] <= 32;
    const bool fp = a->dtype == TL_F64 || a->dtype == TL_F32;
    // few rows, any layout: the box kernel, unless the tuned tile kernels
    // (stream / bulk: first-order-compatible float64 outputs) apply
    if (few_rows && ttm_few_mode() > 0 &&
        (ttm_few_mode() > 1 || !ttm_tile_kernels_apply(*a, *bmat, mode - 1))) {
        int rc = ttm_few_enqueue(*a, a_ptr, *bmat, b_ptr, c_ptr, mode - 1, st);
        if (rc != TL_EUNSUPPORTED) return rc;
    }
    if (few_rows || !fp) {
        int rc = ttm_staged_enqueue(*a, a_ptr, *bmat, b_ptr, c_ptr, mode - 1, st, ssq_out, ssq_ws, ssq_fused);
        if (rc != TL_EUNSUPPORTED) return rc;
    }
    if (fp) {
        int rc = ttm_dmma_enqueue(*a, a_ptr, *bmat, b_ptr, c_ptr, mode - 1, st);
        if (rc != TL_EUNSUPPORTED) return rc;
        if (!few_rows) {
            rc = ttm_staged_enqueue(*a, a_ptr, *bmat, b_ptr, c_ptr, mode - 1, st);
            if (rc != TL_EUNSUPPORTED) return rc;
        }
    }
    return ttm_simt_enqueue(*a, a_ptr, *bmat, b_ptr, c_ptr, mode - 1, st);
}

int tl_ttm(const tl_desc *a, const void *a_ptr, const tl_desc *bmat, const void *b_ptr, const tl_desc *c, void *c_ptr,
           int32_t mode, void *stream) {
    return ttm_dispatch(a, a_ptr, bmat, b_ptr, c, c_ptr, mode, stream, nullptr, nullptr, nullptr);
}

int tl_ttm_ssq(const tl_desc *a, const void *a_ptr, const tl_desc *bmat, const void *b_ptr, const tl_desc *c,
               void *c_ptr, int32_t mode, double *ssq_dev, void *ws, size_t ws_bytes, int32_t *fused, void *stream) {
    if (ssq_dev != nullptr && (ws == nullptr || ws_bytes < reduce_workspace_bytes())) {
        set_error("ttm: workspace of %zu bytes required", reduce_workspace_bytes());
        return TL_EWORKSPACE;
    }
    return ttm_dispatch(a, a_ptr, bmat, b_ptr, c, c_ptr, mode, stream, ssq_dev, ws, fused);
}

size_t tl_reduce_workspace_bytes(void) { return reduce_workspace_bytes(); }

static bool same_shape(const tl_desc &a, const tl_desc &b) {
    if (a.order != b.order) return false;
    for (int r = 0; r < a.order; ++r)
        if (a.extent[r] != b.extent[r]) return false;
    return true;
}

int tl_inner_flat(const tl_desc *a, const void *a_ptr, const tl_desc *b, const void *b_ptr, const void *init,
                  void *result_dev, void *ws, size_t ws_bytes, void *stream) {
    if (!check_desc(a, "inner A") || !check_desc(b, "inner B")) return TL_EINVAL;
    if (!same_shape(*a, *b)) {
        set_error("shape mismatch");
        return TL_EINVAL;
    }
    if (!check_ptrs("inner", {a_ptr, b_ptr, result_dev, ws})) return TL_EINVAL;
    return reduce_enqueue(*a, a_ptr, *b, b_ptr, result_dev, false, ws, ws_bytes, (cudaStream_t)stream, init);
}

int tl_inner(const tl_desc *a, const void *a_ptr, const tl_desc *b, const void *b_ptr, void *result_dev, void *ws,
             size_t ws_bytes, void *stream) {
    return tl_inner_flat(a, a_ptr, b, b_ptr, nullptr, result_dev, ws, ws_bytes, stream);
}

int tl_frobenius_norm(const tl_desc *a, const void *a_ptr, double *result_dev, void *ws, size_t ws_bytes,
                      void *stream) {
    if (!check_desc(a, "norm A")) return TL_EINVAL;
    if (!is_float(a->dtype)) {
        set_error("frobenius_norm requires floating elements");
        return TL_EUNSUPPORTED;
    }
    if (!check_ptrs("frobenius_norm", {a_ptr, result_dev, ws})) return TL_EINVAL;
    return reduce_enqueue(*a, a_ptr, *a, a_ptr, result_dev, true, ws, ws_bytes, (cudaStream_t)stream);
}

int tl_hopm_workspace_bytes(const tl_desc *a, size_t *ws_bytes) {
    if (!check_desc(a, "hopm A") || ws_bytes == nullptr) return TL_EINVAL;
    return hopm_workspace(*a, ws_bytes);
}

static int hopm_check(const tl_desc *a, double *const *u_ptrs, int32_t max_sweeps) {
    if (!check_desc(a, "hopm A")) return TL_EINVAL;
    if (max_sweeps < 1) {
        set_error("max_sweeps must be >= 1");
        return TL_EINVAL;
    }
    if (!is_float(a->dtype)) {
        set_error("hopm requires floating elements");
        return TL_EUNSUPPORTED;
    }
    if (u_ptrs == nullptr) {
        set_error("hopm: null vector array");
        return TL_EINVAL;
    }
    if (a->order > 1) {
        std::vector<int> dims;
        if (!dense_order(*a, dims)) {
            set_error("hopm: A must be a dense permutation layout");
            return TL_EUNSUPPORTED;
        }
    }
    return TL_OK;
}

int tl_hopm(const tl_desc *a, const void *a_ptr, const double *const *u0_ptrs, double *const *u_ptrs,
            int32_t max_sweeps, double tol, double *l_dev, double *hist_dev, int32_t *info_dev, double *resid_dev,
            void *ws, size_t ws_bytes, void *stream) {
    int rc = hopm_check(a, u_ptrs, max_sweeps);
    if (rc != TL_OK) return rc;
    if (!check_ptrs("hopm", {a_ptr, l_dev, hist_dev, info_dev, ws})) return TL_EINVAL;
    return hopm_enqueue(*a, a_ptr, u0_ptrs, u_ptrs, max_sweeps, tol, l_dev, hist_dev, info_dev, resid_dev, ws,
                        ws_bytes, (cudaStream_t)stream);
}

int tl_rank_one_compose(const tl_desc *shape, const double *const *u, const double *scale_dev, double *out,
                        void *stream) {
    if (!check_desc(shape, "rank_one shape") || u == nullptr || scale_dev == nullptr) return TL_EINVAL;
    return rank_one_enqueue(*shape, u, scale_dev, out, (cudaStream_t)stream);
}

int tl_residual(const tl_desc *a, const void *a_ptr, const double *const *u, const double *scale_dev,
                double *result_dev, void *ws, size_t ws_bytes, void *stream) {
    if (!check_desc(a, "residual A") || u == nullptr || scale_dev == nullptr) return TL_EINVAL;
    return residual_enqueue(*a, a_ptr, u, scale_dev, nullptr, 0, result_dev, ws, ws_bytes, (cudaStream_t)stream);
}

struct tl_graph_s {
    cudaGraphExec_t exec;
};

int tl_hopm_graph_create(const tl_desc *a, const void *a_ptr, const double *const *u0_ptrs, double *const *u_ptrs,
                         int32_t max_sweeps, double tol, double *l_dev, double *hist_dev, int32_t *info_dev,
                         double *resid_dev, void *ws, size_t ws_bytes, void *stream, tl_graph *out) {
    int rc = hopm_check(a, u_ptrs, max_sweeps);
    if (rc != TL_OK) return rc;
    if (out == nullptr || !check_ptrs("hopm graph", {a_ptr, l_dev, hist_dev, info_dev, ws})) {
        if (out == nullptr) set_error("hopm graph: null output handle");
        return TL_EINVAL;
    }
    (void)device_info();  // cache device attributes outside the capture
    cudaStream_t st = (cudaStream_t)stream;
    cudaStream_t cap = st;
    bool own = false;
    if (st == nullptr) {  // the legacy stream cannot be captured
        cudaError_t e = cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking);
        if (e != cudaSuccess) return cuda_status(e, "hopm graph stream");
        own = true;
    }
    cudaError_t e = cudaStreamBeginCapture(cap, cudaStreamCaptureModeThreadLocal);
    if (e != cudaSuccess) {
        if (own) cudaStreamDestroy(cap);
        return cuda_status(e, "hopm begin capture");
    }
    rc = hopm_enqueue(*a, a_ptr, u0_ptrs, u_ptrs, max_sweeps, tol, l_dev, hist_dev, info_dev, resid_dev, ws,
                      ws_bytes, cap);
    cudaGraph_t graph = nullptr;
    cudaError_t e2 = cudaStreamEndCapture(cap, &graph);
    if (own) cudaStreamDestroy(cap);
    if (rc != TL_OK) {
        if (graph) cudaGraphDestroy(graph);
        return rc;
    }
    if (e2 != cudaSuccess) return cuda_status(e2, "hopm end capture");
    cudaGraphExec_t exec = nullptr;
    e = cudaGraphInstantiate(&exec, graph, 0);
    cudaGraphDestroy(graph);
    if (e != cudaSuccess) return cuda_status(e, "hopm graph instantiate");
    *out = new tl_graph_s{exec};
    return TL_OK;
}

int tl_graph_launch(tl_graph g, void *stream) {
    if (g == nullptr) return TL_EINVAL;
    return cuda_status(cudaGraphLaunch(g->exec, (cudaStream_t)stream), "graph launch");
}

int tl_graph_destroy(tl_graph g) {
    if (g == nullptr) return TL_OK;
    cudaError_t e = cudaGraphExecDestroy(g->exec);
    delete g;
    return cuda_status(e, "graph destroy");
}

int tl_plan_describe(int32_t op, const tl_desc *a, const tl_desc *bmat, int32_t mode, char *buf, size_t len) {
    if (!check_desc(a, "plan A") || buf == nullptr || len == 0) return TL_EINVAL;
    if (mode < 1 || mode > a->order) {
        set_error("mode %d out of range 1..%d", mode, a->order);
        return TL_EINVAL;
    }
    if (op == 0) return ttv_describe(*a, mode - 1, buf, len);
    if (!check_desc(bmat, "plan matrix") || bmat->order != 2 || bmat->extent[1] != a->extent[mode - 1]) {
        set_error("plan: matrix does not match mode %d", mode);
        return TL_EINVAL;
    }
    // the dispatch order of tl_ttm
    std::string s;
    const bool few_rows = bmat->extent[0] <= 32;
    const bool fp = a->dtype == TL_F64 || a->dtype == TL_F32;
    int rc = TL_EUNSUPPORTED;
    if (few_rows && ttm_few_mode() > 0 && (ttm_few_mode() > 1 || !ttm_tile_kernels_apply(*a, *bmat, mode - 1)))
        rc = ttm_few_describe(*a, *bmat, mode - 1, s);
    if (rc == TL_EUNSUPPORTED && (few_rows || !fp)) rc = ttm_staged_describe(*a, *bmat, mode - 1, s);
    if (rc == TL_EUNSUPPORTED && fp) {
        rc = ttm_dmma_describe(*a, *bmat, mode - 1, s);
        if (rc == TL_EUNSUPPORTED && !few_rows) rc = ttm_staged_describe(*a, *bmat, mode - 1, s);
    }
    if (rc == TL_EUNSUPPORTED) {
        const int64_t F = volume(*a) / a->extent[mode - 1];
        s = std::string("{\"path\": \"simt\", \"F\": ") + std::to_string(F) + "}";
        rc = TL_OK;
    }
    if (rc != TL_OK) return rc;
    snprintf(buf, len, "%s", s.c_str());
    return TL_OK;
}

int tl_copy(const tl_desc *a, const void *a_ptr, const tl_desc *c, void *c_ptr, void *stream) {
    if (!check_desc(a, "copy A") || !check_desc(c, "copy C")) return TL_EINVAL;
    if (!same_shape(*a, *c) || a->dtype != c->dtype) {
        set_error("copy: shape or dtype mismatch");
        return TL_EINVAL;
    }
    if (!check_ptrs("copy", {a_ptr, c_ptr})) return TL_EINVAL;
    return copy_enqueue(*a, a_ptr, *c, c_ptr, (cudaStream_t)stream);
}


// ---------------------------------------------------------------- times_vectors
// The chain of a times_vectors call (contraction.py:481-519): vectors sorted
// by mode, highest first; each step contracts one mode of the previous
// first-order result; an order-1 remainder is contracted as an (n, 1)
// column over mode 1 (the reference's inner_product_flat fold).
struct TvChain {
    int n = 0;
    tl_desc in[TL_MAX_ORDER];
    int m0[TL_MAX_ORDER];
    int vec[TL_MAX_ORDER];  // index into the caller's vector arrays
    int64_t inter_elems = 0;  // largest intermediate (ping-pong halves of the workspace)
};

static int tv_plan(const tl_desc *a, int32_t nvec, const int32_t *modes, const tl_desc *vdescs, TvChain &ch) {
    if (!check_desc(a, "times_vectors A")) return TL_EINVAL;
    const int p = a->order;
    if (nvec < 1 || nvec > p || modes == nullptr || vdescs == nullptr) {
        set_error("times_vectors: %d vectors for order %d", nvec, p);
        return TL_EINVAL;
    }
    int order[TL_MAX_ORDER];
    for (int q = 0; q < nvec; ++q) {
        order[q] = q;
        if (modes[q] < 1 || modes[q] > p) {
            set_error("times_vectors: mode %d out of range 1..%d", modes[q], p);
            return TL_EINVAL;
        }
        if (q && modes[q] <= modes[q - 1]) {
            set_error("times_vectors: modes must be strictly increasing");
            return TL_EINVAL;
        }
    }
    std::sort(order, order + nvec, [&](int x, int y) { return modes[x] > modes[y]; });
    tl_desc cur = *a;
    for (int s = 0; s < nvec; ++s) {
        const int q = order[s];
        int m0 = modes[q] - 1;
        const tl_desc &v = vdescs[q];
        if (!check_desc(&v, "times_vectors vector")) return TL_EINVAL;
        if (cur.order == 1) {  // (n, 1) column over mode 1
            cur.order = 2;
            cur.extent[1] = 1;
            cur.stride[1] = cur.extent[0];
            m0 = 0;
        }
        if (!(v.order == 1 || (v.order == 2 && v.extent[1] == 1)) || v.extent[0] != cur.extent[m0]) {
            set_error("times_vectors vector %d does not match extent %lld", q + 1, (long long)cur.extent[m0]);
            return TL_EINVAL;
        }
        ch.in[s] = cur;
        ch.m0[s] = m0;
        ch.vec[s] = q;
        // next input: cur without dimension m0, first-order float
        tl_desc nx{};
        nx.order = cur.order - 1;
        nx.dtype = a->dtype;
        int64_t run = 1;
        for (int r = 0, t = 0; r < cur.order; ++r) {
            if (r == m0) continue;
            nx.extent[t] = cur.extent[r];
            nx.stride[t] = run;
            run *= cur.extent[r];
            ++t;
        }
        if (s + 1 < nvec) ch.inter_elems = std::max<int64_t>(ch.inter_elems, run);
        cur = nx;
    }
    ch.n = nvec;
    return TL_OK;
}

int tl_times_vectors_workspace_bytes(const tl_desc *a, int32_t nvec, const int32_t *modes, const tl_desc *vdescs,
                                     size_t *bytes) {
    TvChain ch;
    int rc = tv_plan(a, nvec, modes, vdescs, ch);
    if (rc != TL_OK) return rc;
    if (bytes == nullptr) return TL_EINVAL;
    *bytes = 2 * (((size_t)ch.inter_elems * dtype_size(a->dtype) + 255) & ~(size_t)255);
    return TL_OK;
}

int tl_times_vectors(const tl_desc *a, const void *a_ptr, int32_t nvec, const int32_t *modes, const tl_desc *vdescs,
                     const void *const *vptrs, const tl_desc *c, void *c_ptr, void *ws, size_t ws_bytes, void *stream) {
    TvChain ch;
    int rc = tv_plan(a, nvec, modes, vdescs, ch);
    if (rc != TL_OK) return rc;
    if (!check_desc(c, "times_vectors C") || vptrs == nullptr) return TL_EINVAL;
    if (!check_ptrs("times_vectors", {a_ptr, c_ptr})) return TL_EINVAL;
    const size_t half = ((size_t)ch.inter_elems * dtype_size(a->dtype) + 255) & ~(size_t)255;
    if (nvec > 1 && (ws == nullptr || ws_bytes < 2 * half)) {
        set_error("times_vectors: workspace of %zu bytes required", 2 * half);
        return TL_EWORKSPACE;
    }
    const void *srcs[TL_MAX_ORDER];
    void *outs[TL_MAX_ORDER];
    const void *bp[TL_MAX_ORDER];
    int32_t bdt[TL_MAX_ORDER];
    int64_t bst[TL_MAX_ORDER];
    for (int s = 0; s < ch.n; ++s) {
        srcs[s] = s == 0 ? a_ptr : outs[s - 1];
        outs[s] = (s + 1 == ch.n) ? c_ptr : (void *)((unsigned char *)ws + (s % 2) * half);
        const tl_desc &v = vdescs[ch.vec[s]];
        bp[s] = (const unsigned char *)vptrs[ch.vec[s]] + v.offset * (int64_t)dtype_size(v.dtype);
        bdt[s] = v.dtype;
        bst[s] = v.stride[0];
        if (vptrs[ch.vec[s]] == nullptr) {
            set_error("times_vectors: null vector pointer");
            return TL_EINVAL;
        }
    }
    return chain_enqueue(ch.n, ch.in, srcs, outs, ch.m0, bp, bdt, bst, (cudaStream_t)stream);
}

}  // extern "C"
