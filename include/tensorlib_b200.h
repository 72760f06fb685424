/*
 * tensorlib_b200.h -- C ABI of the B200-native tensorlib hot path.
 *
 * This is the drop-in boundary.  The reference (tensorlib 0.1.0, pure
 * Python; /root/reference/pkg/src/tensorlib) has no FFI: its "plugin"
 * surface is the Python function signatures fed by the MultiIterator
 * protocol (iterators.py:80-137).  Each entry point below
 * replaces one of those functions; the cited file:line is the reference
 * interface it stands in for.  Python binds this header with ctypes
 * (paper_1711_10912_b200/_abi.py; INTEGRATION.md shows the binding a
 * tensorlib maintainer would add).
 *
 * Conventions
 *  - Plain pointers and sizes only.  Device pointers are CUDA device
 *    addresses; `stream` is a cudaStream_t passed as void* (0 = legacy).
 *  - A tensor operand is (tl_desc, pointer).  tl_desc carries what the
 *    reference's MultiIterator carries (data, pos, strides, extents):
 *    order, element type, base element offset, extents and ELEMENT strides
 *    indexed by dimension (stride[0] belongs to dimension 1), exactly the
 *    tuple compute_strides() returns (layout.py:113-128).
 *  - Modes are one-based, like the reference.
 *  - Outputs are caller-allocated, dense, first-order with zero offsets
 *    (contraction.py:9-12).  The library never allocates device memory;
 *    scratch comes from a caller workspace which must be zero-filled once
 *    before first use (the library leaves it zeroed again).
 *  - Calls are stream-ordered, never synchronise and never query device
 *    state, so they can be captured into a CUDA graph.
 *  - Return value: TL_OK or a TL_E* code; tl_last_error() (thread-local)
 *    describes the last failure.  Python maps TL_EINVAL -> ValueError,
 *    TL_EUNSUPPORTED -> NotImplementedError, TL_ECUDA -> RuntimeError,
 *    TL_EDEGENERATE -> DegenerateInputError (hopm.py:26-35).
 */
#ifndef TENSORLIB_B200_H
#define TENSORLIB_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TL_MAX_ORDER 16
#define TL_ABI_VERSION 1

typedef enum { TL_F32 = 0, TL_F64 = 1, TL_I64 = 2 } tl_dtype;

typedef enum {
    TL_OK = 0,
    TL_EINVAL = 1,       /* argument violates the reference's contract (ValueError) */
    TL_EUNSUPPORTED = 2, /* legal for the reference but not on this path (e.g. non-dense) */
    TL_ECUDA = 3,        /* CUDA launch/runtime error */
    TL_EWORKSPACE = 4,   /* workspace too small */
    TL_EDEGENERATE = 5   /* reserved: HOPM degeneracy is reported through info[] */
} tl_status;

typedef struct tl_desc {
    int32_t order;                 /* p >= 1 */
    int32_t dtype;                 /* tl_dtype */
    int64_t offset;                /* element offset of the first element */
    int64_t extent[TL_MAX_ORDER];  /* n_1..n_p */
    int64_t stride[TL_MAX_ORDER];  /* w_1..w_p, elements */
} tl_desc;

/* ABI version and the compiled device architecture (e.g. 100 for sm_100a). */
int32_t tl_abi_version(void);
int32_t tl_device_arch(void);
/* Thread-local description of the last error (never NULL). */
const char *tl_last_error(void);

/* Optional: initialise the library's CUDA runtime state on the current
 * device and load its small kernels (a process's first call otherwise pays
 * the lazy-loading cost, ~3-12 ms).  No reference counterpart. */
int tl_init(void);

/* ttv -- contraction.py:113-131 (ttv(a, b, mode)).
 * C(i_1..i_{m-1}, i_{m+1}..i_p) = sum_k A(..k..) * b(k), k sequential.
 * b: order-1 of length n_mode, or an (n_mode, 1) column.  c: dense
 * first-order, order p-1.  Every output element is the reference's left
 * fold from 0 in binary64 (float32 storage is widened exactly, the fold is
 * done in binary64 and rounded once on store), so outputs are bit-identical
 * to the reference.  Needs no workspace. */
int tl_ttv(const tl_desc *a, const void *a_ptr, const tl_desc *b, const void *b_ptr,
           const tl_desc *c, void *c_ptr, int32_t mode, void *stream);

/* ttm -- contraction.py:200-227 (ttm(a, bmat, mode)).
 * C(.., j at mode, ..) = sum_k A(.., k at mode, ..) * B(j, k); B is
 * (n_new x n_mode) with its own layout; c: dense first-order, order p.
 * float64: DMMA tensor-core tiles; float32: FFMA tiles; int64: exact. */
int tl_ttm(const tl_desc *a, const void *a_ptr, const tl_desc *bmat, const void *b_ptr,
           const tl_desc *c, void *c_ptr, int32_t mode, void *stream);

/* tl_ttm, plus (when the chosen kernel supports it) the sum of squares of
 * C computed in the same launch's epilogue: ssq_dev[0] = sum C^2,
 * ssq_dev[1] = sqrt(sum C^2) = frobenius_norm(C) (contraction.py:462-464),
 * deterministic, relative error < 1e-12.  *fused (host) is set to 1 when
 * ssq_dev will be written, else 0 (then only C is produced).  ws: the
 * tl_reduce_workspace_bytes() zeroed scratch.  No reference counterpart:
 * this fuses the config-5 chain's norm into its ttm. */
int tl_ttm_ssq(const tl_desc *a, const void *a_ptr, const tl_desc *bmat, const void *b_ptr,
               const tl_desc *c, void *c_ptr, int32_t mode, double *ssq_dev, void *ws,
               size_t ws_bytes, int32_t *fused, void *stream);

/* Workspace bytes needed by tl_inner / tl_frobenius_norm (fixed size). */
size_t tl_reduce_workspace_bytes(void);

/* inner_product_tensors -- contraction.py:457-459 / inner_product_flat
 * elementwise.py:411-433: *result_dev = sum_i a[i] * b[i] over equal
 * shapes, any layouts.  Floating inputs accumulate in binary64 with a
 * compensated (double-double) sum; int64 accumulates exactly mod 2^64.
 * result_dev: device double (floats) or int64 (int64 operands). */
int tl_inner(const tl_desc *a, const void *a_ptr, const tl_desc *b, const void *b_ptr,
             void *result_dev, void *ws, size_t ws_bytes, void *stream);

/* inner_product_flat(a, b, init) -- elementwise.py:411-414: as tl_inner,
 * with the fold starting at *init (a HOST scalar of the result type:
 * double for floating operands, int64 for int64 operands; NULL = 0).  init
 * enters the compensated sum before its single final rounding, as the
 * reference's `acc = init; acc += a*b` starts from it. */
int tl_inner_flat(const tl_desc *a, const void *a_ptr, const tl_desc *b, const void *b_ptr,
                  const void *init, void *result_dev, void *ws, size_t ws_bytes, void *stream);

/* frobenius_norm -- contraction.py:462-464: *result_dev = sqrt(<a, a>). */
int tl_frobenius_norm(const tl_desc *a, const void *a_ptr, double *result_dev,
                      void *ws, size_t ws_bytes, void *stream);

/* times_vectors -- contraction.py:481-519 (explicit-modes form) as ONE
 * cooperative launch: the vectors are applied highest mode first, each step
 * the reference's left fold over k, each intermediate rounded to A's
 * storage type -- bit-identical to the sequence of tl_ttv calls.  modes:
 * one-based, strictly increasing, one per vector (an order-1 remainder is
 * folded like the reference's inner_product_flat).  c: dense first-order,
 * A's float dtype.  Returns TL_EUNSUPPORTED (nothing enqueued) when a step's
 * output is a permutation of its canonical order (e.g. last-order A) or A
 * is not floating; the caller then issues the tl_ttv sequence.  Scratch for
 * the intermediates: tl_times_vectors_workspace_bytes. */
int tl_times_vectors_workspace_bytes(const tl_desc *a, int32_t nvec, const int32_t *modes,
                                     const tl_desc *vdescs, size_t *ws_bytes);
int tl_times_vectors(const tl_desc *a, const void *a_ptr, int32_t nvec, const int32_t *modes,
                     const tl_desc *vdescs, const void *const *vptrs, const tl_desc *c, void *c_ptr,
                     void *ws, size_t ws_bytes, void *stream);

/* hopm -- hopm.py:63-120.  Gauss-Seidel higher-order power method, run
 * entirely on the device.  u_ptrs[r] (r < p) are device float64 vectors of
 * length n_{r+1}: on entry the (already normalised) start vectors, on exit
 * the result.  l_dev[p] receives the final per-mode norms, hist_dev
 * [max_sweeps] the lambda history, info_dev[4] = {sweeps, converged,
 * degenerate_sweep, degenerate_mode} (degenerate_* = 0 unless a mode
 * update had norm 0, hopm.py:107-108).  u0_ptrs: NULL (u_ptrs hold the
 * start vectors) or p device vectors copied into u_ptrs at the start of the
 * run, which makes a captured graph replayable.  resid_dev: NULL, or
 * [max_sweeps] doubles receiving residual(a, state) after every sweep
 * (track_residuals, hopm.py:114-115).  Every step is the reference's
 * arithmetic (ttv folds, sequential norms, IEEE division), so lambda and the
 * vectors are bit-identical to the reference.  a: float64 or float32. */
int tl_hopm_workspace_bytes(const tl_desc *a, size_t *ws_bytes);
int tl_hopm(const tl_desc *a, const void *a_ptr, const double *const *u0_ptrs, double *const *u_ptrs,
            int32_t max_sweeps, double tol, double *l_dev, double *hist_dev, int32_t *info_dev,
            double *resid_dev, void *ws, size_t ws_bytes, void *stream);

/* The same HOPM run captured once into an executable CUDA graph (no host
 * round trip per sweep); launch it with tl_graph_launch.  Pointers and
 * shapes are baked in. */
typedef struct tl_graph_s *tl_graph;
int tl_hopm_graph_create(const tl_desc *a, const void *a_ptr, const double *const *u0_ptrs,
                         double *const *u_ptrs, int32_t max_sweeps, double tol, double *l_dev,
                         double *hist_dev, int32_t *info_dev, double *resid_dev, void *ws,
                         size_t ws_bytes, void *stream, tl_graph *out);
int tl_graph_launch(tl_graph g, void *stream);
int tl_graph_destroy(tl_graph g);

/* Element-wise copy between two tensors of equal shape and dtype with
 * arbitrary layouts/strides: C(i) = A(i) for every multi-index.  This is
 * relayout (tensor.py:167-184) and view materialisation (contraction.py:
 * 539-542) for the container layer. */
int tl_copy(const tl_desc *a, const void *a_ptr, const tl_desc *c, void *c_ptr, void *stream);

/* rank_one_compose -- hopm.py:123-139: out (dense first-order, shape of
 * `shape`) = scale * u_1(i_1) * ... * u_p(i_p), multiplied left to right like
 * the reference.  u: p device float64 vectors; scale_dev: device double. */
int tl_rank_one_compose(const tl_desc *shape, const double *const *u, const double *scale_dev, double *out,
                        void *stream);

/* residual -- hopm.py:142-147: *result_dev = ||A - scale * u_1 o ... o u_p||_F
 * (elementwise differences exactly as the reference forms them; the sum is
 * double-double).  ws: tl_reduce_workspace_bytes() zeroed bytes. */
int tl_residual(const tl_desc *a, const void *a_ptr, const double *const *u, const double *scale_dev,
                double *result_dev, void *ws, size_t ws_bytes, void *stream);

/* Host only (no device access): the launch plan tl_ttv (op 0) or tl_ttm
 * (op 1, matrix rows J, matrix descriptor bmat) would use for operand a and
 * the one-based mode -- the canonical form A[O][K][I], the
 * kernel regime / GETT digit order -- as a JSON object in buf. */
int tl_plan_describe(int32_t op, const tl_desc *a, const tl_desc *bmat, int32_t mode, char *buf, size_t len);

#ifdef __cplusplus
}
#endif
#endif /* TENSORLIB_B200_H */
