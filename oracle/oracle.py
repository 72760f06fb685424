"""ctypes front-end for the CPU parity oracle (oracle/tl_oracle.c).

TEST INFRASTRUCTURE ONLY -- imported by tests/, __graft_entry__.smoke()
and bench.py's CPU-baseline legs as the checker, never by the product
package.  Every function restates a reference function; see the header of
tl_oracle.c for the file:line map.

Operands are flat numpy buffers plus (shape, element strides by dimension),
i.e. exactly the (data, strides, extents) triple of the reference's
MultiIterator (iterators.py:80-103).  float32 buffers are widened to
float64 (exact) because the reference computes on Python floats.
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "libtloracle.so")
_lib = None

_i64p = ctypes.POINTER(ctypes.c_int64)
_f64p = ctypes.POINTER(ctypes.c_double)
_f32p = ctypes.POINTER(ctypes.c_float)
_i32p = ctypes.POINTER(ctypes.c_int32)


def build() -> str:
    """Compile the oracle with its Makefile (gcc; no GPU needed)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(
            os.path.join(_HERE, "tl_oracle.c")
        ):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        L.tlo_ttv_f64.argtypes = [ctypes.c_int, _i64p, _i64p, _f64p, ctypes.c_int64, _f64p,
                                  ctypes.c_int, _f64p, ctypes.c_int]
        L.tlo_ttv_i64.argtypes = [ctypes.c_int, _i64p, _i64p, _i64p, ctypes.c_int64, _i64p,
                                  ctypes.c_int, _i64p, ctypes.c_int]
        L.tlo_ttv_f32in.argtypes = [ctypes.c_int, _i64p, _i64p, _f32p, ctypes.c_int64, _f32p,
                                    ctypes.c_int, _f64p, ctypes.c_int]
        L.tlo_ttm_f64.argtypes = [ctypes.c_int, _i64p, _i64p, _f64p, ctypes.c_int64,
                                  ctypes.c_int64, ctypes.c_int64, _f64p, ctypes.c_int, _f64p,
                                  _i64p, ctypes.c_int64, ctypes.c_int]
        L.tlo_ttm_canon_f64.argtypes = [ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, _f64p, ctypes.c_int64,
                                        ctypes.c_int64, ctypes.c_int64, _f64p, _f64p, ctypes.c_int, ctypes.c_int]
        L.tlo_ttm_i64.argtypes = [ctypes.c_int, _i64p, _i64p, _i64p, ctypes.c_int64,
                                  ctypes.c_int64, ctypes.c_int64, _i64p, ctypes.c_int, _i64p,
                                  _i64p, ctypes.c_int64, ctypes.c_int]
        L.tlo_inner_f64.argtypes = [ctypes.c_int, _i64p, _i64p, _f64p, _i64p, _f64p, ctypes.c_double]
        L.tlo_inner_f64.restype = ctypes.c_double
        L.tlo_inner_i64.argtypes = [ctypes.c_int, _i64p, _i64p, _i64p, _i64p, _i64p, ctypes.c_int64]
        L.tlo_inner_i64.restype = ctypes.c_int64
        L.tlo_norm_f64.argtypes = [ctypes.c_int, _i64p, _i64p, _f64p]
        L.tlo_norm_f64.restype = ctypes.c_double
        L.tlo_inner_flat_mt_f64.argtypes = [ctypes.c_int64, _f64p, _f64p, ctypes.c_int]
        L.tlo_inner_flat_mt_f64.restype = ctypes.c_double
        L.tlo_inner_flat_mt_f32.argtypes = [ctypes.c_int64, _f32p, _f32p, ctypes.c_int]
        L.tlo_inner_flat_mt_f32.restype = ctypes.c_double
        L.tlo_hopm_f64.argtypes = [ctypes.c_int, _i64p, _i64p, _f64p, ctypes.c_int, ctypes.c_double,
                                   _f64p, _f64p, _f64p, _f64p, _i32p, ctypes.c_int]
        L.tlo_max_threads.restype = ctypes.c_int
        _lib = L
    return _lib


def max_threads() -> int:
    return lib().tlo_max_threads()


def _i64(seq):
    arr = np.ascontiguousarray(np.asarray(seq, dtype=np.int64))
    return arr, arr.ctypes.data_as(_i64p)


def _ptr(arr, kind):
    return arr.ctypes.data_as({"f64": _f64p, "f32": _f32p, "i64": _i64p}[kind])


def _flat(buf, dtype):
    arr = np.asarray(buf)
    if arr.dtype != dtype:
        arr = arr.astype(dtype)
    return np.ascontiguousarray(arr.reshape(-1))


def first_order_strides(shape):
    """compute_strides(shape, (1..p)) -- layout.py:113-128."""
    out, run = [], 1
    for n in shape:
        out.append(run)
        run *= n
    return tuple(out)


def ttv(buf, shape, strides, b, mode, nthreads=0, b_stride=1):
    """contraction.py:113 -- returns the first-order output buffer.

    float64 output for float inputs (the reference computes in binary64),
    int64 for integer inputs."""
    shape = tuple(int(n) for n in shape)
    p = len(shape)
    nout = int(np.prod(shape)) // shape[mode - 1]
    s, sp = _i64(shape)
    w, wp = _i64(strides)
    arr = np.asarray(buf)
    if arr.dtype.kind in "iu":
        a = _flat(arr, np.int64)
        bv = _flat(b, np.int64)
        c = np.empty(nout, dtype=np.int64)
        rc = lib().tlo_ttv_i64(p, sp, wp, _ptr(a, "i64"), b_stride, _ptr(bv, "i64"), mode,
                               _ptr(c, "i64"), nthreads)
    elif arr.dtype == np.float32 and np.asarray(b).dtype == np.float32:
        a = _flat(arr, np.float32)
        bv = _flat(b, np.float32)
        c = np.empty(nout, dtype=np.float64)
        rc = lib().tlo_ttv_f32in(p, sp, wp, _ptr(a, "f32"), b_stride, _ptr(bv, "f32"), mode,
                                 _ptr(c, "f64"), nthreads)
    else:
        a = _flat(arr, np.float64)
        bv = _flat(b, np.float64)
        c = np.empty(nout, dtype=np.float64)
        rc = lib().tlo_ttv_f64(p, sp, wp, _ptr(a, "f64"), b_stride, _ptr(bv, "f64"), mode,
                               _ptr(c, "f64"), nthreads)
    if rc != 0:
        raise ValueError("oracle ttv: invalid arguments")
    return c


def ttm(buf, shape, strides, bmat, bshape, bstrides, mode, nthreads=0, select=None):
    """contraction.py:200 -- first-order output buffer (or the outputs at
    the first-order linear indices in ``select``)."""
    shape = tuple(int(n) for n in shape)
    p = len(shape)
    J = int(bshape[0])
    nout = int(np.prod(shape)) // shape[mode - 1] * J
    s, sp = _i64(shape)
    w, wp = _i64(strides)
    if select is not None:
        sel, selp = _i64(select)
        nsel = len(sel)
        nres = nsel
    else:
        sel, selp, nsel, nres = None, None, 0, nout
    arr = np.asarray(buf)
    if arr.dtype.kind in "iu":
        a = _flat(arr, np.int64)
        bm = _flat(bmat, np.int64)
        c = np.empty(nres, dtype=np.int64)
        rc = lib().tlo_ttm_i64(p, sp, wp, _ptr(a, "i64"), J, int(bstrides[0]), int(bstrides[1]),
                               _ptr(bm, "i64"), mode, _ptr(c, "i64"), selp, nsel, nthreads)
    else:
        a = _flat(arr, np.float64)
        bm = _flat(bmat, np.float64)
        c = np.empty(nres, dtype=np.float64)
        rc = lib().tlo_ttm_f64(p, sp, wp, _ptr(a, "f64"), J, int(bstrides[0]), int(bstrides[1]),
                               _ptr(bm, "f64"), mode, _ptr(c, "f64"), selp, nsel, nthreads)
    if rc != 0:
        raise ValueError("oracle ttm: invalid arguments")
    return c


def inner(abuf, shape, astrides, bbuf, bstrides, init=0):
    """inner_product_flat (elementwise.py:411-433), multi-index order."""
    shape = tuple(int(n) for n in shape)
    s, sp = _i64(shape)
    wa, wap = _i64(astrides)
    wb, wbp = _i64(bstrides)
    A, B = np.asarray(abuf), np.asarray(bbuf)
    if A.dtype.kind in "iu" and B.dtype.kind in "iu":
        a, b = _flat(A, np.int64), _flat(B, np.int64)
        return int(lib().tlo_inner_i64(len(shape), sp, wap, _ptr(a, "i64"), wbp, _ptr(b, "i64"), int(init)))
    a, b = _flat(A, np.float64), _flat(B, np.float64)
    return float(lib().tlo_inner_f64(len(shape), sp, wap, _ptr(a, "f64"), wbp, _ptr(b, "f64"), float(init)))


def norm(abuf, shape, strides):
    """frobenius_norm (contraction.py:462-464)."""
    shape = tuple(int(n) for n in shape)
    s, sp = _i64(shape)
    w, wp = _i64(strides)
    a = _flat(abuf, np.float64)
    return float(lib().tlo_norm_f64(len(shape), sp, wp, _ptr(a, "f64")))


def inner_flat_mt(abuf, bbuf, nthreads=0):
    """Multi-core partial-fold inner product over same-layout buffers (CPU
    baseline timing only; not bit-identical to the reference)."""
    A, B = np.asarray(abuf), np.asarray(bbuf)
    if A.dtype == np.float32 and B.dtype == np.float32:
        a, b = _flat(A, np.float32), _flat(B, np.float32)
        return float(lib().tlo_inner_flat_mt_f32(a.size, _ptr(a, "f32"), _ptr(b, "f32"), nthreads))
    a, b = _flat(A, np.float64), _flat(B, np.float64)
    return float(lib().tlo_inner_flat_mt_f64(a.size, _ptr(a, "f64"), _ptr(b, "f64"), nthreads))


class OracleDegenerate(ArithmeticError):
    def __init__(self, sweep, mode):
        super().__init__(f"zero vector at normalization (sweep {sweep}, mode {mode})")
        self.sweep, self.mode = sweep, mode


def hopm(buf, shape, strides, max_sweeps=50, tol=1e-10, u0=None, nthreads=0):
    """hopm.py:63-120.  Returns dict(u=[...], l=[...], lambda_history,
    sweeps, converged)."""
    shape = tuple(int(n) for n in shape)
    p = len(shape)
    s, sp = _i64(shape)
    w, wp = _i64(strides)
    a = _flat(buf, np.float64)
    tot = sum(shape)
    u_out = np.zeros(tot, dtype=np.float64)
    l_out = np.zeros(p, dtype=np.float64)
    hist = np.zeros(max_sweeps, dtype=np.float64)
    info = np.zeros(4, dtype=np.int32)
    if u0 is not None:
        u0c = np.ascontiguousarray(np.concatenate([np.asarray(v, dtype=np.float64).reshape(-1) for v in u0]))
        u0p = _ptr(u0c, "f64")
    else:
        u0c, u0p = None, None
    rc = lib().tlo_hopm_f64(p, sp, wp, _ptr(a, "f64"), int(max_sweeps), float(tol), u0p,
                            _ptr(u_out, "f64"), _ptr(l_out, "f64"), _ptr(hist, "f64"),
                            info.ctypes.data_as(_i32p), nthreads)
    if rc == 1:
        raise ValueError("oracle hopm: invalid arguments")
    if rc == 2:
        raise ValueError("oracle hopm: zero start vector")
    if rc == 3:
        raise OracleDegenerate(int(info[2]), int(info[3]))
    us, off = [], 0
    for n in shape:
        us.append(u_out[off:off + n].copy())
        off += n
    sweeps = int(info[0])
    return {
        "u": us,
        "l": [float(x) for x in l_out],
        "lambda_history": [float(x) for x in hist[:sweeps]],
        "sweeps": sweeps,
        "converged": bool(info[1]),
    }


# -- small-case pure-Python restatements (no C counterpart needed at these sizes) -----


def _py(buf, kind):
    arr = np.asarray(buf).reshape(-1)
    return [int(x) for x in arr] if kind == "int64" else [float(x) for x in arr.astype(np.float64)]


def _multi(shape):
    """Zero-based multi-indices, last dimension fastest."""
    import itertools

    return itertools.product(*[range(n) for n in shape])


def ttt(abuf, ashape, astrides, bbuf, bshape, bstrides, q, phi, psi, kind="float64"):
    """Tensor-times-tensor (contraction.py:337-418): output = A's free dims
    in phi order then B's in psi order (first-order buffer); each output is
    a left fold over the contracted pairs, the LAST pair innermost (the base
    case of _ttt_rec), as ``acc += a * b`` on Python numbers.  Returns
    (flat first-order output list, out_shape)."""
    a, b = _py(abuf, kind), _py(bbuf, kind)
    phi = [x - 1 for x in phi]
    psi = [x - 1 for x in psi]
    r, s = len(phi) - q, len(psi) - q
    out_shape = tuple(ashape[phi[k]] for k in range(r)) + tuple(bshape[psi[k]] for k in range(s))
    bounds = [ashape[phi[r + k]] for k in range(q)]
    shape = out_shape or (1,)
    fs = first_order_strides(shape)
    out = [0 if kind == "int64" else 0.0] * int(np.prod(shape))
    for ic in _multi(shape):
        pa = sum(ic[k] * astrides[phi[k]] for k in range(r))
        pb = sum(ic[r + k] * bstrides[psi[k]] for k in range(s))
        acc = 0 if kind == "int64" else 0.0
        if q == 0:
            acc = a[pa] * b[pb]
        else:
            for jt in _multi(bounds):  # first contracted pair outermost
                ia = pa + sum(jt[k] * astrides[phi[r + k]] for k in range(q))
                ib = pb + sum(jt[k] * bstrides[psi[s + k]] for k in range(q))
                acc += a[ia] * b[ib]
        out[sum(i * w for i, w in zip(ic, fs)) if out_shape else 0] = acc
    return out, out_shape if out_shape else (1,)


def transpose(abuf, shape, strides, tau, kind="float64"):
    """C(i_1..i_p) = A(i_tau1..i_taup), first-order output (contraction.py:75-107)."""
    a = _py(abuf, kind)
    out_shape = tuple(shape[t - 1] for t in tau)
    fs = first_order_strides(out_shape)
    out = [None] * int(np.prod(out_shape))
    for ic in _multi(out_shape):
        pa = sum(ic[r] * strides[t - 1] for r, t in enumerate(tau))
        out[sum(i * w for i, w in zip(ic, fs))] = a[pa]
    return out, out_shape


def ttm_canon(buf, shape, layout, bmat, bshape, bstrides, mode, absval=False, nthreads=0):
    """Full-size ttm restatement (tlo_ttm_canon_f64): the output buffer in
    A's OWN layout (extent J at ``mode``), every element the reference's
    k-ordered mul-then-add fold; bit-identical to ``ttm``.  With absval the
    fold of |A| |B| (the elementwise error bound)."""
    shape = tuple(int(n) for n in shape)
    layout = tuple(int(x) for x in layout)
    t = layout.index(mode)
    I = int(np.prod([shape[q - 1] for q in layout[:t]], dtype=np.int64)) if t else 1
    K = shape[mode - 1]
    O = int(np.prod(shape, dtype=np.int64)) // (I * K)
    J = int(bshape[0])
    a = _flat(np.asarray(buf), np.float64)
    bm = _flat(bmat, np.float64)
    c = np.empty(O * J * I, dtype=np.float64)
    rc = lib().tlo_ttm_canon_f64(O, K, I, _ptr(a, "f64"), J, int(bstrides[0]), int(bstrides[1]), _ptr(bm, "f64"),
                                 _ptr(c, "f64"), 1 if absval else 0, nthreads)
    if rc != 0:
        raise ValueError("oracle ttm_canon: invalid arguments")
    return c
