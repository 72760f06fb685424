"""Hot-path tensor functions on B200: ttv, ttm, inner product, norm and
the sequenced products.

Same names, argument meaning and errors as the reference suite
(/root/reference/pkg/src/tensorlib/contraction.py): modes are one-based,
outputs are fresh dense first-order tensors with zero offsets, and each
contraction allocates exactly one output (test_contraction.py:398-425).
Every numeric step runs in hand-written sm_100a kernels behind the C ABI
(include/tensorlib_b200.h); there is no CPU fallback.
"""

from __future__ import annotations

import ctypes
import math

import torch

from . import _abi
from .layout import TensorMeta
from .tensor import DenseTensor, _copy

__all__ = [
    "frobenius_norm",
    "inner_product_flat",
    "inner_product_tensors",
    "times_matrices",
    "times_vectors",
    "ttm",
    "ttv",
]


def _operand(x) -> DenseTensor:
    if isinstance(x, DenseTensor):
        return x
    raise TypeError(f"expected a DenseTensor, got {type(x).__name__}")


def _vector(b, expected_len: int, what: str) -> DenseTensor:
    """An order-1 tensor or an (n, 1) column (contraction.py:58-69)."""
    b = _operand(b)
    ext = b.shape
    if len(ext) == 2 and ext[1] == 1:
        ext = ext[:1]
    if len(ext) != 1:
        raise ValueError(f"{what} must be a vector, got extents {b.shape}")
    if ext[0] != expected_len:
        raise ValueError(f"{what} length {ext[0]} does not match extent {expected_len}")
    return b


def _is_float(dt) -> bool:
    return dt in (torch.float32, torch.float64)


def ttv(a, b, mode: int) -> DenseTensor:
    """C(i_1..i_{m-1}, i_{m+1}..i_p) = sum_k A(..k..) b(k)  (contraction.py:113-131).

    Bit-identical to the reference: every output is its left fold in k order
    in binary64 (float32 storage widened exactly, rounded once on store)."""
    A = _operand(a)
    p = A.order
    if p < 2:
        raise ValueError(f"ttv requires order >= 2, got {p}")
    if not 1 <= mode <= p:
        raise ValueError(f"mode {mode} out of range 1..{p}")
    B = _vector(b, A.shape[mode - 1], "ttv vector")
    if _is_float(A.dtype) != _is_float(B.dtype):
        raise NotImplementedError("ttv: mixed integer and floating operands")
    out = DenseTensor(A.shape[: mode - 1] + A.shape[mode:], dtype=A.dtype, device=A.device, fill_value=None)
    L = _abi.lib()
    rc = L.tl_ttv(A.desc(), A.ptr(), B.desc(), B.ptr(), out.desc(), out.ptr(), int(mode), _abi.stream_handle())
    _abi.check(rc, "ttv")
    return out


def ttm(a, bmat, mode: int) -> DenseTensor:
    """C(.., j at mode, ..) = sum_k A(.., k, ..) B(j, k)  (contraction.py:200-227).

    B has shape (n_new, n_mode) -- rows index the new dimension, no implicit
    transpose.  float64 runs on FP64 DMMA tensor-core tiles."""
    A = _operand(a)
    p = A.order
    if p < 2:
        raise ValueError(f"ttm requires order >= 2, got {p}")
    if not 1 <= mode <= p:
        raise ValueError(f"mode {mode} out of range 1..{p}")
    Bm = _operand(bmat)
    if Bm.order != 2:
        raise ValueError(f"ttm matrix must have order 2, got {Bm.order}")
    if Bm.shape[1] != A.shape[mode - 1]:
        raise ValueError(f"matrix columns {Bm.shape[1]} do not match extent {A.shape[mode - 1]} of mode {mode}")
    if Bm.dtype != A.dtype:
        Bm = Bm.to(A.dtype)
    m = mode - 1
    out = DenseTensor(A.shape[:m] + (Bm.shape[0],) + A.shape[m + 1:], dtype=A.dtype, device=A.device, fill_value=None)
    L = _abi.lib()
    rc = L.tl_ttm(A.desc(), A.ptr(), Bm.desc(), Bm.ptr(), out.desc(), out.ptr(), int(mode), _abi.stream_handle())
    _abi.check(rc, "ttm")
    return out


def _reduce_result_buffer(dtype, device) -> torch.Tensor:
    return torch.empty(1, dtype=torch.int64 if dtype == torch.int64 else torch.float64, device=device)


def inner_product_device(a, b) -> torch.Tensor:
    """sum_i a[i] b[i] as a 1-element device tensor (no host sync)."""
    A, B = _operand(a), _operand(b)
    if A.shape != B.shape:
        raise ValueError(f"shape mismatch: {B.shape} vs {A.shape}")
    res = _reduce_result_buffer(A.dtype, A.device)
    ws = _abi.reduce_workspace(A.device)
    L = _abi.lib()
    rc = L.tl_inner(A.desc(), A.ptr(), B.desc(), B.ptr(), res.data_ptr(), ws.data_ptr(), ws.numel(),
                    _abi.stream_handle())
    _abi.check(rc, "inner")
    return res


def inner_product_tensors(a, b):
    """Scalar sum_i a[i] * b[i] over tensors of equal shape (contraction.py:457-459)."""
    return inner_product_device(a, b).item()


def inner_product_flat(a, b, init=0):
    """init + sum_i a[i] * b[i] (elementwise.py:411-414)."""
    return init + inner_product_tensors(a, b)


def frobenius_norm_device(a) -> torch.Tensor:
    A = _operand(a)
    if not _is_float(A.dtype):
        A = A.to(torch.float64)
    res = torch.empty(1, dtype=torch.float64, device=A.device)
    ws = _abi.reduce_workspace(A.device)
    L = _abi.lib()
    rc = L.tl_frobenius_norm(A.desc(), A.ptr(), res.data_ptr(), ws.data_ptr(), ws.numel(), _abi.stream_handle())
    _abi.check(rc, "frobenius_norm")
    return res


def frobenius_norm(a) -> float:
    """sqrt(<a, a>) (contraction.py:462-464)."""
    return frobenius_norm_device(a).item()


def _check_modes(modes, count: int, p: int, what: str):
    modes = [int(m) for m in modes]
    if len(modes) != count:
        raise ValueError(f"{what}: got {count} operands for modes {modes}")
    if any(not 1 <= m <= p for m in modes):
        raise ValueError(f"{what}: modes {modes} out of range 1..{p}")
    if any(m2 <= m1 for m1, m2 in zip(modes, modes[1:])):
        raise ValueError(f"{what}: modes {modes} must be strictly increasing")
    return modes


def times_vectors(a, vectors, modes=None, skip=None) -> DenseTensor:
    """Contract with several vectors, highest mode first (contraction.py:481-519).

    ``skip`` names the one mode left alone (a full-length vector list is
    accepted, the skipped entry ignored).  Contracting every mode returns a
    shape-(1,) tensor; contracting none returns a copy."""
    A = _operand(a)
    p = A.order
    if (modes is None) == (skip is None):
        raise ValueError("provide exactly one of modes or skip")
    vectors = list(vectors)
    if skip is not None:
        if not 1 <= skip <= p:
            raise ValueError(f"skip mode {skip} out of range 1..{p}")
        if len(vectors) == p:
            vectors = vectors[: skip - 1] + vectors[skip:]
        modes = [m for m in range(1, p + 1) if m != skip]
    modes = _check_modes(modes, len(vectors), p, "times_vectors")
    if not vectors:
        return _first_order_copy(A)
    result = A
    for m, vec in sorted(zip(modes, vectors), reverse=True, key=lambda x: x[0]):
        if result.order == 1:
            # Only mode 1 remains: the reference takes inner_product_flat
            # (a sequential fold) and returns shape (1,).  The same fold is
            # a ttv of the (n, 1) column over mode 1, which keeps it exact.
            _vector(vec, result.shape[0], "times_vectors vector")
            col = DenseTensor._wrap(TensorMeta((result.shape[0], 1)), result.buffer)
            result = ttv(col, vec, 1)
        else:
            result = ttv(result, vec, m)
    return result


def times_matrices(a, matrices, modes) -> DenseTensor:
    """ttm for each (matrix, mode), highest mode first (contraction.py:522-536)."""
    A = _operand(a)
    p = A.order
    matrices = list(matrices)
    modes = _check_modes(modes, len(matrices), p, "times_matrices")
    if not matrices:
        return _first_order_copy(A)
    result = A
    for m, mat in sorted(zip(modes, matrices), reverse=True, key=lambda x: x[0]):
        result = ttm(result, mat, m)
    return result


def _first_order_copy(A: DenseTensor) -> DenseTensor:
    out = DenseTensor(A.shape, dtype=A.dtype, device=A.device, fill_value=None)
    _copy(A.desc(), A.buffer, out.desc(), out.buffer)
    return out
