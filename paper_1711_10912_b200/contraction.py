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
import numbers
import os
from dataclasses import dataclass
from typing import Sequence, Tuple

import torch

from . import _abi
from .layout import TensorMeta
from .tensor import DenseTensor, _copy
from .views import as_dense_operand

__all__ = [
    "ContractionSpec",
    "frobenius_norm",
    "inner_product_flat",
    "inner_product_tensors",
    "outer_product",
    "reduce_ttm_to_ttt",
    "reduce_ttv_to_ttt",
    "times_matrices",
    "times_vectors",
    "transpose",
    "ttm",
    "ttt",
    "ttv",
]


def _operand(x) -> DenseTensor:
    """DenseTensor or TensorView operand (contraction.py:52-55) as a DenseTensor."""
    return as_dense_operand(x)


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
    if _is_float(A.dtype) != _is_float(Bm.dtype):
        raise NotImplementedError("ttm: mixed integer and floating operands")
    if A.dtype == torch.float32 and Bm.dtype == torch.float64:
        # keep B's binary64 values: contract in float64, round once to float32
        return ttm(A.to(torch.float64), Bm, mode).to(torch.float32)
    if Bm.dtype != A.dtype:
        Bm = Bm.to(A.dtype)  # float32 matrix, float64 tensor: widening is exact
    m = mode - 1
    out = DenseTensor(A.shape[:m] + (Bm.shape[0],) + A.shape[m + 1:], dtype=A.dtype, device=A.device, fill_value=None)
    L = _abi.lib()
    if A.dtype == torch.float64 and _fuse_norm():
        # the small-J stream kernel also leaves ||C|| (its epilogue's sum of
        # squares) for a following frobenius_norm(C)
        ssq = torch.empty(2, dtype=torch.float64, device=A.device)
        ws = _abi.reduce_workspace(A.device)
        fused = ctypes.c_int32(0)
        rc = L.tl_ttm_ssq(A.desc(), A.ptr(), Bm.desc(), Bm.ptr(), out.desc(), out.ptr(), int(mode), ssq.data_ptr(),
                          ws.data_ptr(), ws.numel(), ctypes.byref(fused), _abi.stream_handle())
        _abi.check(rc, "ttm")
        if fused.value:
            out._ssq = (ssq, out.buffer, out.buffer._version)
        return out
    rc = L.tl_ttm(A.desc(), A.ptr(), Bm.desc(), Bm.ptr(), out.desc(), out.ptr(), int(mode), _abi.stream_handle())
    _abi.check(rc, "ttm")
    return out


def _fuse_norm() -> bool:
    """Fused ||C|| in ttm's epilogue (TL_FUSED_NORM=0 disables)."""
    return os.environ.get("TL_FUSED_NORM", "1") != "0"


def _reduce_result_buffer(dtype, device) -> torch.Tensor:
    return torch.empty(1, dtype=torch.int64 if dtype == torch.int64 else torch.float64, device=device)


def inner_product_device(a, b, init=None) -> torch.Tensor:
    """init + sum_i a[i] b[i] as a 1-element device tensor (no host sync).
    ``init`` (a host scalar, default 0) is the fold's starting value; for
    floating operands it enters the compensated sum before the single final
    rounding, for int64 operands it must be an integer."""
    A, B = _operand(a), _operand(b)
    if A.shape != B.shape:
        raise ValueError(f"shape mismatch: {B.shape} vs {A.shape}")
    res = _reduce_result_buffer(A.dtype, A.device)
    ws = _abi.reduce_workspace(A.device)
    L = _abi.lib()
    init_ref = None
    if init is not None:
        init_ref = ctypes.c_int64(int(init)) if A.dtype == torch.int64 else ctypes.c_double(float(init))
    rc = L.tl_inner_flat(A.desc(), A.ptr(), B.desc(), B.ptr(),
                         ctypes.byref(init_ref) if init_ref is not None else None, res.data_ptr(),
                         ws.data_ptr(), ws.numel(), _abi.stream_handle())
    _abi.check(rc, "inner")
    return res


def inner_product_tensors(a, b):
    """Scalar sum_i a[i] * b[i] over tensors of equal shape (contraction.py:457-459)."""
    return inner_product_device(a, b).item()


def inner_product_flat(a, b, init=0):
    """init + sum_i a[i] * b[i] by multi-index (elementwise.py:411-433).

    The reference folds ``acc = init; acc += a[i]*b[i]``: the device sum
    starts from ``init`` too (it is not added to a rounded total).  An
    integer operand pair with a non-integral ``init`` sums exactly and adds
    ``init`` once on the host, as Python's int + float would."""
    A = _operand(a)
    if A.dtype == torch.int64 and not isinstance(init, numbers.Integral):
        return init + inner_product_tensors(a, b)
    return inner_product_device(a, b, init).item()


def frobenius_norm_device(a) -> torch.Tensor:
    """||a|| as a 1-element device tensor.  When the kernel that produced a's
    current values already computed it (ttm's fused epilogue), that value is
    returned without another pass over a."""
    A = _operand(a)
    fused = A._fused_norm() if isinstance(a, DenseTensor) else None
    if fused is not None:
        return fused[1:2]
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
    if len(vectors) >= 2 and _use_chain() and _is_float(A.dtype):
        out = _times_vectors_chain(A, vectors, modes)
        if out is not None:
            return out
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


def _use_chain() -> bool:
    """times_vectors as one cooperative launch (tl_times_vectors, opt-in with
    TL_TV_CHAIN=1) instead of one tl_ttv launch per vector.  Both are
    bit-identical; the launch sequence is the default because it is faster:
    measured on B200 the chain takes 182-188 vs 164-168 us on config-2
    shaped chains and 141-157 vs 80-83 us on config-4 chains (the tuned pass
    kernels beat a pass inside a cooperative kernel, whose occupancy is set by
    its largest stage; the launches it saves cost ~1 us each in a graph)."""
    return os.environ.get("TL_TV_CHAIN", "0") == "1"


def _times_vectors_chain(A: DenseTensor, vectors, modes):
    """The whole chain in one launch, or None when the library declines it
    (a permuted step output: the caller issues the ttv sequence)."""
    vecs = []
    for m, v in zip(modes, vectors):
        V = _operand(v)
        n = A.shape[m - 1] if A.order > 1 else A.shape[0]
        _vector(V, V.shape[0], "times_vectors vector")
        if _is_float(V.dtype) != _is_float(A.dtype):
            raise NotImplementedError("times_vectors: mixed integer and floating operands")
        vecs.append(V)
    p = A.order
    out_shape = tuple(A.shape[r] for r in range(p) if r + 1 not in modes) or (1,)
    L = _abi.lib()
    n = len(vecs)
    vd = (_abi.TlDesc * n)(*[V.desc() for V in vecs])
    md = (ctypes.c_int32 * n)(*modes)
    need = ctypes.c_size_t(0)
    adesc = A.desc()
    _abi.check(L.tl_times_vectors_workspace_bytes(adesc, n, md, vd, ctypes.byref(need)), "times_vectors")
    ws = torch.empty(max(int(need.value), 16), dtype=torch.uint8, device=A.device)
    out = DenseTensor(out_shape, dtype=A.dtype, device=A.device, fill_value=None)
    vp = (ctypes.c_void_p * n)(*[V.ptr() for V in vecs])
    rc = L.tl_times_vectors(adesc, A.ptr(), n, md, vd, vp, out.desc(), out.ptr(), ws.data_ptr(), ws.numel(),
                            _abi.stream_handle())
    if rc == _abi.TL_EUNSUPPORTED:
        return None
    _abi.check(rc, "times_vectors")
    return out


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


# -- general tensor-times-tensor ------------------------------


@dataclass(frozen=True)
class ContractionSpec:
    """q contracted pairs; one-based permutations phi (A) and psi (B), free
    dimensions first, contracted pairs last (contraction.py:304-334)."""

    q: int
    phi: Tuple[int, ...]
    psi: Tuple[int, ...]

    def __post_init__(self):
        object.__setattr__(self, "phi", tuple(int(x) for x in self.phi))
        object.__setattr__(self, "psi", tuple(int(x) for x in self.psi))
        if self.q < 0:
            raise ValueError("q must be nonnegative")
        for name, perm in (("phi", self.phi), ("psi", self.psi)):
            if sorted(perm) != list(range(1, len(perm) + 1)):
                raise ValueError(f"{name} {perm} is not a permutation")
        if self.q > len(self.phi) or self.q > len(self.psi):
            raise ValueError("q exceeds an operand's order")
        if not self.phi or not self.psi:
            raise ValueError("operands must have at least one dimension")

    @property
    def r(self) -> int:
        return len(self.phi) - self.q

    @property
    def s(self) -> int:
        return len(self.psi) - self.q


def _relayouted(T: DenseTensor, layout) -> DenseTensor:
    """A copy of T stored under ``layout`` (device tl_copy); internal
    scratch, so not a counted DenseTensor allocation (the reference's ttt
    allocates only its output, test_contraction.py:398-425)."""
    if tuple(layout) == T.layout:
        return T
    meta = TensorMeta(T.shape, layout=tuple(layout))
    out = DenseTensor._wrap(meta, torch.empty(T.size, dtype=T.dtype, device=T.device))
    _copy(T.desc(), T.buffer, out.desc(), out.buffer)
    return out


def ttt(a, b, spec: ContractionSpec) -> DenseTensor:
    """General tensor-tensor product (contraction.py:337-369).

    C = A's free dims (phi order) then B's free dims (psi order), summing the
    q contracted pairs.  On the device this is two relayouts and one ttm:
    A is stored as a first-order (F_A x K) matrix and B as a (K x F_B)
    tensor with the contracted index linearised last-pair-fastest -- the
    reference's nesting order (the innermost loop of _ttt_rec is the last
    pair) -- and C = ttm(B', A', 1) is already C's first-order buffer."""
    A, B = _operand(a), _operand(b)
    q, r, s = spec.q, spec.r, spec.s
    if len(spec.phi) != A.order:
        raise ValueError(f"phi length {len(spec.phi)} does not match order {A.order}")
    if len(spec.psi) != B.order:
        raise ValueError(f"psi length {len(spec.psi)} does not match order {B.order}")
    phi = [x - 1 for x in spec.phi]
    psi = [x - 1 for x in spec.psi]
    for k in range(q):
        na, nb = A.shape[phi[r + k]], B.shape[psi[s + k]]
        if na != nb:
            raise ValueError(f"contracted pair {k + 1} has mismatched extents {na} vs {nb}")
    if _is_float(A.dtype) != _is_float(B.dtype):
        raise NotImplementedError("ttt: mixed integer and floating operands")
    if B.dtype != A.dtype:
        B = B.to(A.dtype)
    out_shape = tuple(A.shape[phi[k]] for k in range(r)) + tuple(B.shape[psi[k]] for k in range(s))
    L = _abi.lib()
    code = _abi.DTYPE_CODE[A.dtype]

    def view(T, dims):  # descriptor of T with its dimensions visited in ``dims`` order
        return _abi.make_desc(tuple(T.shape[d] for d in dims), tuple(T.strides[d] for d in dims), code)

    if r == 0 and s == 0:
        # full contraction: the inner product over the paired dimensions
        res = _reduce_result_buffer(A.dtype, A.device)
        ws = _abi.reduce_workspace(A.device)
        _abi.check(L.tl_inner(view(A, phi), A.ptr(), view(B, psi), B.ptr(), res.data_ptr(), ws.data_ptr(),
                              ws.numel(), _abi.stream_handle()), "ttt")
        out = DenseTensor((1,), dtype=A.dtype, device=A.device, fill_value=None)
        out.buffer.copy_(res)
        return out
    if q == 1 and (s == 0 or r == 0):
        # one operand is a vector: ttv over a permuted view, the reference's
        # fold bit for bit (x*y commutes)
        T, perm, v = (A, phi, B) if s == 0 else (B, psi, A)
        out = DenseTensor(out_shape, dtype=A.dtype, device=A.device, fill_value=None)
        _abi.check(L.tl_ttv(view(T, perm), T.ptr(), v.desc(), v.ptr(), out.desc(), out.ptr(), len(perm),
                            _abi.stream_handle()), "ttt")
        return out
    FA = math.prod(A.shape[phi[k]] for k in range(r))
    FB = math.prod(B.shape[psi[k]] for k in range(s))
    Kq = math.prod(A.shape[phi[r + k]] for k in range(q))
    a_layout = tuple(phi[k] + 1 for k in range(r)) + tuple(phi[r + k] + 1 for k in reversed(range(q)))
    b_layout = tuple(psi[s + k] + 1 for k in reversed(range(q))) + tuple(psi[k] + 1 for k in range(s))
    Am = DenseTensor._wrap(TensorMeta((FA, Kq)), _relayouted(A, a_layout).buffer)
    Bt = DenseTensor._wrap(TensorMeta((Kq, FB)), _relayouted(B, b_layout).buffer)
    C = ttm(Bt, Am, 1)  # (FA, FB) first-order == C's first-order buffer
    return DenseTensor._wrap(TensorMeta(out_shape if out_shape else (1,)), C.buffer)


def reduce_ttv_to_ttt(p: int, m: int) -> ContractionSpec:
    """Spec whose ttt equals ttv(a, b, m) for order-p a (contraction.py:421-426)."""
    if not 1 <= m <= p:
        raise ValueError(f"mode {m} out of range 1..{p}")
    return ContractionSpec(1, tuple(k for k in range(1, p + 1) if k != m) + (m,), (1,))


def reduce_ttm_to_ttt(p: int, m: int) -> ContractionSpec:
    """ttm as ttt with the new dimension last (contraction.py:429-440)."""
    if not 1 <= m <= p:
        raise ValueError(f"mode {m} out of range 1..{p}")
    return ContractionSpec(1, tuple(k for k in range(1, p + 1) if k != m) + (m,), (1, 2))


def outer_product(a, b) -> DenseTensor:
    """All-pairs product: ttt with q = 0 (contraction.py:446-454)."""
    A, B = _operand(a), _operand(b)
    return ttt(A, B, ContractionSpec(0, tuple(range(1, A.order + 1)), tuple(range(1, B.order + 1))))


def transpose(a, tau: Sequence[int]) -> DenseTensor:
    """Permuted copy C(i_1..i_p) = A(i_tau1..i_taup), first-order output
    (contraction.py:75-107): one device copy with permuted source strides."""
    A = _operand(a)
    p = A.order
    tau = tuple(int(t) for t in tau)
    if sorted(tau) != list(range(1, p + 1)):
        raise ValueError(f"tau {tau} is not a permutation of 1..{p}")
    out = DenseTensor(tuple(A.shape[t - 1] for t in tau), dtype=A.dtype, device=A.device, fill_value=None)
    src = _abi.make_desc(out.shape, tuple(A.strides[t - 1] for t in tau), _abi.DTYPE_CODE[A.dtype])
    _copy(src, A.buffer, out.desc(), out.buffer)
    return out


def _first_order_copy(A: DenseTensor) -> DenseTensor:
    out = DenseTensor(A.shape, dtype=A.dtype, device=A.device, fill_value=None)
    _copy(A.desc(), A.buffer, out.desc(), out.buffer)
    return out
