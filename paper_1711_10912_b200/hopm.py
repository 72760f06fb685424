"""Higher-order power method on B200 (hopm.py:63-120 of the reference).

The whole Gauss-Seidel loop -- per-mode ttv chains, sequential norms,
normalisation, lambda history, the tol test, degeneracy and (optionally) the
per-sweep residual -- is one CUDA graph built by the C ABI
(tl_hopm_graph_create); the host waits once at the end.  lambda and the
vectors are bit-identical to the reference (csrc/hopm.cu).
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import torch

from . import _abi
from .layout import TensorMeta
from .tensor import DenseTensor
from .views import as_dense_operand

__all__ = ["DegenerateInputError", "HopmState", "hopm", "HopmRunner", "rank_one_compose", "residual"]


class DegenerateInputError(ArithmeticError):
    """A mode update produced the zero vector (hopm.py:26-35)."""

    def __init__(self, sweep: int, mode: int):
        super().__init__(f"zero vector at normalization (sweep {sweep}, mode {mode})")
        self.sweep = sweep
        self.mode = mode


@dataclass
class HopmState:
    """u: unit vectors per dimension; l: per-mode norms of the final sweep;
    scale = l[-1]; histories per sweep (hopm.py:38-56)."""

    u: List[DenseTensor]
    l: List[float]
    sweeps: int
    converged: bool
    lambda_history: List[float] = field(default_factory=list)
    residual_history: List[float] = field(default_factory=list)

    @property
    def scale(self) -> float:
        return self.l[-1]


def _seq_norm(values) -> float:
    """The reference's frobenius_norm of a vector: sqrt of a left fold."""
    acc = 0
    for x in values:
        acc += x * x
    return math.sqrt(acc)


def _start_vectors(shape, u0) -> List[List[float]]:
    """hopm.py:81-98, evaluated in host binary64 exactly as the reference
    does (n ** -0.5, or u0 / frobenius_norm(u0))."""
    p = len(shape)
    if u0 is None:
        return [[n ** -0.5] * n for n in shape]
    vecs = list(u0)
    if len(vecs) != p:
        raise ValueError(f"expected {p} start vectors, got {len(vecs)}")
    out = []
    for r, (v, n) in enumerate(zip(vecs, shape), start=1):
        vshape = tuple(v.shape)
        if len(vshape) != 1 or vshape != (n,):
            raise ValueError(f"start vector {r} must have shape ({n},), got {vshape}")
        vals = [float(x) for x in (v.data if hasattr(v, "data") else v)]
        nrm = _seq_norm(vals)
        if nrm == 0.0:
            raise ValueError(f"start vector {r} is zero")
        out.append([x / nrm for x in vals])
    return out


_EXACT_INT = 1 << 53


def _floating(a: DenseTensor) -> DenseTensor:
    """int64 tensors enter HOPM as float64: the reference multiplies its
    Python ints by float vector entries, i.e. converts each to binary64
    first, which is exact below 2^53 (checked; larger values raise)."""
    if a.dtype in (torch.float32, torch.float64):
        return a
    if a.size and int(a.buffer.abs().max().item()) > _EXACT_INT:
        raise NotImplementedError("hopm: int64 entries beyond 2^53 are not exactly representable in binary64")
    return a.to(torch.float64)


def _vec(t: torch.Tensor) -> DenseTensor:
    return DenseTensor._wrap(TensorMeta((t.numel(),)), t)


class HopmRunner:
    """A captured HOPM graph over a fixed tensor: ``run()`` replays the
    whole max_sweeps loop (start vectors are re-copied each replay)."""

    def __init__(self, a: DenseTensor, max_sweeps: int = 50, u0=None, tol: float = 1e-10,
                 track_residuals: bool = False):
        if max_sweeps < 1:
            raise ValueError("max_sweeps must be >= 1")
        a = _floating(as_dense_operand(a))
        self.a = a
        self.max_sweeps = int(max_sweeps)
        self.tol = float(tol)
        dev = a.device
        starts = _start_vectors(a.shape, u0)
        self.u0 = [torch.tensor(v, dtype=torch.float64, device=dev) for v in starts]
        self.u = [torch.empty(len(v), dtype=torch.float64, device=dev) for v in starts]
        p = a.order
        self.l = torch.zeros(p, dtype=torch.float64, device=dev)
        self.hist = torch.zeros(self.max_sweeps, dtype=torch.float64, device=dev)
        self.info = torch.zeros(4, dtype=torch.int32, device=dev)
        self.resid = torch.zeros(self.max_sweeps, dtype=torch.float64, device=dev) if track_residuals else None
        L = _abi.lib()
        desc = a.desc()
        need = ctypes.c_size_t(0)
        _abi.check(L.tl_hopm_workspace_bytes(desc, ctypes.byref(need)), "hopm workspace")
        self.ws = torch.zeros(max(int(need.value), 256), dtype=torch.uint8, device=dev)
        self._u0p = (ctypes.c_void_p * p)(*[t.data_ptr() for t in self.u0])
        self._up = (ctypes.c_void_p * p)(*[t.data_ptr() for t in self.u])
        self._graph = ctypes.c_void_p(0)
        self.stream = torch.cuda.Stream(device=dev)
        self.stream.wait_stream(torch.cuda.current_stream(dev))
        rc = L.tl_hopm_graph_create(desc, a.ptr(), self._u0p, self._up, self.max_sweeps, self.tol,
                                    self.l.data_ptr(), self.hist.data_ptr(), self.info.data_ptr(),
                                    self.resid.data_ptr() if self.resid is not None else None,
                                    self.ws.data_ptr(), self.ws.numel(), _abi.stream_handle(self.stream),
                                    ctypes.byref(self._graph))
        _abi.check(rc, "hopm graph")

    def launch(self, stream=None) -> None:
        s = stream if stream is not None else torch.cuda.current_stream(self.a.device)
        _abi.check(_abi.lib().tl_graph_launch(self._graph, _abi.stream_handle(s)), "hopm launch")

    def state(self) -> HopmState:
        sweeps, converged, dsweep, dmode = self.info.cpu().tolist()
        if dsweep:
            raise DegenerateInputError(dsweep, dmode)
        resid = self.resid[:sweeps].cpu().tolist() if self.resid is not None else []
        return HopmState(u=[_vec(t.clone()) for t in self.u], l=self.l.cpu().tolist(), sweeps=sweeps,
                         converged=bool(converged), lambda_history=self.hist[:sweeps].cpu().tolist(),
                         residual_history=resid)

    def run(self) -> HopmState:
        self.launch()
        return self.state()

    def close(self) -> None:
        if self._graph:
            _abi.lib().tl_graph_destroy(self._graph)
            self._graph = ctypes.c_void_p(0)

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def hopm(a, max_sweeps: int = 50, u0: Optional[Sequence] = None, tol: float = 1e-10,
         track_residuals: bool = False) -> HopmState:
    """Best rank-one approximation by alternating sweeps (hopm.py:63-120).

    Raises DegenerateInputError when a mode update has norm zero, ValueError
    for max_sweeps < 1 or invalid start vectors.  With track_residuals the
    residual ||a - lambda u_1 o ... o u_p||_F after every sweep is recorded
    (computed on the device inside the same graph)."""
    if max_sweeps < 1:
        raise ValueError("max_sweeps must be >= 1")
    runner = HopmRunner(a, max_sweeps=max_sweeps, u0=u0, tol=tol, track_residuals=track_residuals)
    try:
        return runner.run()
    finally:
        runner.close()


def _vector_ptrs(vectors, device):
    vs = [v.buffer if isinstance(v, DenseTensor) else torch.as_tensor(v) for v in vectors]
    vs = [v.to(device=device, dtype=torch.float64).contiguous() for v in vs]
    return vs, (ctypes.c_void_p * len(vs))(*[v.data_ptr() for v in vs])


def rank_one_compose(scale: float, vectors: Sequence) -> DenseTensor:
    """B(i_1, .., i_p) = scale * u_1(i_1) * ... * u_p(i_p), first-order
    (hopm.py:123-139), multiplied left to right like the reference."""
    if len(vectors) == 0:
        raise ValueError("need at least one vector")
    shape = tuple(int(v.size) if isinstance(v, DenseTensor) else len(v) for v in vectors)
    out = DenseTensor(shape, fill_value=None)
    vs, ptrs = _vector_ptrs(vectors, out.device)
    sc = torch.tensor([float(scale)], dtype=torch.float64, device=out.device)
    rc = _abi.lib().tl_rank_one_compose(out.desc(), ptrs, sc.data_ptr(), out.ptr(), _abi.stream_handle())
    _abi.check(rc, "rank_one_compose")
    return out


def residual(a, state: HopmState) -> float:
    """||a - rank_one_compose(state.scale, state.u)||_F (hopm.py:142-147)."""
    a = _floating(as_dense_operand(a))
    vs, ptrs = _vector_ptrs(state.u, a.device)
    sc = torch.tensor([float(state.l[-1])], dtype=torch.float64, device=a.device)
    res = torch.empty(1, dtype=torch.float64, device=a.device)
    ws = _abi.reduce_workspace(a.device)
    rc = _abi.lib().tl_residual(a.desc(), a.ptr(), ptrs, sc.data_ptr(), res.data_ptr(), ws.data_ptr(), ws.numel(),
                                _abi.stream_handle())
    _abi.check(rc, "residual")
    return res.item()
