"""ctypes binding of libtlb200.so (include/tensorlib_b200.h).

The product path has no fallback: if the shared library is missing or no
CUDA device is visible, every operation raises.  PyTorch supplies device
buffers and the current stream only.
"""

from __future__ import annotations

import ctypes
import os
import threading

import torch

_PKG = os.path.dirname(os.path.abspath(__file__))
# TL_LIB: an alternative build of the same library (A/B measurements only)
LIB_PATH = os.environ.get("TL_LIB") or os.path.join(_PKG, "_lib", "libtlb200.so")

TL_MAX_ORDER = 16
TL_F32, TL_F64, TL_I64 = 0, 1, 2
TL_OK, TL_EINVAL, TL_EUNSUPPORTED, TL_ECUDA, TL_EWORKSPACE, TL_EDEGENERATE = range(6)

DTYPE_CODE = {torch.float32: TL_F32, torch.float64: TL_F64, torch.int64: TL_I64}

EXPORTS = (
    "tl_abi_version",
    "tl_device_arch",
    "tl_last_error",
    "tl_init",
    "tl_ttv",
    "tl_ttm",
    "tl_ttm_ssq",
    "tl_reduce_workspace_bytes",
    "tl_inner",
    "tl_inner_flat",
    "tl_frobenius_norm",
    "tl_hopm_workspace_bytes",
    "tl_hopm",
    "tl_hopm_graph_create",
    "tl_graph_launch",
    "tl_graph_destroy",
    "tl_copy",
    "tl_rank_one_compose",
    "tl_residual",
    "tl_plan_describe",
    "tl_times_vectors_workspace_bytes",
    "tl_times_vectors",
)


class TlDesc(ctypes.Structure):
    _fields_ = [
        ("order", ctypes.c_int32),
        ("dtype", ctypes.c_int32),
        ("offset", ctypes.c_int64),
        ("extent", ctypes.c_int64 * TL_MAX_ORDER),
        ("stride", ctypes.c_int64 * TL_MAX_ORDER),
    ]


def make_desc(shape, strides, dtype_code, offset=0) -> TlDesc:
    d = TlDesc()
    d.order = len(shape)
    d.dtype = dtype_code
    d.offset = offset
    for r, (n, w) in enumerate(zip(shape, strides)):
        d.extent[r] = int(n)
        d.stride[r] = int(w)
    return d


_lib = None
_lock = threading.Lock()
_vp = ctypes.c_void_p
_dp = ctypes.POINTER(TlDesc)


def load_library(path: str = LIB_PATH):
    """Load and type the shared library (works without a GPU)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            raise RuntimeError(
                f"{path} is missing: build the CUDA extension first "
                "(python -m paper_1711_10912_b200._build or __graft_entry__.build()); "
                "there is no CPU fallback"
            )
        L = ctypes.CDLL(path)
        L.tl_abi_version.restype = ctypes.c_int32
        L.tl_device_arch.restype = ctypes.c_int32
        L.tl_last_error.restype = ctypes.c_char_p
        L.tl_init.restype = ctypes.c_int
        L.tl_ttv.argtypes = [_dp, _vp, _dp, _vp, _dp, _vp, ctypes.c_int32, _vp]
        L.tl_ttm.argtypes = [_dp, _vp, _dp, _vp, _dp, _vp, ctypes.c_int32, _vp]
        L.tl_ttm_ssq.argtypes = [_dp, _vp, _dp, _vp, _dp, _vp, ctypes.c_int32, _vp, _vp, ctypes.c_size_t,
                                 ctypes.POINTER(ctypes.c_int32), _vp]
        L.tl_reduce_workspace_bytes.restype = ctypes.c_size_t
        L.tl_inner.argtypes = [_dp, _vp, _dp, _vp, _vp, _vp, ctypes.c_size_t, _vp]
        L.tl_inner_flat.argtypes = [_dp, _vp, _dp, _vp, _vp, _vp, _vp, ctypes.c_size_t, _vp]
        L.tl_frobenius_norm.argtypes = [_dp, _vp, _vp, _vp, ctypes.c_size_t, _vp]
        L.tl_hopm_workspace_bytes.argtypes = [_dp, ctypes.POINTER(ctypes.c_size_t)]
        vpp = ctypes.POINTER(_vp)
        L.tl_hopm.argtypes = [_dp, _vp, vpp, vpp, ctypes.c_int32, ctypes.c_double, _vp, _vp, _vp, _vp, _vp,
                              ctypes.c_size_t, _vp]
        L.tl_hopm_graph_create.argtypes = [_dp, _vp, vpp, vpp, ctypes.c_int32, ctypes.c_double, _vp, _vp, _vp, _vp,
                                           _vp, ctypes.c_size_t, _vp, ctypes.POINTER(_vp)]
        L.tl_graph_launch.argtypes = [_vp, _vp]
        L.tl_graph_destroy.argtypes = [_vp]
        L.tl_copy.argtypes = [_dp, _vp, _dp, _vp, _vp]
        L.tl_rank_one_compose.argtypes = [_dp, vpp, _vp, _vp, _vp]
        L.tl_residual.argtypes = [_dp, _vp, vpp, _vp, _vp, _vp, ctypes.c_size_t, _vp]
        i32p = ctypes.POINTER(ctypes.c_int32)
        L.tl_times_vectors_workspace_bytes.argtypes = [_dp, ctypes.c_int32, i32p, _dp, ctypes.POINTER(ctypes.c_size_t)]
        L.tl_times_vectors.argtypes = [_dp, _vp, ctypes.c_int32, i32p, _dp, vpp, _dp, _vp, _vp, ctypes.c_size_t, _vp]
        L.tl_plan_describe.argtypes = [ctypes.c_int32, _dp, _dp, ctypes.c_int32, ctypes.c_char_p, ctypes.c_size_t]
        for name in ("tl_ttv", "tl_ttm", "tl_ttm_ssq", "tl_inner", "tl_inner_flat", "tl_frobenius_norm", "tl_hopm_workspace_bytes", "tl_hopm",
                     "tl_hopm_graph_create", "tl_graph_launch", "tl_graph_destroy", "tl_copy", "tl_rank_one_compose",
                     "tl_residual", "tl_plan_describe", "tl_times_vectors_workspace_bytes", "tl_times_vectors"):
            getattr(L, name).restype = ctypes.c_int
        _lib = L
        return L


def lib():
    """The library, for a compute call: requires a CUDA device."""
    if not torch.cuda.is_available():
        raise RuntimeError("paper_1711_10912_b200 needs a CUDA (sm_100a) device; there is no CPU fallback")
    return load_library()


_warm_devices = set()


def warm(device) -> None:
    """Once per device: tl_init (the library's runtime state and its small
    kernels), so the first hot-path call of a process is not ms-slow.  Runs
    when the first DenseTensor is placed on ``device``."""
    if device.type != "cuda":
        raise RuntimeError(f"paper_1711_10912_b200 tensors live on a CUDA device, not {device}; there is no CPU fallback")
    idx = device.index if device.index is not None else torch.cuda.current_device()
    if idx in _warm_devices:
        return
    L = lib()
    with torch.cuda.device(idx):
        check(L.tl_init(), "init")
    _warm_devices.add(idx)


def check(rc: int, what: str = "") -> None:
    if rc == TL_OK:
        return
    msg = _lib.tl_last_error().decode() if _lib is not None else "unknown error"
    if rc == TL_EINVAL:
        raise ValueError(msg)
    if rc == TL_EUNSUPPORTED:
        raise NotImplementedError(msg)
    if rc == TL_EWORKSPACE:
        raise RuntimeError(f"workspace: {msg}")
    raise RuntimeError(f"CUDA error in {what}: {msg}")


def stream_handle(stream=None) -> ctypes.c_void_p:
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


_ws_cache = {}


def reduce_workspace(device) -> torch.Tensor:
    """Zero-filled scratch for inner/norm; the kernels leave it zeroed."""
    key = (device.index if device.index is not None else torch.cuda.current_device())
    ws = _ws_cache.get(key)
    if ws is None:
        n = int(load_library().tl_reduce_workspace_bytes())
        ws = torch.zeros(n, dtype=torch.uint8, device=device)
        _ws_cache[key] = ws
    return ws
