"""DenseTensor on B200 device memory -- the container of the hot path.

API of the reference container (tensor.py:33-284 of tensorlib): runtime
shape, one-based layout, offsets; a buffer in memory-index order; outputs
of contractions are fresh first-order tensors with zero offsets.  What
differs, by design:

* the buffer is a 1-D torch CUDA tensor (``.buffer``), not a Python list;
* the element type is explicit: ``dtype`` in {float64 (default), float32,
  int64}.  ``from_memory`` infers it (all-int -> int64, else float64,
  float32 only when the source is float32);
* ``.data`` is a host snapshot list in memory-index order whose element and
  slice writes go through to the device buffer (``t.data[j] = v`` works as
  on the reference's storage list, hopm.py:138, views.py:222); operations
  that would change the length raise, since the storage size is fixed;
* relayout/assign run on the device (tl_copy).
"""

from __future__ import annotations

import numbers

import numpy as np
import torch

from . import _abi
from .iterators import MultiIterator, StrideIterator
from .layout import TensorMeta, memory_index, validate_layout, validate_shape, volume

__all__ = ["DenseTensor", "tensors_equal", "as_dtype"]

_NAMES = {
    "float64": torch.float64, "f64": torch.float64, "double": torch.float64,
    "float32": torch.float32, "f32": torch.float32, "float": torch.float32,
    "int64": torch.int64, "i64": torch.int64, "int": torch.int64,
}


def as_dtype(dtype) -> torch.dtype:
    if dtype is None:
        return torch.float64
    if isinstance(dtype, torch.dtype):
        out = dtype
    elif isinstance(dtype, str):
        out = _NAMES[dtype]
    else:
        out = {np.dtype(np.float64): torch.float64, np.dtype(np.float32): torch.float32,
               np.dtype(np.int64): torch.int64}.get(np.dtype(dtype))
    if out not in _abi.DTYPE_CODE:
        raise TypeError(f"unsupported dtype {dtype!r}; use float64, float32 or int64")
    return out


def _default_device():
    if not torch.cuda.is_available():
        raise RuntimeError("paper_1711_10912_b200 needs a CUDA (sm_100a) device; there is no CPU fallback")
    return torch.device("cuda", torch.cuda.current_device())


def _device(device) -> torch.device:
    dev = torch.device(device) if device is not None else _default_device()
    _abi.warm(dev)
    return dev


def _checked_scalar(dtype: torch.dtype, value):
    """A value about to be stored into an element of ``dtype``.  Integer
    storage refuses values it cannot hold exactly (the reference's list
    would keep them; torch would truncate silently)."""
    if dtype == torch.int64 and not isinstance(value, numbers.Integral):
        f = float(value)
        if not f.is_integer():
            raise TypeError(f"cannot store {value!r} in an int64 tensor exactly; convert it with .to('float64')")
        return int(f)
    return value


class _DataList(list):
    """Snapshot of a device buffer in memory-index order whose writes go
    through to the buffer (the reference's ``.data`` *is* the storage list,
    tensor.py:46).  Reads are the values at the time ``.data`` was taken;
    every element or same-length slice write updates both this list and
    the device buffer.  Length-changing operations raise TypeError."""

    __slots__ = ("_buf",)

    def __init__(self, buf: torch.Tensor):
        super().__init__(buf.cpu().tolist())
        self._buf = buf

    def __setitem__(self, key, value):
        n = len(self)
        if isinstance(key, slice):
            idx = range(n)[key]
            vals = list(value)
            if len(vals) != len(idx):
                raise TypeError("tensor storage has a fixed size: slice assignment must keep the length")
            vals = [_checked_scalar(self._buf.dtype, v) for v in vals]
            list.__setitem__(self, key, vals)
            if vals:
                pos = torch.as_tensor(list(idx), dtype=torch.int64).to(self._buf.device)
                self._buf[pos] = torch.as_tensor(vals, dtype=self._buf.dtype).to(self._buf.device)
            return
        j = key.__index__()
        if not -n <= j < n:
            raise IndexError("list assignment index out of range")
        j %= n
        v = _checked_scalar(self._buf.dtype, value)
        list.__setitem__(self, j, v)
        self._buf[j] = v

    def _fixed(self, *args, **kwargs):
        raise TypeError("tensor storage has a fixed size; assign whole-list data through the .data setter")

    append = extend = insert = pop = remove = clear = __delitem__ = __iadd__ = __imul__ = _fixed

    def _write_all(self):
        self._buf.copy_(torch.as_tensor(list(self), dtype=self._buf.dtype))

    def sort(self, *args, **kwargs):
        list.sort(self, *args, **kwargs)
        self._write_all()

    def reverse(self):
        list.reverse(self)
        self._write_all()


def _infer_dtype(data) -> torch.dtype:
    if isinstance(data, torch.Tensor):
        if data.dtype in (torch.float32, torch.float64, torch.int64):
            return data.dtype
        return torch.float64 if data.is_floating_point() else torch.int64
    if isinstance(data, np.ndarray):
        if data.dtype == np.float32:
            return torch.float32
        if data.dtype.kind in "iub":
            return torch.int64
        return torch.float64
    seq = list(data)
    if seq and all(isinstance(x, numbers.Integral) and not isinstance(x, bool) for x in seq):
        return torch.int64
    return torch.float64


class DenseTensor:
    """Dense array with runtime order, extents, offsets and layout, stored
    on the GPU in memory-index order."""

    # _ssq: (device [sum C^2, ||C||], the buffer it describes, its version)
    # when a kernel computed the Frobenius norm of this tensor's values as it
    # produced them (ttm's fused epilogue); valid while the buffer is the
    # same object at the same torch version (every in-place write through
    # this API -- .data, item/element setters, fill, copy_ -- bumps it)
    __slots__ = ("meta", "buffer", "_ssq")

    def __init__(self, shape, offsets=None, layout=None, fill_value=0, dtype=None, device=None):
        """Value-initialised like the reference (tensor.py:44-46).
        ``fill_value=None`` leaves the buffer uninitialised (contraction
        outputs, which the kernels overwrite completely)."""
        self.meta = TensorMeta(shape, offsets, layout)
        self._ssq = None
        dt = as_dtype(dtype)
        dev = _device(device)
        if fill_value is None:
            self.buffer = torch.empty((self.meta.size,), dtype=dt, device=dev)
        else:
            self.buffer = torch.full((self.meta.size,), fill_value, dtype=dt, device=dev)

    # -- construction -------------------------------------------------------------
    @classmethod
    def _wrap(cls, meta: TensorMeta, buffer: torch.Tensor) -> "DenseTensor":
        t = cls.__new__(cls)
        t.meta = meta
        t.buffer = buffer
        t._ssq = None
        return t

    def _fused_norm(self):
        """The device [sum of squares, norm] a producing kernel left for this
        exact buffer state, or None."""
        f = getattr(self, "_ssq", None)
        if f is None or f[1] is not self.buffer or f[2] != self.buffer._version:
            return None
        return f[0]

    @classmethod
    def from_memory(cls, shape, data, offsets=None, layout=None, dtype=None, device=None) -> "DenseTensor":
        """Copy a flat element sequence in memory order (tensor.py:48-59).

        ``data`` may be a list/tuple, a numpy array or a torch tensor (host
        or device; a pinned host tensor is copied asynchronously)."""
        meta = TensorMeta(shape, offsets, layout)
        dt = as_dtype(dtype) if dtype is not None else _infer_dtype(data)
        dev = _device(device)
        if isinstance(data, torch.Tensor):
            src = data.reshape(-1)
            buf = torch.empty(src.numel(), dtype=dt, device=dev)
            buf.copy_(src, non_blocking=src.is_pinned())
        else:
            arr = np.asarray(data if isinstance(data, np.ndarray) else list(data))
            np_dt = {torch.float64: np.float64, torch.float32: np.float32, torch.int64: np.int64}[dt]
            buf = torch.from_numpy(np.ascontiguousarray(arr.reshape(-1), dtype=np_dt)).to(dev)
        if buf.numel() != meta.size:
            raise ValueError(f"data length {buf.numel()} does not match volume {meta.size}")
        return cls._wrap(meta, buf)

    # -- structure ----------------------------------------------------------------
    @property
    def shape(self):
        return self.meta.shape

    @property
    def order(self) -> int:
        return self.meta.order

    @property
    def layout(self):
        return self.meta.layout

    @property
    def offsets(self):
        return self.meta.offsets

    @property
    def strides(self):
        return self.meta.strides

    @property
    def size(self) -> int:
        return self.buffer.numel()

    @property
    def dtype(self) -> torch.dtype:
        return self.buffer.dtype

    @property
    def device(self) -> torch.device:
        return self.buffer.device

    def desc(self) -> _abi.TlDesc:
        """The device layout descriptor (plays the MultiIterator's role)."""
        return _abi.make_desc(self.shape, self.strides, _abi.DTYPE_CODE[self.dtype])

    def ptr(self) -> int:
        return self.buffer.data_ptr()

    # -- host interchange ------------------------------------------------------------
    @property
    def data(self) -> list:
        """The buffer in memory-index order as a host list whose element and
        slice writes go through to the device (see ``_DataList``)."""
        return _DataList(self.buffer)

    @data.setter
    def data(self, values) -> None:
        """Replace every element (memory-index order).  An int64 tensor that
        is given non-integral values becomes float64, as the reference's
        list would simply hold them."""
        if isinstance(values, torch.Tensor):
            src = values.reshape(-1)
        else:
            arr = values if isinstance(values, np.ndarray) else np.asarray(list(values))
            src = torch.as_tensor(np.ascontiguousarray(arr.reshape(-1)))
        if src.numel() != self.meta.size:
            raise ValueError(f"data length {src.numel()} does not match volume {self.meta.size}")
        if self.dtype == torch.int64 and src.is_floating_point() and not bool(torch.all(src == torch.round(src))):
            self.buffer = torch.empty(self.meta.size, dtype=torch.float64, device=self.device)
        self.buffer.copy_(src.to(self.dtype))

    def numpy(self) -> np.ndarray:
        return self.buffer.cpu().numpy()

    def copy(self) -> "DenseTensor":
        return DenseTensor._wrap(self.meta, self.buffer.clone())

    # -- element access (host round trips; for tests and small tensors) -----------------
    def _key(self, key) -> tuple:
        key = (key,) if isinstance(key, numbers.Integral) else tuple(key)
        if len(key) != self.order:
            raise ValueError(f"expected {self.order} indices, got {len(key)}")
        for r, (i, o, n) in enumerate(zip(key, self.offsets, self.shape)):
            if not o <= i < o + n:
                raise IndexError(f"index {i} out of bounds [{o}, {o + n}) in dimension {r + 1}")
        return key

    def __getitem__(self, key):
        return self.buffer[memory_index(self.strides, self._key(key), self.offsets)].item()

    def __setitem__(self, key, value):
        self.buffer[memory_index(self.strides, self._key(key), self.offsets)] = _checked_scalar(self.dtype, value)

    def get_memory(self, j: int):
        if not 0 <= j < self.size:
            raise IndexError(f"memory index {j} out of range [0, {self.size})")
        return self.buffer[j].item()

    def set_memory(self, j: int, value) -> None:
        if not 0 <= j < self.size:
            raise IndexError(f"memory index {j} out of range [0, {self.size})")
        self.buffer[j] = _checked_scalar(self.dtype, value)

    def item(self):
        if self.size != 1:
            raise ValueError(f"item() requires volume 1, got {self.size}")
        return self.buffer[0].item()

    # -- whole-tensor operations ---------------------------------------------------------
    def fill(self, value) -> None:
        self.buffer.fill_(value)

    def relayout(self, new_layout) -> None:
        """Physically reorder to ``new_layout`` keeping index -> value
        (tensor.py:167-184), with the device copy kernel."""
        new_layout = validate_layout(new_layout, self.order)
        if new_layout == self.layout:
            return
        new_meta = TensorMeta(self.shape, self.offsets, new_layout)
        out = torch.empty_like(self.buffer)
        _copy(self.desc(), self.buffer, _abi.make_desc(self.shape, new_meta.strides, _abi.DTYPE_CODE[self.dtype]), out)
        self.meta = new_meta
        self.buffer = out

    def assign(self, src) -> None:
        """Copy src's values per zero-based multi-index (tensor.py:141-165)."""
        if src is self:
            return
        if self.order == src.order:
            meta = TensorMeta(src.shape, self.offsets, self.layout)
        else:
            meta = TensorMeta(src.shape, src.offsets, src.layout)
        out = torch.empty(meta.size, dtype=src.dtype, device=src.device)
        _copy(src.desc(), src.buffer, _abi.make_desc(meta.shape, meta.strides, _abi.DTYPE_CODE[src.dtype]), out)
        self.meta = meta
        self.buffer = out

    def reshape(self, new_shape) -> None:
        """Adopt a same-volume shape keeping the memory sequence (tensor.py:186-200)."""
        new_shape = validate_shape(new_shape)
        if volume(new_shape) != self.size:
            raise ValueError(f"reshape to {new_shape} changes volume ({volume(new_shape)} != {self.size})")
        self.meta = self.meta.with_shape(new_shape)

    def to(self, dtype) -> "DenseTensor":
        return DenseTensor._wrap(self.meta, self.buffer.to(as_dtype(dtype)))

    # -- iterators (tensor.py:204-235) ----------------------------------------------------
    def miter(self) -> MultiIterator:
        """Cursor at the first element over the device buffer; accepted by
        every hot-path function as an operand (contraction.py:52-55)."""
        return MultiIterator(self.buffer, 0, self.strides, self.shape)

    def dim_begin(self, dim: int, at=None) -> StrideIterator:
        """Stride iterator over dimension ``dim`` (one-based); ``at`` fixes
        the other coordinates as an absolute multi-index."""
        return StrideIterator(self.buffer, self._dim_base(dim, at), self.strides[dim - 1])

    def dim_end(self, dim: int, at=None) -> StrideIterator:
        w = self.strides[dim - 1]
        return StrideIterator(self.buffer, self._dim_base(dim, at) + self.shape[dim - 1] * w, w)

    def _dim_base(self, dim: int, at) -> int:
        if not 1 <= dim <= self.order:
            raise ValueError(f"dimension {dim} out of range 1..{self.order}")
        if at is None:
            return 0
        if len(at) != self.order:
            raise ValueError(f"expected {self.order} indices, got {len(at)}")
        return sum(self.strides[r] * (at[r] - self.offsets[r]) for r in range(self.order) if r != dim - 1)

    def view(self, *ranges):
        """Rectangular view (tensor.py:237-250): one range per dimension, or
        one sequence of them."""
        from .views import TensorView

        if len(ranges) == 1 and isinstance(ranges[0], (list, tuple)):
            ranges = tuple(ranges[0])
        return TensorView(self, ranges)

    # -- interchange -------------------------------------------------------------------
    def to_dict(self) -> dict:
        return {"shape": list(self.shape), "layout": list(self.layout), "offsets": list(self.offsets),
                "data": self.buffer.cpu().tolist()}

    @classmethod
    def from_dict(cls, obj: dict) -> "DenseTensor":
        try:
            shape, data = obj["shape"], obj["data"]
            layout, offsets = obj.get("layout"), obj.get("offsets")
        except (TypeError, KeyError) as exc:
            raise ValueError(f"malformed tensor object: missing {exc}") from exc
        return cls.from_memory(shape, data, offsets, layout)

    def __eq__(self, other):
        if not isinstance(other, DenseTensor):
            return NotImplemented
        return tensors_equal(self, other)

    __hash__ = None

    def __repr__(self):
        return f"DenseTensor(shape={self.shape}, offsets={self.offsets}, layout={self.layout}, dtype={self.dtype})"


def _copy(adesc, abuf: torch.Tensor, cdesc, cbuf: torch.Tensor) -> None:
    L = _abi.lib()
    rc = L.tl_copy(adesc, abuf.data_ptr(), cdesc, cbuf.data_ptr(), _abi.stream_handle())
    _abi.check(rc, "copy")


def tensors_equal(a, b) -> bool:
    """Equal order, shape and elements per zero-based multi-index; layout
    and offsets are ignored; tensors and views alike (tensor.py:287-304)."""
    if a.order != b.order or a.shape != b.shape:
        return False
    if not isinstance(a, DenseTensor) or not isinstance(b, DenseTensor):
        from .views import as_dense_operand

        a, b = as_dense_operand(a), as_dense_operand(b)
    if a.layout == b.layout:
        return bool(torch.equal(a.buffer, b.buffer.to(a.dtype)))
    tmp = torch.empty_like(b.buffer)
    _copy(b.desc(), b.buffer, _abi.make_desc(b.shape, a.strides, _abi.DTYPE_CODE[b.dtype]), tmp)
    return bool(torch.equal(a.buffer, tmp.to(a.dtype)))
