"""CPU-only checks: the C-ABI library loads and exports every symbol the
header declares, its argument validation mirrors the reference's errors
(no device work is reached), and the host-side layout algebra."""

import ctypes
import os
import re

import pytest

from paper_1711_10912_b200 import _abi
from paper_1711_10912_b200.layout import (
    TensorMeta,
    compute_strides,
    first_order_layout,
    inverse_memory_index,
    last_order_layout,
    memory_index,
    zero_indices,
)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    text = open(os.path.join(ROOT, "include", "tensorlib_b200.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(tl_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_header_symbols():
    L = _abi.load_library()
    names = header_functions()
    assert len(names) >= 14
    for n in names:
        assert hasattr(L, n), n
    assert set(_abi.EXPORTS) <= set(names)
    assert L.tl_abi_version() == 1
    assert L.tl_device_arch() == 100


def test_library_is_sm100a_cubin():
    import subprocess

    out = subprocess.run(["cuobjdump", "--list-elf", _abi.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def desc(shape, strides=None, dtype=_abi.TL_F64):
    if strides is None:
        strides = compute_strides(shape, first_order_layout(len(shape)))
    return _abi.make_desc(shape, strides, dtype)


def test_abi_validation_mirrors_reference_errors():
    L = _abi.load_library()
    a = desc((3, 4))
    # mode out of range (contraction.py:125-126)
    assert L.tl_ttv(a, None, desc((4,)), None, desc((3,)), None, 3, None) == _abi.TL_EINVAL
    assert b"out of range" in L.tl_last_error()
    # vector length mismatch (contraction.py:65-68)
    assert L.tl_ttv(a, None, desc((5,)), None, desc((3,)), None, 2, None) == _abi.TL_EINVAL
    # order-1 tensor (contraction.py:123-124)
    assert L.tl_ttv(desc((4,)), None, desc((4,)), None, desc((1,)), None, 1, None) == _abi.TL_EINVAL
    # ttm matrix columns mismatch / order (contraction.py:216-222)
    assert L.tl_ttm(a, None, desc((2, 5)), None, desc((3, 2)), None, 2, None) == _abi.TL_EINVAL
    assert L.tl_ttm(a, None, desc((2, 4, 1)), None, desc((3, 2)), None, 2, None) == _abi.TL_EINVAL
    # inner shape mismatch (elementwise.py:69-70)
    assert L.tl_inner(desc((2, 3)), None, desc((3, 2)), None, None, None, 0, None) == _abi.TL_EINVAL
    # non-first-order output
    assert L.tl_ttv(a, None, desc((4,)), None, desc((3, 1), (3, 1)), None, 2, None) == _abi.TL_EINVAL
    # hopm max_sweeps < 1 (hopm.py:79-80)
    ptrs = (ctypes.c_void_p * 2)()
    assert L.tl_hopm(a, None, None, ptrs, 0, 0.0, None, None, None, None, 0, None) == _abi.TL_EINVAL


def test_compute_strides_rule_and_erratum():
    # the rule gives (6,3,1) for (4,2,3) under (3,2,1) -- not the paper's (6,2,1)
    assert compute_strides((4, 2, 3), (3, 2, 1)) == (6, 3, 1)
    assert compute_strides((4, 2, 3), (1, 2, 3)) == (1, 4, 8)
    assert compute_strides((128,) * 4, (3, 1, 2, 4)) == (128, 16384, 1, 2097152)
    assert compute_strides((3, 33, 5, 17, 9, 2, 640), (5, 3, 2, 1, 6, 4, 7)) == (1485, 45, 9, 8910, 1, 4455, 151470)
    assert first_order_layout(3) == (1, 2, 3) and last_order_layout(3) == (3, 2, 1)


def test_meta_and_index_round_trip():
    m = TensorMeta((3, 4, 2), offsets=(1, -2, 0), layout=(2, 3, 1))
    with pytest.raises(AttributeError):
        m.shape = (1,)
    seen = set()
    for idx in zero_indices(m.shape):
        j = memory_index(m.strides, tuple(i + o for i, o in zip(idx, m.offsets)), m.offsets)
        assert inverse_memory_index(m, j) == idx
        seen.add(j)
    assert seen == set(range(24))
    with pytest.raises(ValueError):
        TensorMeta((2, 0))
    with pytest.raises(ValueError):
        TensorMeta((2, 2), layout=(1, 1))
