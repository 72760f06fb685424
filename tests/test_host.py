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
    assert L.tl_hopm(a, None, None, ptrs, 0, 0.0, None, None, None, None, None, 0, None) == _abi.TL_EINVAL
    # null data pointers are refused before any device work
    assert L.tl_ttv(a, None, desc((4,)), None, desc((3,)), None, 2, None) == _abi.TL_EINVAL
    assert b"null data pointer" in L.tl_last_error()
    assert L.tl_copy(a, None, a, None, None) == _abi.TL_EINVAL
    # host-only plan query rejects a bad mode
    buf = ctypes.create_string_buffer(256)
    assert L.tl_plan_describe(0, a, None, 5, buf, 256) == _abi.TL_EINVAL


def plan(op, shape, layout, mode, dtype=_abi.TL_F32, bshape=None):
    import json

    L = _abi.load_library()
    L.tl_plan_describe.argtypes = [ctypes.c_int32, ctypes.POINTER(_abi.TlDesc), ctypes.POINTER(_abi.TlDesc),
                                   ctypes.c_int32, ctypes.c_char_p, ctypes.c_size_t]
    buf = ctypes.create_string_buffer(2048)
    b = desc(bshape, dtype=dtype) if bshape else None
    rc = L.tl_plan_describe(op, desc(shape, compute_strides(shape, layout), dtype), b, mode, buf, 2048)
    assert rc == 0, L.tl_last_error()
    return json.loads(buf.value.decode())


# SURVEY.md §8a canonical forms (A: contracted stride 1 -> staged; B: strided).
CFG2_TABLE = {
    (1, 2, 3, 4): [("staged", 2**21, 1, True), ("strided", 2**14, 128, True), ("strided", 128, 2**14, True),
                   ("strided", 1, 2**21, True)],
    (4, 3, 2, 1): [("strided", 1, 2**21, False), ("strided", 128, 2**14, False), ("strided", 2**14, 128, False),
                   ("staged", 2**21, 1, False)],
    (3, 1, 2, 4): [("strided", 2**14, 128, False), ("strided", 128, 2**14, False), ("staged", 2**21, 1, True),
                   ("strided", 1, 2**21, False)],
}


@pytest.mark.parametrize("layout", list(CFG2_TABLE))
def test_ttv_canonical_forms_match_survey(layout):
    for mode, (regime, O, I, ident) in enumerate(CFG2_TABLE[layout], start=1):
        p = plan(0, (128,) * 4, layout, mode)
        # permuted outputs of regime B take the boxed variant of the strided kernel
        got = "strided" if p["regime"] == "strided-box" else p["regime"]
        assert (got, p["O"], p["K"], p["I"], bool(p["ident"])) == (regime, O, 128, I, ident), (layout, mode)
        assert p["regime"] != "strided-box", (layout, mode)  # K = 128: the plain strided kernel


def test_ttv_plans_for_other_configs():
    # config 1: O=64, K=96, I=128 -- 8192 outputs of a 6 MB operand: latency-bound,
    # whole-block small kernel
    p = plan(0, (128, 96, 64), (1, 2, 3), 2, _abi.TL_F64)
    assert (p["regime"], p["O"], p["K"], p["I"]) == ("small-cols", 64, 96, 128)
    # a large operand with as few outputs (64 x 128 fibres of 4096 terms):
    # 2-D TMA column boxes (the per-thread ring where the driver's tensor-map
    # encoder is unavailable, e.g. this CPU-only host)
    assert plan(0, (128, 4096, 64), (1, 2, 3), 2, _abi.TL_F64)["regime"] in ("cols-tma", "deep-ring")
    # config 5 seed 0 layout: contracted stride 1, K=9, permuted output, TMA bulk tiles
    shape5 = (3, 33, 5, 17, 9, 2, 640)
    p = plan(0, shape5, (5, 3, 2, 1, 6, 4, 7), 5, _abi.TL_F64)
    assert (p["regime"], p["O"], p["K"], p["I"], p["ident"]) == ("staged-bulk", 10771200, 9, 1, 0)
    # config 5 seed 5 layout: O=1, I=10.7M (regime B)
    p = plan(0, shape5, (7, 4, 2, 1, 6, 3, 5), 5, _abi.TL_F64)
    assert (p["regime"], p["O"], p["I"]) == ("strided-box", 1, 10771200)
    # HOPM's 400x400 intermediates use the small-problem kernels
    assert plan(0, (400, 400), (1, 2), 1, _abi.TL_F64)["regime"] == "small-rows"
    assert plan(0, (400, 400), (1, 2), 2, _abi.TL_F64)["regime"] == "small-cols"


def test_ttv_plans_on_the_config5_shape_round2():
    """Planner rules added in round 2 ("The configs' own shapes"), on the
    order-7 config-5 shape in layouts of the every-layout sweep."""
    shape = (3, 33, 5, 17, 9, 2, 640)
    # rows of 2 elements x 640 k-rows: the staged tiles with fewer rows per tile, not one thread per fibre
    p = plan(0, shape, (6, 7, 3, 4, 5, 1, 2), 7, _abi.TL_F64)
    assert (p["regime"], p["K"], p["I"]) == ("staged", 640, 2)
    # unaligned rows (33 doubles = 264 bytes): 96 rows per tile stream as one TMA bulk copy
    p = plan(0, shape, (2, 5, 3, 4, 7, 6, 1), 2, _abi.TL_F64)
    assert (p["regime"], p["K"], p["I"], p["block"]) == ("staged-bulk", 33, 1, 96)
    # short folds with scattered outputs: the tile-fold kernel with flattened chains -- also when the
    # C-fastest digit is A's fastest one (extent 3), when a chain extent is ragged (33, 85), and for
    # 4 < K <= 8 on the strided regime
    for layout, mode, K, I in [((1, 6, 7, 3, 5, 2, 4), 6, 2, 3), ((6, 1, 2, 5, 3, 7, 4), 1, 3, 2),
                               ((3, 4, 1, 6, 5, 2, 7), 1, 3, 85), ((2, 3, 1, 6, 5, 4, 7), 3, 5, 33)]:
        p = plan(0, shape, layout, mode, _abi.TL_F64)
        assert (p["regime"], p["K"], p["I"]) == ("tile-fold", K, I), (layout, mode, p)
    # K = 9 (config 5's own mode) stays on the boxed / strided kernels
    assert plan(0, shape, (7, 4, 2, 1, 6, 3, 5), 5, _abi.TL_F64)["regime"] in ("strided", "strided-box")


def test_ttm_gett_plans():
    # config 3 on the GETT: operand majors and the free-digit order sigma
    p = plan(1, (512,) * 3, (1, 2, 3), 1, _abi.TL_F64, (384, 512))
    assert p["path"] == "gett" and p["a_kmajor"] == 1 and p["jstride"] == 1 and p["pairs"] == 1
    p = plan(1, (512,) * 3, (1, 2, 3), 2, _abi.TL_F64, (384, 512))
    assert (p["O"], p["K"], p["I"], p["a_kmajor"]) == (512, 512, 512, 0)
    # last-order mode 2: A's and C's fastest free dims differ -> 2-D box 8 x 16
    p = plan(1, (512,) * 3, (3, 2, 1), 2, _abi.TL_F64, (384, 512))
    assert p["sigma"][0] == [8, 1, 196608] and p["sigma"][1] == [16, 262144, 1]
    # config 5's ttm (J = 16) is HBM-bound -> the warp-specialised stream
    # kernel: 8-slab tiles (24 positions = 3 whole n8 tiles), 8 consumer warps
    # with 3 private slots each inside the 220 KB budget
    p = plan(1, (3, 33, 5, 17, 2, 640), (1, 2, 3, 4, 5, 6), 2, _abi.TL_F64, (16, 33))
    assert (p["path"], p["O"], p["K"], p["I"], p["J"]) == ("stream", 108800, 33, 3, 16)
    assert (p["R"], p["NT"], p["warps"], p["slots_per_warp"]) == (8, 3, 8, 3) and p["smem"] <= 220 * 1024


def test_ttm_small_j_plans():
    # J = 32 on a (5, 37, 20001) tensor: tiles sized so all 8 warps keep 2 slots
    p = plan(1, (5, 37, 20001), (1, 2, 3), 2, _abi.TL_F64, (32, 37))
    assert p["path"] == "stream" and p["warps"] == 8 and p["slots_per_warp"] >= 2
    assert (p["R"] * p["I"]) <= 8 * p["NT"] and p["R"] * p["K"] * p["I"] % 2 == 0
    # Where the stream / bulk tile kernels do not apply (R*I = 256 positions
    # exceed a warp and a bulk plan would need 512 threads: the wide-fuzz
    # regression; permuted outputs; float32 / int64), the few-row box kernel
    # of csrc/ttm_few.cu takes J <= 32 with K <= 128 (round 2)
    p = plan(1, (2, 8, 16, 7, 5, 2, 8), (1, 2, 3, 4, 5, 6, 7), 4, _abi.TL_F64, (25, 7))
    assert (p["path"], p["store"], p["ba"] * p["bc"]) == ("few", "direct", 128)
    # permuted output whose fastest free digit differs from A's: a 2-D box written along C
    p = plan(1, (20, 60, 3), (2, 1, 3), 1, _abi.TL_F64, (32, 20))
    assert (p["path"], p["store"]) == ("few", "along-j")  # mode 1: C is contiguous along j
    p = plan(1, (3, 33, 5, 17, 2, 640), (4, 3, 6, 5, 1, 2), 2, _abi.TL_F64, (16, 33))
    assert (p["path"], p["store"], p["ba"] * p["bc"]) == ("few", "along-y", 128)
    assert p["X"] * p["Y"] == 3 * 5 * 17 * 2 * 640 and p["ba"] == 32  # K >= 2 J: long runs along A
    p = plan(1, (3, 33, 5, 17, 2, 640), (4, 3, 6, 5, 1, 2), 5, _abi.TL_F64, (16, 2))
    assert (p["path"], p["store"], p["ba"]) == ("few", "along-y", 4)  # K < J / 2: long runs along C
    # long folds (K > 128) keep the GETT, now with a 16- / 32-row tile
    assert plan(1, (200, 60, 3), (2, 1, 3), 1, _abi.TL_F64, (32, 200))["path"] == "gett"
    assert plan(1, (3, 33, 5, 17), (1, 2, 3, 4), 2, _abi.TL_F32, (16, 33))["path"] == "few"
    assert plan(1, (9, 31, 4), (1, 2, 3), 3, _abi.TL_F64, (15, 4))["path"] == "few"
    # more than 32 rows: GETT / staged / SIMT as before
    assert plan(1, (9, 31, 4), (1, 2, 3), 3, _abi.TL_F64, (40, 4))["path"] == "simt"


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


def test_range_and_spec_validation_host():
    """Host-side argument rules of views.py:25-80 and contraction.py:304-334,
    421-440 (no device needed)."""
    from paper_1711_10912_b200 import ContractionSpec, Range, reduce_ttm_to_ttt, reduce_ttv_to_ttt

    assert Range().is_full
    r = Range(2, 3, 9)
    assert (r.first, r.step, r.last) == (2, 3, 9)
    assert r.resolve(0, 10, 1) == (2, 3, 9)
    assert Range(4).resolve(1, 5, 1) == (4, 1, 4)
    for bad in [(3, 1), (1, 0, 4), (1, 2, 3, 4)]:
        with pytest.raises(ValueError):
            Range(*bad)
    with pytest.raises(IndexError):
        Range(0, 10).resolve(0, 10, 1)
    s = ContractionSpec(2, [3, 1, 2], [3, 2, 1])
    assert (s.q, s.r, s.s, s.phi, s.psi) == (2, 1, 1, (3, 1, 2), (3, 2, 1))
    for bad in [(1, (1, 1), (1,)), (2, (1,), (1, 2)), (-1, (1,), (1,)), (0, (), (1,))]:
        with pytest.raises(ValueError):
            ContractionSpec(*bad)
    assert reduce_ttv_to_ttt(3, 2) == ContractionSpec(1, (1, 3, 2), (1,))
    assert reduce_ttm_to_ttt(4, 1) == ContractionSpec(1, (2, 3, 4, 1), (1, 2))
    with pytest.raises(ValueError):
        reduce_ttm_to_ttt(2, 0)


def test_gett_tile_store_order():
    # 64-wide tiles hold 8 A-fast x 8 C-fast positions of the 8 x 16 box; the
    # staged epilogue writes them in C order
    p = plan(1, (512,) * 3, (3, 2, 1), 2, _abi.TL_F64, (384, 512))
    assert p["box"] == 64
    assert plan(1, (512,) * 3, (1, 2, 3), 2, _abi.TL_F64, (384, 512))["box"] == 0
    # J = 32 with a small K stays on the small-J family (the stream kernel)
    assert plan(1, (5, 37, 2001), (1, 2, 3), 2, _abi.TL_F64, (32, 37))["path"] == "stream"


def test_product_package_never_touches_the_oracle():
    """The oracle is test infrastructure only: no module of the package
    imports, loads or names it, and the package has no CPU compute path."""
    pkg = os.path.join(ROOT, "paper_1711_10912_b200")
    for fn in os.listdir(pkg):
        if fn.endswith(".py"):
            text = open(os.path.join(pkg, fn)).read()
            assert "oracle" not in text, fn
            assert "tl_oracle" not in text and "libtloracle" not in text, fn


def test_exact_dot_matches_fractions():
    """The normwise inner-product reference (tests/tolerance.py) is exact."""
    import fractions

    import numpy as np
    from tolerance import exact_dot

    rng = np.random.default_rng(7)
    for n in (1, 7, 300):
        a, b = rng.standard_normal(n) * 1e3, rng.standard_normal(n) * 1e-3
        want = float(sum(fractions.Fraction(x) * fractions.Fraction(y) for x, y in zip(a, b)) + fractions.Fraction(0.5))
        assert exact_dot(a, b, 0.5) == want


def test_walk_positions_host_cursor():
    """Iterator bookkeeping needs no device: the reference recursion's visit
    order (iterators.py:165-182) over a host-list cursor."""
    from paper_1711_10912_b200 import MultiIterator, walk_positions

    it = MultiIterator([0] * 24, 0, (1, 4, 12), (4, 3, 2))
    assert walk_positions(it) == list(range(24))
    it = MultiIterator([0] * 24, 1, (6, 1), (4, 2))
    assert walk_positions(it) == [1 + 6 * i + j for j in range(2) for i in range(4)]
    assert it.begin(1).stride == 1 and it.end(0).pos == 1 + 24
