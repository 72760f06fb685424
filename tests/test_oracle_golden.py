"""Pin the CPU oracle to the reference: every golden output produced by
running the reference implementation (tests/golden/make_golden.py) must be
reproduced BIT FOR BIT by oracle/tl_oracle.c.  CPU only."""

import hashlib
import math

import numpy as np
import pytest

import workloads as W
from oracle import oracle as O


def sha(arr):
    return hashlib.sha256(np.ascontiguousarray(arr).tobytes()).hexdigest()


def strides_of(case, key="layout"):
    return W.compute_strides(case["shape"], case[key])


def test_oracle_ttv_small(small_golden):
    n = 0
    for c in small_golden["cases"]:
        if c["op"] != "ttv":
            continue
        got = O.ttv(c["a"], c["shape"], strides_of(c), c["b"], c["mode"])
        want = c["out"]
        assert got.dtype == want.dtype
        assert np.array_equal(got.view(np.uint64 if got.dtype == np.float64 else np.int64),
                              want.view(np.uint64 if want.dtype == np.float64 else np.int64)), c
        n += 1
    assert n >= 100


def test_oracle_ttm_small(small_golden):
    n = 0
    for c in small_golden["cases"]:
        if c["op"] != "ttm":
            continue
        bstr = W.compute_strides(c["bshape"], c["blayout"])
        got = O.ttm(c["a"], c["shape"], strides_of(c), c["bmat"], c["bshape"], bstr, c["mode"])
        assert np.array_equal(got, c["out"]) and got.tobytes() == c["out"].tobytes(), c
        # sampled evaluation agrees with the full one
        sel = np.arange(0, got.size, 3)
        part = O.ttm(c["a"], c["shape"], strides_of(c), c["bmat"], c["bshape"], bstr, c["mode"], select=sel)
        assert part.tobytes() == got[sel].tobytes()
        n += 1
    assert n >= 60


def test_oracle_ttm_canon_small(small_golden):
    """The full-size (canonical-form, vectorised) ttm restatement equals the
    reference's outputs bit for bit on every float golden case."""
    n = 0
    for c in small_golden["cases"]:
        if c["op"] != "ttm" or np.asarray(c["a"]).dtype.kind != "f":
            continue
        bstr = W.compute_strides(c["bshape"], c["blayout"])
        layout = tuple(c["layout"])
        got = O.ttm_canon(c["a"], c["shape"], layout, c["bmat"], c["bshape"], bstr, c["mode"])
        out_shape = list(c["shape"])
        out_shape[c["mode"] - 1] = c["bshape"][0]
        first = W.from_buffer(got, tuple(out_shape), layout).ravel(order="F")
        assert first.tobytes() == np.asarray(c["out"], dtype=np.float64).tobytes(), c
        n += 1
    assert n >= 20


def test_oracle_inner_norm_small(small_golden):
    for c in small_golden["cases"]:
        if c["op"] == "inner":
            got = O.inner(c["a"], c["shape"], strides_of(c), c["b"], strides_of(c, "blayout"))
            assert got == c["value"] and type(got) is type(c["value"]), c
        elif c["op"] == "norm":
            got = O.norm(c["a"], c["shape"], strides_of(c))
            assert got == c["value"], c


def test_oracle_hopm_small(small_golden):
    n = 0
    for c in small_golden["cases"]:
        if c["op"] != "hopm":
            continue
        u0 = None
        if "u0" in c:
            u0, off = [], 0
            for k in c["shape"]:
                u0.append(c["u0"][off:off + k])
                off += k
        r = O.hopm(c["a"], c["shape"], strides_of(c), max_sweeps=c["max_sweeps"], tol=c["tol"], u0=u0)
        assert r["sweeps"] == c["sweeps"] and r["converged"] == c["converged"]
        assert np.concatenate(r["u"]).tobytes() == c["u"].tobytes()
        assert np.asarray(r["l"]).tobytes() == c["l"].tobytes()
        assert np.asarray(r["lambda_history"]).tobytes() == c["lambda_history"].tobytes()
        n += 1
    assert n >= 8


def test_oracle_kats(small_golden):
    kat = small_golden["kat"]
    # ttv(I_2, ones, 2) == [1, 1]   (test_contraction.py:78-80)
    eye = np.array([1, 0, 0, 1], dtype=np.int64)
    assert O.ttv(eye, (2, 2), (1, 2), np.ones(2, dtype=np.int64), 2).tolist() == kat["ttv_identity_row_sums"]
    ones = np.ones(12, dtype=np.int64)
    assert O.ttv(ones, (2, 3, 2), (1, 2, 6), np.ones(3, dtype=np.int64), 2).tolist() == kat["ttv_counting"]
    assert O.norm(np.ones(8), (2, 2, 2), (1, 2, 4)) == kat["norm_all_ones_222"] == math.sqrt(8)
    r = O.hopm(np.array([3.0, 0.0, 4.0]), (3,), (1,))
    assert r["l"] == kat["hopm_order_one"]["l"] and r["u"][0].tolist() == kat["hopm_order_one"]["u"]
    with pytest.raises(O.OracleDegenerate) as e:
        O.hopm(np.zeros(6), (2, 3), (1, 2))
    assert [e.value.sweep, e.value.mode] == kat["hopm_zero_degenerate"]


def test_oracle_cfg1(configs_golden):
    g = configs_golden["cfg1"]
    T, b = W.cfg1()
    assert sha(T) == g["input_sha256"]
    got = O.ttv(W.layout_buffer(T, (1, 2, 3)), T.shape, (1, 128, 128 * 96), b, 2)
    assert sha(got) == g["sha256"]


@pytest.mark.parametrize("seed", [0, 5])
def test_oracle_cfg5_chain(configs_golden, seed):
    key = f"cfg5_seed{seed}"
    if key not in configs_golden:
        pytest.skip(f"{key} not generated")
    g = configs_golden[key]
    T, v, M, layout = W.cfg5(seed)
    assert list(layout) == g["layout"]
    buf = W.layout_buffer(T, layout)
    c1 = O.ttv(buf, T.shape, W.compute_strides(T.shape, layout), v, 5)
    assert sha(c1) == g["ttv_sha256"]
    shp1 = g["ttv_shape"]
    c2 = O.ttm(c1, shp1, W.compute_strides(shp1, W.first_order(6)), W.layout_buffer(M, (1, 2)), M.shape, (1, 16), 2)
    assert sha(c2) == g["ttm_sha256"]
    assert O.norm(c2, g["ttm_shape"], W.compute_strides(g["ttm_shape"], W.first_order(6))) == g["norm"]


def test_oracle_cfg2(configs_golden):
    if "cfg2" not in configs_golden:
        pytest.skip("cfg2 not generated")
    g = configs_golden["cfg2"]
    T, vecs, T2 = W.cfg2()
    for name, layout in W.CFG2_LAYOUTS.items():
        buf = W.layout_buffer(T, layout)
        st = W.compute_strides(T.shape, layout)
        for mode in (1, 2, 3, 4):
            key = f"ttv_{name}_q{mode}"
            if key not in g:
                continue
            got = O.ttv(buf, T.shape, st, vecs[mode - 1], mode)
            assert sha(got) == g[key]["sha256"], key
    if "norm_first" in g:
        st = W.compute_strides(T.shape, (1, 2, 3, 4))
        assert O.norm(W.layout_buffer(T, (1, 2, 3, 4)), T.shape, st) == g["norm_first"]["value"]


def test_oracle_cfg4(configs_golden):
    if "cfg4" not in configs_golden:
        pytest.skip("cfg4 not generated")
    g = configs_golden["cfg4"]
    T, _ = W.cfg4()
    r = O.hopm(W.layout_buffer(T, (1, 2, 3)), T.shape, (1, 400, 160000), max_sweeps=50, tol=0.0)
    assert r["lambda_history"] == g["lambda_history"]
    assert r["l"] == g["l"]
    for u, want in zip(r["u"], g["u"]):
        assert u.tolist() == want


def test_oracle_ttt_transpose_small(small_golden):
    """The pure-Python ttt / transpose restatements reproduce the
    reference's outputs bit for bit (contraction.py:75-107, 337-454)."""
    n = 0
    for c in small_golden["cases"]:
        if c["op"] == "ttt":
            out, shape = O.ttt(c["a"], c["shape"], strides_of(c), c["b"], c["bshape"],
                               W.compute_strides(c["bshape"], c["blayout"]), c["q"], c["phi"], c["psi"], c["kind"])
        elif c["op"] == "outer":
            sa, sb = c["shape"], c["bshape"]
            out, shape = O.ttt(c["a"], sa, O.first_order_strides(sa), c["b"], sb, O.first_order_strides(sb), 0,
                               range(1, len(sa) + 1), range(1, len(sb) + 1))
        elif c["op"] == "transpose":
            out, shape = O.transpose(c["a"], c["shape"], strides_of(c), c["tau"], c["kind"])
        else:
            continue
        want = c["out"]
        assert list(shape) == c["out_shape"]
        assert np.asarray(out, dtype=want.dtype).tobytes() == want.tobytes(), c
        n += 1
    assert n >= 60
