"""GPU parity: the B200 path through the public API / C ABI against the
reference's golden outputs and the pinned CPU oracle.

ttv, times_vectors, hopm and the exact ttm fold are BIT-IDENTICAL to the
reference; DMMA ttm, inner and norm are checked against the stated
tolerances (float64 1e-12, float32 1e-5) relative to the a-priori bound
sum_k |a_k||b_k|."""

import hashlib

import numpy as np
import pytest
import torch

import workloads as W
from oracle import oracle as O
from tolerance import check_inner, check_ttm

pytestmark = pytest.mark.gpu

RTOL64 = 1e-12
RTOL32 = 1e-5


def tl():
    import paper_1711_10912_b200 as m

    return m


def dev_tensor(buf, shape, layout, dtype=None):
    return tl().DenseTensor.from_memory(tuple(shape), np.asarray(buf), layout=tuple(layout), dtype=dtype)


def bits(arr):
    a = np.ascontiguousarray(arr)
    return a.view(np.uint64 if a.dtype.itemsize == 8 else np.uint32)


def test_ttv_golden_bit_exact(gpu, small_golden):
    n = 0
    for c in small_golden["cases"]:
        if c["op"] != "ttv":
            continue
        A = dev_tensor(c["a"], c["shape"], c["layout"])
        n_m = c["shape"][c["mode"] - 1]
        if c["column"]:
            B = tl().DenseTensor.from_memory((n_m, 1), np.asarray(c["b"]))
        else:
            B = tl().DenseTensor.from_memory((n_m,), np.asarray(c["b"]))
        C = tl().ttv(A, B, c["mode"])
        assert list(C.shape) == c["out_shape"] and C.layout == tuple(range(1, len(C.shape) + 1))
        got = C.numpy()
        want = c["out"]
        if c["kind"] == "float32":
            assert got.dtype == np.float32
            want = want.astype(np.float32)  # reference binary64 fold, rounded once
        assert np.array_equal(bits(got), bits(want)), c
        n += 1
    assert n >= 100


def test_ttm_golden(gpu, small_golden):
    for c in small_golden["cases"]:
        if c["op"] != "ttm":
            continue
        A = dev_tensor(c["a"], c["shape"], c["layout"])
        Bm = dev_tensor(c["bmat"], c["bshape"], c["blayout"])
        C = tl().ttm(A, Bm, c["mode"])
        assert list(C.shape) == c["out_shape"]
        got, want = C.numpy(), c["out"]
        if c["kind"] == "int64":
            assert np.array_equal(got, want), c
        else:
            # a-priori bound: sum_k |A||B| per output, via the oracle on |A|, |B|
            bstr = W.compute_strides(c["bshape"], c["blayout"])
            bound = O.ttm(np.abs(c["a"]), c["shape"], W.compute_strides(c["shape"], c["layout"]),
                          np.abs(c["bmat"]), c["bshape"], bstr, c["mode"])
            check_ttm(got, want, bound)


def test_inner_norm_golden(gpu, small_golden):
    for c in small_golden["cases"]:
        if c["op"] == "inner":
            A = dev_tensor(c["a"], c["shape"], c["layout"])
            B = dev_tensor(c["b"], c["shape"], c["blayout"])
            got = tl().inner_product_tensors(A, B)
            if c["kind"] == "int64":
                assert got == c["value"] and isinstance(got, int)
            else:
                shp = tuple(c["shape"])
                check_inner(got, c["value"], W.from_buffer(c["a"], shp, c["layout"]).ravel(order="F"),
                            W.from_buffer(c["b"], shp, c["blayout"]).ravel(order="F"))
        elif c["op"] == "norm":
            A = dev_tensor(c["a"], c["shape"], c["layout"])
            got = tl().frobenius_norm(A)
            assert abs(got - c["value"]) <= RTOL64 * c["value"], c


def test_times_vectors_golden_bit_exact(gpu, small_golden):
    for c in small_golden["cases"]:
        if c["op"] != "times_vectors":
            continue
        A = dev_tensor(c["a"], c["shape"], c["layout"])
        vs, off = [], 0
        for n in c["shape"]:
            vs.append(tl().DenseTensor.from_memory((n,), c["vectors"][off:off + n]))
            off += n
        if c["skip"] is not None:
            C = tl().times_vectors(A, vs, skip=c["skip"])
        else:
            C = tl().times_vectors(A, [vs[m - 1] for m in c["modes"]], c["modes"])
        assert list(C.shape) == c["out_shape"]
        assert np.array_equal(bits(C.numpy()), bits(c["out"])), c


def test_hopm_golden_bit_exact(gpu, small_golden):
    n = 0
    for c in small_golden["cases"]:
        if c["op"] != "hopm":
            continue
        A = dev_tensor(c["a"], c["shape"], c["layout"])
        u0 = None
        if "u0" in c:
            u0, off = [], 0
            for k in c["shape"]:
                u0.append(tl().DenseTensor.from_memory((k,), c["u0"][off:off + k]))
                off += k
        st = tl().hopm(A, max_sweeps=c["max_sweeps"], tol=c["tol"], u0=u0)
        assert st.sweeps == c["sweeps"] and st.converged == c["converged"]
        assert np.array_equal(bits(np.concatenate([u.numpy() for u in st.u])), bits(c["u"])), c
        assert np.array_equal(bits(np.asarray(st.l)), bits(c["l"]))
        assert np.array_equal(bits(np.asarray(st.lambda_history)), bits(c["lambda_history"]))
        n += 1
    assert n >= 8


def test_hopm_residuals_and_rank_one_golden(gpu, small_golden):
    """track_residuals / residual / rank_one_compose (hopm.py:114-147): lambda
    and vectors bit-exact, the composed tensor bit-exact (same product order),
    residuals (a parallel sum) within 1e-12 relative."""
    m = tl()
    n = 0
    for c in small_golden["cases"]:
        if c["op"] != "hopm_resid":
            continue
        A = dev_tensor(c["a"], c["shape"], c["layout"])
        st = m.hopm(A, max_sweeps=c["max_sweeps"], tol=c["tol"], track_residuals=True)
        assert np.array_equal(bits(np.asarray(st.lambda_history)), bits(c["lambda_history"]))
        assert np.array_equal(bits(np.concatenate([u.numpy() for u in st.u])), bits(c["u"]))
        assert len(st.residual_history) == len(c["residual_history"])
        for got, want in zip(st.residual_history, c["residual_history"]):
            assert abs(got - want) <= 1e-12 * max(1.0, abs(want))
        B = m.rank_one_compose(st.scale, st.u)
        assert B.shape == tuple(c["shape"]) and np.array_equal(bits(B.numpy()), bits(c["compose"]))
        assert abs(m.residual(A, st) - c["residual"]) <= 1e-12 * max(1.0, c["residual"])
        n += 1
    assert n == 3


def test_cli_hopm(gpu, tmp_path, capsys):
    """`python -m paper_1711_10912_b200 hopm` mirrors cli.py:139-164."""
    import json

    from paper_1711_10912_b200 import cli

    rng = np.random.default_rng(8)
    us = [rng.standard_normal(n) for n in (3, 4, 2)]
    us = [u / np.linalg.norm(u) for u in us]
    T = 2.0 * np.einsum("i,j,k->ijk", *us)
    path = tmp_path / "t.json"
    path.write_text(json.dumps({"shape": [3, 4, 2], "layout": [1, 2, 3], "offsets": [0, 0, 0],
                                "data": T.ravel("F").tolist()}))
    assert cli.main(["hopm", "--in", str(path), "--json"]) == 0
    out = json.loads(capsys.readouterr().out)
    assert out["converged"] and abs(out["scale"] - 2.0) < 1e-10 and out["residual"] < 1e-10
    path.write_text(json.dumps({"shape": [2, 3], "data": [0.0] * 6}))
    assert cli.main(["hopm", "--in", str(path)]) == 3
    path.write_text(json.dumps({"shape": [3, 3, 3], "data": rng.uniform(-1, 1, 27).tolist()}))
    assert cli.main(["hopm", "--in", str(path), "--sweeps", "1"]) == 2
    assert "sweep 1: lambda" in capsys.readouterr().out
    path.write_text("{not json")
    with pytest.raises(SystemExit) as e:
        cli.main(["hopm", "--in", str(path)])
    assert e.value.code == 1


def test_kats(gpu, small_golden):
    m = tl()
    kat = small_golden["kat"]
    eye = m.DenseTensor((2, 2))
    eye[0, 0] = 1
    eye[1, 1] = 1
    assert m.ttv(eye, m.DenseTensor((2,), fill_value=1), 2).data == kat["ttv_identity_row_sums"]
    c = m.ttv(m.DenseTensor((2, 3, 2), fill_value=1), m.DenseTensor((3,), fill_value=1), 2)
    assert c.shape == (2, 2) and c.data == kat["ttv_counting"]
    assert m.frobenius_norm(m.DenseTensor((2, 2, 2), fill_value=1)) == kat["norm_all_ones_222"]
    full = m.times_vectors(m.DenseTensor((2, 3, 2), fill_value=1), [m.DenseTensor((n,), fill_value=1) for n in (2, 3, 2)],
                           [1, 2, 3])
    assert full.shape == (1,) and full.item() == 12
    st = m.hopm(m.DenseTensor.from_memory((3,), [3.0, 0.0, 4.0]))
    assert st.l[0] == 5.0 and st.u[0].data == [0.6, 0.0, 0.8]
    with pytest.raises(m.DegenerateInputError) as e:
        m.hopm(m.DenseTensor((2, 3)))
    assert [e.value.sweep, e.value.mode] == kat["hopm_zero_degenerate"]


# ----------------------------------------------------------------- regimes sweep
@pytest.mark.parametrize("dtype", ["float64", "float32", "int64"])
def test_ttv_random_layouts_vs_oracle(gpu, dtype):
    """Random orders 2..6, odd extents, every mode, random layouts: exact."""
    rng = np.random.default_rng(7)
    import random

    prng = random.Random(7)
    for t in range(60):
        p = prng.randint(2, 6)
        shape = tuple(prng.choice([1, 2, 3, 5, 7, 9, 16, 33, 40, 64]) for _ in range(p))
        while np.prod(shape) > 2_000_000:
            shape = tuple(max(1, s // 2) for s in shape)
        layout = W.random_layout(p, prng.randint(0, 1 << 30))
        mode = prng.randint(1, p)
        if dtype == "int64":
            T = rng.integers(-50, 50, size=shape)
            b = rng.integers(-50, 50, size=shape[mode - 1])
        else:
            T = rng.uniform(-1, 1, size=shape).astype(dtype)
            b = rng.uniform(-1, 1, size=shape[mode - 1]).astype(dtype)
        buf = W.layout_buffer(T, layout)
        A = dev_tensor(buf, shape, layout)
        C = tl().ttv(A, tl().DenseTensor.from_memory((shape[mode - 1],), b), mode)
        want = O.ttv(buf, shape, W.compute_strides(shape, layout), b, mode)
        if dtype == "float32":
            want = want.astype(np.float32)
        assert np.array_equal(bits(C.numpy()), bits(want)), (shape, layout, mode)


def test_cfg1_bit_exact(gpu, configs_golden):
    T, b = W.cfg1()
    A = dev_tensor(W.layout_buffer(T, (1, 2, 3)), T.shape, (1, 2, 3))
    C = tl().ttv(A, tl().DenseTensor.from_memory((96,), b), 2)
    assert C.shape == (128, 64)
    assert hashlib.sha256(C.numpy().tobytes()).hexdigest() == configs_golden["cfg1"]["sha256"]


def test_cfg5_chain(gpu, configs_golden):
    for seed in (0, 5):
        key = f"cfg5_seed{seed}"
        if key not in configs_golden:
            continue
        g = configs_golden[key]
        T, v, M, layout = W.cfg5(seed)
        A = dev_tensor(W.layout_buffer(T, layout), T.shape, layout)
        del T
        C1 = tl().ttv(A, tl().DenseTensor.from_memory((9,), v), 5)
        c1 = C1.numpy()
        assert hashlib.sha256(c1.tobytes()).hexdigest() == g["ttv_sha256"]
        Bm = tl().DenseTensor.from_memory(M.shape, W.layout_buffer(M, (1, 2)))
        C2 = tl().ttm(C1, Bm, 2)
        got = C2.numpy()
        shp1 = g["ttv_shape"]
        bound = O.ttm(np.abs(c1), shp1, W.compute_strides(shp1, W.first_order(6)), np.abs(W.layout_buffer(M, (1, 2))),
                      M.shape, (1, 16), 2)
        want = O.ttm(c1, shp1, W.compute_strides(shp1, W.first_order(6)), W.layout_buffer(M, (1, 2)), M.shape, (1, 16), 2)
        assert hashlib.sha256(want.tobytes()).hexdigest() == g["ttm_sha256"]
        assert np.all(np.abs(got - want) <= RTOL64 * bound)
        nrm = tl().frobenius_norm(C2)
        assert abs(nrm - g["norm"]) <= RTOL64 * g["norm"]


def test_cfg2_ttv_bit_exact(gpu, configs_golden):
    if "cfg2" not in configs_golden:
        pytest.skip("cfg2 golden missing")
    g = configs_golden["cfg2"]
    T, vecs, T2 = W.cfg2()
    for name, layout in W.CFG2_LAYOUTS.items():
        A = dev_tensor(W.layout_buffer(T, layout), T.shape, layout)
        for mode in (1, 2, 3, 4):
            key = f"ttv_{name}_q{mode}"
            C = tl().ttv(A, tl().DenseTensor.from_memory((128,), vecs[mode - 1]), mode)
            got = hashlib.sha256(C.numpy().tobytes()).hexdigest()
            if key in g:
                assert got == g[key]["f32_sha256"], key
            else:
                want = O.ttv(W.layout_buffer(T, layout), T.shape, W.compute_strides(T.shape, layout), vecs[mode - 1], mode)
                assert got == hashlib.sha256(want.astype(np.float32).tobytes()).hexdigest(), key
        del A
        torch.cuda.empty_cache()
    # norm and inner products (float32 storage, binary64 accumulation): 1e-5
    A = dev_tensor(W.layout_buffer(T, (1, 2, 3, 4)), T.shape, (1, 2, 3, 4))
    nrm = tl().frobenius_norm(A)
    ref_n = g["norm_first"]["value"] if "norm_first" in g else O.norm(T.ravel("F"), T.shape, (1, 128, 128**2, 128**3))
    # the reference's own sequential fold of 2^28 squares carries ~1e-12
    # relative rounding error; the stated float32 bar is 1e-5
    assert abs(nrm - ref_n) <= RTOL32 * ref_n
    assert abs(nrm - ref_n) <= 1e-10 * ref_n
    B = dev_tensor(W.layout_buffer(T2, (1, 2, 3, 4)), T.shape, (1, 2, 3, 4))
    absbound = float(np.dot(np.abs(T.ravel("F")).astype(np.float64), np.abs(T2.ravel("F")).astype(np.float64)))
    ip = tl().inner_product_tensors(A, B)
    if "inner_first_first" in g:
        assert abs(ip - g["inner_first_first"]["value"]) <= RTOL32 * absbound
    Bl = dev_tensor(W.layout_buffer(T2, (4, 3, 2, 1)), T.shape, (4, 3, 2, 1))
    ip2 = tl().inner_product_tensors(A, Bl)
    assert abs(ip2 - ip) <= 1e-13 * absbound  # layout invariance
    if "inner_first_last" in g:
        assert abs(ip2 - g["inner_first_last"]["value"]) <= RTOL32 * absbound


def test_cfg4_hopm_bit_exact(gpu, configs_golden):
    if "cfg4" not in configs_golden:
        pytest.skip("cfg4 golden missing")
    g = configs_golden["cfg4"]
    T, _ = W.cfg4()
    A = dev_tensor(W.layout_buffer(T, (1, 2, 3)), T.shape, (1, 2, 3))
    st = tl().hopm(A, max_sweeps=50, tol=0.0)
    assert st.sweeps == 50 and not st.converged
    assert st.lambda_history == g["lambda_history"]
    assert st.l == g["l"]
    for u, want in zip(st.u, g["u"]):
        assert u.data == want
