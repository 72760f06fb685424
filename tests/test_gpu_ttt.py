"""GPU parity for the general tensor-times-tensor product and its named
special cases (contraction.py:75-107, 304-454).

ttt runs as device relayouts plus one ttm tile kernel.  int64 and float32
results are exact (float32: binary64 fold rounded once); float64 results
of the DMMA path hold the ttm tolerance 1e-12 * sum_k |a||b|.  The
vector-operand and full-contraction specs route to ttv / inner, so the
reference's identities ttv == ttt(reduce_ttv_to_ttt) and
ttt(full) == inner_product_tensors hold exactly."""

import random

import numpy as np
import pytest

import workloads as W
from oracle import oracle as O

pytestmark = pytest.mark.gpu

RTOL64 = 1e-12


def tl():
    import paper_1711_10912_b200 as m

    return m


def dev(buf, shape, layout=None):
    shape = tuple(shape)
    return tl().DenseTensor.from_memory(shape, np.asarray(buf), layout=tuple(layout or range(1, len(shape) + 1)))


def bits(arr):
    a = np.ascontiguousarray(arr)
    return a.view({8: np.uint64, 4: np.uint32}[a.dtype.itemsize])


def check(got, want, kind, bound=None):
    got = np.asarray(got)
    want = np.asarray(want)
    if kind == "int64":
        assert np.array_equal(got, want.astype(np.int64))
    elif kind == "float32":
        assert got.dtype == np.float32
        assert np.array_equal(bits(got), bits(want.astype(np.float32)))
    else:
        assert np.all(np.abs(got - want) <= RTOL64 * bound + 1e-300), np.max(np.abs(got - want))


def test_ttt_golden(gpu, small_golden):
    n = 0
    for c in small_golden["cases"]:
        if c["op"] != "ttt":
            continue
        A = dev(c["a"], c["shape"], c["layout"])
        B = dev(c["b"], c["bshape"], c["blayout"])
        C = tl().ttt(A, B, tl().ContractionSpec(c["q"], c["phi"], c["psi"]))
        assert list(C.shape) == c["out_shape"] and C.dtype == A.dtype
        bound = None
        if c["kind"] == "float64":
            bound, _ = O.ttt(np.abs(c["a"]), c["shape"], W.compute_strides(c["shape"], c["layout"]),
                             np.abs(c["b"]), c["bshape"], W.compute_strides(c["bshape"], c["blayout"]),
                             c["q"], c["phi"], c["psi"])
        check(C.numpy(), c["out"], c["kind"], np.asarray(bound))
        n += 1
    assert n >= 40


def test_transpose_and_outer_golden_exact(gpu, small_golden):
    n = 0
    for c in small_golden["cases"]:
        if c["op"] == "transpose":
            C = tl().transpose(dev(c["a"], c["shape"], c["layout"]), c["tau"])
        elif c["op"] == "outer":
            C = tl().outer_product(dev(c["a"], c["shape"]), dev(c["b"], c["bshape"]))
        else:
            continue
        assert list(C.shape) == c["out_shape"] and C.layout == tuple(range(1, len(C.shape) + 1))
        assert np.asarray(C.numpy()).tobytes() == c["out"].astype(C.numpy().dtype).tobytes(), c
        n += 1
    assert n >= 16


def test_ttt_known_answers(gpu):
    """test_contraction.py:167-190 restated."""
    m = tl()
    u = m.DenseTensor.from_memory((2,), [2, 3])
    v = m.DenseTensor.from_memory((3,), [1, 10, 100])
    c = m.ttt(u, v, m.ContractionSpec(0, (1,), (1,)))
    assert c.shape == (2, 3) and c.data == [2, 3, 20, 30, 200, 300]
    ones = m.DenseTensor((2, 2, 2), fill_value=1)
    c = m.ttt(ones, ones, m.ContractionSpec(3, (1, 2, 3), (1, 2, 3)))
    assert c.shape == (1,) and c.item() == 8
    c = m.ttt(m.DenseTensor((3, 4, 2), fill_value=1), m.DenseTensor((4, 3, 5), fill_value=1),
              m.ContractionSpec(2, (3, 1, 2), (3, 2, 1)))
    assert c.shape == (2, 5) and c.data == [12] * 10


def test_spec_validation(gpu):
    m = tl()
    for args in [(1, (1, 1), (1,)), (2, (1,), (1, 2)), (-1, (1,), (1,))]:
        with pytest.raises(ValueError):
            m.ContractionSpec(*args)
    a, b = m.DenseTensor((2, 3)), m.DenseTensor((4,))
    with pytest.raises(ValueError):
        m.ttt(a, b, m.ContractionSpec(1, (1, 2), (1,)))
    with pytest.raises(ValueError):
        m.ttt(a, b, m.ContractionSpec(1, (1,), (1,)))
    with pytest.raises(ValueError):
        m.transpose(m.DenseTensor((2, 2)), (1, 1))
    assert m.reduce_ttv_to_ttt(3, 2) == m.ContractionSpec(1, (1, 3, 2), (1,))
    assert m.reduce_ttm_to_ttt(3, 1) == m.ContractionSpec(1, (2, 3, 1), (1, 2))
    with pytest.raises(ValueError):
        m.reduce_ttv_to_ttt(2, 3)


@pytest.mark.parametrize("dtype", [np.float64, np.float32, np.int64])
def test_reduction_identities_exact(gpu, dtype):
    """ttv == ttt(reduce_ttv_to_ttt) and ttt(full) == inner, bit for bit
    (test_contraction.py:263-273, test_acceptance.py:138-177)."""
    m = tl()
    rng = random.Random(10)
    nrng = np.random.default_rng(10)

    def draw(shape):
        if dtype == np.int64:
            return nrng.integers(-9, 10, size=shape)
        return nrng.uniform(-1, 1, size=shape).astype(dtype)

    for _ in range(40):
        p = rng.randint(2, 4)
        shape = tuple(rng.randint(1, 6) for _ in range(p))
        mode = rng.randint(1, p)
        lay = W.random_layout(p, rng.randint(0, 10**6))
        T = draw(shape)
        a = dev(W.layout_buffer(T, lay), shape, lay)
        b = dev(draw((shape[mode - 1],)), (shape[mode - 1],))
        assert m.tensors_equal(m.ttv(a, b, mode), m.ttt(a, b, m.reduce_ttv_to_ttt(p, mode)))
        # vector on the left: sum_k b(k) A(..k..) folds the same products
        spec = m.ContractionSpec(1, (1,), tuple(d for d in range(1, p + 1) if d != mode) + (mode,))
        assert m.tensors_equal(m.ttv(a, b, mode), m.ttt(b, a, spec))
        c = dev(draw(shape), shape)
        full = m.ContractionSpec(p, tuple(range(1, p + 1)), tuple(range(1, p + 1)))
        want = m.inner_product_tensors(a, c)
        if dtype == np.float32:
            want = float(np.float32(want))  # float32 storage: the binary64 result rounded once
        assert m.ttt(a, c, full).item() == want


def test_ttm_reduction_spec(gpu):
    """ttt(reduce_ttm_to_ttt(p, m)) is ttm with the new dimension cycled to
    the back (contraction.py:429-440); exact on int64."""
    m = tl()
    rng = random.Random(12)
    nrng = np.random.default_rng(12)
    for _ in range(20):
        p = rng.randint(2, 4)
        shape = tuple(rng.randint(1, 5) for _ in range(p))
        mode = rng.randint(1, p)
        J = rng.randint(1, 5)
        T = nrng.integers(-9, 10, size=shape)
        M = nrng.integers(-9, 10, size=(J, shape[mode - 1]))
        a = dev(W.layout_buffer(T, range(1, p + 1)), shape)
        bm = dev(W.layout_buffer(M, (1, 2)), (J, shape[mode - 1]))
        via = m.ttt(a, bm, m.reduce_ttm_to_ttt(p, mode)).numpy()
        direct = m.ttm(a, bm, mode).numpy()
        dshape = shape[: mode - 1] + (J,) + shape[mode:]
        cyc = np.moveaxis(direct.reshape(dshape, order="F"), mode - 1, -1)
        assert np.array_equal(via, cyc.reshape(-1, order="F"))


@pytest.mark.parametrize("case", [
    # (A shape, A layout, B shape, B layout, q, phi, psi) -- GETT-sized
    ((64, 48, 40), (1, 2, 3), (40, 48, 96), (1, 2, 3), 2, (1, 3, 2), (3, 1, 2)),
    ((33, 70, 9), (3, 1, 2), (9, 130), (2, 1), 1, (1, 2, 3), (2, 1)),
    ((128, 256), (2, 1), (256, 64, 3), (1, 3, 2), 1, (1, 2), (2, 3, 1)),
    ((20, 30), (1, 2), (40, 50), (1, 2), 0, (2, 1), (1, 2)),
])
def test_ttt_large_vs_numpy(gpu, case):
    sa, la, sb, lb, q, phi, psi = case
    nrng = np.random.default_rng(3)
    Ta = nrng.uniform(-1, 1, size=sa)
    Tb = nrng.uniform(-1, 1, size=sb)
    m = tl()
    C = m.ttt(dev(W.layout_buffer(Ta, la), sa, la), dev(W.layout_buffer(Tb, lb), sb, lb), m.ContractionSpec(q, phi, psi))
    r, s = len(sa) - q, len(sb) - q
    ax_a = [phi[r + k] - 1 for k in range(q)]
    ax_b = [psi[s + k] - 1 for k in range(q)]
    want = np.tensordot(Ta, Tb, axes=(ax_a, ax_b))  # free axes in natural order
    free_a = sorted(d - 1 for d in phi[:r])
    free_b = sorted(d - 1 for d in psi[:s])
    order = [free_a.index(phi[k] - 1) for k in range(r)] + [r + free_b.index(psi[k] - 1) for k in range(s)]
    want = np.transpose(want, order)
    bound = np.tensordot(np.abs(Ta), np.abs(Tb), axes=(ax_a, ax_b)).transpose(order)
    got = C.numpy().reshape(C.shape, order="F")
    assert got.shape == want.shape
    assert np.all(np.abs(got - want) <= RTOL64 * bound + 1e-300)


@pytest.mark.parametrize("dtype", ["float32", "float64", "int64"])
def test_transpose_shared_fastest_dim_rows(gpu, dtype):
    """Relayouts whose source and destination share the fastest dimension
    copy whole 16-byte vectors per row (copy_rows_kernel): exact, including
    rows that are not a multiple of the vector width (element path)."""
    m = tl()
    rng = np.random.default_rng(5)
    for shape, tau in (((16, 5, 7, 3), (1, 3, 2, 4)), ((8, 33, 9), (1, 3, 2)), ((6, 4, 5), (1, 3, 2)),
                       ((128, 3, 2, 5), (1, 4, 3, 2))):
        T = rng.integers(-9, 9, size=shape) if dtype == "int64" else rng.standard_normal(shape).astype(dtype)
        A = m.DenseTensor.from_memory(shape, T.ravel(order="F"))
        got = m.transpose(A, tau).numpy()
        want = np.transpose(T, [t - 1 for t in tau]).ravel(order="F")
        assert got.tobytes() == want.astype(got.dtype).tobytes(), (shape, tau)
        B = A.copy()
        B.relayout(tau)
        assert m.tensors_equal(A, B)
