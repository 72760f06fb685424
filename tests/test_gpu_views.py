"""Views as hot-path operands (views.py of the reference; SURVEY.md §8b
"operand polymorphism"): the reference's own tests draw every operand as a
dense tensor or a stepped view into a larger parent, 50/50
(conftest.py:38-55).  Each result is checked against the oracle evaluated on
the parent buffer through the view's (gamma, strides) address law."""

import random

import numpy as np
import pytest

import workloads as W
from oracle import oracle as O

pytestmark = pytest.mark.gpu


def tl():
    import paper_1711_10912_b200 as m

    return m


def bits(arr):
    a = np.ascontiguousarray(arr)
    return a.view({8: np.uint64, 4: np.uint32}[a.dtype.itemsize])


def rand_operand(rng, nrng, shape, kind, want_view=None):
    """(operand, flat buffer seen from the operand's base, its strides):
    a dense tensor with a random layout or a stepped view into a parent."""
    m = tl()
    view = rng.random() < 0.5 if want_view is None else want_view
    p = len(shape)

    def draw(shp):
        if kind == "int64":
            return nrng.integers(-9, 10, size=shp)
        return nrng.uniform(-1, 1, size=shp).astype(kind)

    if not view:
        lay = W.random_layout(p, rng.randint(0, 10**6))
        buf = W.layout_buffer(draw(shape), lay)
        t = m.DenseTensor.from_memory(shape, buf, layout=lay)
        return t, buf, t.strides
    steps = [rng.randint(1, 2) for _ in range(p)]
    leads = [rng.randint(0, 1) for _ in range(p)]
    pshape = tuple(lead + t * (n - 1) + 1 + rng.randint(0, 1) for n, t, lead in zip(shape, steps, leads))
    offs = tuple(rng.randint(-2, 2) for _ in range(p))
    lay = W.random_layout(p, rng.randint(0, 10**6))
    pbuf = W.layout_buffer(draw(pshape), lay)
    parent = m.DenseTensor.from_memory(pshape, pbuf, layout=lay, offsets=offs)
    ranges = [m.Range(o + lead, t, o + lead + t * (n - 1)) for o, lead, t, n in zip(offs, leads, steps, shape)]
    v = m.TensorView(parent, ranges)
    assert v.shape == tuple(shape)
    return v, pbuf[v.gamma:], v.strides


def test_view_structure_and_access(gpu):
    m = tl()
    a = m.DenseTensor.from_memory((4, 5, 3), np.arange(60, dtype=np.float64), layout=(2, 1, 3), offsets=(1, 0, -1))
    v = m.TensorView(a, [m.Range(1, 2, 3), m.Range(), m.Range(0)])
    assert v.shape == (2, 5, 1)
    assert v.strides == tuple(w * t for w, t in zip(a.strides, (2, 1, 1)))
    assert v.gamma == (1 - 1) * a.strides[0] + (0 - 0) * a.strides[1] + (0 + 1) * a.strides[2]
    for i in range(2):
        for j in range(5):
            assert v[1 + i, j, -1] == a[1 + 2 * i, j, 0]
    v[2, 4, -1] = -7.0
    assert a[3, 4, 0] == -7.0
    assert m.classify_view(m.TensorView(a, [m.Range(), m.Range(), m.Range(0)])) == "slice"
    assert m.classify_view(m.TensorView(a, [m.Range(2), m.Range(), m.Range(0)])) == "fiber"
    with pytest.raises(IndexError):
        m.TensorView(a, [m.Range(0, 9), m.Range(), m.Range()])
    with pytest.raises(ValueError):
        m.Range(3, 1)
    with pytest.raises(ValueError):
        m.TensorView(a, [m.Range()])
    mat = v.materialize()
    assert mat.shape == v.shape and mat.layout == (1, 2, 3)
    assert m.tensors_equal(mat, v)


def test_dense_views_are_not_copied(gpu):
    m = tl()
    from paper_1711_10912_b200.views import as_dense_operand

    a = m.DenseTensor.from_memory((6, 4, 5), np.arange(120, dtype=np.float64), layout=(3, 1, 2))
    full = m.TensorView(a, [m.Range(), m.Range(), m.Range()])
    slab = m.TensorView(a, [m.Range(), m.Range(1, 2), m.Range()])  # dim 2 is slowest in (3,1,2)
    for v in (full, slab):
        assert v.is_dense()
        d = as_dense_operand(v)
        assert d.buffer.data_ptr() == a.buffer.data_ptr() + 8 * v.gamma
        assert m.tensors_equal(d, v.materialize())
    strided = m.TensorView(a, [m.Range(0, 2, 4), m.Range(), m.Range()])
    assert not strided.is_dense()


@pytest.mark.parametrize("kind", ["float64", "float32", "int64"])
def test_ttv_on_views_bit_exact(gpu, kind):
    m = tl()
    rng, nrng = random.Random(3), np.random.default_rng(3)
    for _ in range(40):
        p = rng.randint(2, 4)
        shape = tuple(rng.randint(1, 5) for _ in range(p))
        mode = rng.randint(1, p)
        a, abuf, astr = rand_operand(rng, nrng, shape, kind)
        b, bbuf, bstr = rand_operand(rng, nrng, (shape[mode - 1],), kind)
        got = m.ttv(a, b, mode).numpy()
        bvec = np.asarray([bbuf[k * bstr[0]] for k in range(shape[mode - 1])])
        want = O.ttv(abuf, shape, astr, bvec, mode)
        if kind == "float32":
            want = want.astype(np.float32)
        assert np.array_equal(bits(got), bits(want))


def test_ttm_inner_norm_on_views(gpu):
    m = tl()
    rng, nrng = random.Random(4), np.random.default_rng(4)
    for _ in range(30):
        p = rng.randint(2, 4)
        shape = tuple(rng.randint(1, 5) for _ in range(p))
        mode = rng.randint(1, p)
        J = rng.randint(1, 4)
        a, abuf, astr = rand_operand(rng, nrng, shape, "int64")
        bm, bbuf, bstr = rand_operand(rng, nrng, (J, shape[mode - 1]), "int64")
        got = m.ttm(a, bm, mode).numpy()
        assert np.array_equal(got, O.ttm(abuf, shape, astr, bbuf, (J, shape[mode - 1]), bstr, mode))
        c, cbuf, cstr = rand_operand(rng, nrng, shape, "int64")
        assert m.inner_product_tensors(a, c) == O.inner(abuf, shape, astr, cbuf, cstr)
        f, fbuf, fstr = rand_operand(rng, nrng, shape, "float64")
        assert abs(m.frobenius_norm(f) - O.norm(fbuf, shape, fstr)) <= 1e-13 * max(1.0, O.norm(fbuf, shape, fstr))


def test_ttt_times_vectors_hopm_on_views(gpu):
    m = tl()
    rng, nrng = random.Random(5), np.random.default_rng(5)
    a, abuf, astr = rand_operand(rng, nrng, (3, 4, 2), "int64", want_view=True)
    b, bbuf, bstr = rand_operand(rng, nrng, (4, 3, 5), "int64", want_view=True)
    spec = m.ContractionSpec(2, (3, 1, 2), (3, 2, 1))
    out, shape = O.ttt(abuf, (3, 4, 2), astr, bbuf, (4, 3, 5), bstr, 2, (3, 1, 2), (3, 2, 1), "int64")
    got = m.ttt(a, b, spec)
    assert got.shape == shape and got.data == out
    vs = [m.DenseTensor.from_memory((n,), nrng.uniform(-1, 1, n)) for n in (3, 4, 2)]
    f, fbuf, fstr = rand_operand(rng, nrng, (3, 4, 2), "float64", want_view=True)
    tv = m.times_vectors(f, vs, skip=2)
    ref = m.times_vectors(f.materialize(), vs, skip=2)
    assert np.array_equal(bits(tv.numpy()), bits(ref.numpy()))
    st_v = m.hopm(f, max_sweeps=5, tol=0.0)
    st_d = m.hopm(f.materialize(), max_sweeps=5, tol=0.0)
    assert st_v.lambda_history == st_d.lambda_history
