"""Conformance: the reference's contraction suite, restated on the B200 path.

Every case below is drawn with the same seeds and the same draw order as
/root/reference/pkg/tests/test_contraction.py (cited per test), so the GPU
path sees the very operands -- views, offsets, random layouts, integer data
-- that the reference's own tests check.  Expected values come from an
independent element-by-element evaluation of the defining sums; integer
data makes every comparison exact.  The unmodified reference file itself
is run against this package by tools/ref_suite/ (see INTEGRATION.md).
"""

import math
import random

import pytest

from .refcases import all_idx, box, dense_draw, eye, operand_draw, tl

pytestmark = pytest.mark.gpu


def _ttv_expect(abox, shape, bvals, m):
    out_shape = shape[: m - 1] + shape[m:]
    return {i: sum(abox[i[: m - 1] + (k,) + i[m - 1:]] * bvals[k] for k in range(shape[m - 1]))
            for i in all_idx(out_shape)}


def _ttt_expect(abox, bbox, na, nb, q, phi, psi):
    r, s = len(phi) - q, len(psi) - q
    out_shape = tuple(na[phi[k] - 1] for k in range(r)) + tuple(nb[psi[k] - 1] for k in range(s))
    sums = [na[phi[r + k] - 1] for k in range(q)]
    want = {}
    for ic in all_idx(out_shape or (1,)):
        acc = 0
        for jt in all_idx(sums):
            ia, ib = [0] * len(na), [0] * len(nb)
            for k in range(r):
                ia[phi[k] - 1] = ic[k]
            for k in range(s):
                ib[psi[k] - 1] = ic[r + k]
            for k in range(q):
                ia[phi[r + k] - 1] = ib[psi[s + k] - 1] = jt[k]
            acc += abox[tuple(ia)] * bbox[tuple(ib)]
        want[ic if out_shape else (0,)] = acc
    return want


def _ttt_draw(rng):
    """One random (A, B, spec) triple in the reference's draw order
    (test_contraction.py:173-193, test_numpy_crosscheck.py:82-100)."""
    pa = rng.randint(1, 4)
    q = rng.randint(0, pa)
    r = pa - q
    s_min = 0 if q else 1
    s = rng.randint(s_min, max(s_min, 4 - q))
    pb = q + s
    na = tuple(rng.randint(1, 4) for _ in range(pa))
    phi = list(range(1, pa + 1))
    rng.shuffle(phi)
    psi = list(range(1, pb + 1))
    rng.shuffle(psi)
    nb = [0] * pb
    for k in range(s):
        nb[psi[k] - 1] = rng.randint(1, 4)
    for k in range(q):
        nb[psi[s + k] - 1] = na[phi[r + k] - 1]
    a = operand_draw(rng, na)
    b = operand_draw(rng, tuple(nb))
    return a, b, na, tuple(nb), q, tuple(phi), tuple(psi)


# -- transpose (test_contraction.py:42-78) ---------------------------------------------


def test_transpose_matrix(gpu):
    m = tl()
    a = dense_draw(random.Random(0), (2, 3))
    c = m.transpose(a, (2, 1))
    ab = box(a)
    assert c.shape == (3, 2)
    assert all(box(c)[(j, i)] == ab[(i, j)] for i in range(2) for j in range(3))


def test_transpose_identity_and_random(gpu):
    m = tl()
    a = dense_draw(random.Random(1), (2, 3, 2))
    assert m.tensors_equal(m.transpose(a, (1, 2, 3)), a)
    rng = random.Random(2)
    for _ in range(15):
        shape = tuple(rng.randint(1, 3) for _ in range(4))
        a = operand_draw(rng, shape)
        tau = list(range(1, 5))
        rng.shuffle(tau)
        got, ab = box(m.transpose(a, tau)), box(a)
        for ic, v in got.items():
            ia = [0] * 4
            for r, t in enumerate(tau):
                ia[t - 1] = ic[r]
            assert v == ab[tuple(ia)]
    with pytest.raises(ValueError):
        m.transpose(m.DenseTensor((2, 2)), (1, 1))


# -- ttv (test_contraction.py:81-117) ----------------------------------------------------


def test_ttv_known_answers(gpu):
    m = tl()
    c = m.ttv(eye(2), m.DenseTensor((2,), fill_value=1), 2)
    assert c.shape == (2,) and c.data == [1, 1]
    c = m.ttv(m.DenseTensor((2, 3, 2), fill_value=1), m.DenseTensor((3,), fill_value=1), 2)
    assert c.shape == (2, 2) and c.data == [3] * 4


def test_ttv_random_operands_all_modes(gpu):
    m = tl()
    rng = random.Random(3)
    for _ in range(40):
        p = rng.randint(2, 4)
        shape = tuple(rng.randint(1, 4) for _ in range(p))
        md = rng.randint(1, p)
        a = operand_draw(rng, shape)
        b = operand_draw(rng, (shape[md - 1],))
        bvals = [box(b)[(k,)] for k in range(shape[md - 1])]
        assert box(m.ttv(a, b, md)) == _ttv_expect(box(a), shape, bvals, md)


def test_ttv_column_vector_and_errors(gpu):
    m = tl()
    a = dense_draw(random.Random(4), (3, 4))
    col, flat = m.DenseTensor((4, 1)), m.DenseTensor((4,))
    for k in range(4):
        col[k, 0] = k + 1
        flat[k] = k + 1
    assert m.tensors_equal(m.ttv(a, col, 2), m.ttv(a, flat, 2))
    z = m.DenseTensor((3, 4))
    for bad in ((z, m.DenseTensor((4,)), 3), (z, m.DenseTensor((5,)), 2),
                (m.DenseTensor((4,)), m.DenseTensor((4,)), 1)):
        with pytest.raises(ValueError):
            m.ttv(*bad)


# -- ttm (test_contraction.py:120-163) ---------------------------------------------------


def test_ttm_identity_and_single_row(gpu):
    m = tl()
    rng = random.Random(5)
    for md in (1, 2, 3):
        a = dense_draw(rng, (3, 4, 2))
        assert m.tensors_equal(m.ttm(a, eye(a.shape[md - 1]), md), a)
    rng = random.Random(6)
    a = dense_draw(rng, (3, 4, 2))
    row = dense_draw(rng, (1, 4))
    c = m.ttm(a, row, 2)
    assert c.shape == (3, 1, 2)
    vec = m.DenseTensor((4,))
    for k in range(4):
        vec[k] = row[row.offsets[0], k + row.offsets[1]]
    c.reshape((3, 2))
    assert m.tensors_equal(c, m.ttv(a, vec, 2))


def test_ttm_random_operands(gpu):
    m = tl()
    rng = random.Random(7)
    for _ in range(30):
        p = rng.randint(2, 4)
        shape = tuple(rng.randint(1, 4) for _ in range(p))
        md = rng.randint(1, p)
        n_new = rng.randint(1, 4)
        a = operand_draw(rng, shape)
        bm = operand_draw(rng, (n_new, shape[md - 1]))
        ab, bb = box(a), box(bm)
        for ic, v in box(m.ttm(a, bm, md)).items():
            assert v == sum(ab[ic[: md - 1] + (k,) + ic[md:]] * bb[(ic[md - 1], k)] for k in range(shape[md - 1]))


def test_ttm_dimension_mismatch(gpu):
    m = tl()
    with pytest.raises(ValueError):
        m.ttm(m.DenseTensor((3, 4)), m.DenseTensor((2, 5)), 2)
    with pytest.raises(ValueError):
        m.ttm(m.DenseTensor((3, 4)), m.DenseTensor((2, 4, 1)), 2)


# -- ttt (test_contraction.py:166-244) ---------------------------------------------------


def test_ttt_known_answers(gpu):
    m = tl()
    u = m.DenseTensor.from_memory((2,), [2, 3])
    v = m.DenseTensor.from_memory((3,), [1, 10, 100])
    c = m.ttt(u, v, m.ContractionSpec(0, (1,), (1,)))
    assert c.shape == (2, 3) and box(c) == {(i, j): u[i] * v[j] for i in range(2) for j in range(3)}
    ones = lambda s: m.DenseTensor(s, fill_value=1)  # noqa: E731
    c = m.ttt(ones((2, 2, 2)), ones((2, 2, 2)), m.ContractionSpec(3, (1, 2, 3), (1, 2, 3)))
    assert c.shape == (1,) and c.item() == 8
    c = m.ttt(ones((3, 4, 2)), ones((4, 3, 5)), m.ContractionSpec(2, (3, 1, 2), (3, 2, 1)))
    assert c.shape == (2, 5) and c.data == [12] * 10


def test_ttt_random_specs(gpu):
    m = tl()
    rng = random.Random(8)
    for _ in range(30):
        a, b, na, nb, q, phi, psi = _ttt_draw(rng)
        got = box(m.ttt(a, b, m.ContractionSpec(q, phi, psi)))
        assert got == _ttt_expect(box(a), box(b), na, nb, q, phi, psi)


def test_ttt_spec_validation(gpu):
    m = tl()
    for args in ((1, (1, 1), (1,)), (2, (1,), (1, 2)), (-1, (1,), (1,))):
        with pytest.raises(ValueError):
            m.ContractionSpec(*args)
    a, b = m.DenseTensor((2, 3)), m.DenseTensor((4,))
    with pytest.raises(ValueError):
        m.ttt(a, b, m.ContractionSpec(1, (1, 2), (1,)))
    with pytest.raises(ValueError):
        m.ttt(a, b, m.ContractionSpec(1, (1,), (1,)))


# -- reduction specs (test_contraction.py:247-290) ---------------------------------------


def test_reduction_specs(gpu):
    m = tl()
    spec = m.reduce_ttv_to_ttt(3, 2)
    assert (spec.phi, spec.psi, spec.q) == ((1, 3, 2), (1,), 1)
    rng = random.Random(9)
    a, b = dense_draw(rng, (3, 4)), dense_draw(rng, (3,))
    assert m.tensors_equal(m.ttv(a, b, 1), m.ttt(a, b, m.reduce_ttv_to_ttt(2, 1)))
    rng = random.Random(10)
    for _ in range(60):
        p = rng.randint(2, 4)
        shape = tuple(rng.randint(1, 4) for _ in range(p))
        md = rng.randint(1, p)
        a = operand_draw(rng, shape)
        b = operand_draw(rng, (shape[md - 1],))
        assert m.tensors_equal(m.ttv(a, b, md), m.ttt(a, b, m.reduce_ttv_to_ttt(p, md)))
    rng = random.Random(11)
    a, b = dense_draw(rng, (3, 2, 4)), dense_draw(rng, (5, 4))
    assert m.tensors_equal(m.ttm(a, b, 3), m.ttt(a, b, m.reduce_ttm_to_ttt(3, 3)))
    rng = random.Random(12)
    for _ in range(20):
        p = rng.randint(2, 4)
        shape = tuple(rng.randint(1, 4) for _ in range(p))
        md = rng.randint(1, p)
        a = dense_draw(rng, shape)
        b = dense_draw(rng, (rng.randint(1, 4), shape[md - 1]))
        cycled = tuple(k for k in range(1, p + 1) if k != md) + (md,)
        assert m.tensors_equal(m.ttt(a, b, m.reduce_ttm_to_ttt(p, md)), m.transpose(m.ttm(a, b, md), cycled))


# -- named special cases (test_contraction.py:293-322) -----------------------------------


def test_norm_inner_outer(gpu):
    m = tl()
    assert m.frobenius_norm(m.DenseTensor((2, 2, 2), fill_value=1)) == math.sqrt(8)
    t = dense_draw(random.Random(13), (3, 2), kind="float")
    assert m.inner_product_tensors(t, t) >= 0
    z = m.DenseTensor((3, 2))
    assert m.inner_product_tensors(z, z) == 0
    rng = random.Random(14)
    a, b = operand_draw(rng, (2, 3)), operand_draw(rng, (4,))
    c = m.outer_product(a, b)
    ab, bb, got = box(a), box(b), box(c)
    assert c.shape == (2, 3, 4)
    assert all(got[(i, j, k)] == ab[(i, j)] * bb[(k,)] for i in range(2) for j in range(3) for k in range(4))
    with pytest.raises(ValueError):
        m.inner_product_tensors(m.DenseTensor((2, 3)), m.DenseTensor((3, 2)))


# -- times_vectors / times_matrices (test_contraction.py:325-395) ------------------------


def test_times_vectors(gpu):
    m = tl()
    a = m.DenseTensor((2, 3, 2), fill_value=1)
    c = m.times_vectors(a, [m.DenseTensor((n,), fill_value=1) for n in (2, 3, 2)], [1, 2, 3])
    assert c.shape == (1,) and c.item() == 12
    rng = random.Random(15)
    a, b = dense_draw(rng, (3, 4, 2)), dense_draw(rng, (4,))
    assert m.tensors_equal(m.times_vectors(a, [b], [2]), m.ttv(a, b, 2))
    rng = random.Random(16)
    for _ in range(10):
        p = rng.randint(2, 4)
        shape = tuple(rng.randint(1, 4) for _ in range(p))
        skip = rng.randint(1, p)
        a = dense_draw(rng, shape)
        full = [dense_draw(rng, (n,)) for n in shape]
        modes = [md for md in range(1, p + 1) if md != skip]
        assert m.tensors_equal(m.times_vectors(a, full, skip=skip),
                               m.times_vectors(a, [full[md - 1] for md in modes], modes))
    rng = random.Random(17)
    a, u, w = dense_draw(rng, (3, 4, 2)), dense_draw(rng, (3,)), dense_draw(rng, (2,))
    both = m.times_vectors(a, [u, w], [1, 3])
    assert m.tensors_equal(both, m.ttv(m.ttv(a, w, 3), u, 1))
    assert m.tensors_equal(both, m.ttv(m.ttv(a, u, 1), w, 2))
    a, v = m.DenseTensor((2, 3)), m.DenseTensor((2,))
    for args, kw in ((([v, v], [1, 1]), {}), (([v], [3]), {}), (([v], [1]), {"skip": 2})):
        with pytest.raises(ValueError):
            m.times_vectors(a, *args, **kw)


def test_times_matrices(gpu):
    m = tl()
    rng = random.Random(18)
    a = dense_draw(rng, (2, 3, 2))
    assert m.tensors_equal(m.times_matrices(a, [eye(n) for n in a.shape], [1, 2, 3]), a)
    rng = random.Random(19)
    a, b = dense_draw(rng, (2, 3, 2)), dense_draw(rng, (4, 3))
    assert m.tensors_equal(m.times_matrices(a, [b], [2]), m.ttm(a, b, 2))
    rng = random.Random(20)
    a, u, v = dense_draw(rng, (2, 3, 2)), dense_draw(rng, (4, 2)), dense_draw(rng, (5, 2))
    both = m.times_matrices(a, [u, v], [1, 3])
    assert m.tensors_equal(both, m.ttm(m.ttm(a, v, 3), u, 1))
    assert m.tensors_equal(both, m.ttm(m.ttm(a, u, 1), v, 3))


# -- allocation discipline (test_contraction.py:398-425) ---------------------------------


def test_each_contraction_allocates_only_its_output(gpu, monkeypatch):
    m = tl()
    calls = [0]
    init = m.DenseTensor.__init__

    def counted(self, *args, **kw):
        calls[0] += 1
        return init(self, *args, **kw)

    monkeypatch.setattr(m.DenseTensor, "__init__", counted)
    rng = random.Random(21)
    a, b = operand_draw(rng, (3, 4, 2)), operand_draw(rng, (4,))
    mat, t2 = operand_draw(rng, (5, 4)), operand_draw(rng, (4, 3))
    for fn in (lambda: m.ttv(a, b, 2), lambda: m.ttm(a, mat, 2),
               lambda: m.ttt(a, t2, m.ContractionSpec(2, (3, 1, 2), (2, 1))), lambda: m.transpose(a, (2, 3, 1))):
        calls[0] = 0
        fn()
        assert calls[0] == 1
