"""Conformance: the reference's HOPM suite, restated on the B200 path
(/root/reference/pkg/tests/test_hopm.py, same seeds and draw order).

Rank-one tensors are composed from seeded unit vectors; HOPM must recover
scale and vectors to 1e-10, keep unit norms to 1e-12, report degeneracy
at (sweep 1, mode 1) for a zero tensor and keep a monotone residual."""

import math
import random

import pytest

from .refcases import tl

pytestmark = pytest.mark.gpu


def unit(rng, n):
    m = tl()
    v = [rng.uniform(-1.0, 1.0) for _ in range(n)]
    s = math.sqrt(sum(x * x for x in v))
    return m.DenseTensor.from_memory((n,), [x / s for x in v])


def rank_one(rng, shape, scale):
    us = [unit(rng, n) for n in shape]
    return tl().rank_one_compose(scale, us), us


def uniform_tensor(rng, shape):
    a = tl().DenseTensor(shape)
    a.data = [rng.uniform(-1, 1) for _ in range(a.size)]
    return a


def test_recovery_of_exact_rank_one(gpu):  # test_hopm.py:30-36, 77-81, 140-145
    m = tl()
    for seed, shape, scale in ((0, (3, 4, 2), 3.0), (4, (3, 2, 4), 1.5), (9, (4, 2, 3), 4.5)):
        a, _ = rank_one(random.Random(seed), shape, scale)
        st = m.hopm(a, max_sweeps=50)
        assert st.converged and abs(st.scale - scale) < 1e-10
        assert m.residual(a, st) < 1e-10
        assert max(st.l) - min(st.l) < 1e-10


def test_vectors_up_to_sign_and_custom_start(gpu):  # test_hopm.py:38-44, 83-87
    m = tl()
    a, us = rank_one(random.Random(1), (4, 3), 2.0)
    st = m.hopm(a)
    for got, want in zip(st.u, us):
        assert abs(abs(sum(x * y for x, y in zip(got.data, want.data))) - 1.0) < 1e-10
    a, us = rank_one(random.Random(5), (3, 3), 2.5)
    st = m.hopm(a, u0=us)
    assert st.converged and abs(st.scale - 2.5) < 1e-10


def test_order_one_and_degenerate(gpu):  # test_hopm.py:46-55
    m = tl()
    st = m.hopm(m.DenseTensor.from_memory((3,), [3.0, 0.0, 4.0]))
    assert st.l[0] == 5.0 and st.u[0].data == [0.6, 0.0, 0.8]
    with pytest.raises(m.DegenerateInputError) as err:
        m.hopm(m.DenseTensor((2, 3)))
    assert (err.value.sweep, err.value.mode) == (1, 1)


def test_unit_norms_monotone_residual_sweep_limit(gpu):  # test_hopm.py:57-74, 97-102
    m = tl()
    st = m.hopm(uniform_tensor(random.Random(2), (3, 3, 2)), max_sweeps=10, tol=0.0)
    assert all(abs(m.frobenius_norm(u) - 1.0) < 1e-12 for u in st.u)
    rng = random.Random(3)
    for _ in range(5):
        shape = tuple(rng.randint(2, 4) for _ in range(rng.randint(2, 3)))
        hist = m.hopm(uniform_tensor(rng, shape), max_sweeps=20, tol=0.0, track_residuals=True).residual_history
        assert all(b <= a + 1e-10 for a, b in zip(hist, hist[1:]))
    st = m.hopm(uniform_tensor(random.Random(6), (3, 3, 3)), max_sweeps=1)
    assert st.sweeps == 1 and not st.converged


def test_start_vector_validation(gpu):  # test_hopm.py:89-95
    m = tl()
    a = m.DenseTensor((3, 2), fill_value=1.0)
    for kw in ({"u0": [m.DenseTensor((3,), fill_value=1.0)]},
               {"u0": [m.DenseTensor((3,)), m.DenseTensor((2,), fill_value=1.0)]}, {"max_sweeps": 0}):
        with pytest.raises(ValueError):
            m.hopm(a, **kw)


def test_rank_one_compose_and_residual(gpu):  # test_hopm.py:105-145
    m = tl()
    e1 = m.DenseTensor.from_memory((3,), [1.0, 0.0, 0.0])
    e2 = m.DenseTensor.from_memory((2,), [1.0, 0.0])
    b = m.rank_one_compose(1.0, [e1, e2])
    assert b[0, 0] == 1.0 and sum(abs(x) for x in b.data) == 1.0
    rng = random.Random(7)
    us = [unit(rng, n) for n in (3, 4, 2)]
    assert abs(m.frobenius_norm(m.rank_one_compose(2.25, us)) - 2.25) < 1e-12
    rng = random.Random(8)
    us = [unit(rng, n) for n in (2, 3, 2)]
    first = m.DenseTensor.from_memory(us[0].shape, [3.0 * x for x in us[0].data])
    assert m.tensors_equal(m.rank_one_compose(3.0, us), m.outer_product(m.outer_product(first, us[1]), us[2]))
    rng = random.Random(10)
    a = uniform_tensor(rng, (3, 2))
    us = [unit(rng, n) for n in a.shape]
    st = m.HopmState(u=us, l=[0.0, 0.0], sweeps=0, converged=False)
    assert abs(m.residual(a, st) - m.frobenius_norm(a)) < 1e-12
