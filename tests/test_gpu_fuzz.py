"""Randomised sweep over every kernel regime: random order (2..7), extents
(including 1 and odd sizes), layout, mode, J and dtype, at sizes that reach
the staged/strided/small ttv kernels, the GETT / bulk / staged / SIMT ttm
kernels and the flat/tiled reductions.  Every case is checked against the
CPU oracle: bit-exact for ttv (all dtypes), int64 ttm and float32 ttm;
float64 ttm within 1e-12 of sum|A||B|; inner/norm within the double-double
bounds."""

import os
import random

import numpy as np
import pytest

import workloads as W
from oracle import oracle as O
from tolerance import check_ttm

pytestmark = pytest.mark.gpu

# TL_FUZZ_SEEDS=N widens every sweep (default: the few seeds the suite runs)
EXTRA = int(os.environ.get("TL_FUZZ_SEEDS", "0"))


def tl():
    import paper_1711_10912_b200 as m

    return m


def bits(a):
    a = np.ascontiguousarray(a)
    return a.view({8: np.uint64, 4: np.uint32}[a.dtype.itemsize])


def rand_shape(rng, max_vol):
    p = rng.randint(2, 7)
    choices = [1, 2, 3, 4, 5, 7, 8, 9, 16, 17, 31, 32, 33, 40, 64, 100, 128, 257]
    while True:
        shape = tuple(rng.choice(choices) for _ in range(p))
        if np.prod(shape) <= max_vol:
            return shape


def draw(nrng, shape, kind):
    if kind == "int64":
        return nrng.integers(-20, 20, size=shape)
    return nrng.uniform(-1, 1, size=shape).astype(kind)


@pytest.mark.parametrize("seed", range(max(4, EXTRA)))
def test_fuzz_ttv(gpu, seed):
    m = tl()
    rng, nrng = random.Random(100 + seed), np.random.default_rng(100 + seed)
    for t in range(60):
        kind = ["float64", "float32", "int64"][t % 3]
        shape = rand_shape(rng, 3_000_000)
        p = len(shape)
        layout = W.random_layout(p, rng.randint(0, 1 << 30))
        mode = rng.randint(1, p)
        T = draw(nrng, shape, kind)
        b = draw(nrng, (shape[mode - 1],), kind)
        buf = W.layout_buffer(T, layout)
        C = m.ttv(m.DenseTensor.from_memory(shape, buf, layout=layout), m.DenseTensor.from_memory((shape[mode - 1],), b),
                  mode).numpy()
        want = O.ttv(buf, shape, W.compute_strides(shape, layout), b, mode)
        if kind == "float32":
            want = want.astype(np.float32)
        assert np.array_equal(bits(C), bits(want)), (shape, layout, mode, kind)


@pytest.mark.parametrize("seed", range(max(4, EXTRA)))
def test_fuzz_ttm(gpu, seed):
    m = tl()
    rng, nrng = random.Random(200 + seed), np.random.default_rng(200 + seed)
    for t in range(40):
        kind = ["float64", "float64", "float32", "int64"][t % 4]
        shape = rand_shape(rng, 400_000)
        p = len(shape)
        layout = W.random_layout(p, rng.randint(0, 1 << 30))
        mode = rng.randint(1, p)
        J = rng.choice([1, 3, 8, 16, 17, 24, 32, 33, 48, 64, 100])
        blayout = (1, 2) if rng.random() < 0.5 else (2, 1)
        T = draw(nrng, shape, kind)
        M = draw(nrng, (J, shape[mode - 1]), kind)
        buf, mbuf = W.layout_buffer(T, layout), W.layout_buffer(M, blayout)
        C = m.ttm(m.DenseTensor.from_memory(shape, buf, layout=layout),
                  m.DenseTensor.from_memory(M.shape, mbuf, layout=blayout), mode).numpy()
        st, bst = W.compute_strides(shape, layout), W.compute_strides(M.shape, blayout)
        want = O.ttm(buf, shape, st, mbuf, M.shape, bst, mode)
        if kind == "float64":
            bound = O.ttm(np.abs(buf), shape, st, np.abs(mbuf), M.shape, bst, mode)
            check_ttm(C, want, bound)
        else:
            if kind == "float32":
                want = want.astype(np.float32)
            assert np.array_equal(bits(C), bits(want)), (shape, layout, mode, J, kind)


@pytest.mark.parametrize("seed", range(max(2, EXTRA)))
def test_fuzz_inner_norm(gpu, seed):
    m = tl()
    rng, nrng = random.Random(300 + seed), np.random.default_rng(300 + seed)
    for t in range(40):
        kind = ["float64", "float32", "int64"][t % 3]
        shape = rand_shape(rng, 3_000_000)
        p = len(shape)
        la = W.random_layout(p, rng.randint(0, 1 << 30))
        lb = la if rng.random() < 0.5 else W.random_layout(p, rng.randint(0, 1 << 30))
        Ta, Tb = draw(nrng, shape, kind), draw(nrng, shape, kind)
        ba, bb = W.layout_buffer(Ta, la), W.layout_buffer(Tb, lb)
        A = m.DenseTensor.from_memory(shape, ba, layout=la)
        B = m.DenseTensor.from_memory(shape, bb, layout=lb)
        sa, sb = W.compute_strides(shape, la), W.compute_strides(shape, lb)
        got = m.inner_product_tensors(A, B)
        want = O.inner(ba, shape, sa, bb, sb)
        if kind == "int64":
            assert got == want
            continue
        # the oracle (= the reference's sequential fold) carries up to n*u of
        # sum|ab| itself; ours is a double-double / short-chain sum
        n = int(np.prod(shape))
        tol = 1e-13 + n * 2.0 ** -53
        scale = float(np.sum(np.abs(Ta.astype(np.float64) * Tb.astype(np.float64))))
        assert abs(got - want) <= tol * scale + 1e-300, (shape, la, lb)
        nrm = m.frobenius_norm(A)
        wn = O.norm(ba, shape, sa)
        assert abs(nrm - wn) <= tol * wn + 1e-300, (shape, la)


@pytest.mark.parametrize("seed", range(max(3, EXTRA)))
def test_fuzz_ttm_small_j_first_order(gpu, seed):
    """float64 ttm with J <= 32 on first-order tensors (outputs in A's order):
    the warp-specialised stream kernel and its fallbacks, including partial
    last tiles, odd R*K*I (8-byte tails) and tiny O."""
    m = tl()
    rng, nrng = random.Random(400 + seed), np.random.default_rng(400 + seed)
    for t in range(30):
        shape = rand_shape(rng, 2_000_000)
        p = len(shape)
        layout = tuple(range(1, p + 1))
        mode = rng.randint(1, p)
        J = rng.randint(1, 32)
        T = nrng.standard_normal(shape)
        M = nrng.standard_normal((J, shape[mode - 1]))
        buf, mbuf = W.layout_buffer(T, layout), W.layout_buffer(M, (1, 2))
        C = m.ttm(m.DenseTensor.from_memory(shape, buf, layout=layout),
                  m.DenseTensor.from_memory(M.shape, mbuf), mode).numpy()
        st, bst = W.compute_strides(shape, layout), W.compute_strides(M.shape, (1, 2))
        want = O.ttm(buf, shape, st, mbuf, M.shape, bst, mode)
        bound = O.ttm(np.abs(buf), shape, st, np.abs(mbuf), M.shape, bst, mode)
        check_ttm(C, want, bound)
