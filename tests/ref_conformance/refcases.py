"""Seeded case builders for the conformance suite.

These restate the instance builders of the reference suite's conftest
(/root/reference/pkg/tests/conftest.py:13-70) with the SAME consumption of
``random.Random`` draws, so a seed here yields the very tensors, views,
layouts and offsets the reference's own tests draw.  The drop-in's
defaults apply: ``DenseTensor(shape)`` is float64, and the integer-valued
data below is exact in it.  Test infrastructure only.
"""

from __future__ import annotations

import itertools


def tl():
    import paper_1711_10912_b200 as m

    return m


def layout_draw(rng, p):
    perm = list(range(1, p + 1))
    rng.shuffle(perm)
    return tuple(perm)


def offsets_draw(rng, p):
    return tuple(rng.randint(-2, 2) for _ in range(p))


def dense_draw(rng, shape, kind="int"):
    """A tensor with random offsets and layout; integer values in [-9, 9]
    or floats in [0.5, 2] (conftest.py:28-35)."""
    m = tl()
    p = len(shape)
    t = m.DenseTensor(shape, offsets_draw(rng, p), layout_draw(rng, p))
    n = t.size
    t.data = [rng.randint(-9, 9) for _ in range(n)] if kind == "int" else [rng.uniform(0.5, 2.0) for _ in range(n)]
    return t


def operand_draw(rng, shape, kind="int"):
    """Half the time a tensor, else a stepped view of this shape into a
    larger parent (conftest.py:38-58)."""
    m = tl()
    if rng.random() < 0.5:
        return dense_draw(rng, shape, kind)
    p = len(shape)
    steps = [rng.randint(1, 2) for _ in range(p)]
    leads = [rng.randint(0, 1) for _ in range(p)]
    parent_shape = tuple(ld + st * (n - 1) + 1 + rng.randint(0, 1) for n, st, ld in zip(shape, steps, leads))
    parent = dense_draw(rng, parent_shape, kind)
    ranges = []
    for r in range(p):
        lo = parent.offsets[r] + leads[r]
        ranges.append(m.Range(lo, steps[r], lo + steps[r] * (shape[r] - 1)))
    return m.TensorView(parent, ranges)


def box(x) -> dict:
    """Zero-based multi-index -> value, read element by element through the
    operand's own indexing (conftest.py:61-66)."""
    o = x.offsets
    return {i: x[tuple(a + b for a, b in zip(i, o))] for i in itertools.product(*(range(n) for n in x.shape))}


def all_idx(shape):
    return itertools.product(*(range(n) for n in shape))


def eye(n):
    m = tl()
    t = m.DenseTensor((n, n))
    for i in range(n):
        t[i, i] = 1
    return t
