"""Conformance: the storage and iterator contract of the reference
(tensor.py:33-284, iterators.py:28-182, views.py:181-209) on device
buffers -- write-through ``.data``, ``miter()`` cursors as hot-path
operands (contraction.py:52-55), stride-iterator ranges and the
recursion's visit order (test_iterators.py)."""

import itertools
import random

import numpy as np
import pytest

from .refcases import box, dense_draw, operand_draw, tl

pytestmark = pytest.mark.gpu


def iota(shape, **kw):
    m = tl()
    t = m.DenseTensor(shape, **kw)
    t.data = list(range(t.size))
    return t


def test_data_writes_go_through(gpu):
    m = tl()
    t = m.DenseTensor((2, 3), layout=(2, 1))
    d = t.data
    d[4] = 7.5  # the reference's out.data[j] = v (hopm.py:138, views.py:222)
    assert t.get_memory(4) == 7.5 and t.data[4] == 7.5
    d[0:2] = [1, 2]
    assert t.data[:2] == [1.0, 2.0]
    assert t[1, 1] == t.get_memory(m.memory_index(t.strides, (1, 1), t.offsets))
    for bad in (lambda: d.append(1), lambda: d.pop(), lambda: d.extend([1]), lambda: d.__delitem__(0)):
        with pytest.raises(TypeError):
            bad()
    i = m.DenseTensor.from_memory((3,), [1, 2, 3])
    assert i.dtype.is_floating_point is False
    with pytest.raises(TypeError):
        i.data[0] = 0.5  # int64 storage cannot hold it exactly: refused, never truncated
    i.data = [0.5, 1, 2]  # whole-list assignment keeps the values (the tensor becomes float64)
    assert i.data == [0.5, 1.0, 2.0]


def test_miter_and_views_are_operands(gpu):
    m = tl()
    rng = random.Random(31)
    for _ in range(20):
        p = rng.randint(2, 4)
        shape = tuple(rng.randint(1, 4) for _ in range(p))
        md = rng.randint(1, p)
        a = operand_draw(rng, shape)
        b = dense_draw(rng, (shape[md - 1],))
        want = m.ttv(a, b, md)
        assert m.tensors_equal(m.ttv(a.miter(), b.miter(), md), want)
    # a cursor over a host list (user code building a MultiIterator by hand)
    host = list(range(24))
    it = m.MultiIterator(host, 0, (1, 4, 12), (4, 3, 2))
    a = m.DenseTensor.from_memory((4, 3, 2), host)
    v = m.DenseTensor.from_memory((3,), [1, -2, 3])
    assert m.tensors_equal(m.ttv(it, v, 2), m.ttv(a, v, 2))


def test_stride_iterators(gpu):
    m = tl()
    a = m.DenseTensor((4, 3, 2))
    first, last = a.dim_begin(2), a.dim_end(2)
    assert (first.pos, first.stride, last.pos) == (0, 4, 12)
    m.fill_range(first, last, 5.0)
    assert sorted(j for j, x in enumerate(a.data) if x == 5.0) == [0, 4, 8]
    t = m.DenseTensor((3,))
    t.dim_begin(1).value = 9
    assert t.data[0] == 9
    a = iota((4, 3, 2), offsets=(0, -1, 0))
    it, end = a.dim_begin(2, at=(1, -1, 1)), a.dim_end(2, at=(1, -1, 1))
    seq = []
    while it != end:
        seq.append(it.value)
        it.advance()
    assert seq == [a[1, k - 1, 1] for k in range(3)]
    with pytest.raises(ValueError):
        a.dim_begin(4)


def test_inner_product_range_and_flat_init(gpu):
    m = tl()
    a = iota((2, 3, 3))
    b = iota((4, 3), layout=(2, 1))
    got = m.inner_product_range(a.dim_begin(3), a.dim_end(3), b.dim_begin(2), 0.0)
    assert got == sum(a[0, 0, k] * b[0, k] for k in range(3))
    # init enters the compensated sum: the result is init + sum rounded once
    x = m.DenseTensor.from_memory((2,), [1.0, 1.0])
    assert m.inner_product_flat(x, x, 1e16) == 1e16 + 2.0
    assert m.inner_product_flat(x, x, 0.5) == 2.5
    k = m.DenseTensor.from_memory((3,), [1, 2, 3])
    assert m.inner_product_flat(k, k, 10) == 24
    assert m.inner_product_flat(k, k, 0.25) == 14.25


def test_visit_order_and_completeness(gpu):
    m = tl()
    for p in (1, 2, 3):
        for layout in itertools.permutations(range(1, p + 1)):
            a = m.DenseTensor((3, 2, 4)[:p], layout=layout)
            assert sorted(m.walk_positions(a.miter())) == list(range(a.size))
    a = iota((5, 4, 3), layout=(3, 1, 2))
    v = a.view(m.Range(1, 2, 4), m.Range(0, 2, 3), None)
    got = m.walk_positions(v.miter())
    firsts = [r[0] for r in v.ranges]
    steps = [r[1] for r in v.ranges]
    want = {m.memory_index(a.strides, tuple(f + t * k for f, t, k in zip(firsts, steps, i)), a.offsets)
            for i in itertools.product(*(range(n) for n in v.shape))}
    assert len(got) == len(want) and set(got) == want
    # the recursion order: depth p-1 outermost, depth 0 innermost
    it = m.MultiIterator([0] * 24, 0, (1, 4, 12), (4, 3, 2))
    assert m.walk_positions(it) == list(range(24))


def test_nested_fill_through_cursors(gpu):
    m = tl()
    for layout in itertools.permutations((1, 2, 3)):
        a = m.DenseTensor((3, 2, 4), layout=layout)
        it = a.miter()
        f2, e2 = it.begin(2), it.end(2)
        while f2 != e2:
            it.move_to(f2)
            f1, e1 = it.begin(1), it.end(1)
            while f1 != e1:
                it.move_to(f1)
                m.fill_range(it.begin(0), it.end(0), 7)
                f1.advance()
            f2.advance()
        assert a.data == [7] * a.size


def test_view_box_reads_match_materialize(gpu):
    rng = random.Random(41)
    for _ in range(10):
        shape = tuple(rng.randint(1, 4) for _ in range(3))
        v = operand_draw(rng, shape)
        if isinstance(v, tl().TensorView):
            mat = v.materialize()
            assert box(mat) == {i: x for i, x in box(v).items()}
            assert np.array_equal(v.numpy(), mat.numpy())
