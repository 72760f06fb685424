"""Inner product of two tensors that share their fastest dimension but order
the others differently (e.g. layouts (1,2,3,4) x (1,4,2,3)): the vectorised
row walk of csrc/reduce.cu (16-byte loads, row starts through b's digit map)
and its scalar fallback for odd rows, against the oracle's fold
(elementwise.py:411-433) within the double-double bounds."""

import numpy as np
import pytest

import workloads as W
from oracle import oracle as O
from tolerance import check_inner

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("kind", ["float64", "float32", "int64"])
@pytest.mark.parametrize("shape,la,lb", [
    ((64, 12, 10, 9), (1, 2, 3, 4), (1, 4, 2, 3)),      # whole vectors per row
    ((64, 12, 10, 9), (1, 3, 2, 4), (1, 4, 3, 2)),
    ((30, 7, 11, 5), (1, 2, 3, 4), (1, 4, 2, 3)),       # float64 vectors only (30 % 4 != 0)
    ((33, 8, 6), (1, 2, 3), (1, 3, 2)),                 # odd rows: scalar walk
    ((128, 40, 3, 17, 2), (1, 2, 3, 4, 5), (1, 5, 3, 2, 4)),
])
def test_inner_shared_fastest_dimension(gpu, kind, shape, la, lb):
    import paper_1711_10912_b200 as m

    nrng = np.random.default_rng(abs(hash((kind, shape, lb))) % (1 << 31))
    if kind == "int64":
        Ta, Tb = nrng.integers(-50, 50, size=shape), nrng.integers(-50, 50, size=shape)
    else:
        Ta, Tb = nrng.uniform(-1, 1, size=shape).astype(kind), nrng.uniform(-1, 1, size=shape).astype(kind)
    ba, bb = W.layout_buffer(Ta, la), W.layout_buffer(Tb, lb)
    A = m.DenseTensor.from_memory(shape, ba, layout=la)
    B = m.DenseTensor.from_memory(shape, bb, layout=lb)
    got = m.inner_product_tensors(A, B)
    want = O.inner(ba, shape, W.compute_strides(shape, la), bb, W.compute_strides(shape, lb))
    if kind == "int64":
        assert got == want
    else:
        check_inner(got, want, Ta.astype(np.float64), Tb.astype(np.float64))
