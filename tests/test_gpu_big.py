"""Index space past 2^32 elements (the reference's cap is 2^63 - 1,
layout.py:48).  A 180 GB B200 holds such tensors; the kernels' 32-bit digit
maps do not cover them, so these cases run on the 64-bit fallback kernels
(copy64, ttv_generic64, the 64-bit one-thread-per-output ttm, and the
64-bit reduction walk).  Each check compares against the same computation
on slices below 2^32 (bit-exact for ttv/ttm/copy) or an accurate float64
sum (inner).  Tensors are float32, 17-34 GB each; data is generated on the
device (torch's RNG) -- no oracle is needed, only self-consistency with the
tuned paths that the rest of the suite pins to the reference."""

import pytest
import torch

pytestmark = pytest.mark.gpu

BIG = (1 << 32) + 1


def tl():
    import paper_1711_10912_b200 as m

    return m


def wrap(buf, shape, layout=None):
    m = tl()
    from paper_1711_10912_b200.layout import TensorMeta

    return m.DenseTensor._wrap(TensorMeta(shape, layout=layout), buf)


def big_uniform(n, seed):
    g = torch.Generator(device="cuda")
    g.manual_seed(seed)
    t = torch.empty(n, device="cuda", dtype=torch.float32)
    return t.uniform_(-1.0, 1.0, generator=g)  # in place: no 2^32-element temporaries


@pytest.fixture(autouse=True)
def _free():
    yield
    torch.cuda.synchronize()
    torch.cuda.empty_cache()


def test_plan_reports_generic64(gpu):
    m = tl()
    L = m._abi.lib()
    import ctypes

    buf = ctypes.create_string_buffer(512)
    a = m._abi.make_desc((2, BIG), (1, 2), m._abi.TL_F32)
    assert L.tl_plan_describe(0, a, None, 1, buf, 512) == 0
    assert b'"generic64"' in buf.value


def test_ttv_outer_past_2_32(gpu):
    """(2, 2^32+1) first-order, mode 1: O = 2^32 + 1 outputs."""
    m = tl()
    A = wrap(big_uniform(2 * BIG, 1), (2, BIG))
    v = m.DenseTensor.from_memory((2,), [0.75, -1.25])
    C = m.ttv(A, v, 1)
    n = 1 << 20
    for o0 in (0, BIG - n):
        part = m.ttv(wrap(A.buffer[2 * o0: 2 * (o0 + n)], (2, n)), v, 1)
        assert torch.equal(C.buffer[o0: o0 + n], part.buffer)


def test_ttv_inner_past_2_32(gpu):
    """(2^32+1, 2) first-order, mode 2: I = 2^32 + 1; out[i] = (0 + a_i b0) + a_{i+I} b1."""
    m = tl()
    A = wrap(big_uniform(2 * BIG, 2), (BIG, 2))
    v = m.DenseTensor.from_memory((2,), [0.5, 3.0])
    C = m.ttv(A, v, 2)
    idx = torch.randint(0, BIG, (1 << 20,), device="cuda")
    x0, x1 = A.buffer[idx].double(), A.buffer[idx + BIG].double()
    want = ((0.0 + x0 * 0.5) + x1 * 3.0).float()
    assert torch.equal(C.buffer[idx], want)


def test_ttm_outer_past_2_32(gpu):
    """(2, 2^32+1) mode 1 with a 2 x 2 matrix: the 64-bit ttm path."""
    m = tl()
    A = wrap(big_uniform(2 * BIG, 3), (2, BIG))
    M = m.DenseTensor.from_memory((2, 2), [1.5, -0.5, 2.0, 0.25], dtype="float32")
    C = m.ttm(A, M, 1)
    n = 1 << 20
    for o0 in (0, BIG - n):
        part = m.ttm(wrap(A.buffer[2 * o0: 2 * (o0 + n)], (2, n)), M, 1)
        assert torch.equal(C.buffer[2 * o0: 2 * (o0 + n)], part.buffer)


def test_relayout_past_2_32(gpu):
    """(8, 3, 2^28 + 1) relayout (1,2,3) -> (1,3,2): 6.4e9 elements, one copy."""
    m = tl()
    shape = (8, 3, (1 << 28) + 1)
    n = shape[0] * shape[1] * shape[2]
    A = wrap(big_uniform(n, 4), shape)
    B = A.copy()
    B.relayout((1, 3, 2))
    idx = [torch.randint(0, e, (1 << 20,), device="cuda") for e in shape]
    sa, sb = A.strides, B.strides
    pa = idx[0] * sa[0] + idx[1] * sa[1] + idx[2] * sa[2]
    pb = idx[0] * sb[0] + idx[1] * sb[1] + idx[2] * sb[2]
    assert torch.equal(A.buffer[pa], B.buffer[pb])


def test_inner_past_2_32_rows(gpu):
    """(2, 2^30+1, 2) first-order x layout (1,3,2): 2^32+ elements whose
    b offsets need the 64-bit map."""
    m = tl()
    from paper_1711_10912_b200.tensor import _copy

    shape = (2, (1 << 30) + 1, 2)
    n = shape[0] * shape[1] * shape[2]
    A = wrap(big_uniform(n, 5), shape)
    Bf = wrap(big_uniform(n, 6), shape)  # B's values in first order
    B = m.DenseTensor(shape, layout=(1, 3, 2), dtype="float32", fill_value=None)
    _copy(Bf.desc(), Bf.buffer, B.desc(), B.buffer)
    got = m.inner_product_tensors(A, B)
    want = 0.0
    absb = 0.0
    step = 1 << 28
    for s in range(0, n, step):
        a, b = A.buffer[s: s + step].double(), Bf.buffer[s: s + step].double()
        want += float(torch.sum(a * b))
        absb += float(torch.sum(torch.abs(a * b)))
    assert abs(got - want) <= 1e-12 * absb
