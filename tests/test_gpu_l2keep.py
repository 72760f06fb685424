"""ttv over tensors at least twice the L2 size: these take the L2 streaming
policy (loads evict-first except the part a pass reads last, which keeps the
normal policy for the next pass over the same tensor; ttv.cu TtvParams::keep_*)
-- in every instantiation it touches: the strided kernel for float32 (VEC 4 /
2 / 1), float64 (VEC 2 / 1) and int64 (VEC 2 / 1) on one-wave and multi-wave
grids, and the 2-D TMA rows kernel.  The policy must not change a result:
integer-valued data makes every fold exact in any order, so each output is
compared bit for bit with a float64 tensordot of the same data."""

import pytest
import torch

pytestmark = pytest.mark.gpu


def tl():
    import paper_1711_10912_b200 as m

    return m


def wrap(buf, shape, layout=None):
    from paper_1711_10912_b200.layout import TensorMeta

    return tl().DenseTensor._wrap(TensorMeta(shape, layout=layout), buf)


def small_ints(n, dtype, seed):
    g = torch.Generator(device="cuda")
    g.manual_seed(seed)
    return torch.randint(-4, 5, (n,), generator=g, device="cuda").to(dtype)


@pytest.fixture(autouse=True)
def _free():
    yield
    torch.cuda.synchronize()
    torch.cuda.empty_cache()


CASES = [
    # (shape, dtype, modes): first-order layout, >= 252 MB
    ((128, 128, 128, 40), torch.float32, (1, 2, 3, 4)),  # rows TMA, VEC 4 multi-wave, one wave (O = 1)
    ((130, 128, 128, 40), torch.float32, (2,)),  # I = 130: VEC 2
    ((127, 128, 128, 41), torch.float32, (2,)),  # I = 127: VEC 1 (32-bit hinted loads)
    ((128, 128, 128, 20), torch.float64, (1, 2, 3, 4)),
    ((129, 128, 128, 20), torch.float64, (2,)),  # VEC 1 (64-bit hinted loads)
    ((128, 128, 128, 20), torch.int64, (2, 4)),
    ((129, 128, 128, 20), torch.int64, (2,)),
]


@pytest.mark.parametrize("shape,dtype,modes", CASES, ids=lambda v: str(v))
def test_ttv_large_tensor_l2_policy_exact(gpu, shape, dtype, modes):
    m = tl()
    n = 1
    for e in shape:
        n *= e
    buf = small_ints(n, dtype, seed=sum(shape))
    A = wrap(buf, shape)
    # torch view of the first-order buffer with dimension 1 fastest
    At = buf.view(tuple(reversed(shape))).permute(*reversed(range(len(shape)))).to(torch.float64)
    for mode in modes:
        v = small_ints(shape[mode - 1], dtype, seed=mode)
        C = m.ttv(A, wrap(v, (shape[mode - 1],)), mode)
        want = torch.tensordot(At, v.to(torch.float64), dims=([mode - 1], [0]))
        got = C.buffer.view(tuple(reversed(want.shape))).permute(*reversed(range(want.dim()))).to(torch.float64)
        assert torch.equal(got, want), f"{shape} {dtype} mode {mode}"
