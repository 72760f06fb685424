"""Large-tensor ttv paths, each checked bit for bit on integer-valued data
(every fold exact in any order) against a float64 tensordot:

* tensors at least twice the L2 size: these take the L2 streaming
policy (loads evict-first except the part a pass reads last, which keeps the
normal policy for the next pass over the same tensor; ttv.cu TtvParams::keep_*)
-- in every instantiation it touches: the strided kernel for float32 (VEC 4 /
2 / 1), float64 (VEC 2 / 1) and int64 (VEC 2 / 1) on one-wave and multi-wave
grids, and the 2-D TMA rows kernel -- the policy must not change a result;
* short folds (K <= 16, >= 64 MB operands): the elementwise short-fold stream,
  into C in canonical order or through the digit maps when C's fastest
  canonical digit is contiguous;
* long folds over few fibres: one-warp CTAs streaming 2-D TMA boxes of k-rows x
  32 columns when rows are 16-byte aligned, else the per-thread cp.async ring
  kernel, columns (VEC 4 / 1) and rows (16-byte chunks, and element pieces
  when rows are not 16-byte aligned)."""

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


CASES2 = [
    # (shape, layout, dtype, mode, expected regime)
    ((1848, 2, 21263), (2, 1, 3), torch.float64, 2, "short-fold"),  # K = 2, I = 1, ident
    ((237, 10, 2, 11277), (3, 1, 4, 2), torch.float64, 3, "short-fold"),  # K = 2, permuted, fast digit C-contiguous
    ((907, 24, 3, 1001), (1, 2, 3, 4), torch.float32, 3, "short-fold"),  # K = 3, I > 1
    ((90, 4305, 336), (3, 2, 1), torch.float32, 2, "cols-tma"),  # few column fibres, long fold, aligned rows
    ((128, 4096, 64), (1, 2, 3), torch.float64, 2, "cols-tma"),  # float64 boxes; last slab zero-padded by TMA past I
    ((101, 3000, 97), (1, 2, 3), torch.float64, 2, "deep-ring"),  # I*8 not 16-byte aligned: the ring
    ((45, 4305, 333), (3, 2, 1), torch.float32, 2, "deep-ring"),  # VEC 1 columns
    ((201, 333367 // 4), (2, 1), torch.float64, 2, "deep-ring"),  # rows, odd K: element pieces
    ((200, 83336), (2, 1), torch.float64, 2, "deep-ring"),  # rows, 16-byte chunks
    # short folds with scattered permuted outputs: the fused transpose-fold
    ((7, 3, 6, 3, 20, 36, 551), (3, 5, 1, 4, 7, 6, 2), torch.float32, 4, "tile-fold"),  # K = 3, short X chain
    ((5, 4, 532, 801, 2, 8), (2, 6, 4, 3, 5, 1), torch.float32, 2, "tile-fold"),  # rows of K = 4
    ((2, 5, 4305, 56, 6, 9), (5, 4, 3, 1, 2, 6), torch.float32, 1, "tile-fold"),  # K = 2, long inner block
    ((6, 29, 7, 11, 2, 634, 10), (7, 5, 3, 6, 1, 2, 4), torch.float32, 5, "tile-fold"),  # K = 2, I = 10
    ((15, 42, 2, 4, 22, 5, 147), (5, 1, 2, 3, 7, 6, 4), torch.float64, 3, "tile-fold"),  # float64, K = 2
]


@pytest.mark.parametrize("shape,layout,dtype,mode,regime", CASES2, ids=lambda v: str(v))
def test_ttv_short_and_deep_paths_exact(gpu, shape, layout, dtype, mode, regime):
    import ctypes
    import json

    m = tl()
    n = 1
    for e in shape:
        n *= e
    buf = small_ints(n, dtype, seed=n % 1000)
    A = wrap(buf, shape, layout)
    info = ctypes.create_string_buffer(512)
    assert m._abi.lib().tl_plan_describe(0, A.desc(), None, mode, info, 512) == 0
    assert json.loads(info.value.decode())["regime"] == regime
    # torch view of the buffer: storage order = layout (dimension layout[0] fastest)
    p = len(shape)
    At = buf.view(tuple(shape[d - 1] for d in reversed(layout)))
    perm = [0] * p
    for pos, d in enumerate(reversed(layout)):
        perm[d - 1] = pos
    At = At.permute(*perm).to(torch.float64)
    v = small_ints(shape[mode - 1], dtype, seed=7)
    C = m.ttv(A, wrap(v, (shape[mode - 1],)), mode)
    want = torch.tensordot(At, v.to(torch.float64), dims=([mode - 1], [0]))
    got = C.buffer.view(tuple(reversed(want.shape))).permute(*reversed(range(want.dim()))).to(torch.float64)
    assert torch.equal(got, want)
