"""ttm with few rows (J <= 32) on ANY permutation layout and mode: the box
kernel of csrc/ttm_few.cu (x along A, y along C, masked odd extents; direct /
along-y / along-j stores) against the CPU oracle -- bit-exact for float32 and
int64, float64 within 1e-12 of sum|A||B| and 1e-12 normwise.  Run once with
the default dispatch (the stream / bulk tile kernels keep first-order-compatible
float64 outputs) and once in a child process with TL_TTM_FEW=2 (every J <= 32
ttm on the box kernel).

    python tests/test_gpu_ttm_few.py        # the sweep under the current environment
"""

import ctypes
import json
import os
import random
import subprocess
import sys

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
for p in (ROOT, HERE):
    if p not in sys.path:
        sys.path.insert(0, p)

import workloads as W  # noqa: E402
from oracle import oracle as O  # noqa: E402
from tolerance import check_ttm  # noqa: E402

pytestmark = pytest.mark.gpu


def bits(a):
    a = np.ascontiguousarray(a)
    return a.view({8: np.uint64, 4: np.uint32}[a.dtype.itemsize])


def rand_shape(rng, max_vol):
    p = rng.randint(2, 7)
    choices = [1, 2, 3, 4, 5, 7, 8, 9, 16, 17, 31, 32, 33, 40, 64, 100, 128, 257, 640]
    while True:
        shape = tuple(rng.choice(choices) for _ in range(p))
        if 1 <= np.prod(shape) <= max_vol:
            return shape


def plan_path(m, A, B, mode):
    info = ctypes.create_string_buffer(1024)
    rc = m._abi.lib().tl_plan_describe(1, A.desc(), B.desc(), mode, info, 1024)
    assert rc == 0
    return json.loads(info.value.decode())


def sweep(seeds=(0, 1, 2), cases=40, max_vol=600_000):
    import paper_1711_10912_b200 as m

    taken = {}
    for seed in seeds:
        rng, nrng = random.Random(700 + seed), np.random.default_rng(700 + seed)
        for t in range(cases):
            kind = ["float64", "float64", "float32", "int64"][t % 4]
            shape = rand_shape(rng, max_vol)
            p = len(shape)
            layout = W.random_layout(p, rng.randint(0, 1 << 30))
            mode = rng.randint(1, p)
            J = rng.randint(1, 32)
            blayout = (1, 2) if rng.random() < 0.5 else (2, 1)
            if kind == "int64":
                T = nrng.integers(-20, 20, size=shape)
                M = nrng.integers(-20, 20, size=(J, shape[mode - 1]))
            else:
                T = nrng.uniform(-1, 1, size=shape).astype(kind)
                M = nrng.standard_normal((J, shape[mode - 1])).astype(kind)
            buf, mbuf = W.layout_buffer(T, layout), W.layout_buffer(M, blayout)
            A = m.DenseTensor.from_memory(shape, buf, layout=layout)
            B = m.DenseTensor.from_memory(M.shape, mbuf, layout=blayout)
            d = plan_path(m, A, B, mode)
            key = d.get("path", "?") + ("/" + d["store"] if "store" in d else "")
            taken[key] = taken.get(key, 0) + 1
            C = m.ttm(A, B, mode).numpy()
            st, bst = W.compute_strides(shape, layout), W.compute_strides(M.shape, blayout)
            want = O.ttm(buf, shape, st, mbuf, M.shape, bst, mode)
            what = (shape, layout, mode, J, kind, d)
            if kind == "float64":
                bound = O.ttm(np.abs(buf), shape, st, np.abs(mbuf), M.shape, bst, mode)
                try:
                    check_ttm(C, want, bound)
                except AssertionError as e:
                    raise AssertionError(f"{what}: {e}")
            else:
                if kind == "float32":
                    want = want.astype(np.float32)
                assert np.array_equal(bits(C), bits(want)), what
    return taken


def test_few_rows_any_layout_default_dispatch(gpu):
    taken = sweep()
    # the box kernel takes the permuted / strided cases in all three store orders
    for key in ("few/direct", "few/along-y", "few/along-j"):
        assert taken.get(key, 0) > 0, taken


def test_few_rows_any_layout_forced(gpu):
    env = dict(os.environ, TL_TTM_FEW="2")
    r = subprocess.run([sys.executable, os.path.abspath(__file__)], env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    taken = json.loads(r.stdout.strip().splitlines()[-1])
    # (the box kernel keeps B in shared memory: K * J images past 64 KB stay on the other paths)
    assert sum(v for k, v in taken.items() if k.startswith("few/")) >= 0.9 * sum(taken.values()), taken


def test_few_rows_config5_shape_every_mode(gpu):
    """The cfg5 ttm operand shape (3,33,5,17,2,640) in a random layout, J = 16,
    every mode: results equal the first-order layout's (same k-ordered chains)."""
    import torch

    import paper_1711_10912_b200 as m

    shape = (3, 33, 5, 17, 2, 64)
    nrng = np.random.default_rng(5)
    T = nrng.uniform(-1, 1, size=shape)
    A0 = m.DenseTensor.from_memory(shape, W.layout_buffer(T, tuple(range(1, 7))))
    for lay in [(4, 3, 6, 5, 1, 2), (3, 6, 5, 2, 4, 1), (6, 5, 4, 3, 2, 1)]:
        A = m.DenseTensor.from_memory(shape, W.layout_buffer(T, lay), layout=lay)
        for mode in range(1, 7):
            M = nrng.standard_normal((16, shape[mode - 1]))
            B = m.DenseTensor.from_memory(M.shape, W.layout_buffer(M, (1, 2)))
            got, ref = m.ttm(A, B, mode), m.ttm(A0, B, mode)
            assert torch.equal(got.buffer, ref.buffer), (lay, mode)


if __name__ == "__main__":
    print(json.dumps(sweep()))
