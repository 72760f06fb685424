"""The configs' shapes under EVERY permutation layout and EVERY mode: north_star's
"across all layouts and modes" as a table.

  ttv    128^4 float32 (cfg2)            24 layouts x 4 modes
  ttv    400^3 float64 (cfg4)             6 layouts x 3 modes
  ttv    3x33x5x17x9x2x640 float64 (cfg5) NL seeded random layouts x 7 modes
  ttm    512^3 float64 x 384x512 (cfg3)   6 layouts x 3 modes
  ttm    3x33x5x17x2x640 float64, J = 16  NL seeded random layouts x 6 modes
  inner  128^4 float32, first x every 24th layout
  norm   128^4 float32 / 400^3 float64 (layout-independent walk)

Every result is compared with the first-order layout's result of the same
logical tensor: ttv/ttm outputs are first-order tensors whose every element is
the same k-ordered fold, so they must be bit-identical across layouts.

    python tools/experiments/config_sweep.py [what,...] [NL]
"""
import itertools
import json
import os
import statistics
import sys

import numpy as np
import torch

R = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path[:0] = [R, os.path.join(R, "tests"), os.path.join(R, "tools", "experiments")]
import ctypes  # noqa: E402

import paper_1711_10912_b200 as tl  # noqa: E402
from paper_1711_10912_b200.layout import TensorMeta  # noqa: E402
from sweep_ttm5 import timeit  # noqa: E402


def peaks():
    try:
        return float(json.load(open(os.path.join(R, "MEASURED_PEAKS.json")))["hbm_gbs"])
    except Exception:
        return 6545.6


PK = peaks()
FP64_PEAK = 37.05
L = tl._abi.lib()


def describe(A, mode, B=None):
    info = ctypes.create_string_buffer(512)
    L.tl_plan_describe(1 if B is not None else 0, A.desc(), B.desc() if B is not None else None, mode, info, 512)
    try:
        d = json.loads(info.value.decode())
        return d.get("regime", d.get("path", "?")) + ("/" + d["store"] if "store" in d else "")
    except Exception:
        return info.value.decode()[:60]


def first_order(shape, dtype, seed):
    g = torch.Generator(device="cuda").manual_seed(seed)
    n = int(np.prod(shape))
    buf = torch.rand(n, dtype=dtype, device="cuda", generator=g) * 2 - 1
    return tl.DenseTensor._wrap(TensorMeta(tuple(shape)), buf)


def in_layout(A0, layout):
    A = tl.DenseTensor._wrap(TensorMeta(A0.shape), A0.buffer.clone())
    A.relayout(tuple(layout))
    return A


def vec(n, dtype, seed):
    g = torch.Generator(device="cuda").manual_seed(1000 + seed)
    return tl.DenseTensor._wrap(TensorMeta((n,)), torch.rand(n, dtype=dtype, device="cuda", generator=g) * 2 - 1)


def mat(j, k, dtype, seed):
    g = torch.Generator(device="cuda").manual_seed(2000 + seed)
    return tl.DenseTensor._wrap(TensorMeta((j, k)), torch.randn(j * k, dtype=dtype, device="cuda", generator=g))


def emit(rows, **row):
    rows.append(row)
    print(json.dumps(row), flush=True)


def sweep_ttv(rows, name, shape, dtype, layouts, reps=5):
    s = 4 if dtype == torch.float32 else 8
    n = int(np.prod(shape))
    A0 = first_order(shape, dtype, 0)
    vs = [vec(shape[m], dtype, m) for m in range(len(shape))]
    ref = [tl.ttv(A0, vs[m], m + 1).buffer.clone() for m in range(len(shape))]
    for lay in layouts:
        A = in_layout(A0, lay)
        for m in range(len(shape)):
            C = tl.ttv(A, vs[m], m + 1)
            same = bool(torch.equal(C.buffer, ref[m]))
            us = timeit(lambda: tl.ttv(A, vs[m], m + 1), n=reps)
            nbytes = s * (n + shape[m]) + C.buffer.element_size() * (n // shape[m])
            emit(rows, op="ttv", cfg=name, layout=list(lay), mode=m + 1, us=round(us, 1),
                 frac=round(nbytes / us / 1e3 / PK, 3), kernel=describe(A, m + 1), bit_identical=same)
        del A
        torch.cuda.empty_cache()


def sweep_ttm(rows, name, shape, J, layouts, reps=5):
    n = int(np.prod(shape))
    A0 = first_order(shape, torch.float64, 3)
    Bs = [mat(J, shape[m], torch.float64, m) for m in range(len(shape))]
    ref = [tl.ttm(A0, Bs[m], m + 1).buffer.clone() for m in range(len(shape))]
    for lay in layouts:
        A = in_layout(A0, lay)
        for m in range(len(shape)):
            C = tl.ttm(A, Bs[m], m + 1)
            diff = (C.buffer - ref[m]).abs().max().item()
            scale = ref[m].abs().max().item()
            us = timeit(lambda: tl.ttm(A, Bs[m], m + 1), n=reps)
            flops = 2.0 * n * J
            nbytes = 8 * (n + J * shape[m] + n // shape[m] * J)
            emit(rows, op="ttm", cfg=name, layout=list(lay), mode=m + 1, us=round(us, 1),
                 tflops=round(flops / us / 1e6, 2), frac_fp64=round(flops / us / 1e6 / FP64_PEAK, 3),
                 frac_hbm=round(nbytes / us / 1e3 / PK, 3), kernel=describe(A, m + 1, Bs[m]),
                 max_abs_diff_vs_first=diff, scale=scale)
        del A
        torch.cuda.empty_cache()


def sweep_inner(rows, name, shape, dtype, layouts, reps=5):
    s = 4 if dtype == torch.float32 else 8
    n = int(np.prod(shape))
    A0 = first_order(shape, dtype, 5)
    B0 = first_order(shape, dtype, 6)
    ref = tl.inner_product_tensors(A0, B0)
    for lay in layouts:
        B = in_layout(B0, lay)
        val = tl.inner_product_tensors(A0, B)
        us = timeit(lambda: tl.contraction.inner_product_device(A0, B), n=reps)
        emit(rows, op="inner", cfg=name, layout=list(lay), us=round(us, 1), frac=round(2 * s * n / us / 1e3 / PK, 3),
             rel_diff_vs_first=abs(val - ref) / abs(ref))
        del B
        torch.cuda.empty_cache()
    us = timeit(lambda: tl.contraction.frobenius_norm_device(A0), n=reps)
    emit(rows, op="norm", cfg=name, us=round(us, 1), frac=round(s * n / us / 1e3 / PK, 3))


def random_layouts(p, count):
    out = []
    for seed in range(count):
        out.append(tuple(int(x) + 1 for x in np.random.default_rng(seed).permutation(p)))
    return out


def main():
    what = sys.argv[1].split(",") if len(sys.argv) > 1 else ["ttv2", "ttv4", "ttv5", "ttm3", "ttm5", "inner"]
    NL = int(sys.argv[2]) if len(sys.argv) > 2 else 8
    rows = []
    if "ttv2" in what:
        sweep_ttv(rows, "cfg2", (128,) * 4, torch.float32, list(itertools.permutations(range(1, 5))))
    if "ttv4" in what:
        sweep_ttv(rows, "cfg4", (400,) * 3, torch.float64, list(itertools.permutations(range(1, 4))))
    if "ttv5" in what:
        sweep_ttv(rows, "cfg5", (3, 33, 5, 17, 9, 2, 640), torch.float64, random_layouts(7, NL))
    if "ttm3" in what:
        sweep_ttm(rows, "cfg3", (512,) * 3, 384, list(itertools.permutations(range(1, 4))))
    if "ttm5" in what:
        sweep_ttm(rows, "cfg5", (3, 33, 5, 17, 2, 640), 16, [tuple(range(1, 7))] + random_layouts(6, max(1, NL // 2)))
    if "inner" in what:
        lays = list(itertools.permutations(range(1, 5)))
        sweep_inner(rows, "cfg2", (128,) * 4, torch.float32, lays[::4] + [lays[-1]])
    for op, cfg in sorted({(r["op"], r["cfg"]) for r in rows}):
        key = "frac_fp64" if (op == "ttm" and cfg == "cfg3") else ("frac_hbm" if op == "ttm" else "frac")
        fr = sorted(r[key] for r in rows if r["op"] == op and r["cfg"] == cfg)
        bad = [r for r in rows if r["op"] == op and r["cfg"] == cfg and r.get("bit_identical") is False]
        print(json.dumps({"summary": f"{op} {cfg}", "cases": len(fr), "min": fr[0], "p10": fr[len(fr) // 10],
                          "median": statistics.median(fr), "max": fr[-1], "below_0.8": sum(f < 0.8 for f in fr),
                          "below_0.7": sum(f < 0.7 for f in fr), "not_bit_identical": len(bad), "key": key}))


if __name__ == "__main__":
    main()
