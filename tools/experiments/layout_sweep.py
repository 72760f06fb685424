"""ttv over random orders / extents / permutation layouts / modes at HBM-bound
sizes (about 512 MB per tensor): achieved GB/s of algorithmic bytes and the
kernel regime each case took.  Evidence for north_star's "across all layouts
and modes" (config 2 and config 5 cover only a few).  Seeded; prints one JSON
line per case and a summary line.

    python tools/experiments/layout_sweep.py [n_cases] [seed]
"""
import json
import os
import statistics
import sys

import numpy as np
import torch

R = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path[:0] = [R, os.path.join(R, "tests"), os.path.join(R, "tools", "experiments")]
import paper_1711_10912_b200 as tl  # noqa: E402
from paper_1711_10912_b200.layout import TensorMeta  # noqa: E402
from sweep_ttm5 import timeit  # noqa: E402


def peak():
    try:
        return float(json.load(open(os.path.join(R, "MEASURED_PEAKS.json")))["hbm_gbs"])
    except Exception:
        return 6545.6


def random_shape(rng, p, target):
    """p extents in [2, 1000] whose product is close to target."""
    while True:
        logs = rng.dirichlet(np.ones(p)) * np.log(target)
        ext = [max(2, int(round(np.exp(x)))) for x in logs]
        n = int(np.prod(ext))
        if 0.7 * target <= n <= 1.3 * target and max(ext) <= 1 << 20:
            return tuple(ext)


def main():
    n_cases = int(sys.argv[1]) if len(sys.argv) > 1 else 24
    rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 7)
    pk = peak()
    L = tl._abi.lib()
    import ctypes

    rows = []
    for c in range(n_cases):
        dtype = torch.float32 if c % 2 == 0 else torch.float64
        s = 4 if dtype == torch.float32 else 8
        p = int(rng.integers(2, 8))
        shape = random_shape(rng, p, (512 << 20) // s)
        layout = tuple(int(x) + 1 for x in rng.permutation(p))
        n = int(np.prod(shape))
        buf = torch.rand(n, dtype=dtype, device="cuda")
        check = os.environ.get("TL_SWEEP_CHECK") is not None
        if check:
            # the same logical tensor in first-order layout: every ttv output must be bit-identical
            A0 = tl.DenseTensor._wrap(TensorMeta(shape), buf)
            A = tl.DenseTensor._wrap(TensorMeta(shape), buf.clone())
            A.relayout(layout)
        else:
            A = tl.DenseTensor._wrap(TensorMeta(shape, layout=layout), buf)
        for mode in range(1, p + 1):
            v = tl.DenseTensor._wrap(TensorMeta((shape[mode - 1],)), torch.rand(shape[mode - 1], dtype=dtype, device="cuda"))
            if check:
                same = bool(torch.equal(tl.ttv(A, v, mode).buffer, tl.ttv(A0, v, mode).buffer))
                if not same:
                    print(json.dumps({"MISMATCH": True, "shape": shape, "layout": layout, "mode": mode}), flush=True)
                    raise SystemExit(1)
            us = timeit(lambda: tl.ttv(A, v, mode), n=5)
            nbytes = s * (n + shape[mode - 1] + n // shape[mode - 1])
            info = ctypes.create_string_buffer(512)
            L.tl_plan_describe(0, A.desc(), None, mode, info, 512)
            try:
                d = json.loads(info.value.decode())
                regime = f"{d['regime']} O={d['O']} K={d['K']} I={d['I']} ident={d['ident']}"
            except Exception:
                regime = info.value.decode()[:80]
            row = {"case": c, "dtype": "f32" if s == 4 else "f64", "shape": shape, "layout": layout, "mode": mode,
                   "us": round(us, 1), "gbs": round(nbytes / us / 1e3, 0), "frac": round(nbytes / us / 1e3 / pk, 3),
                   "kernel": regime}
            rows.append(row)
            print(json.dumps(row), flush=True)
        del A, buf
        if check:
            del A0
        torch.cuda.empty_cache()
    fr = [r["frac"] for r in rows]
    print(json.dumps({"summary": True, "cases": len(rows), "min_frac": min(fr), "median_frac": statistics.median(fr),
                      "p10_frac": sorted(fr)[len(fr) // 10], "below_0.8": sum(f < 0.8 for f in fr), "peak_gbs": pk}))


if __name__ == "__main__":
    main()
