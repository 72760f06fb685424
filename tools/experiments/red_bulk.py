"""Cold-L2 timing of norm / inner across sizes (compare TL_RED_BULK_MIN_KB=0 vs default)."""
import json
import statistics
import sys

import numpy as np
import torch

import paper_1711_10912_b200 as tl
import paper_1711_10912_b200.contraction as C

peak = json.load(open("MEASURED_PEAKS.json")).get("hbm_gbs", 6500) if __import__("os").path.exists("MEASURED_PEAKS.json") else 6500
flush = torch.empty(128 << 20, dtype=torch.float32, device="cuda")


def cold(fn, iters=9):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    ts = []
    for k in range(iters):
        flush.fill_(float(k))
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    return statistics.median(ts)


rng = np.random.default_rng(0)
res = {}
for name, n, dt, op in [("norm_f64_42MB", 5222400, np.float64, "norm"), ("norm_f64_8MB", 1 << 20, np.float64, "norm"),
                        ("norm_f64_2MB", 1 << 18, np.float64, "norm"),
                        ("norm_f32_1GiB", 128 ** 4, np.float32, "norm"), ("inner_f32_2GiB", 128 ** 4, np.float32, "inner"),
                        ("inner_f64_256MB", 1 << 24, np.float64, "inner"), ("inner_f64_42MB", 5222400 // 2, np.float64, "inner"),
                        ("norm_i64_64MB", 1 << 23, np.int64, "inner")]:
    if dt == np.int64:
        x = rng.integers(-9, 9, n)
    else:
        x = rng.standard_normal(n).astype(dt)
    A = tl.DenseTensor.from_memory((n,), x)
    B = tl.DenseTensor.from_memory((n,), x[::-1].copy()) if op == "inner" else A
    if op == "norm":
        f = lambda: C.frobenius_norm_device(A)
        nbytes = x.nbytes
    else:
        f = lambda: C.inner_product_device(A, B)
        nbytes = 2 * x.nbytes
    us = cold(f)
    val = f().item()
    res[name] = {"us": round(us, 2), "frac": round(nbytes / (us * 1e-6) / 1e9 / peak, 3), "value": val}
    del A, B
    torch.cuda.empty_cache()
print(json.dumps(res))
