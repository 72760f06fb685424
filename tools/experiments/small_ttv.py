import os, sys, json
R = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, R); sys.path.insert(0, os.path.join(R, "tools", "experiments"))
import torch
import paper_1711_10912_b200 as tl
import paper_1711_10912_b200.contraction as C
from sweep_ttm5 import timeit
out = {}
for n in (400, 1000):
    P = tl.DenseTensor.from_memory((n, n), torch.randn(n * n, dtype=torch.float64, device="cuda"))
    v = tl.DenseTensor.from_memory((n,), torch.randn(n, dtype=torch.float64, device="cuda"))
    out[f"ttv{n}_m1"] = round(timeit(lambda: tl.ttv(P, v, 1)), 2)
    out[f"ttv{n}_m2"] = round(timeit(lambda: tl.ttv(P, v, 2)), 2)
    out[f"norm{n}"] = round(timeit(lambda: C.frobenius_norm_device(v)), 2)
x = tl.DenseTensor.from_memory((1,), torch.ones(1, dtype=torch.float64, device="cuda"))
out["empty_norm"] = round(timeit(lambda: C.frobenius_norm_device(x)), 2)
print(json.dumps(out))
