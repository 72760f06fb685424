import os, sys, json
R = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, R); sys.path.insert(0, os.path.join(R, "tests"))
import numpy as np, torch
import paper_1711_10912_b200 as tl
import paper_1711_10912_b200.contraction as C
sys.path.insert(0, os.path.join(R, "tools", "experiments"))
from sweep_ttm5 import timeit
out = {}
for n in (5222400, 5222400 * 4, 64 << 20):
    X = tl.DenseTensor.from_memory((n,), torch.randn(n, dtype=torch.float64, device="cuda"))
    Y = tl.DenseTensor.from_memory((n,), torch.randn(n, dtype=torch.float64, device="cuda"))
    t = timeit(lambda: C.frobenius_norm_device(X))
    out[f"norm_{n}"] = (round(t, 2), round(8 * n / t / 1e3, 0))
    t = timeit(lambda: C.inner_product_device(X, Y))
    out[f"inner_{n}"] = (round(t, 2), round(16 * n / t / 1e3, 0))
print(json.dumps(out))
