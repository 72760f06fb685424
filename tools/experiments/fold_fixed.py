"""Small-fold cost vs fold length: ttv of a (400, K) float64 tensor over mode 2
(COLS block) and of a (K, 400) tensor over mode 1 (ROWS block), graph replays."""
import os, sys, json
R = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, R); sys.path.insert(0, os.path.join(R, "tools", "experiments"))
import numpy as np, torch
import paper_1711_10912_b200 as tl
from sweep_ttm5 import timeit
rng = np.random.default_rng(0)
out = {}
for K in (8, 50, 100, 200, 400, 800):
    A = tl.DenseTensor.from_memory((400, K), rng.standard_normal(400 * K))
    v = tl.DenseTensor.from_memory((K,), rng.standard_normal(K))
    out[f"cols_K{K}"] = round(timeit(lambda: tl.ttv(A, v, 2)), 2)
    B = tl.DenseTensor.from_memory((K, 400), rng.standard_normal(400 * K))
    out[f"rows_K{K}"] = round(timeit(lambda: tl.ttv(B, v, 1)), 2)
x = torch.zeros(1, device="cuda")
out["torch_fill_1"] = round(timeit(lambda: x.fill_(1.0)), 2)
print(json.dumps(out))
