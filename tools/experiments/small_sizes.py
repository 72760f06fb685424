"""Device time of ttv on small problems (config 1 and neighbours)."""
import os, sys, json
R = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, R); sys.path.insert(0, os.path.join(R, "tests")); sys.path.insert(0, os.path.join(R, "tools", "experiments"))
import numpy as np, torch
import paper_1711_10912_b200 as tl
from sweep_ttm5 import timeit
out = {}
for shape, mode in [((128, 96, 64), 2), ((64, 64, 64), 2), ((256, 64, 32), 2), ((96, 96, 96), 1), ((32, 512, 64), 3)]:
    A = tl.DenseTensor.from_memory(shape, torch.randn(int(np.prod(shape)), dtype=torch.float64, device="cuda"))
    v = tl.DenseTensor.from_memory((shape[mode - 1],), torch.randn(shape[mode - 1], dtype=torch.float64, device="cuda"))
    out[f"{shape}m{mode}"] = round(timeit(lambda: tl.ttv(A, v, mode), n=20), 2)
print(json.dumps(out))
