"""float64 strided ttv vs inner-block width (HOPM's second pass is I = K = O = 400)."""
import os, sys, json
R = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, R); sys.path.insert(0, os.path.join(R, "tools", "experiments"))
import torch
import paper_1711_10912_b200 as tl
from sweep_ttm5 import timeit
out = {}
buf = torch.randn(400 ** 3, dtype=torch.float64, device="cuda")
for shape, mode in [((400, 400, 400), 2), ((400, 400, 400), 3), ((160000, 400), 2), ((200, 400, 800), 2), ((800, 400, 200), 2), ((512, 400, 312), 2)]:
    A = tl.DenseTensor.from_memory(shape, buf[: shape[0] * shape[1] * (shape[2] if len(shape) > 2 else 1)])
    v = tl.DenseTensor.from_memory((shape[mode - 1],), torch.randn(shape[mode - 1], dtype=torch.float64, device="cuda"))
    us = timeit(lambda: tl.ttv(A, v, mode), n=5)
    out[f"{shape}m{mode}"] = (round(us, 1), round(8 * A.size / us / 1e3, 0))
print(json.dumps(out))
