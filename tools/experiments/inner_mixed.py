"""Inner product of two 1 GiB float32 tensors stored in different layouts."""
import os, sys, json
R = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, R); sys.path.insert(0, os.path.join(R, "tests")); sys.path.insert(0, os.path.join(R, "tools", "experiments"))
import torch
import paper_1711_10912_b200 as tl
import paper_1711_10912_b200.contraction as C
from sweep_ttm5 import timeit
n = 128 ** 4
buf = torch.randn(n, dtype=torch.float32, device="cuda")
buf2 = torch.randn(n, dtype=torch.float32, device="cuda")
out = {}
for la, lb in [((1, 2, 3, 4), (1, 2, 3, 4)), ((1, 2, 3, 4), (4, 3, 2, 1)), ((1, 2, 3, 4), (3, 1, 2, 4)), ((4, 3, 2, 1), (3, 1, 2, 4))]:
    A = tl.DenseTensor.from_memory((128,) * 4, buf, layout=la)
    B = tl.DenseTensor.from_memory((128,) * 4, buf2, layout=lb)
    us = timeit(lambda: C.inner_product_device(A, B), n=5)
    out[f"{la}x{lb}"] = (round(us, 1), round(8 * n / us / 1e3, 0))
print(json.dumps(out))
