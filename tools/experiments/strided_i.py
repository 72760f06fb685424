"""Strided ttv (contracted mode in the middle) vs the inner-block width I, 1 GiB float32."""
import os, sys, json
R = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, R); sys.path.insert(0, os.path.join(R, "tools", "experiments"))
import torch
import paper_1711_10912_b200 as tl
from sweep_ttm5 import timeit
out = {}
buf = torch.randn(1 << 28, dtype=torch.float32, device="cuda")
v = tl.DenseTensor.from_memory((128,), torch.randn(128, dtype=torch.float32, device="cuda"))
for I in (32, 64, 96, 128, 160, 192, 256, 512, 1024, 4096, 16384):
    O = (1 << 28) // (I * 128)
    A = tl.DenseTensor.from_memory((I, 128, O), buf[: I * 128 * O])
    us = timeit(lambda: tl.ttv(A, v, 2), n=5)
    out[I] = (round(us, 1), round(4 * I * 128 * O / us / 1e3, 0))
print(json.dumps(out))
