import os, sys, json
R = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, R); sys.path.insert(0, os.path.join(R, "tools", "experiments"))
import torch
import paper_1711_10912_b200 as tl
import paper_1711_10912_b200.contraction as C
from sweep_ttm5 import timeit
out = {}
for n in (1024, 65536, 1 << 20, 5222400, 20889600):
    X = tl.DenseTensor.from_memory((n,), torch.randn(n, dtype=torch.float64, device="cuda"))
    t = timeit(lambda: C.frobenius_norm_device(X))
    out[n] = round(t, 2)
print(json.dumps(out))
