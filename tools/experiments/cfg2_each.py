import os, sys, json
R = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, R); sys.path.insert(0, os.path.join(R, "tests")); sys.path.insert(0, os.path.join(R, "tools", "experiments"))
import numpy as np, torch
import paper_1711_10912_b200 as tl
import workloads as W
from sweep_ttm5 import timeit
T, vecs, T2 = W.cfg2()
vs = [tl.DenseTensor.from_memory((128,), v) for v in vecs]
out = {}
for n, l in W.CFG2_LAYOUTS.items():
    A = tl.DenseTensor.from_memory(T.shape, W.layout_buffer(T, l), layout=l)
    for m in (1, 2, 3, 4):
        us = timeit(lambda: tl.ttv(A, vs[m - 1], m), n=5)
        out[f"{n}_q{m}"] = (round(us, 1), round(1082130944 / us / 1e3, 0))
    del A; torch.cuda.empty_cache()
print(json.dumps(out))
