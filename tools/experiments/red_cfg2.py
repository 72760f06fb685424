"""Device time of config 2's norm and inner product (1 GiB float32 operands)."""
import os, sys, json
R = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, R); sys.path.insert(0, os.path.join(R, "tests")); sys.path.insert(0, os.path.join(R, "tools", "experiments"))
import torch
import paper_1711_10912_b200 as tl
import paper_1711_10912_b200.contraction as C
import workloads as W
from sweep_ttm5 import timeit
T, vecs, T2 = W.cfg2()
A = tl.DenseTensor.from_memory(T.shape, W.layout_buffer(T, (1, 2, 3, 4)))
B = tl.DenseTensor.from_memory(T.shape, W.layout_buffer(T2, (1, 2, 3, 4)))
n = 128 ** 4
tn = timeit(lambda: C.frobenius_norm_device(A), n=5)
ti = timeit(lambda: C.inner_product_device(A, B), n=5)
print(json.dumps({"norm_us": round(tn, 1), "norm_tbs": round(4 * n / tn / 1e6, 2), "inner_us": round(ti, 1),
                  "inner_tbs": round(8 * n / ti / 1e6, 2), "norm": C.frobenius_norm(A)}))
