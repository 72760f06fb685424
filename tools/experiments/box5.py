"""Time config 5's ttv for both seeded layouts under the current env knobs."""
import os, sys, json, hashlib
R = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, R); sys.path.insert(0, os.path.join(R, "tests")); sys.path.insert(0, os.path.join(R, "tools", "experiments"))
import paper_1711_10912_b200 as tl
import workloads as W
from sweep_ttm5 import timeit
out = {}
for seed in (5, 0):
    T, v, M, layout = W.cfg5(seed)
    A = tl.DenseTensor.from_memory(T.shape, W.layout_buffer(T, layout), layout=layout)
    del T
    V = tl.DenseTensor.from_memory((9,), v)
    out[f"seed{seed}_ttv_us"] = round(timeit(lambda: tl.ttv(A, V, 5), n=10), 2)
    out[f"seed{seed}_sha"] = hashlib.sha256(tl.ttv(A, V, 5).numpy().tobytes()).hexdigest()[:12]
    del A
print(json.dumps(out))
