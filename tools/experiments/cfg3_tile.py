import os, sys, json
R = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, R); sys.path.insert(0, os.path.join(R, "tests")); sys.path.insert(0, os.path.join(R, "tools", "experiments"))
import numpy as np, torch
import paper_1711_10912_b200 as tl
import workloads as W
A_, B_ = W.cfg3()
Bm = tl.DenseTensor.from_memory(B_.shape, W.layout_buffer(B_, (1, 2)))
out = {}
for lname, layout in (("first", (1, 2, 3)), ("last", (3, 2, 1))):
    A = tl.DenseTensor.from_memory(A_.shape, W.layout_buffer(A_, layout), layout=layout)
    for mode in (1, 2, 3):
        C = tl.ttm(A, Bm, mode); torch.cuda.synchronize()
        best = 1e9
        for _ in range(3):
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record(); C = tl.ttm(A, Bm, mode); e.record(); torch.cuda.synchronize()
            best = min(best, s.elapsed_time(e))
        out[f"{lname}_q{mode}"] = round(2 * 512**3 * 384 / (best * 1e-3) / 1e12, 2)
        del C
    del A; torch.cuda.empty_cache()
print(json.dumps(out))
