"""Is the box kernel of ttm_few.cu (J = 1) a faster ttv for the layouts where the ttv kernels are weak?
Times tl.ttv against tl.ttm with a 1 x K matrix (TL_TTM_FEW=2) on the cfg5 shape, random layouts, every mode."""
import json, os, sys
import numpy as np, torch
R = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path[:0] = [R, os.path.join(R, "tests"), os.path.join(R, "tools", "experiments")]
import paper_1711_10912_b200 as tl
from paper_1711_10912_b200.layout import TensorMeta
from sweep_ttm5 import timeit
from config_sweep import first_order, in_layout, vec, random_layouts, describe, PK

shape = (3, 33, 5, 17, 9, 2, 640)
n = int(np.prod(shape))
A0 = first_order(shape, torch.float64, 0)
vs = [vec(shape[m], torch.float64, m) for m in range(7)]
Ms = [tl.DenseTensor._wrap(TensorMeta((1, shape[m])), vs[m].buffer.clone()) for m in range(7)]
for lay in random_layouts(7, int(sys.argv[1]) if len(sys.argv) > 1 else 6):
    A = in_layout(A0, lay)
    for m in range(7):
        t1 = timeit(lambda: tl.ttv(A, vs[m], m + 1), n=5)
        t2 = timeit(lambda: tl.ttm(A, Ms[m], m + 1), n=5)
        nbytes = 8 * (n + shape[m] + n // shape[m])
        print(json.dumps({"layout": list(lay), "mode": m + 1, "ttv_us": round(t1, 1), "ttv_frac": round(nbytes / t1 / 1e3 / PK, 3),
                          "ttv_kernel": describe(A, m + 1), "few_us": round(t2, 1), "few_frac": round(nbytes / t2 / 1e3 / PK, 3),
                          "few_kernel": describe(A, m + 1, Ms[m])}), flush=True)
    del A
    torch.cuda.empty_cache()
