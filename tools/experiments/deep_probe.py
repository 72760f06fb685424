import os, sys, json, torch
sys.path[:0]=['.', 'tests', 'tools/experiments']
import paper_1711_10912_b200 as tl
from paper_1711_10912_b200.layout import TensorMeta
from sweep_ttm5 import timeit
for shape, mode, dt in [((128, 4096, 64), 2, torch.float64), ((128, 4096, 64), 2, torch.float32), ((256, 2048, 64), 2, torch.float64), ((64, 8192, 128), 2, torch.float32), ((400, 400, 400), 2, torch.float64)]:
    n=1
    for e in shape: n*=e
    A=tl.DenseTensor._wrap(TensorMeta(shape), torch.rand(n, dtype=dt, device='cuda'))
    v=tl.DenseTensor._wrap(TensorMeta((shape[mode-1],)), torch.rand(shape[mode-1], dtype=dt, device='cuda'))
    us=timeit(lambda: tl.ttv(A, v, mode), n=5)
    s=4 if dt==torch.float32 else 8
    print(os.environ.get('TL_TTV_DEEP_MIN_K','256'), shape, dt, round(us,1), round(s*n/us/1e3/6549,3))
